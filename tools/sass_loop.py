"""Report the hot loop (the block containing the 256-bit streaming loads) of a kernel's SASS:
instruction count per element and any local-memory spills inside it."""
import re, subprocess, sys
lib, fn, elems = sys.argv[1], sys.argv[2], int(sys.argv[3]) if len(sys.argv) > 3 else 16
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
# find backward branches (loops): target < pc
loops = []
for pc, txt in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < pc:
        loops.append((int(m.group(1), 16), pc))
for lo, hi in loops:
    body = [t for p, t in ins if lo <= p <= hi]
    if any("LDG" in t and ".256" in t for t in body):
        ops = {}
        for t in body:
            op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0]
            ops[op.split(".")[0]] = ops.get(op.split(".")[0], 0) + 1
        spills = sum(1 for t in body if "LDL" in t or "STL" in t)
        print(f"loop {lo:#x}-{hi:#x}: {len(body)} instr, {len(body)/elems:.1f}/elem (if {elems} elems), spills {spills}")
        print("  ", sorted(ops.items(), key=lambda x: -x[1])[:14])
