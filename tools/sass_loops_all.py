"""List every loop (backward branch) of a kernel's SASS with its instruction count and opcode mix."""
import re, subprocess, sys
lib, fn = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
for pc, txt in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < pc:
        lo = int(m.group(1), 16)
        body = [t for p, t in ins if lo <= p <= pc]
        ops = {}
        for t in body:
            op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
            ops[op] = ops.get(op, 0) + 1
        print(f"loop {lo:#x}-{pc:#x}: {len(body)} instr", sorted(ops.items(), key=lambda x: -x[1])[:16])
