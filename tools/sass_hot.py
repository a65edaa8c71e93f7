"""Instruction mix of every backward-branch loop of a kernel's SASS (largest first):
python tools/sass_hot.py lib.so mangled_name [n_loops]"""
import re, subprocess, sys
lib, fn = sys.argv[1], sys.argv[2]
nl = int(sys.argv[3]) if len(sys.argv) > 3 else 3
out = subprocess.run(["cuobjdump", "-sass", "-fun", fn, lib], capture_output=True, text=True).stdout
ins = []
for line in out.splitlines():
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m:
        ins.append((int(m.group(1), 16), m.group(2).strip()))
loops = []
for pc, txt in ins:
    m = re.search(r"BRA (?:\S+ )?0x([0-9a-f]+)", txt)
    if m and int(m.group(1), 16) < pc:
        loops.append((int(m.group(1), 16), pc))
loops.sort(key=lambda x: -(x[1] - x[0]))
for lo, hi in loops[:nl]:
    body = [t for p, t in ins if lo <= p <= hi]
    ops = {}
    for t in body:
        op = re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0]
        ops[op] = ops.get(op, 0) + 1
    print(f"loop {lo:#x}-{hi:#x}: {len(body)} instr; spills {sum(1 for t in body if 'LDL' in t or 'STL' in t)}")
    print("  ", sorted(ops.items(), key=lambda x: -x[1])[:18])
