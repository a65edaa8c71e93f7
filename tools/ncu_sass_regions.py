"""Where a kernel's warp-stall samples fall, by SASS address range: the innermost loops (backward
branches) and the code between them.  python tools/ncu_sass_regions.py report.ncu-rep kernel_regex"""
import csv
import io
import re
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "--kernel-name", f"regex:{sys.argv[2]}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = rows[1]
ia, isrc, iss, iex = (hdr.index(k) for k in ("Address", "Source", "Warp Stall Sampling (All Samples)",
                                              "Instructions Executed"))
ins = []
for r in rows[2:]:
    if len(r) <= iex or not r[ia].startswith("0x"):
        continue
    ins.append((int(r[ia], 16), r[isrc].strip(), int(r[iss] or 0), int(r[iex] or 0)))
base = ins[0][0]
tot_s = sum(x[2] for x in ins)
tot_e = sum(x[3] for x in ins)
# regions: split at backward-branch targets and branch sources
cuts = {0}
for pc, src, _, _ in ins:
    m = re.search(r"BRA (?:\S+ )?(0x[0-9a-f]+)", src)
    if m:
        tgt = int(m.group(1), 16)
        tgt = tgt - base if tgt >= base else tgt  # absolute or kernel-relative
        if tgt < pc - base:
            cuts.add(tgt)
            cuts.add(pc - base + 16)
cuts = sorted(cuts)
regs = []
for a, b in zip(cuts, cuts[1:] + [1 << 40]):
    sel = [x for x in ins if a <= x[0] - base < b]
    if sel:
        regs.append((a, b, sum(x[2] for x in sel), sum(x[3] for x in sel), len(sel)))
print(f"total samples {tot_s}, warp instructions {tot_e}")
for a, b, s, e, n in sorted(regs, key=lambda r: -r[2])[:12]:
    print(f"  {a:#07x}-{min(b, ins[-1][0] - base):#07x}  {n:5d} instr  samples {100 * s / tot_s:5.1f}%  executed {100 * e / tot_e:5.1f}%")
