"""Per-kernel limiter summary from an ncu --set full report: duration, DRAM GB/s, issue, pipes, top stalls.
    python tools/ncu_pipes.py report.ncu-rep"""
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, units = rows[0], rows[1]


def val(row, name):
    try:
        return float(row[hdr.index(name)].replace(",", ""))
    except (ValueError, IndexError):
        return float("nan")


for row in rows[2:]:
    name = row[hdr.index("Kernel Name")][:48]
    dur = val(row, "gpu__time_duration.sum") * {"ms": 1e6, "us": 1e3, "usecond": 1e3, "msecond": 1e6}.get(units[hdr.index("gpu__time_duration.sum")], 1.0)
    dram = (val(row, "dram__bytes_read.sum") + val(row, "dram__bytes_write.sum")) * {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3}.get(units[hdr.index("dram__bytes_read.sum")], 1.0)
    print(f"== {name}  {dur / 1e3:.1f} us  DRAM {dram / 1e9:.2f} GB  {dram / dur:.0f} GB/s  "
          f"inst {val(row, 'smsp__inst_executed.sum') / 1e9:.2f} G  issue {val(row, 'sm__inst_issued.avg.pct_of_peak_sustained_active'):.0f}%")
    pipes = []
    for h in hdr:
        if h.startswith("sm__inst_executed_pipe_") and h.endswith(".avg.pct_of_peak_sustained_active"):
            v = val(row, h)
            if v >= 5:
                pipes.append((h[len("sm__inst_executed_pipe_"):-len(".avg.pct_of_peak_sustained_active")], v))
    for h in ("sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active",
              "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed",
              "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"):
        if h in hdr:
            pipes.append((h.split("__")[1].split(".")[0], val(row, h)))
    print("   pipes: " + ", ".join(f"{k} {v:.0f}%" for k, v in pipes))
    st = []
    for h in hdr:
        if h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio"):
            v = val(row, h)
            if v == v and v > 0.2:
                st.append((h[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], v))
    st.sort(key=lambda x: -x[1])
    print("   stalls/issue: " + ", ".join(f"{k} {v:.2f}" for k, v in st[:8]))
