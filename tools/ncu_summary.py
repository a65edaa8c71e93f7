"""Summarise ncu outputs into profiles/: a launch list (per-kernel device time, DRAM bytes, share of
the step) and the key `--set full` counters of each kernel.

    python tools/ncu_summary.py --launches gpurun_out/r01_launches_bench.csv \
        --full gpurun_out/r01_full.ncu-rep --weights 6738149376 --tag r01
"""
import argparse
import csv
import io
import json
import os
import subprocess
from collections import OrderedDict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SHORT = [("f1_hist", "F1"), ("tf_kernel", "TF"), ("f2_gather", "F2"), ("b1_bucket", "B1"), ("tgamma", "TGAMMA"),
         ("tb_kernel", "TB"), ("tb_split", "TB"), ("b2_dw", "B2")]
ALG = {"F1": 2, "F2": 4, "B1": 4, "B2": 6}
FULL_METRICS = [
    ("gpu__time_duration.sum", "time"), ("dram__bytes_read.sum", "dram_read"), ("dram__bytes_write.sum", "dram_write"),
    ("sm__cycles_elapsed.avg.per_second", "sm_clock"), ("smsp__inst_executed.sum", "inst"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue_active_pct"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps_active_pct"),
    ("l1tex__throughput.avg.pct_of_peak_sustained_active", "l1tex_pct"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_atom.sum", "smem_atom_conflicts"),
    ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block"),
    ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem_throughput_pct"),
]


def short(name):
    for k, v in SHORT:
        if k in name:
            return v
    return name[:30]


def read_csv_text(txt):
    rows = list(csv.reader(io.StringIO(txt)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            return rows[i], rows[i + 1:]
    return rows[0], rows[1:]


def launches(path):
    hdr, rows = read_csv_text(open(path).read())
    ix = {k: j for j, k in enumerate(hdr)}
    per = OrderedDict()
    for r in rows:
        if len(r) < len(hdr):
            continue
        key = (r[ix["ID"]], short(r[ix["Kernel Name"]]))
        per.setdefault(key, {})[r[ix["Metric Name"]]] = float(r[ix["Metric Value"]].replace(",", ""))
    return per


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    ix = {k: j for j, k in enumerate(hdr)}
    out = OrderedDict()
    for r in data:
        k = short(r[ix["Kernel Name"]])
        d = {}
        for m, nm in FULL_METRICS:
            if m in ix and r[ix[m]] not in ("", "n/a"):
                try:
                    v = float(r[ix[m]].replace(",", ""))
                except ValueError:
                    continue
                u = units[ix[m]]
                scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-9, "us": 1e-6, "usecond": 1e-6,
                         "ms": 1e-3, "msecond": 1e-3, "nsecond": 1e-9, "Ghz": 1e9, "Mhz": 1e6, "hz": 1}.get(u, 1)
                d[nm] = v * scale
        out[k] = d
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--weights", type=float, default=6738149376)
    ap.add_argument("--tag", default="r01")
    ap.add_argument("--peak", type=float, default=None,
                    help="HBM GB/s (default: hbm_gbs of MEASURED_PEAKS.json, the driver's measurement)")
    a = ap.parse_args()
    if a.peak is None:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            a.peak = float(json.load(f)["hbm_gbs"])
    os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
    lines = [f"# ncu summary {a.tag}", ""]
    js = {"tag": a.tag, "weights": a.weights, "peak_gbs": a.peak, "kernels": {}}
    if a.launches:
        per = launches(a.launches)
        # last occurrence of each kernel (steady state)
        last = OrderedDict()
        for (lid, k), m in per.items():
            last[k] = m
        tot = sum(m.get("gpu__time_duration.sum", 0) for m in last.values())
        lines += ["## Launch list (`--metrics gpu__time_duration.sum,dram__bytes_*` `--clock-control none`; "
                  "cold-cache, serialised: compare shares)", "",
                  "| kernel | time (us) | share of step | DRAM read+write (GB) | DRAM GB/s | alg. bytes/weight | alg. GB/s | alg./peak |",
                  "|---|---|---|---|---|---|---|---|"]
        for k, m in last.items():
            t = m.get("gpu__time_duration.sum", 0) * 1e-9
            b = m.get("dram__bytes_read.sum", 0) + m.get("dram__bytes_write.sum", 0)
            alg = ALG.get(k)
            ag = alg * a.weights / t / 1e9 if alg and t else None
            lines.append(f"| {k} | {t*1e6:.1f} | {t*1e9/tot:.1%} | {b/1e9:.2f} | {b/t/1e9 if t else 0:.0f} | "
                         f"{alg if alg else '-'} | {'%.0f' % ag if ag else '-'} | {'%.1f%%' % (100*ag/a.peak) if ag else '-'} |")
            js["kernels"].setdefault(k, {}).update({"time_s": t, "dram_bytes": b,
                                                    "dram_bytes_per_weight": b / a.weights})
        lines += ["", f"sum of kernel times: {tot/1e6:.3f} ms", ""]
    if a.full:
        f = full(a.full)
        lines += ["## `--set full` (one launch of each kernel of one CFG3 step: tools/round_profile.sh)", "",
                  "| kernel | time (us) | DRAM GB | DRAM B/weight | SM clk GHz | inst/weight | issue active | warps active | L1tex/SMEM pipe | regs | grid x block |",
                  "|---|---|---|---|---|---|---|---|---|---|---|"]
        for k, d in f.items():
            b = d.get("dram_read", 0) + d.get("dram_write", 0)
            lines.append(f"| {k} | {d.get('time',0)*1e6:.1f} | {b/1e9:.2f} | {b/a.weights:.3f} | {d.get('sm_clock',0)/1e9:.2f} | "
                         f"{d.get('inst',0)*32/a.weights:.1f} | {d.get('issue_active_pct',0):.0f}% | {d.get('warps_active_pct',0):.0f}% | "
                         f"{d.get('l1tex_pct',0):.0f}% | {d.get('regs',0):.0f} | {d.get('grid',0):.0f}x{d.get('block',0):.0f} |")
            js["kernels"].setdefault(k, {}).update({"full_" + kk: v for kk, v in d.items()})
            if k in ALG:
                js["kernels"][k]["dram_bytes_per_weight"] = b / a.weights
        lines.append("")
    open(os.path.join(ROOT, "profiles", f"ncu_summary_{a.tag}.md"), "w").write("\n".join(lines) + "\n")
    json.dump(js, open(os.path.join(ROOT, "profiles", "ncu_full_summary.json"), "w"), indent=1)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
