"""Per-rank work of the sharded step at N ranks, measured on ONE B200: rank 0's share through the
same seven kernels bench.py times.  --mode tensor (bench.py's default at N > 1): rank 0's whole
tensors (dist.assign_tensors) -- that IS the whole per-rank step, since nothing crosses ranks in
that mode (the step time's max over ranks aside, and every rank's load is within 1% of rank 0's
for LLaMA-7B at N = 8).  --mode slice: rank 0's contiguous slice of every tensor with the
table phase replicated, without the count / gamma all-reduces, which need the GPUs.

    python tools/rank_sim.py [--workload cfg3] [--ranks 1 2 4 8] [--steps 10]
Prints one JSON line per N."""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

from paper_2309_00964_b200 import edkm as E, synth  # noqa: E402
from paper_2309_00964_b200.dist import assign_tensors, shard_range  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg3")
    ap.add_argument("--ranks", type=int, nargs="+", default=[1, 2, 4, 8])
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--mode", default="tensor", choices=["tensor", "slice"],
                    help="tensor: rank 0's whole tensors (bench.py's default at N > 1); slice: its slices")
    a = ap.parse_args()
    dev = torch.device("cuda", 0)
    wl = synth.workload(a.workload)
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter, wl.eps)
    full_w = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
    full_g = [synth.grads(wl, t, dev) for t in range(len(wl.shapes))]
    for n in a.ranks:
        if a.mode == "tensor":
            mine = assign_tensors([w.numel() for w in full_w], n)[0]
            Ws = [full_w[t] for t in mine]
            Gs = [full_g[t] for t in mine]
        else:
            rng = [shard_range(w.numel(), 0, n) for w in full_w]
            Ws = [w[lo:hi].contiguous() for w, (lo, hi) in zip(full_w, rng)]
            Gs = [g[lo:hi].contiguous() for g, (lo, hi) in zip(full_g, rng)]
        C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
        Wt = [torch.empty_like(w) for w in Ws]
        dW = [torch.empty_like(w) for w in Ws]
        plan = E.Plan([w.numel() for w in Ws], p, dev)
        stream = torch.cuda.current_stream()
        ev = [[torch.cuda.Event(enable_timing=True) for _ in range(8)] for _ in range(a.steps)]

        def step(e=None):
            def mark(i):
                if e is not None:
                    e[i].record(stream)
            mark(0)
            plan.uniquify(Ws)
            mark(1)
            plan.forward(C0)
            mark(2)
            plan.reconstruct(Ws, Wt, E.SOFT)
            mark(3)
            plan.backward_buckets(Ws, Gs)
            mark(4)
            plan.backward_gamma()
            mark(5)
            plan.backward_table()
            mark(6)
            plan.backward_dw(Ws, Gs, dW)
            mark(7)

        for _ in range(a.warmup):
            step()
        torch.cuda.synchronize()
        for s in range(a.steps):
            step(ev[s])
        torch.cuda.synchronize()
        names = ["F1", "TF", "F2", "B1", "TGAMMA", "TB", "B2"]
        ph = {k: sum(ev[s][i].elapsed_time(ev[s][i + 1]) for s in range(a.steps)) / a.steps for i, k in enumerate(names)}
        ms = sum(ph.values())
        n_local = sum(w.numel() for w in Ws)
        ideal = 16 * n_local / (json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                                           "MEASURED_PEAKS.json")))["hbm_gbs"] * 1e9) * 1e3
        print(json.dumps({"workload": wl.name, "mode": a.mode, "ranks": n, "rank0_tensors": len(Ws), "rank0_weights": n_local, "ms_per_step_compute": ms,
                          "hbm_roofline_ms": ideal, "compute_frac_of_roofline": ideal / ms,
                          "table_phase_ms": ph["TF"] + ph["TGAMMA"] + ph["TB"],
                          "phases_ms": {k: round(v, 4) for k, v in ph.items()},
                          "note": ("rank 0's whole tensors (dist.assign_tensors) on one GPU: the whole per-rank step "
                                   "(no exchange exists in this mode)" if a.mode == "tensor" else
                                   "rank 0's slices on one GPU; no all-reduces (counts are local, so the table phase "
                                   "runs on this rank's patterns: U is ~the same as at N = 1 for these sizes)")}))
        del plan, Ws, Gs, Wt, dW
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
