"""Experiment: overlap F1 (SMEM-atomic bound) with TF+F2 (HBM bound), and B1 with TGAMMA+TB+B2,
by pipelining tensor groups over two streams with the streaming kernels capped to disjoint SM sets.

    python tools/pipeline_exp.py [--workload cfg3]
Prints one line per configuration: forward ms, backward ms (CUDA events, median of reps).
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_00964_b200 import edkm as E  # noqa: E402
from paper_2309_00964_b200 import synth  # noqa: E402
from paper_2309_00964_b200.pipeline import _groups  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg3")
ap.add_argument("--reps", type=int, default=5)
a = ap.parse_args()
wl = synth.workload(a.workload)
dev = torch.device("cuda")
p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
Ws = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
Gs = [synth.grads(wl, t, dev) for t in range(len(wl.shapes))]
numels = [w.numel() for w in Ws]
C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
Wt = [torch.empty_like(w) for w in Ws]
dW = [torch.empty_like(w) for w in Ws]
main = torch.cuda.current_stream()
sB = torch.cuda.Stream()
plans_cache = {}


def plans_for(ng):
    if ng not in plans_cache:
        gr = _groups(numels, ng)
        plans_cache[ng] = (gr, [E.Plan([numels[t] for t in g], p, dev) for g in gr])
    return plans_cache[ng]


def run(ng, c1, c2, c3, c4):
    gr, plans = plans_for(ng)
    sel = lambda L, g: [L[t] for t in g]  # noqa: E731
    e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    e0.record(main)
    evs = []
    for g, pl in zip(gr, plans):
        E.set_max_ctas(c1)
        pl.uniquify(sel(Ws, g), main)
        ev = torch.cuda.Event()
        ev.record(main)
        evs.append(ev)
    for g, pl, ev in zip(gr, plans, evs):
        sB.wait_event(ev)
        pl.forward(C0[g[0]:g[-1] + 1], sB)
        E.set_max_ctas(c2)
        pl.reconstruct(sel(Ws, g), sel(Wt, g), E.SOFT, sB)
    main.wait_stream(sB)
    e1.record(main)
    evs = []
    for g, pl in zip(gr, plans):
        E.set_max_ctas(c3)
        pl.backward_buckets(sel(Ws, g), sel(Gs, g), main)
        ev = torch.cuda.Event()
        ev.record(main)
        evs.append(ev)
    for g, pl, ev in zip(gr, plans, evs):
        sB.wait_event(ev)
        pl.backward_gamma(sB)
        pl.backward_table(sB)
        E.set_max_ctas(c4)
        pl.backward_dw(sel(Ws, g), sel(Gs, g), sel(dW, g), sB)
    main.wait_stream(sB)
    e2.record(main)
    E.set_max_ctas(0)
    return e0, e1, e2


def bench(cfg):
    run(*cfg)
    torch.cuda.synchronize()
    f, b = [], []
    for _ in range(a.reps):
        e0, e1, e2 = run(*cfg)
        torch.cuda.synchronize()
        f.append(e0.elapsed_time(e1))
        b.append(e1.elapsed_time(e2))
    f.sort()
    b.sort()
    return f[len(f) // 2], b[len(b) // 2]


cfgs = [(1, 0, 0, 0, 0)]
for ng in (4, 8, 16):
    for c1, c2 in ((148, 148), (74, 74), (64, 84), (84, 64), (56, 92)):
        cfgs.append((ng, c1, c2, c1, c2))
for ng in (8, 16):
    for c3, c4 in ((60, 88), (50, 98), (40, 108)):
        cfgs.append((ng, 74, 74, c3, c4))
for cfg in cfgs:
    fm, bm = bench(cfg)
    print(f"groups={cfg[0]:2d} F1={cfg[1]:3d} F2={cfg[2]:3d} B1={cfg[3]:3d} B2={cfg[4]:3d}  "
          f"fwd {fm:7.3f} ms  bwd {bm:7.3f} ms  total {fm + bm:7.3f} ms", flush=True)
