"""Host-side timing of the page-compact count exchange on one GPU (no collective): where does the
GPU idle between F1 and the unpack come from?  python tools/dbg_compact_timing.py"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_00964_b200 import edkm as E, synth
from paper_2309_00964_b200.dist import union_pages

wl = synth.workload("cfg3")
dev = torch.device("cuda")
p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
Ws = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
plan = E.Plan([w.numel() for w in Ws], p, dev)
for it in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    plan.uniquify(Ws)
    t1 = time.perf_counter()
    mask = plan.count_pages()
    t2 = time.perf_counter()
    host = union_pages(mask)
    t3 = time.perf_counter()
    pages = host.to(dev)
    t4 = time.perf_counter()
    comp = plan.pack_counts(pages)
    t5 = time.perf_counter()
    plan.unpack_counts(pages, comp)
    t6 = time.perf_counter()
    torch.cuda.synchronize()
    t7 = time.perf_counter()
    print(f"launch F1 {1e3*(t1-t0):.3f}  count_pages {1e3*(t2-t1):.3f}  union_pages (sync+nonzero) {1e3*(t3-t2):.3f}  "
          f"H2D {1e3*(t4-t3):.3f}  pack {1e3*(t5-t4):.3f}  unpack {1e3*(t6-t5):.3f}  tail {1e3*(t7-t6):.3f} ms  "
          f"pages {host.numel()}")
m = mask.reshape(-1).cpu()
t = time.perf_counter(); torch.nonzero(m); print("nonzero alone", 1e3 * (time.perf_counter() - t), "ms")
