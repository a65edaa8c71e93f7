"""ncu target: run `--steps` eDKM steps of a workload (default cfg2) through the C ABI, no timing."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_00964_b200 import edkm as E  # noqa: E402
from paper_2309_00964_b200 import synth  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="cfg2")
ap.add_argument("--steps", type=int, default=2)
a = ap.parse_args()
wl = synth.workload(a.workload)
dev = torch.device("cuda")
p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
Ws = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
Gs = [synth.grads(wl, t, dev) for t in range(len(wl.shapes))]
C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
plan = E.Plan([w.numel() for w in Ws], p, dev)
Wt = [torch.empty_like(w) for w in Ws]
dW = [torch.empty_like(w) for w in Ws]
for _ in range(a.steps):
    plan.step(Ws, Gs, C0, Wt, dW)
torch.cuda.synchronize()
print("done", wl.name, sum(w.numel() for w in Ws))
