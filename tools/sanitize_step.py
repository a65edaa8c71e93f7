"""compute-sanitizer target: one small multi-tensor eDKM step (ragged sizes, misaligned slice, fp32 outputs)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_00964_b200 import edkm as E, synth

for wd, bits in ((torch.bfloat16, 3), (torch.float16, 4), (torch.bfloat16, 8)):
    sizes = [1, 17, 4097, 100_003, 0, 65_536 + 9]
    p = E.Params(wd, bits, 1e-3, 3)
    base = synth.normal_tensor(sum(sizes) + 8, 1.0, wd, 5).cuda()
    Ws, off = [], 3
    for n in sizes:
        Ws.append(base[off:off + n]); off += n
    Gs = [synth.normal_tensor(n, 1e-3, wd, 6 + i).cuda() for i, n in enumerate(sizes)]
    C0 = torch.tensor([synth.quantile_centroids(1 << bits, 1.0)] * len(sizes), dtype=torch.float32, device="cuda")
    plan = E.Plan(sizes, p, "cuda")
    for odt in (wd, torch.float32):
        Wt = [torch.empty(n, dtype=odt, device="cuda") for n in sizes]
        dW = [torch.empty(n, dtype=odt, device="cuda") for n in sizes]
        plan.step(Ws, Gs, C0, Wt, dW)
        plan.reconstruct(Ws, [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes], E.HARD_INDEX)
        plan.reconstruct(Ws, [torch.empty(n, dtype=odt, device="cuda") for n in sizes], E.HARD_VALUE)
    torch.cuda.synchronize()
print("sanitize step done")
