"""compute-sanitizer target: small multi-tensor eDKM steps (ragged sizes incl. empty, a misaligned slice,
16-bit and fp32 outputs, soft/hard/index reconstruct) over bf16 k=2/8/256 and fp16 k=4/16, Gaussian,
heavy-tailed (both B1 banks) and fp32 (split) gradients, plus the page-compact exchange kernels."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2309_00964_b200 import edkm as E, synth

cases = [(torch.bfloat16, 3, "normal"), (torch.float16, 4, "normal"), (torch.bfloat16, 8, "normal"),
         (torch.bfloat16, 1, "cauchy"), (torch.float16, 2, "lognormal3"), (torch.bfloat16, 3, "fp32")]
for wd, bits, glaw in cases:
    sizes = [1, 17, 4097, 100_003, 0, 65_536 + 9]
    p = E.Params(wd, bits, 1e-3, 3)
    base = synth.normal_tensor(sum(sizes) + 8, 1.0, wd, 5).cuda()
    Ws, off = [], 3
    for n in sizes:
        Ws.append(base[off:off + n]); off += n
    if glaw == "normal":
        Gs = [synth.normal_tensor(n, 1e-3, wd, 6 + i).cuda() for i, n in enumerate(sizes)]
    elif glaw == "fp32":
        Gs = [synth.normal_tensor(n, 1e-3, torch.float32, 6 + i).cuda() for i, n in enumerate(sizes)]
    else:
        Gs = [synth.heavy_tailed(n, glaw, 1e-3, wd, 6 + i).cuda() for i, n in enumerate(sizes)]
    C0 = torch.tensor([synth.quantile_centroids(1 << bits, 1.0)] * len(sizes), dtype=torch.float32, device="cuda")
    plan = E.Plan(sizes, p, "cuda")
    for odt in (wd, torch.float32):
        Wt = [torch.empty(n, dtype=odt, device="cuda") for n in sizes]
        dW = [torch.empty(n, dtype=odt, device="cuda") for n in sizes]
        plan.step(Ws, Gs, C0, Wt, dW)
        plan.reconstruct(Ws, [torch.empty(n, dtype=torch.uint8, device="cuda") for n in sizes], E.HARD_INDEX)
        plan.reconstruct(Ws, [torch.empty(n, dtype=odt, device="cuda") for n in sizes], E.HARD_VALUE)
    mask = plan.count_pages()
    pages = torch.nonzero(mask.reshape(-1)).reshape(-1).to(torch.int32)
    comp = plan.pack_counts(pages)
    plan.unpack_counts(pages, comp)
    torch.cuda.synchronize()
print("sanitize step done")
