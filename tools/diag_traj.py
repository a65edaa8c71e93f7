"""Diagnostic: per-iteration centroid trajectory of the GPU table phase vs the oracle."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle import oracle as O
from paper_2309_00964_b200 import edkm as E, synth

def run(dtype, bits, tau, T, sigma, n, seed):
    k = 1 << bits
    W = synth.normal_tensor(n, sigma, dtype, seed)
    C0 = np.float32(synth.quantile_centroids(k, sigma))
    p = E.Params(dtype, bits, tau, T)
    plan = E.Plan([n], p, "cuda")
    Wd = W.cuda()
    plan.uniquify([Wd]); plan.forward(torch.tensor([C0], device="cuda"))
    torch.cuda.synchronize()
    sv = plan.saved.cpu().numpy()
    off = (128 + 255) // 256 * 256
    ct = sv[off: off + (T + 1) * k * 8].view(np.float64).reshape(T + 1, k)
    bits_ = W.view(torch.int16).numpy().view(np.uint16)
    w = O.decode16(bits_, O.BF16 if dtype == torch.bfloat16 else O.FP16)
    Ct, St, _ = O.dkm_forward(w, C0.astype(np.float64), tau, T)
    for t in range(T + 1):
        print(t, "max rel err C_t:", np.max(np.abs(ct[t] - Ct[t])) / np.max(np.abs(Ct[t])), " minS/N", (St[t].min() / n) if t < T else "")

#run(torch.bfloat16, 3, 1e-5, 5, 0.02, 250_000, 80)
#run(torch.bfloat16, 3, 1e-3, 5, 1.0, 1 << 20, 0)

def table_err(dtype, bits, tau, T, sigma, n, seed):
    k = 1 << bits
    W = synth.normal_tensor(n, sigma, dtype, seed)
    C0 = np.float32(synth.quantile_centroids(k, sigma))
    p = E.Params(dtype, bits, tau, T)
    plan = E.Plan([n], p, "cuda")
    plan.uniquify([W.cuda()]); plan.forward(torch.from_numpy(C0[None]).cuda())
    torch.cuda.synchronize()
    sv = plan.saved.cpu().numpy()
    off = (128 + 255) // 256 * 256
    ct = sv[off: off + (T + 1) * k * 8].view(np.float64).reshape(T + 1, k)
    dt = O.BF16 if dtype == torch.bfloat16 else O.FP16
    counts = plan.counts.cpu().numpy()[0]
    u = np.nonzero(counts)[0]
    v = O.decode16(u.astype(np.uint16), dt)
    fin = np.isfinite(v); u, v = u[fin], v[fin]
    tab_gpu = plan.table.cpu().numpy()[0][u]
    tab_ref_gpuC = O.reconstruct(v, ct[-1], tau)          # oracle W~ with the GPU's own C_T
    w = O.decode16(W.view(torch.int16).numpy().view(np.uint16), dt)
    Ct, St, _ = O.dkm_forward(w, C0.astype(np.float64), tau, T)
    tab_ref = O.reconstruct(v, Ct[-1], tau)
    e1 = np.abs(tab_gpu - tab_ref_gpuC); e2 = np.abs(tab_gpu - tab_ref)
    i = np.argmax(e2)
    print(f"{dtype} b{bits} tau{tau} T{T}: C_T rel err {np.max(np.abs(ct[-1]-Ct[-1]))/np.max(np.abs(Ct[-1])):.2e}; "
          f"table err vs own-C {e1.max()/np.abs(tab_ref).max():.2e}, vs oracle {e2.max()/np.abs(tab_ref).max():.2e}")
    print("   worst v", v[i], "gpu", tab_gpu[i], "ref", tab_ref[i], "refownC", tab_ref_gpuC[i], "C_T", Ct[-1])

table_err(torch.float16, 3, 1e-3, 5, 1.0, 131_075, 80)
table_err(torch.bfloat16, 3, 1e-5, 5, 0.02, 250_000, 80)
table_err(torch.bfloat16, 3, 1e-3, 5, 1.0, 1 << 20, 0)
