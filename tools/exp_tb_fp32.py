"""CPU experiment: can TB's per-row arithmetic (and TF's row sums) run in fp32 with fp64 only for
the sums over rows, at the 1e-5 normwise dC_0 / C_T bar?  Emulates the table-form backward in numpy
(vectorised over rows, per iteration, in the kernel's operation order) and compares dC_0 with the
fp64 oracle (oracle.dkm_backward_table).  Variants:
  f64   A in fp32 (as the kernel), everything after it in fp64 (the round-2 kernel)
  n32   everything per row in fp32, gh_j = g1_j v - g2_j, dz_l = h1 v - h2_l (naive)
  s32   fp32 with gh measured from the nearest centroid's gh_m (gh'_m = 0 exactly) and
        dz_l = h1 ((v - C_hi) - C_lo)
Row sums: per-row fp64 (flush 1) or fp32 partials over R consecutive rows of a thread.
    python tools/exp_tb_fp32.py"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import oracle as O  # noqa: E402
from paper_2309_00964_b200 import synth  # noqa: E402

f32 = np.float32


def attention32(v, C, tau):
    v32 = v.astype(f32)
    d = (v[:, None] - C[None, :]) ** 2
    m = np.argmin(d, axis=1)
    lg = (-(d - d[np.arange(len(v)), m][:, None]) / tau).astype(f32)
    A = np.exp2(lg * f32(1.4426950408889634)).astype(f32)
    A = (A / A.sum(axis=1, dtype=f32)[:, None]).astype(f32)
    return A, m, v32


def rowsum(x, n, R):
    """sum over rows of n * x (rows x k) -> k, fp64 per row (R=1) or fp32 partials of R rows."""
    if R == 1:
        return (n.astype(np.float64)[:, None] * x.astype(np.float64)).sum(0)
    nr = x.shape[0]
    pad = (-nr) % R
    y = (n.astype(f32)[:, None] * x.astype(f32)).astype(f32)
    y = np.concatenate([y, np.zeros((pad, y.shape[1]), f32)])
    y = y.reshape(-1, R, y.shape[1])
    part = np.zeros((y.shape[0], y.shape[2]), f32)
    for i in range(R):
        part = (part + y[:, i]).astype(f32)  # sequential in fp32, as a thread does
    return part.astype(np.float64).sum(0)


def forward(v, n, C0, tau, T, R):
    C = np.array(C0, np.float64)
    Ct, St = [C.copy()], []
    for _ in range(T):
        A, _, _ = attention32(v, C, tau)
        if R == 0:
            S = (n[:, None] * A.astype(np.float64)).sum(0)
            M = (n[:, None] * A.astype(np.float64) * v[:, None]).sum(0)
        else:
            S = rowsum(A, n, R)
            M = rowsum(A * v.astype(f32)[:, None], n, R)
        Cn = np.where(S != 0, M / np.where(S != 0, S, 1), C)
        St.append(S)
        C = Cn
        Ct.append(C.copy())
    return np.array(Ct), np.array(St)


def backward(v, n, Ct, St, gamma, tau, mode, R):
    T, k = Ct.shape[0] - 1, Ct.shape[1]
    G = gamma.copy()
    h1 = 2.0 / tau
    psi = np.zeros(len(v))
    for it in range(T - 1, -1, -1):
        C, cn, S = Ct[it], Ct[it + 1], St[it]
        is_ = np.where(S != 0, 1.0 / np.where(S != 0, S, 1), 0.0)
        g1, g2, h2 = G * is_, G * cn * is_, h1 * C
        A, m, v32 = attention32(v, C, tau)
        if mode == "f64":
            A6 = A.astype(np.float64)
            gh = g1[None] * v[:, None] - g2[None]
            s = (A6 * gh).sum(1)
            q = A6 * (gh - s[:, None]) * (h1 * v[:, None] - h2[None])
            dpsi = (A6 * g1[None]).sum(1) - q.sum(1)
        else:
            g1f, g2f, h1f, h2f = g1.astype(f32), g2.astype(f32), f32(h1), h2.astype(f32)
            gh = (g1f[None] * v32[:, None] - g2f[None]).astype(f32)
            if mode in ("dz32", "gz32"):
                # float-float h1 C_l and g1 cn_j: dz = fma(h1, v, -h2hi) - h2lo, gh likewise
                h2 = np.float64(h1f) * C
                h2hi = h2.astype(f32)
                h2lo = (h2 - h2hi.astype(np.float64)).astype(f32)
                dz = ((h1f * v32[:, None]).astype(np.float64) - h2hi[None].astype(np.float64)).astype(f32)
                dz = (dz - h2lo[None]).astype(f32)
                if mode == "gz32":
                    g2 = g1f.astype(np.float64) * cn
                    g2hi = g2.astype(f32)
                    g2lo = (g2 - g2hi.astype(np.float64)).astype(f32)
                    gh = ((g1f[None].astype(np.float64) * v32[:, None]) - g2hi[None]).astype(f32)
                    gh = (gh - g2lo[None]).astype(f32)
            elif mode in ("sh32", "sf32"):
                gh = (gh - gh[np.arange(len(v)), m][:, None]).astype(f32)
                if mode == "sf32":
                    h2 = np.float64(h1f) * C
                    h2hi = h2.astype(f32)
                    h2lo = (h2 - h2hi.astype(np.float64)).astype(f32)
                    dz = ((h1f * v32[:, None]).astype(np.float64) - h2hi[None].astype(np.float64)).astype(f32)
                    dz = (dz - h2lo[None]).astype(f32)
                else:
                    dz = ((h1f * v32[:, None]).astype(np.float64) - h2f[None]).astype(f32)
            elif mode == "s32":
                gh = (gh - gh[np.arange(len(v)), m][:, None]).astype(f32)
                chi = C.astype(f32)
                clo = (C - chi.astype(np.float64)).astype(f32)
                dz = (h1f * ((v32[:, None] - chi[None]).astype(f32) - clo[None])).astype(f32)
            else:
                dz = ((h1f * v32[:, None]).astype(np.float64) - h2f[None]).astype(f32)  # one FMA rounding
            s = (A * gh).sum(1, dtype=f32)
            q = (A * (gh - s[:, None]) * dz).astype(f32)
            dpsi = (A * g1f[None]).sum(1, dtype=f32) - q.sum(1, dtype=f32)
        acc = rowsum(q, n, R) if mode != "f64" else (n[:, None] * q).sum(0)
        psi += dpsi
        G = acc + np.where(is_ == 0, G, 0.0)
    return G


def case(dtype, bits, tau, T, sigma, n, seed=0, glaw="normal"):
    k = 1 << bits
    W = synth.normal_tensor(n, sigma, dtype, 77 + seed)
    G = (synth.normal_tensor(n, 1e-3, torch.float32, 99 + seed) if glaw == "normal"
         else synth.heavy_tailed(n, glaw, 1e-3, torch.float32, 500 + seed)).double().numpy()
    wb = W.view(torch.int16).numpy().view(np.uint16)
    cnt = O.histogram(wb)
    u = np.nonzero(cnt)[0]
    v = O.decode16(u.astype(np.uint16), O.BF16 if dtype == torch.bfloat16 else O.FP16)
    fin = np.isfinite(v)
    u, v = u[fin], v[fin]
    nn = cnt[u].astype(np.float64)
    B = np.zeros(65536)
    np.add.at(B, wb.astype(np.int64), G)
    B = B[u]
    C0 = synth.quantile_centroids(k, sigma)
    Ct, St, TT = O.dkm_forward(v, C0, tau, T, mult=nn)
    _, _, dC_ref = O.dkm_backward_table(v, nn, B, Ct, St, tau)
    _, _, gam = O.dkm_backward_table(v, nn, B, Ct[TT:TT + 1], np.zeros((0, k)), tau)
    out = {}
    for R in (0, 8, 32):
        Cf, Sf = forward(v, nn, C0, tau, T, R)
        out[f"CT_R{R}"] = np.linalg.norm(Cf[-1] - Ct[-1]) / np.linalg.norm(Ct[-1])
    nrm = np.linalg.norm(dC_ref)
    for mode in ("f64", "n32", "s32", "sh32", "sf32"):
        for R in ((1,) if mode == "f64" else (32,)):
            dC = backward(v, nn, Ct, St, gam, tau, mode, R)
            out[f"dC_{mode}_R{R}"] = np.linalg.norm(dC - dC_ref) / nrm
    print(f"{glaw} {str(dtype)[6:]:8s} b={bits} tau={tau:g} T={T} sigma={sigma} n={n} U={len(v)}: " +
          " ".join(f"{a}={b:.1e}" for a, b in out.items()), flush=True)


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "heavy":
        for law in ("cauchy", "student_t1.2", "spike"):
            for seed in (0, 1):
                case(torch.bfloat16, 3, 1e-3, 5, 1.0, 1 << 20, seed, law)
        sys.exit(0)
    for args in [(torch.float16, 4, 1e-5, 30, 0.02, 400_000), (torch.float16, 2, 1e-5, 30, 0.02, 400_000),
                 (torch.bfloat16, 3, 1e-5, 5, 0.02, 250_000), (torch.bfloat16, 3, 1e-6, 5, 0.02, 200_003),
                 (torch.bfloat16, 1, 1e-3, 3, 1.0, 100_000), (torch.bfloat16, 4, 3e-3, 7, 1.0, 150_000),
                 (torch.float16, 4, 1e-8, 10, 0.02, 200_000), (torch.bfloat16, 3, 1e-8, 5, 0.02, 200_000),
                 (torch.float16, 3, 1e-3, 5, 1.0, 131_075)]:
        case(*args)
