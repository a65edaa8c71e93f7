"""CUDA path (libedkm.so through the C ABI) vs the CPU oracle, element by element.

Bars:
  * counts, hard indices, hard values: bit-exact;
  * C_T, W~ (fp32 output), dW (fp32 output), dC_0: normwise
    ||x - x_ref||_inf <= 1e-5 ||x_ref||_inf per tensor (north star tolerance);
  * 16-bit outputs: within 1 ulp of round-to-nearest-even of the oracle value
    (double rounding / fp64 reordering can flip a tie, R8), plus 1e-5 ||ref|| for dW.
The oracle runs dense over all |W| x |C| entries (CFG1 sizes) or, at full
BASELINE sizes, in its pinned attention-table form from exact CPU counts.
"""
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2309_00964_b200 import synth
from paper_2309_00964_b200 import edkm as E

pytestmark = pytest.mark.gpu
TOL = 1e-5
# An oracle S_s[j] below DEAD * N marks a dead cluster (R6; see check_tensor): 2^-100 leaves a
# factor 2^26 between it and the GPU's fp32 flush-to-zero level 2^-126 per attention entry, so
# above it the flushed entries change S_s[j] by < 2^-26 relative and every value is compared.
DEAD = 2.0 ** -100


ERRS = []  # (test, quantity, value): written to $EDKM_PARITY_REPORT by conftest (measured error distribution)


def record(quantity, value):
    ERRS.append((os.environ.get("PYTEST_CURRENT_TEST", "?").split(" ")[0], quantity, float(value)))


def bits_of(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().contiguous().view(torch.int16).numpy().view(np.uint16).ravel()


def odt(dtype):
    return O.BF16 if dtype == torch.bfloat16 else O.FP16


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)) if b.size else 0.0


def ulp16(x: np.ndarray, dtype) -> np.ndarray:
    t = torch.from_numpy(np.abs(x)).to(dtype).to(torch.float64).numpy()
    mant = 7 if dtype == torch.bfloat16 else 10
    tiny = 2.0 ** (-133 if dtype == torch.bfloat16 else -24)
    e = np.floor(np.log2(np.maximum(t, 1e-300)))
    return np.maximum(2.0 ** (e - mant), tiny)


def as16_values(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().to(torch.float64).numpy().ravel()


def run_gpu(Ws, Gs, C0, p: E.Params, out_f32=True):
    """One full step through the C ABI.  Returns dict of numpy results."""
    dev = torch.device("cuda")
    Wd = [w.to(dev).reshape(-1) for w in Ws]
    Gd = [g.to(dev).reshape(-1) for g in Gs]
    plan = E.Plan([w.numel() for w in Wd], p, dev)
    C0d = torch.tensor(np.asarray(C0), dtype=torch.float32, device=dev)
    plan.uniquify(Wd)
    plan.forward(C0d)
    odtype = torch.float32 if out_f32 else p.wdtype
    Wt = [torch.empty(w.numel(), dtype=odtype, device=dev) for w in Wd]
    plan.reconstruct(Wd, Wt, E.SOFT)
    Wt16 = [torch.empty(w.numel(), dtype=p.wdtype, device=dev) for w in Wd]
    plan.reconstruct(Wd, Wt16, E.SOFT)
    idx = [torch.empty(w.numel(), dtype=torch.uint8, device=dev) for w in Wd]
    plan.reconstruct(Wd, idx, E.HARD_INDEX)
    hv = [torch.empty(w.numel(), dtype=torch.float32, device=dev) for w in Wd]
    plan.reconstruct(Wd, hv, E.HARD_VALUE)
    hv16 = [torch.empty(w.numel(), dtype=p.wdtype, device=dev) for w in Wd]
    plan.reconstruct(Wd, hv16, E.HARD_VALUE)
    plan.backward_reduce(Wd, Gd)
    dW = [torch.empty(w.numel(), dtype=odtype, device=dev) for w in Wd]
    plan.backward_apply(Wd, Gd, dW)
    dW16 = [torch.empty(w.numel(), dtype=p.wdtype, device=dev) for w in Wd]
    plan.backward_apply(Wd, Gd, dW16)
    torch.cuda.synchronize()
    nonfin, iters = E.read_status(plan.saved, plan.nt, p)
    v = plan.views()
    ctraj = v["ctraj"].contiguous().view(torch.float64).view(max(plan.nt, 1), p.max_iter + 1, p.k).cpu().numpy()
    straj = v["straj"].contiguous().view(torch.float64).view(max(plan.nt, 1), max(p.max_iter, 1), p.k).cpu().numpy()
    return dict(counts=plan.counts.cpu().numpy(), C=plan.C_out.cpu().numpy(), table=plan.table.cpu().numpy(),
                ctraj=ctraj, straj=straj,
                Wt=[x.cpu().double().numpy() for x in Wt], Wt16=[as16_values(x) for x in Wt16],
                idx=[x.cpu().numpy() for x in idx], hv=[x.cpu().numpy() for x in hv],
                hv16=[bits_of(x) for x in hv16], dW=[x.cpu().double().numpy() for x in dW],
                dW16=[as16_values(x) for x in dW16], dC0=plan.dC0.cpu().numpy(), gamma=plan.gamma.cpu().numpy(),
                nonfinite=nonfin, iters=iters)


def oracle_dense(w_bits, G, C0, p: E.Params):
    C0 = np.asarray(C0, np.float32).astype(np.float64)  # the C ABI takes fp32 centroids: same input
    w = O.decode16(w_bits, odt(p.wdtype))
    Ct, St, T = O.dkm_forward(w, C0, p.tau, p.max_iter, p.eps)
    Wt = O.reconstruct(w, Ct[-1], p.tau)
    dW, dC = O.dkm_backward(w, G, Ct, St, p.tau)
    return dict(w=w, Ct=Ct, St=St, T=T, Wt=Wt, dW=dW, dC=dC)


def within(got, ref, lim, what):
    bad = ~(np.abs(got - ref) <= lim)
    if bad.any():
        i = np.flatnonzero(bad)[:5]
        raise AssertionError(f"{what}: {bad.sum()} of {bad.size} outside the bound; e.g. got {got[i]} ref {ref[i]} "
                             f"lim {np.broadcast_to(lim, ref.shape)[i]}")


def check_tensor(gpu, t, w_bits, G, ref, p: E.Params, dense=True):
    w = ref["w"]
    fin = np.isfinite(w)
    # counts: bit-exact (F1)
    assert np.array_equal(gpu["counts"][t], O.histogram(w_bits).astype(np.int32))
    assert gpu["iters"][t] == ref["T"]
    assert gpu["nonfinite"][t] == int((~fin).sum())
    CT = ref["Ct"][-1]
    nfin = max(int(fin.sum()), 1)
    dead = [s for s in range(ref["T"]) if np.min(ref["St"][s]) < DEAD * nfin]
    if dead:
        # Dead cluster (R6): some S_s[j] of the oracle is below 2^-100 N.  The GPU's fp32 exponent
        # flushes every attention entry below 2^-126 to zero (R7), so such an S_s[j] can only be
        # matched to an absolute N 2^-126; where it is exactly 0 the GPU keeps C_s[j] (R6) while the
        # fp64 oracle moves it onto the nearest weight, and every later iteration may differ.
        # Everything up to and including iteration s0 = the first dead one is compared; after it
        # only what is still defined (counts, finiteness, hard assignment vs the GPU's own C).
        s0 = dead[0]
        Cg, Sg = gpu["ctraj"][t], gpu["straj"][t]
        for s in range(s0 + 1):
            assert normwise(Cg[s], ref["Ct"][s]) <= TOL, ("C_s before the dead iteration", s)
        for s in range(s0 + 1):
            lim = TOL * np.max(ref["St"][s]) + nfin * 2.0 ** -126
            assert np.all(np.abs(Sg[s] - ref["St"][s]) <= lim), ("S_s", s, Sg[s], ref["St"][s])
        assert np.all(np.isfinite(gpu["C"][t]))
        C32 = gpu["C"][t].astype(np.float32)
        idx_ref = O.hard_assign(w, C32)
        idx_ref[~fin] = 0
        assert np.array_equal(gpu["idx"][t].astype(np.int32), idx_ref)
        return
    # the C and S trajectories of every iteration (saved for the backward pass)
    for s in range(ref["T"] + 1):
        assert normwise(gpu["ctraj"][t][s], ref["Ct"][s]) <= TOL, ("C_s", s)
    for s in range(ref["T"]):
        assert normwise(gpu["straj"][t][s], ref["St"][s]) <= TOL, ("S_s", s)
    record("C_T", normwise(gpu["C"][t], CT))
    assert normwise(gpu["C"][t], CT) <= TOL, ("C", normwise(gpu["C"][t], CT))
    # table for every populated finite pattern
    u = np.nonzero(gpu["counts"][t])[0]
    uf = u[np.isfinite(O.decode16(u.astype(np.uint16), odt(p.wdtype)))]
    tab_ref = O.reconstruct(O.decode16(uf.astype(np.uint16), odt(p.wdtype)), CT, p.tau)
    assert normwise(gpu["table"][t][uf], tab_ref) <= TOL
    if not dense:
        return
    Wt_ref, dW_ref = ref["Wt"], ref["dW"]
    assert np.all(np.isnan(gpu["Wt"][t][~fin])) and np.all(np.isnan(gpu["dW"][t][~fin]))
    record("W~ fp32", normwise(gpu["Wt"][t][fin], Wt_ref[fin]))
    record("dW fp32", normwise(gpu["dW"][t][fin], dW_ref[fin]))
    record("dC_0", normwise(gpu["dC0"][t], ref["dC"]))
    if fin.any():
        record("W~ 16-bit ulps", float(np.max(np.abs(gpu["Wt16"][t][fin] - Wt_ref[fin]) / ulp16(Wt_ref[fin], p.wdtype))))
        record("dW 16-bit ulps", float(np.max(np.abs(gpu["dW16"][t][fin] - dW_ref[fin]) / ulp16(dW_ref[fin], p.wdtype))))
    assert normwise(gpu["Wt"][t][fin], Wt_ref[fin]) <= TOL, ("Wt", normwise(gpu["Wt"][t][fin], Wt_ref[fin]))
    assert normwise(gpu["dW"][t][fin], dW_ref[fin]) <= TOL, ("dW", normwise(gpu["dW"][t][fin], dW_ref[fin]))
    # dC_0 normwise; its floor is set by the size of the summands (~sum |G|), below which the
    # fp64 oracle itself only carries cancellation residue (e.g. tiny tensors where every
    # cluster collapses onto its own weights and dL/dC_0 ~ 1e-26)
    floor = 1e-9 * float(np.sum(np.abs(G[fin]))) if G is not None else 0.0
    assert np.max(np.abs(gpu["dC0"][t] - ref["dC"])) <= TOL * max(np.max(np.abs(ref["dC"])), floor) + 1e-37, \
        ("dC", gpu["dC0"][t], ref["dC"])
    # 16-bit outputs: <= 1 ulp of the fp64 oracle value, plus the normwise 1e-5 allowance where
    # W~ cancels to ~0 between centroids of opposite sign (R7, R8)
    within(gpu["Wt16"][t][fin], Wt_ref[fin], ulp16(Wt_ref[fin], p.wdtype) + TOL * np.max(np.abs(Wt_ref[fin])),
           "W~ 16-bit")
    lim = ulp16(dW_ref[fin], p.wdtype) + TOL * np.max(np.abs(dW_ref[fin]))
    within(gpu["dW16"][t][fin], dW_ref[fin], lim, "dW 16-bit")
    # hard assignment against the GPU's own fp32 lookup table (R9): bit-exact
    C32 = gpu["C"][t].astype(np.float32)
    idx_ref = O.hard_assign(w, C32)
    idx_ref[~fin] = 0
    assert np.array_equal(gpu["idx"][t].astype(np.int32), idx_ref)
    hv_ref = C32[idx_ref]
    assert np.array_equal(gpu["hv"][t][fin].view(np.uint32), hv_ref[fin].view(np.uint32))
    hv16_ref = bits_of(torch.from_numpy(hv_ref).to(p.wdtype))
    assert np.array_equal(gpu["hv16"][t][fin], hv16_ref[fin])


# --------------------------------------------------------------------------- CFG1 in full (BASELINE configs[0])
def test_cfg1_full_parity():
    wl = synth.workload("cfg1")
    W = synth.weights(wl, 0)
    G = synth.grads(wl, 0)
    C0 = synth.quantile_centroids(wl.k, wl.sigma)
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    ref = oracle_dense(wb, G.double().numpy(), C0, p)
    assert np.min(ref["St"]) >= 1e-6 * W.numel()
    check_tensor(gpu, 0, wb, G.double().numpy(), ref, p)


# --------------------------------------------------------------------------- sweeps at oracle-friendly sizes
@pytest.mark.parametrize("dtype,bits,tau,T,sigma,n", [
    (torch.bfloat16, 3, 1e-4, 5, 0.02, 300_001),
    (torch.bfloat16, 3, 1e-5, 5, 0.02, 250_000),
    (torch.bfloat16, 3, 1e-6, 5, 0.02, 200_003),
    (torch.bfloat16, 1, 1e-3, 3, 1.0, 100_000),
    (torch.bfloat16, 2, 1e-2, 0, 1.0, 100_000),
    (torch.bfloat16, 4, 3e-3, 7, 1.0, 150_000),
    (torch.float16, 4, 1e-5, 30, 0.02, 200_000),
    (torch.float16, 2, 1e-5, 30, 0.02, 120_007),
    (torch.float16, 3, 1e-3, 5, 1.0, 131_075),
    # bits 5..8 (warp-per-row table kernels; 8-bit embeddings)
    (torch.bfloat16, 5, 1e-3, 4, 1.0, 300_000),
    (torch.bfloat16, 6, 2e-6, 3, 0.02, 200_001),
    (torch.float16, 7, 1e-4, 3, 1.0, 150_000),
    (torch.bfloat16, 8, 1e-8, 3, 0.02, 400_000),
])
def test_parity_sweep(dtype, bits, tau, T, sigma, n):
    k = 1 << bits
    W = synth.normal_tensor(n, sigma, dtype, 77 + bits)
    G = synth.normal_tensor(n, 1e-3, dtype, 99 + bits)
    C0 = synth.quantile_centroids(k, sigma)
    p = E.Params(dtype, bits, tau, T)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    ref = oracle_dense(wb, G.double().numpy(), C0, p)
    if T > 0:
        assert np.min(ref["St"]) >= 1e-6 * n
    check_tensor(gpu, 0, wb, G.double().numpy(), ref, p)


def test_fp32_gradients():
    n = 100_000
    W = synth.normal_tensor(n, 0.02, torch.bfloat16, 5)
    G = synth.normal_tensor(n, 1e-3, torch.float32, 6)
    C0 = synth.quantile_centroids(8, 0.02)
    p = E.Params(torch.bfloat16, 3, 1e-5, 5)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    check_tensor(gpu, 0, wb, G.double().numpy(), oracle_dense(wb, G.double().numpy(), C0, p), p)


# --------------------------------------------------------------------------- heavy-tailed gradients (B1 buckets)
# LLM gradients are heavy-tailed.  B1 sums G per pattern in fixed point (DESIGN S4 "B1"); a
# scale tied to one sample max alone rounds small elements in absolute terms, which put dC_0
# over the 1e-5 bar for these laws.  CFG1 in full against the dense oracle.
@pytest.mark.parametrize("gdtype,seed", [(torch.bfloat16, 0), (torch.bfloat16, 1), (torch.bfloat16, 2),
                                         (torch.float32, 0), (torch.float16, 0)])
@pytest.mark.parametrize("kind", synth.HEAVY_TAILS)
def test_heavy_tailed_gradients_cfg1(kind, gdtype, seed):
    wl = synth.workload("cfg1")
    # 16-bit G must have the weights' dtype (C ABI): fp16 G runs with the CFG1 weights in fp16
    wdt = torch.float16 if gdtype == torch.float16 else wl.wdtype
    W = synth.normal_tensor(wl.shapes[0][1] * wl.shapes[0][2], wl.sigma, wdt, wl.seed_base)
    G = synth.heavy_tailed(W.numel(), kind, 1e-3, gdtype, 500 + seed)
    assert torch.isfinite(G.float()).all()
    C0 = synth.quantile_centroids(wl.k, wl.sigma)
    p = E.Params(wdt, wl.bits, wl.tau, wl.max_iter)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    Gd = G.double().numpy()
    ref = oracle_dense(wb, Gd, C0, p)
    check_tensor(gpu, 0, wb, Gd, ref, p)
    assert normwise(gpu["dC0"][0], ref["dC"]) <= TOL, ("dC_0", gpu["dC0"][0], ref["dC"])
    # gamma_T = sum_u B[u] dW~_u/dC_T (the B1 + TGAMMA output) against the dense definition
    # (the per-learner partial that the all-reduce sums); T = 0 makes dC_0 = gamma_T
    p0 = E.Params(wdt, wl.bits, wl.tau, 0)
    g0 = run_gpu([W], [G], [C0], p0)
    r0 = oracle_dense(wb, Gd, C0, p0)
    assert normwise(g0["dC0"][0], r0["dC"]) <= TOL, ("gamma_T", g0["dC0"][0], r0["dC"])


@pytest.mark.parametrize("kind", synth.HEAVY_TAILS)
def test_heavy_tailed_gradients_cfg2_tensor(kind):
    """One CFG2 tensor (q_proj, 4096 x 4096 bf16, k=8, tau=1e-5, T=5) with heavy-tailed G: dC_0
    and dW against the oracle's pinned attention-table form (exact per-pattern sums B[u])."""
    wl = synth.workload("cfg2")
    W = synth.weights(wl, 0)
    G = synth.heavy_tailed(W.numel(), kind, 1e-3, torch.bfloat16, 700)
    C0 = synth.quantile_centroids(wl.k, wl.sigma)
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    c = O.histogram(wb)
    assert np.array_equal(gpu["counts"][0], c.astype(np.int32))
    u = np.nonzero(c)[0]
    v = O.decode16(u.astype(np.uint16), O.BF16)
    Ct, St, _ = O.dkm_forward(v, np.float32(C0).astype(np.float64), wl.tau, wl.max_iter, mult=c[u])
    assert normwise(gpu["C"][0], Ct[-1]) <= TOL
    pos = np.searchsorted(u, wb)
    Gd = G.double().numpy()
    B = np.bincount(pos, weights=Gd, minlength=u.size)
    phi, psi, dC = O.dkm_backward_table(v, c[u].astype(np.float64), B, Ct, St, wl.tau)
    assert normwise(gpu["dC0"][0], dC) <= TOL, (kind, gpu["dC0"][0], dC)
    dw_ref = Gd * phi[pos] + psi[pos]
    assert normwise(gpu["dW"][0], dw_ref) <= TOL


@pytest.mark.parametrize("dtype,bits,lo,hi,n", [(torch.bfloat16, 3, -40, 12, 60_000),
                                                  (torch.float16, 4, -10, 4, 200_000)])
def test_rows_beyond_the_shared_stage(dtype, bits, lo, hi, n):
    """38 tensors (so the table kernels run CFG3/CFG4's cluster size: 2 CTAs per bf16 tensor, 4 per
    fp16 tensor) whose weights are log-uniform over many binades, so every CTA holds more populated
    patterns than it stages in shared memory (4,608 bf16 / 6,400 fp16 rows): the rows beyond the
    stage take the global-memory path in TF, TGAMMA and TB (value, count and psi).  C_0: the
    quantiles of N(0, 2^2) (well separated), tau = 1e-2."""
    nt = 38
    rng = np.random.default_rng(7)
    Ws = []
    for i in range(nt):
        x = np.exp2(rng.uniform(lo, hi, n)) * np.where(rng.random(n) < 0.5, -1.0, 1.0)
        Ws.append(torch.from_numpy(x).to(dtype))
    Gs = [synth.normal_tensor(n, 1e-3, dtype, 900 + i) for i in range(nt)]
    C0s = [synth.quantile_centroids(1 << bits, 2.0)] * nt
    p = E.Params(dtype, bits, 1e-2, 3)
    gpu = run_gpu(Ws, Gs, C0s, p)
    stage = 4608 if dtype == torch.bfloat16 else 6400
    cl = 2 if dtype == torch.bfloat16 else 4
    beyond = 0
    for t in range(nt):
        wb = bits_of(Ws[t])
        beyond += np.unique(wb).size > cl * stage
        if t % 6 == 0:  # the dense oracle on every sixth tensor (each one runs the same kernels)
            ref = oracle_dense(wb, Gs[t].double().numpy(), C0s[t], p)
            check_tensor(gpu, t, wb, Gs[t].double().numpy(), ref, p)
    assert beyond == nt  # every tensor has rows beyond its CTAs' stages


@pytest.mark.parametrize("dtype,bits", [(torch.bfloat16, 3), (torch.float16, 4), (torch.bfloat16, 6)])
def test_absent_pattern_entries_are_never_read(dtype, bits):
    """TF writes the W~ tables (fp32, 16-bit, hard index) only for populated and non-finite
    patterns (include/edkm.h); every output must come out bit-identical whatever the other entries
    hold: one plan's saved/table/workspace buffers start as 0xFF bytes (stale index bytes past k),
    the other's as zeros; soft (16-bit and fp32), hard-value and hard-index outputs and dW compared."""
    n = 300_001
    W = synth.normal_tensor(n, 0.02, dtype, 61)
    W[[3, 99]] = torch.tensor([float("nan"), -float("inf")], dtype=dtype)
    G = synth.normal_tensor(n, 1e-3, dtype, 62).cuda()
    Wd = W.cuda()
    p = E.Params(dtype, bits, 1e-5, 4)
    C0 = torch.tensor([synth.quantile_centroids(1 << bits, 0.02)], dtype=torch.float32, device="cuda")
    res = []
    for fill in (0xFF, 0x00):
        plan = E.Plan([n], p, "cuda")
        for buf in (plan.saved, plan.ws, plan.table.view(torch.uint8)):
            buf.fill_(fill)
        outs = {}
        for odt in (dtype, torch.float32):
            wt = torch.empty(n, dtype=odt, device="cuda")
            dw = torch.empty(n, dtype=odt, device="cuda")
            plan.step([Wd], [G], C0, [wt], [dw])
            outs[f"soft_{odt}"], outs[f"dw_{odt}"] = wt.cpu(), dw.cpu()
        hv = torch.empty(n, dtype=dtype, device="cuda")
        plan.reconstruct([Wd], [hv], E.HARD_VALUE)
        hi = torch.empty(n, dtype=torch.uint8, device="cuda")
        plan.reconstruct([Wd], [hi], E.HARD_INDEX)
        torch.cuda.synchronize()
        outs["hard_value"], outs["hard_index"] = hv.cpu(), hi.cpu()
        res.append(outs)
    for k in res[0]:
        a, b = res[0][k], res[1][k]
        assert torch.equal(a.view(torch.uint8), b.view(torch.uint8)), k


def test_many_ragged_tensors_and_empty():
    sizes = [0, 1, 17, 4097, 65536 * 3 + 5, 0, 250_001, 2, 31, 33]
    p = E.Params(torch.bfloat16, 3, 1e-3, 4)
    Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 300 + i) for i, n in enumerate(sizes)]
    Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 400 + i) for i, n in enumerate(sizes)]
    # C_0 = k distinct weights of the tensor where it has >= k distinct values (no cluster starts
    # empty, so every value is compared); n = 1, 2 < k necessarily leaves dead clusters (R6)
    C0s = [synth.data_quantile_centroids(w, 8) if n >= 8 else synth.quantile_centroids(8, 1.0)
           for w, n in zip(Ws, sizes)]
    gpu = run_gpu(Ws, Gs, C0s, p)
    compared = 0
    for t, n in enumerate(sizes):
        wb = bits_of(Ws[t])
        if n == 0:
            assert gpu["counts"][t].sum() == 0
            assert np.allclose(gpu["C"][t], C0s[t], rtol=1e-7)  # no data: centroids unchanged (R6)
            continue
        ref = oracle_dense(wb, Gs[t].double().numpy(), C0s[t], p)
        if n >= 8:
            assert np.min(ref["St"]) >= DEAD * n
            compared += 1
        check_tensor(gpu, t, wb, Gs[t].double().numpy(), ref, p)
    assert compared == 6


def test_misaligned_slices():
    base = synth.normal_tensor(200_000, 1.0, torch.bfloat16, 11)
    gbase = synth.normal_tensor(200_000, 1e-3, torch.bfloat16, 12)
    p = E.Params(torch.bfloat16, 2, 1e-2, 3)
    for off in (1, 3, 5, 8, 15):
        W = base[off:off + 150_001]
        G = gbase[off:off + 150_001]
        C0 = synth.quantile_centroids(4, 1.0)
        gpu = run_gpu([W], [G], [C0], p)
        wb = bits_of(W)
        check_tensor(gpu, 0, wb, G.double().numpy(), oracle_dense(wb, G.double().numpy(), C0, p), p)
    # gradient misaligned relative to the weights: scalar path
    W = base[:150_000]
    G = gbase[3:150_003]
    C0 = synth.quantile_centroids(4, 1.0)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    check_tensor(gpu, 0, wb, G.double().numpy(), oracle_dense(wb, G.double().numpy(), C0, p), p)


def test_narrow_window_tail_outliers():
    """Weights whose populated pages span more than the per-weight kernels' window cap (55
    magnitude pages): TF then picks the narrowest window holding all but ~1e-6 of the weights
    (common.cuh choose_window), so a handful of tiny-magnitude outliers fall outside it and take
    the generic paths of B1 (fp64 global bucket), B2 (global (phi, psi)) and F1/F2 -- the
    results must still match the oracle element by element."""
    n = 1 << 23
    W = synth.normal_tensor(n, 1.0, torch.bfloat16, 21).clone()
    G = synth.normal_tensor(n, 1e-3, torch.bfloat16, 22)
    for i, v in zip((5, 77_777, 1_000_003, 4_000_001, 6_543_210, n - 1), (1e-30, -2e-35, 3e-25, -1e-37, 5e-33, -7e-28)):
        W[i] = v
    wb = bits_of(W)
    pages = np.unique((wb >> 8) & 0x7F)
    assert pages.max() - pages.min() + 1 > 55  # the window must be narrowed
    p = E.Params(torch.bfloat16, 3, 1e-3, 5)
    C0 = synth.quantile_centroids(8, 1.0)
    gpu = run_gpu([W], [G], [C0], p)
    check_tensor(gpu, 0, wb, G.double().numpy(), oracle_dense(wb, G.double().numpy(), C0, p), p)


def test_cuda_graph_replay_matches_eager():
    """Plan.graph: the whole step captured once and replayed on new input values gives the
    eager step's results (counts, W~ bit-exact; the gradients to fp64 atomic-order rounding)."""
    dev = torch.device("cuda")
    sizes = [300_001, 1 << 20, 4097]
    p = E.Params(torch.bfloat16, 3, 1e-3, 5)
    C0 = torch.tensor([synth.quantile_centroids(8, 1.0)] * len(sizes), dtype=torch.float32, device=dev)

    def inputs(seed):
        return ([synth.normal_tensor(n, 1.0, torch.bfloat16, seed + i).to(dev) for i, n in enumerate(sizes)],
                [synth.normal_tensor(n, 1e-3, torch.bfloat16, seed + 50 + i).to(dev) for i, n in enumerate(sizes)])

    Ws, Gs = inputs(100)
    outs = [torch.empty(n, dtype=torch.float32, device=dev) for n in sizes]
    dW = [torch.empty(n, dtype=torch.float32, device=dev) for n in sizes]
    plan = E.Plan(sizes, p, dev)
    g = plan.graph(Ws, Gs, C0, outs, dW)
    W2, G2 = inputs(200)  # new values in the captured buffers
    for a, b in zip(Ws + Gs, W2 + G2):
        a.copy_(b)
    g.replay()
    torch.cuda.synchronize()
    ref = E.Plan(sizes, p, dev)
    outs2 = [torch.empty_like(o) for o in outs]
    dW2 = [torch.empty_like(d) for d in dW]
    ref.step(W2, G2, C0, outs2, dW2)
    torch.cuda.synchronize()
    assert torch.equal(plan.counts, ref.counts)
    assert all(torch.equal(a, b) for a, b in zip(outs, outs2))
    for a, b in zip(dW, dW2):
        assert normwise(a.cpu().double().numpy(), b.cpu().double().numpy()) <= 1e-12
    assert normwise(plan.dC0.cpu().double().numpy(), ref.dC0.cpu().double().numpy()) <= 1e-9


# --------------------------------------------------------------------------- histogram edge cases (bit-exact)
@pytest.mark.parametrize("case", ["constant", "every_pattern", "random_bits", "signed_zero", "tiny", "big"])
def test_uniquify_edge_cases(case):
    if case == "constant":
        b = np.full(300_000, 0x3F80, np.uint16)                     # one bin > 65535 (32-way collisions)
    elif case == "every_pattern":
        b = np.random.default_rng(0).permutation(65536).astype(np.uint16)
    elif case == "random_bits":
        b = np.random.default_rng(1).integers(0, 65536, 1_000_003).astype(np.uint16)  # incl. >= 0xE000 (L2 path)
    elif case == "signed_zero":
        b = np.array([0x0000, 0x8000] * 50_001, np.uint16)
    elif case == "tiny":
        b = np.array([0xBA45, 0xCB1F, 0xBA45], np.uint16)            # Fig. 3
    else:
        b = np.random.default_rng(2).integers(0x3000, 0x3100, (1 << 22) + 3).astype(np.uint16)
    W = torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16).cuda()
    counts = E.uniquify([W], E.Params(torch.bfloat16))
    torch.cuda.synchronize()
    assert np.array_equal(counts.cpu().numpy()[0], O.histogram(b).astype(np.int32))


@pytest.mark.parametrize("ctas", [1, 3])
@pytest.mark.parametrize("case", ["const_pos", "const_neg", "normal_plus_outliers", "two_signs_one_row"])
def test_uniquify_lane_private_folds(case, ctas):
    """F1's lane-private path: segments of several 2M-element chunks per CTA (folds of the 16-bit
    copies at their limit, 32 x 127 x 16 = 65024 increments of one counter), both counter halves,
    and patterns outside the sampled window (global atomics) -- bit-exact."""
    n = 5_000_003
    rng = np.random.default_rng(11)
    if case == "const_pos":
        b = np.full(n, 0x3F80, np.uint16)
    elif case == "const_neg":
        b = np.full(n, 0xBF80, np.uint16)
    elif case == "two_signs_one_row":
        b = np.where(rng.random(n) < 0.5, 0x3C12, 0xBC12).astype(np.uint16)
    else:
        w = (rng.standard_normal(n) * 0.02).astype(np.float32)
        b = (w.view(np.uint32) >> 16).astype(np.uint16)  # truncation: any bf16 pattern law will do
        idx = rng.integers(0, n, 5000)
        b[idx] = rng.choice(np.array([0x0000, 0x8000, 0x0001, 0x7F80, 0xFFC1, 0x7000, 0x1234], np.uint16), idx.size)
    W = torch.from_numpy(b.view(np.int16).copy()).view(torch.bfloat16).cuda()
    old = E.set_max_ctas(ctas)
    try:
        counts = E.uniquify([W], E.Params(torch.bfloat16))
        torch.cuda.synchronize()
    finally:
        E.set_max_ctas(old)
    assert np.array_equal(counts.cpu().numpy()[0], O.histogram(b).astype(np.int32))


@pytest.mark.parametrize("dtype,bits", [(torch.bfloat16, 3), (torch.float16, 4), (torch.bfloat16, 6)])
def test_nonfinite_patterns_flagged_and_excluded(dtype, bits):
    """NaN/Inf weights: counted, excluded from clustering, W~ and dW NaN (R10) -- for bf16 and fp16
    (different non-finite pattern blocks) and for the warp-per-row kernels (k = 64)."""
    n = 100_000
    W = synth.normal_tensor(n, 1.0, dtype, 21)
    bad = torch.tensor([5, 77, 1000, 99_999])
    W[bad] = torch.tensor([float("nan"), float("inf"), -float("inf"), float("nan")], dtype=dtype)
    G = synth.normal_tensor(n, 1e-3, dtype, 22)
    C0 = synth.quantile_centroids(1 << bits, 1.0)
    p = E.Params(dtype, bits, 1e-3, 5)
    gpu = run_gpu([W], [G], [C0], p)
    wb = bits_of(W)
    ref = oracle_dense(wb, G.double().numpy(), C0, p)
    check_tensor(gpu, 0, wb, G.double().numpy(), ref, p)
    assert gpu["nonfinite"][0] == 4


def test_eps_mode_iteration_count():
    # eps stop is "parity unpinned" (R4): check the GPU stops where the oracle does when no near-tie
    n = 200_000
    W = synth.normal_tensor(n, 1.0, torch.bfloat16, 31)
    G = synth.normal_tensor(n, 1e-3, torch.bfloat16, 32)
    C0 = synth.quantile_centroids(8, 1.0)
    wb = bits_of(W)
    w = O.decode16(wb, O.BF16)
    full, _, _ = O.dkm_forward(w, C0, 1e-3, 60)
    d = np.max(np.abs(np.diff(full, axis=0)), axis=1)
    eps = float(np.sqrt(d[10] * d[11]))          # between two iterations, far from either delta
    assert min(abs(d - eps)) > 1e-9 * np.max(np.abs(full))
    p = E.Params(torch.bfloat16, 3, 1e-3, 60, eps)
    gpu = run_gpu([W], [G], [C0], p)
    ref = oracle_dense(wb, G.double().numpy(), C0, p)
    check_tensor(gpu, 0, wb, G.double().numpy(), ref, p)


def test_eps_mode_pinned_to_lloyd():
    """The GPU's eps stop (R4) on the exact-Lloyd data of tests/test_oracle.py::test_eps_stop_pinned_to_lloyd:
    at tau = 1e-9 every delta is an exact dyadic number (69/8, 7, 5/2, 3/2, 5/4, 0), so the iteration count
    for eps equal to, or just below, a delta is fixed by textbook Lloyd -- and must match the oracle's."""
    from fractions import Fraction
    w = torch.tensor([25, 9, 22, 16, 25, 14, 21, 17], dtype=torch.bfloat16)
    deltas = [Fraction(69, 8), Fraction(7), Fraction(5, 2), Fraction(3, 2), Fraction(5, 4), Fraction(0)]
    for eps in [float(d) for d in deltas[:5]] + [float(np.nextafter(float(d), 0.0)) for d in deltas[:5]] + [1e-300]:
        T_exp = next(t + 1 for t, d in enumerate(deltas) if d <= Fraction(eps))
        p = E.Params(torch.bfloat16, 1, 1e-9, 10, eps)
        gpu = run_gpu([w], [torch.ones(8, dtype=torch.bfloat16)], [[2.0, 10.0]], p)
        assert gpu["iters"][0] == T_exp, (eps, gpu["iters"][0], T_exp)
        ref = oracle_dense(bits_of(w), np.ones(8), [2.0, 10.0], p)
        assert ref["T"] == T_exp
        np.testing.assert_array_equal(gpu["ctraj"][0][: T_exp + 1], ref["Ct"])


def test_autograd_function_matches_oracle():
    n = 65_537
    W = synth.normal_tensor(n, 1.0, torch.bfloat16, 41).cuda().requires_grad_()
    C0 = torch.tensor(synth.quantile_centroids(4, 1.0), device="cuda", requires_grad=True)
    Wt = E.edkm(W, C0, bits=2, tau=1e-2, max_iter=3)
    G = synth.normal_tensor(n, 1e-3, torch.bfloat16, 42).cuda()
    Wt.backward(G)
    ref = oracle_dense(bits_of(W), G.double().cpu().numpy(), C0.detach().cpu().numpy(), E.Params(torch.bfloat16, 2, 1e-2, 3))
    assert np.all(np.abs(as16_values(Wt) - ref["Wt"]) <= ulp16(ref["Wt"], torch.bfloat16))
    assert normwise(C0.grad.cpu().numpy(), ref["dC"]) <= TOL
    dw = as16_values(W.grad)
    assert np.all(np.abs(dw - ref["dW"]) <= ulp16(ref["dW"], torch.bfloat16) + TOL * np.max(np.abs(ref["dW"])))


@pytest.mark.parametrize("dtype,tol", [(torch.float64, 1e-9), (torch.float32, 5e-3)])
def test_dense_baseline_computes_the_oracle(dtype, tol):
    """tools/dense_baseline.py (the dense |W|x|C| map of P:39 under torch autograd)
    computes the oracle's W~, dW and dC_0 on CFG1: to 1e-9 with an fp64 map; with the fp32 map the
    paper's PyTorch path would use, within 5e-3 (all-fp32 DKM loses ~1e-5..1e-3 here, DESIGN R7)."""
    from tools.dense_baseline import dense_step
    wl = synth.workload("cfg1")
    W = synth.weights(wl, 0)
    G = synth.grads(wl, 0)
    C0 = synth.quantile_centroids(wl.k, wl.sigma)
    Wt, dW, dC = dense_step(W.cuda(), G.cuda(), np.float32(C0).astype(np.float64), wl.tau, wl.max_iter, dtype)
    ref = oracle_dense(bits_of(W), G.double().numpy(), C0, E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter))
    assert normwise(Wt.double().cpu().numpy(), ref["Wt"]) <= tol
    assert normwise(dW.double().cpu().numpy(), ref["dW"]) <= tol
    assert normwise(dC.double().cpu().numpy(), ref["dC"]) <= tol


def test_launch_counts_are_native():
    W = synth.normal_tensor(10_000, 1.0, torch.bfloat16, 51).cuda()
    p = E.Params(torch.bfloat16, 3, 1e-3, 2)
    E.uniquify([W], p)
    assert E.last_launch_count() == 1


def test_host_pipeline_matches_oracle():
    """pipeline.HostPipeline: host-resident W, G through three overlapped streams, per tensor group."""
    from paper_2309_00964_b200.pipeline import HostPipeline
    sizes = [50_000, 7, 120_001, 65_536, 3_000, 90_000]
    p = E.Params(torch.bfloat16, 2, 1e-2, 3)
    Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 900 + i) for i, n in enumerate(sizes)]
    Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 950 + i) for i, n in enumerate(sizes)]
    C0 = torch.tensor([synth.data_quantile_centroids(w, 4) for w in Ws], dtype=torch.float32, device="cuda")
    hW = [w.pin_memory() for w in Ws]
    hG = [g.pin_memory() for g in Gs]
    hWt = [torch.empty_like(w).pin_memory() for w in Ws]
    hdW = [torch.empty_like(w).pin_memory() for w in Ws]
    pipe = HostPipeline(sizes, p, "cuda", n_groups=3)
    assert len(pipe.groups) == 3 and sorted(sum(pipe.groups, [])) == list(range(len(sizes)))
    dC = pipe.step(hW, hG, C0, hWt, hdW)
    torch.cuda.synchronize()
    dC = torch.cat([d.cpu() for d in dC]).numpy()
    for t in range(len(sizes)):
        ref = oracle_dense(bits_of(Ws[t]), Gs[t].double().numpy(), C0[t].cpu().numpy(), p)
        assert np.min(ref["St"]) >= DEAD * sizes[t]  # data-quantile C_0: no dead cluster, all compared
        assert np.all(np.abs(as16_values(hWt[t]) - ref["Wt"]) <= ulp16(ref["Wt"], torch.bfloat16)
                      + TOL * np.max(np.abs(ref["Wt"])))
        lim = ulp16(ref["dW"], torch.bfloat16) + TOL * np.max(np.abs(ref["dW"]))
        assert np.all(np.abs(as16_values(hdW[t]) - ref["dW"]) <= lim)
        assert np.max(np.abs(dC[t] - ref["dC"])) <= TOL * np.max(np.abs(ref["dC"])) + 1e-37
