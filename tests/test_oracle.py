"""Pins of the CPU oracle (oracle/) against what the paper and mathematics fix.

Nothing here compares the oracle with itself or with the CUDA path.  Each test
names the passage (PAPER.md line, "P:<n>") or DESIGN.md reading it checks, and
is chosen so that a plausible slip in the oracle (a dropped term, a sign, a
transposed index, a wrong power of tau) fails at least one of them:

  decode          vs numpy float16 / torch bfloat16 for all 65,536 patterns
  histogram       brute force; Fig. 3 worked example
  attention       rows sum to 1; equal patterns give equal rows
  forward         tau->0 == textbook Lloyd k-means; tau->inf and k=1 closed
                  forms; exact scale law; permutation invariance; golden case
  backward        torch fp64 autograd of an independently written graph;
                  central finite differences; k=1 / tau->inf closed forms
  table form      attention table + index list == dense map
  hard assign     brute-force argmin, lowest index on ties (R9)
  non-finite      NaN/Inf weights excluded from clustering (R10)
  eps stop        self-consistency only ("parity unpinned", R4)
"""
import json
import os

import numpy as np
import pytest
import torch

from oracle import oracle as O

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def bf16_bits(x: np.ndarray) -> np.ndarray:
    return torch.tensor(x, dtype=torch.float32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def normwise(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


# --------------------------------------------------------------------------- decode
def test_decode_all_patterns_match_library_formats():
    u = np.arange(65536, dtype=np.uint16)
    ref16 = u.view(np.float16).astype(np.float64)
    refbf = torch.from_numpy(u.view(np.int16).copy()).view(torch.bfloat16).to(torch.float64).numpy()
    for dt, ref in ((O.FP16, ref16), (O.BF16, refbf)):
        got = O.decode16(u, dt)
        nan = np.isnan(ref)
        assert np.array_equal(np.isnan(got), nan)
        assert np.array_equal(got[~nan], ref[~nan])
        # signed zeros are distinct patterns with the same value (R10)
        assert np.array_equal(np.signbit(got[~nan]), np.signbit(ref[~nan]))


def test_decode_fig3_patterns():
    # P:69 Fig. 3 uses the patterns BA45 and CB1F; their exact bf16/fp16 values
    got_bf = O.decode16(np.array([0xBA45, 0xCB1F], np.uint16), O.BF16)
    got_h = O.decode16(np.array([0xBA45, 0xCB1F], np.uint16), O.FP16)
    assert got_bf[0] == -(1 + 0x45 / 128) * 2.0 ** (0x74 - 127)
    assert got_bf[1] == -(1 + 0x1F / 128) * 2.0 ** (0x96 - 127)
    assert got_h[0] == -(1 + 0x245 / 1024) * 2.0 ** (0x0E - 15)
    assert got_h[1] == -(1 + 0x31F / 1024) * 2.0 ** (0x12 - 15)


# --------------------------------------------------------------------------- histogram (Fig. 3)
def test_histogram_fig3_worked_example():
    g = json.load(open(os.path.join(GOLD, "fig3_uniquify.json")))
    bits = np.array([int(b, 16) for b in g["bits"]], np.uint16)
    c = O.histogram(bits)
    exp = {int(k, 16): v for k, v in g["expected_counts"].items()}
    assert {int(u): int(c[u]) for u in np.nonzero(c)[0]} == exp
    assert c.sum() == bits.size
    # the index list is the pattern itself: nothing to compute, the offsets are the bits
    assert [int(b) for b in bits] == [int(b, 16) for b in g["expected_index_list"]]
    v = O.decode16(bits, O.BF16)
    A = O.attention(v, [-1e-3, 0.0, 2e-3, -2e7], 1e-6)
    for i, j in g["identical_rows"]:
        assert np.array_equal(A[i], A[j])          # same bits => same attention


@pytest.mark.parametrize("seed", [0, 1])
def test_histogram_brute_force(seed):
    rng = np.random.default_rng(seed)
    n = 5000
    bits = np.concatenate([rng.integers(0, 65536, n), np.full(300, 0x3F80), [0, 0x8000, 0xFFFF]]).astype(np.uint16)
    rng.shuffle(bits)
    c = O.histogram(bits)
    ref = {}
    for b in bits.tolist():
        ref[b] = ref.get(b, 0) + 1
    assert all(int(c[u]) == ref.get(u, 0) for u in range(65536))
    assert int(c.sum()) == bits.size
    assert O.histogram(np.zeros(0, np.uint16)).sum() == 0


# --------------------------------------------------------------------------- attention (north star, R1)
def test_attention_rows_sum_to_one_and_are_softmax_of_neg_sq_distance():
    rng = np.random.default_rng(3)
    w = rng.normal(0, 1, 300)
    C = np.sort(rng.normal(0, 1, 8))
    for tau in (1e-4, 1e-2, 1.0, 1e3):
        A = O.attention(w, C, tau)
        assert np.all(A >= 0)
        assert np.max(np.abs(A.sum(1) - 1)) < 4e-16 * 8
        # ratios are exp(-(d_a - d_b)/tau) where both are representable
        i = 5
        d = (w[i] - C) ** 2
        a, b = np.argsort(d)[:2]
        if (d[b] - d[a]) / tau < 600:
            assert np.isclose(A[i, b] / A[i, a], np.exp(-(d[b] - d[a]) / tau), rtol=1e-12)
    # nearest centroid gets the largest weight (distance is squared Euclidean, R1)
    A = O.attention(w, C, 1e-2)
    assert np.array_equal(np.argmax(A, 1), np.argmin((w[:, None] - C[None]) ** 2, 1))


# --------------------------------------------------------------------------- forward
def lloyd(w, C0, T):
    """Textbook Lloyd k-means: nearest centroid (lowest index on ties), then means; empty cluster keeps C."""
    C = np.array(C0, np.float64)
    traj = [C.copy()]
    for _ in range(T):
        a = np.argmin(np.abs(w[:, None] - C[None, :]), axis=1)
        Cn = C.copy()
        for j in range(C.size):
            if np.any(a == j):
                Cn[j] = np.mean(w[a == j])
        C = Cn
        traj.append(C.copy())
    return np.array(traj)


@pytest.mark.parametrize("k,T", [(2, 3), (4, 5), (8, 5), (16, 4)])
def test_forward_tau_to_zero_is_lloyd_kmeans(k, T):
    rng = np.random.default_rng(k)
    w = rng.normal(0, 1, 2000)
    C0 = np.sort(rng.normal(0, 1, k))
    Ct, St, Tout = O.dkm_forward(w, C0, 1e-9, T)
    assert Tout == T
    np.testing.assert_allclose(Ct, lloyd(w, C0, T), rtol=1e-13, atol=1e-15)
    # S_t counts the members of each cluster
    a = np.argmin(np.abs(w[:, None] - Ct[T - 1][None, :]), axis=1)
    np.testing.assert_array_equal(St[T - 1], np.bincount(a, minlength=k))


def test_forward_tau_to_infinity_closed_form():
    rng = np.random.default_rng(5)
    w = rng.normal(0.3, 1, 1000)
    G = rng.normal(0, 1, 1000)
    C0 = np.array([-1.0, -0.2, 0.4, 2.0])
    Ct, St, T = O.dkm_forward(w, C0, 1e30, 3)
    assert np.allclose(Ct[1:], w.mean(), rtol=0, atol=1e-14)
    assert np.allclose(St, w.size / 4, rtol=1e-14)
    Wt = O.reconstruct(w, Ct[-1], 1e30)
    assert np.allclose(Wt, w.mean(), atol=1e-14)
    dW, dC = O.dkm_backward(w, G, Ct, St, 1e30)
    assert np.allclose(dW, G.sum() / w.size, atol=1e-12)
    assert np.max(np.abs(dC)) < 1e-20


@pytest.mark.parametrize("T", [0, 1, 4])
def test_single_centroid_closed_form(T):
    rng = np.random.default_rng(7)
    w = rng.normal(0, 2, 777)
    G = rng.normal(0, 1, 777)
    Ct, St, Tout = O.dkm_forward(w, [0.5], 0.37, T)
    Wt = O.reconstruct(w, Ct[-1], 0.37)
    dW, dC = O.dkm_backward(w, G, Ct, St, 0.37)
    if T == 0:
        assert np.all(Wt == 0.5) and np.all(dW == 0) and np.isclose(dC[0], G.sum(), rtol=1e-13)
    else:
        assert np.allclose(Ct[1:, 0], w.mean(), rtol=1e-13)
        assert np.all(St == w.size)
        assert np.allclose(Wt, w.mean(), rtol=1e-13)
        assert np.allclose(dW, G.sum() / w.size, rtol=1e-11)
        assert abs(dC[0]) < 1e-12


def test_scale_law_is_exact():
    # (W, C0, tau) -> (sW, sC0, s^2 tau) gives (sC, sW~) and unchanged dW, dC0, bit for bit for s = 2^m
    rng = np.random.default_rng(11)
    w = rng.normal(0, 1, 500)
    G = rng.normal(0, 1, 500)
    C0 = np.sort(rng.normal(0, 1, 8))
    tau, T, s = 3e-2, 4, 4.0
    Ct, St, _ = O.dkm_forward(w, C0, tau, T, nthreads=1)
    Ct2, St2, _ = O.dkm_forward(s * w, s * C0, s * s * tau, T, nthreads=1)
    assert np.array_equal(Ct2, s * Ct) and np.array_equal(St2, St)
    assert np.array_equal(O.reconstruct(s * w, Ct2[-1], s * s * tau), s * O.reconstruct(w, Ct[-1], tau))
    dW, dC = O.dkm_backward(w, G, Ct, St, tau, nthreads=1)
    dW2, dC2 = O.dkm_backward(s * w, G, Ct2, St2, s * s * tau, nthreads=1)
    assert np.array_equal(dW2, dW) and np.array_equal(dC2, dC)


def test_permutation_invariance():
    rng = np.random.default_rng(12)
    w = rng.normal(0, 1, 1500)
    G = rng.normal(0, 1, 1500)
    C0 = np.sort(rng.normal(0, 1, 4))
    p = rng.permutation(w.size)
    Ct, St, _ = O.dkm_forward(w, C0, 0.05, 3)
    Ctp, Stp, _ = O.dkm_forward(w[p], C0, 0.05, 3)
    np.testing.assert_allclose(Ctp, Ct, rtol=1e-13)
    dW, dC = O.dkm_backward(w, G, Ct, St, 0.05)
    dWp, dCp = O.dkm_backward(w[p], G[p], Ctp, Stp, 0.05)
    np.testing.assert_allclose(dWp, dW[p], rtol=1e-10, atol=1e-12)
    np.testing.assert_allclose(dCp, dC, rtol=1e-10)


def test_thread_count_does_not_change_results_beyond_rounding():
    rng = np.random.default_rng(13)
    w = rng.normal(0, 1, 20000)
    C0 = np.sort(rng.normal(0, 1, 8))
    a = O.dkm_forward(w, C0, 1e-2, 5, nthreads=1)[0]
    b = O.dkm_forward(w, C0, 1e-2, 5, nthreads=7)[0]
    np.testing.assert_allclose(a, b, rtol=1e-13)


# --------------------------------------------------------------------------- golden tiny case
def test_golden_tiny_case():
    g = json.load(open(os.path.join(GOLD, "survey_tiny_case.json")))
    bits = np.array([int(b, 16) for b in g["w_bf16_bits"]], np.uint16)
    w = O.decode16(bits, O.BF16)
    assert np.array_equal(w, np.array(g["w"]))
    rt = g["printed_digits_rtol"]
    Ct, St, T = O.dkm_forward(w, g["C0"], g["tau"], g["T"])
    np.testing.assert_allclose(Ct, np.array(g["C_traj"]), rtol=rt, atol=1e-12)
    Wt = O.reconstruct(w, Ct[-1], g["tau"])
    np.testing.assert_allclose(Wt, g["W_tilde"], rtol=rt, atol=1e-12)
    dW, dC = O.dkm_backward(w, g["G"], Ct, St, g["tau"])
    np.testing.assert_allclose(dW, g["dW"], rtol=rt, atol=1e-12)
    np.testing.assert_allclose(dC, g["dC0"], rtol=rt, atol=1e-12)
    idx = O.hard_assign(w, Ct[-1].astype(np.float32))
    assert idx.tolist() == g["hard_idx_vs_C3"]


# --------------------------------------------------------------------------- backward
def torch_dkm(w, G, C0, tau, T):
    """DKM written independently with torch ops; autograd derives the backward."""
    wt = torch.tensor(w, dtype=torch.float64, requires_grad=True)
    C0t = torch.tensor(C0, dtype=torch.float64, requires_grad=True)
    C = C0t
    for _ in range(T):
        A = torch.softmax(-((wt[:, None] - C[None, :]) ** 2) / tau, dim=1)
        C = (A * wt[:, None]).sum(0) / A.sum(0)
    A = torch.softmax(-((wt[:, None] - C[None, :]) ** 2) / tau, dim=1)
    Wt = A @ C
    (Wt * torch.tensor(G, dtype=torch.float64)).sum().backward()
    return C.detach().numpy(), Wt.detach().numpy(), wt.grad.numpy(), C0t.grad.numpy()


@pytest.mark.parametrize("k,tau,T", [(2, 0.3, 0), (4, 0.05, 1), (8, 1e-2, 3), (8, 1e-3, 5), (16, 3e-3, 2)])
def test_backward_matches_torch_autograd(k, tau, T):
    rng = np.random.default_rng(100 + k)
    n = 300
    w = rng.normal(0, 1, n)
    G = rng.normal(0, 1, n)
    C0 = np.quantile(w, (np.arange(k) + 0.5) / k)
    Ct, St, _ = O.dkm_forward(w, C0, tau, T)
    Wt = O.reconstruct(w, Ct[-1], tau)
    dW, dC = O.dkm_backward(w, G, Ct, St, tau)
    C_ref, Wt_ref, dW_ref, dC_ref = torch_dkm(w, G, C0, tau, T)
    assert normwise(Ct[-1], C_ref) < 1e-13
    assert normwise(Wt, Wt_ref) < 1e-13
    assert normwise(dW, dW_ref) < 1e-10
    assert normwise(dC, dC_ref) < 1e-10


@pytest.mark.parametrize("k,T", [(2, 0), (2, 2), (4, 3), (8, 4)])
def test_backward_central_finite_differences(k, T):
    rng = np.random.default_rng(200 + k + T)
    n, tau, h = 16, 0.05, 1e-6
    w = rng.normal(0, 0.5, n)
    G = rng.normal(0, 1, n)
    C0 = np.sort(rng.normal(0, 0.5, k))

    def loss(w_, C0_):
        Ct_, _, _ = O.dkm_forward(w_, C0_, tau, T, nthreads=1)
        return float(np.dot(G, O.reconstruct(w_, Ct_[-1], tau)))

    Ct, St, _ = O.dkm_forward(w, C0, tau, T, nthreads=1)
    dW, dC = O.dkm_backward(w, G, Ct, St, tau, nthreads=1)
    fdW = np.array([(loss(w + h * e, C0) - loss(w - h * e, C0)) / (2 * h) for e in np.eye(n)])
    fdC = np.array([(loss(w, C0 + h * e) - loss(w, C0 - h * e)) / (2 * h) for e in np.eye(k)])
    assert normwise(dW, fdW) < 1e-6
    assert normwise(dC, fdC) < 1e-6


# --------------------------------------------------------------------------- table form
@pytest.mark.parametrize("k,tau,T", [(8, 1e-3, 5), (4, 1e-2, 2), (16, 5e-3, 3)])
def test_attention_table_form_equals_dense_map(k, tau, T):
    rng = np.random.default_rng(300 + k)
    n = 40000
    bits = bf16_bits(rng.normal(0, 1, n))          # many repeated 16-bit patterns
    w = O.decode16(bits, O.BF16)
    G = rng.normal(0, 1, n)
    C0 = np.quantile(w, (np.arange(k) + 0.5) / k)
    u, inv, cnt = np.unique(bits, return_inverse=True, return_counts=True)
    assert u.size < n / 4
    v = O.decode16(u, O.BF16)
    Ct, St, _ = O.dkm_forward(w, C0, tau, T)
    Ctu, Stu, _ = O.dkm_forward(v, C0, tau, T, mult=cnt)
    assert normwise(Ctu, Ct) < 1e-13 and normwise(Stu, St) < 1e-13
    Wt = O.reconstruct(w, Ct[-1], tau)
    assert np.array_equal(O.reconstruct(v, Ct[-1], tau)[inv], Wt)
    dW, dC = O.dkm_backward(w, G, Ct, St, tau)
    B = np.bincount(inv, weights=G, minlength=u.size)
    phi, psi, dCu = O.dkm_backward_table(v, cnt, B, Ct, St, tau)
    assert normwise(G * phi[inv] + psi[inv], dW) < 1e-11
    assert normwise(dCu, dC) < 1e-11
    # gamma_T is linear in B: sharding the weights into two halves and summing the
    # per-half gamma_T (T = 0 call returns gamma_T) reproduces the unsharded backward
    half = n // 2
    g_parts = []
    for sl in (slice(0, half), slice(half, n)):
        Bp = np.bincount(inv[sl], weights=G[sl], minlength=u.size)
        g_parts.append(O.dkm_backward_table(v, cnt, Bp, Ct[-1:], St[:0], tau)[2])
    phi2, psi2, dC2 = O.dkm_backward_table(v, cnt, None, Ct, St, tau, gammaT=g_parts[0] + g_parts[1])
    assert normwise(dC2, dC) < 1e-11 and normwise(G * phi2[inv] + psi2[inv], dW) < 1e-11
    # phi is the direct path: G-independent and non-negative, phi = (2/tau) Var_A(C)
    A = O.attention(v, Ct[-1], tau)
    var = (A * (Ct[-1][None] - (A @ Ct[-1])[:, None]) ** 2).sum(1)
    assert normwise(phi, 2 / tau * var) < 1e-10


# --------------------------------------------------------------------------- hard assignment (R9)
def test_hard_assign_brute_force_and_ties():
    rng = np.random.default_rng(400)
    C = np.sort(rng.normal(0, 1, 8)).astype(np.float32)
    w = np.concatenate([rng.normal(0, 1, 1000), (C[:-1].astype(np.float64) + C[1:]) / 2, C])
    idx = O.hard_assign(w, C)
    d = (w[:, None] - C.astype(np.float64)[None]) ** 2
    assert np.array_equal(idx, np.argmin(d, 1))          # numpy returns the first (lowest) index
    Cdup = np.array([0.5, -1.0, 0.5, 2.0], np.float32)   # duplicated centroid: lowest j wins
    assert O.hard_assign(np.array([0.5, 0.4, 1.9]), Cdup).tolist() == [0, 0, 3]


# --------------------------------------------------------------------------- non-finite patterns (R10)
def test_nonfinite_weights_are_excluded():
    rng = np.random.default_rng(500)
    w = rng.normal(0, 1, 1000)
    G = rng.normal(0, 1, 1000)
    bad = np.array([3, 50, 999])
    wn = w.copy()
    wn[bad] = [np.nan, np.inf, -np.inf]
    keep = np.setdiff1d(np.arange(w.size), bad)
    C0 = [-1.0, 0.0, 1.0, 2.0]
    Ct, St, _ = O.dkm_forward(wn, C0, 0.02, 3)
    Ctk, Stk, _ = O.dkm_forward(w[keep], C0, 0.02, 3)
    np.testing.assert_allclose(Ct, Ctk, rtol=1e-14)
    Wt = O.reconstruct(wn, Ct[-1], 0.02)
    assert np.all(np.isnan(Wt[bad])) and np.all(np.isfinite(Wt[keep]))
    dW, dC = O.dkm_backward(wn, G, Ct, St, 0.02)
    dWk, dCk = O.dkm_backward(w[keep], G[keep], Ctk, Stk, 0.02)
    assert np.all(np.isnan(dW[bad]))
    np.testing.assert_allclose(dW[keep], dWk, rtol=1e-12, atol=1e-14)
    np.testing.assert_allclose(dC, dCk, rtol=1e-12)


# --------------------------------------------------------------------------- eps stop (R4, parity unpinned)
def test_eps_stop_self_consistent():
    rng = np.random.default_rng(600)
    w = rng.normal(0, 1, 3000)
    C0 = np.sort(rng.normal(0, 1, 8))
    full, _, _ = O.dkm_forward(w, C0, 1e-2, 60)
    deltas = np.max(np.abs(np.diff(full, axis=0)), axis=1)
    eps = float(deltas[15])
    T_expected = int(np.argmax(deltas <= eps)) + 1
    Ct, St, T = O.dkm_forward(w, C0, 1e-2, 60, eps=eps)
    assert T == T_expected <= 16
    np.testing.assert_array_equal(Ct, full[: T + 1])
    assert deltas[T - 1] <= eps and np.all(deltas[: T - 1] > eps)


def _lloyd_exact(w, C0, T):
    """Textbook Lloyd k-means in exact rational arithmetic (fractions), independent of the oracle."""
    from fractions import Fraction
    C = [Fraction(c) for c in C0]
    traj = [list(C)]
    for _ in range(T):
        a = []
        for x in w:
            d = [abs(Fraction(x) - c) for c in C]
            assert d.count(min(d)) == 1  # no ties: the assignment is unique
            a.append(d.index(min(d)))
        C = [sum(Fraction(x) for x, aj in zip(w, a) if aj == j) / max(1, a.count(j)) if j in a else C[j]
             for j in range(len(C))]
        traj.append(list(C))
    return traj


@pytest.mark.parametrize("max_iter", [10, 4])
def test_eps_stop_pinned_to_lloyd(max_iter):
    """R4 against an independent reference: at tau = 1e-9 the oracle IS Lloyd's k-means (pinned above),
    so an eps-stopped run must stop after the first update t whose max_j |C_t - C_{t-1}| <= eps, with the
    deltas taken from textbook Lloyd in exact arithmetic -- not from the oracle's own trajectory.  The
    data (integers, two clusters whose sizes make every mean dyadic) give exact fp64 deltas 69/8, 7, 5/2,
    3/2, 5/4, 0, so eps equal to a delta separates `<=` from `<`, and eps just below it from off-by-one."""
    w = np.array([25, 9, 22, 16, 25, 14, 21, 17], np.float64)
    C0 = np.array([2.0, 10.0])
    traj = _lloyd_exact(w.tolist(), C0.tolist(), 10)
    deltas = [max(abs(a - b) for a, b in zip(traj[t + 1], traj[t])) for t in range(10)]
    assert [str(d) for d in deltas[:6]] == ["69/8", "7", "5/2", "3/2", "5/4", "0"]

    def expected_T(eps):
        for t, d in enumerate(deltas[:max_iter]):
            if d <= eps:
                return t + 1
        return max_iter

    cases = [float(d) for d in deltas[:5]]                              # eps exactly a delta
    cases += [float(np.nextafter(float(d), 0.0)) for d in deltas[:5]]   # just below it
    cases += [1e-300, 100.0]
    from fractions import Fraction
    for eps in cases:
        Ct, St, T = O.dkm_forward(w, C0, 1e-9, max_iter, eps=eps)
        assert T == expected_T(Fraction(eps)), (eps, T)
        np.testing.assert_array_equal(Ct, np.array([[float(c) for c in C] for C in traj[: T + 1]]))
    # eps = 0 disables the test: exactly max_iter updates
    _, _, T = O.dkm_forward(w, C0, 1e-9, max_iter, eps=0.0)
    assert T == max_iter


def test_bad_arguments_are_rejected():
    with pytest.raises(ValueError):
        O.dkm_forward([0.0], [0.0], -1.0, 1)
    with pytest.raises(ValueError):
        O.dkm_forward([0.0], [0.0], 1.0, -1)
    with pytest.raises(ValueError):
        O.decode16(np.zeros(1, np.uint16), 7)
