"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

CFG3 (full LLaMA-7B: 226 tensors, 6,738,149,376 bf16 weights, k=8, tau=1e-5, T=5), CFG2
(one decoder layer), CFG4 (the CFG3 shapes in fp16, k=16 and k=4, T=30) and CFG5 (LLaMA-13B,
282 tensors) run through one edkm.Plan exactly as bench.py does (16-bit W~ and dW).
Checked against the oracle on sampled tensors, in the attention-table form that
tests/test_oracle.py pins to the dense definition: exact counts (bit-exact), C_T,
the W~ table of every populated pattern, dC_0, and 200,000 sampled elements of W~ and dW
computed one by one from the oracle's (phi, psi).  Every tensor: counts bit-exact against
the oracle's histogram and no non-finite weights.
"""
import numpy as np
import pytest
import torch

from oracle import oracle as O
from paper_2309_00964_b200 import edkm as E
from paper_2309_00964_b200 import synth

pytestmark = pytest.mark.gpu
TOL = 1e-5


def ulp16(x, dtype):
    """One unit in the last place of the 16-bit output format at |x| (the rounding of W~ / dW)."""
    mant, tiny = (7, 2.0 ** -133) if dtype == torch.bfloat16 else (10, 2.0 ** -24)
    t = torch.from_numpy(np.abs(x)).to(dtype).to(torch.float64).numpy()
    return np.maximum(2.0 ** (np.floor(np.log2(np.maximum(t, 1e-300))) - mant), tiny)


def run(name, sample):
    wl = synth.workload(name)
    dev = torch.device("cuda")
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
    Ws = [synth.weights(wl, t, dev) for t in range(len(wl.shapes))]
    Gs = [synth.grads(wl, t, dev) for t in range(len(wl.shapes))]
    C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)] * len(Ws), dtype=torch.float32, device=dev)
    plan = E.Plan([w.numel() for w in Ws], p, dev)
    Wt = [torch.empty_like(w) for w in Ws]
    dW = [torch.empty_like(w) for w in Ws]
    plan.step(Ws, Gs, C0, Wt, dW)
    torch.cuda.synchronize()
    nonfin, iters = E.read_status(plan.saved, plan.nt, p)
    counts = plan.counts.cpu().numpy()
    assert set(iters) == {wl.max_iter} and not any(nonfin)
    # counts of EVERY tensor bit-exact against the oracle's histogram (F1 is integer work)
    hist = {}
    for t in range(len(Ws)):
        c = O.histogram(Ws[t].view(torch.int16).cpu().numpy().view(np.uint16))
        assert np.array_equal(counts[t], c.astype(np.int32)), wl.shapes[t][0]
        if t in sample:
            hist[t] = c
    rng = np.random.default_rng(7)
    for t in sample:
        bits = Ws[t].view(torch.int16).cpu().numpy().view(np.uint16)
        G = Gs[t].double().cpu().numpy()
        c = hist[t]
        u = np.nonzero(c)[0]
        v = O.decode16(u.astype(np.uint16), O.BF16 if wl.wdtype == torch.bfloat16 else O.FP16)
        C0t = np.float32(C0[t].cpu().numpy()).astype(np.float64)
        Ct, St, _ = O.dkm_forward(v, C0t, wl.tau, wl.max_iter, mult=c[u])
        assert np.min(St) >= 1e-6 * bits.size
        CT = Ct[-1]
        gC = plan.C_out[t].cpu().numpy()
        assert np.max(np.abs(gC - CT)) <= TOL * np.max(np.abs(CT)), wl.shapes[t][0]
        tab = O.reconstruct(v, CT, wl.tau)
        gtab = plan.table[t].cpu().numpy()[u]
        assert np.max(np.abs(gtab - tab)) <= TOL * np.max(np.abs(tab))
        pos = np.searchsorted(u, bits)
        B = np.bincount(pos, weights=G, minlength=u.size)
        phi, psi, dC = O.dkm_backward_table(v, c[u].astype(np.float64), B, Ct, St, wl.tau)
        gdC = plan.dC0[t].cpu().numpy()
        assert np.max(np.abs(gdC - dC)) <= TOL * np.max(np.abs(dC)), (wl.shapes[t][0], gdC, dC)
        idx = rng.integers(0, bits.size, 200_000)
        wt_ref = tab[pos[idx]]
        wt_gpu = Wt[t].view(-1)[torch.from_numpy(idx).to(dev)].double().cpu().numpy()
        assert np.all(np.abs(wt_gpu - wt_ref) <= ulp16(wt_ref, wl.wdtype))
        dw_all = G * phi[pos] + psi[pos]
        dw_ref = dw_all[idx]
        dw_gpu = dW[t].view(-1)[torch.from_numpy(idx).to(dev)].double().cpu().numpy()
        assert np.all(np.abs(dw_gpu - dw_ref) <= ulp16(dw_ref, wl.wdtype) + TOL * np.max(np.abs(dw_all)))


def test_cfg2_decoder_layer_all_tensors():
    run("cfg2", sample=range(7))


@pytest.mark.slow
def test_cfg3_llama7b_sampled_tensors():
    wl = synth.workload("cfg3")
    names = [s[0] for s in wl.shapes]
    sample = [0, names.index("layers.0.q_proj"), names.index("layers.17.gate_proj"),
              names.index("layers.31.down_proj"), len(names) - 1]
    run("cfg3", sample=sample)


def _sample(name):
    names = [s[0] for s in synth.workload(name).shapes]
    return [0, names.index("layers.0.q_proj"), names.index("layers.17.gate_proj"),
            names.index("layers.31.down_proj"), len(names) - 1]


@pytest.mark.slow
@pytest.mark.parametrize("name", ["cfg4", "cfg4_b2"])
def test_cfg4_fp16_sweep_sampled_tensors(name):
    run(name, sample=_sample(name))


@pytest.mark.slow
def test_cfg5_llama13b_sampled_tensors():
    run("cfg5", sample=_sample("cfg5"))
