"""Dense-map DKM on B200 with torch autograd -- the design eDKM starts from (PAPER.md P:39 S2: an
|W| x |C| attention map per iteration, kept for backward), run on the same GPU for comparison
(SURVEY.md S8(f) NEXT #4).  Not part of the product path: plain torch ops (library kernels).

For each weight matrix of the workload it times forward (T unrolled iterations + W~) and
backward (autograd) and records the peak memory -- the quantities of the paper's Table 2
(one attention layer of LLaMA-7B on A100 + CPU offload, "8.67 s" dense vs "14.9 s"
eDKM; memory in MiB) -- and, in the same run, the same tensors through the table path
(edkm.Plan, the C ABI), so one JSON line carries both.  tests/test_gpu_parity.py checks that
dkm_dense computes the oracle's W~, dW and dC_0 (fp64 map) on CFG1.
Usage:  python tools/dense_baseline.py [--workload cfg2] [--steps 3] [--dtype fp32|fp64]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_00964_b200 import synth  # noqa: E402

TABLE2 = ("PAPER.md Table 2 (P:97-107; S3.2 P:134-136; hardware P:87: 8x A100-80GB node): one attention layer "
          "of the LLaMA-7B decoder, 3-bit, forward+backward: dense DKM 1600 MB / 8.67 s; marshaling 544 MB / 8.97 s; "
          "+ sharding 68 MB / 9.5 s; + uniquification 97 MB / 15.9 s; all three (eDKM) 12 MB / 14.9 s, i.e. "
          "129.9x less memory at 1.7x the runtime")


def dkm_dense(W, C0, tau, T):
    """W~ = attn(W, C_T) . C_T with T soft k-means updates, every step on the dense |W| x k map (R1-R3;
    softmax subtracts the row max of the logits, as the oracle subtracts min_l d)."""
    w = W.reshape(-1, 1)
    C = C0
    for _ in range(T):
        A = torch.softmax(-(w - C[None, :]) ** 2 / tau, dim=1)     # |W| x |C| map
        C = (A * w).sum(0) / A.sum(0)
    A = torch.softmax(-(w - C[None, :]) ** 2 / tau, dim=1)
    return (A @ C).reshape(W.shape)


def dense_step(W16, G, C0, tau, T, dtype=torch.float32):
    """One fwd+bwd of dkm_dense in `dtype`: returns (W~, dW, dC_0)."""
    W = W16.to(dtype).requires_grad_()
    C = torch.as_tensor(C0, dtype=dtype, device=W16.device).clone().requires_grad_()
    Wt = dkm_dense(W, C, tau, T)
    Wt.backward(G.to(dtype))
    return Wt.detach(), W.grad, C.grad


def time_table_path(Ws, Gs, wl, steps):
    """The same tensors through edkm.Plan, one tensor per call like the dense loop (ms per tensor, peak)."""
    from paper_2309_00964_b200 import edkm as E
    p = E.Params(wl.wdtype, wl.bits, wl.tau, wl.max_iter)
    out = []
    for W, G in zip(Ws, Gs):
        torch.cuda.reset_peak_memory_stats()
        base = torch.cuda.memory_allocated()
        plan = E.Plan([W.numel()], p, W.device)
        C0 = torch.tensor([synth.quantile_centroids(wl.k, wl.sigma)], dtype=torch.float32, device=W.device)
        Wt, dW = [torch.empty_like(W)], [torch.empty_like(W)]
        times = []
        for s in range(steps + 1):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            plan.step([W], [G], C0, Wt, dW)
            e1.record()
            torch.cuda.synchronize()
            if s:
                times.append(e0.elapsed_time(e1))
        out.append({"ms_fwd_bwd": sorted(times)[len(times) // 2],
                    "extra_peak_mem_GiB": (torch.cuda.max_memory_allocated() - base) / 2**30})
        del plan
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--dtype", default="fp32", choices=["fp32", "fp64"])
    a = ap.parse_args()
    wl = synth.workload(a.workload)
    dt = torch.float32 if a.dtype == "fp32" else torch.float64
    dev = torch.device("cuda")
    res, Ws, Gs = [], [], []
    for t, (name, r, c) in enumerate(wl.shapes):
        W16 = synth.weights(wl, t, dev)
        G = synth.grads(wl, t, dev)
        Ws.append(W16)
        Gs.append(G)
        C0 = synth.quantile_centroids(wl.k, wl.sigma)
        times = []
        for s in range(a.steps + 1):
            torch.cuda.reset_peak_memory_stats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            dense_step(W16.reshape(r, c), G.reshape(r, c), C0, wl.tau, wl.max_iter, dt)
            e1.record()
            torch.cuda.synchronize()
            if s:
                times.append(e0.elapsed_time(e1))
        ms = sorted(times)[len(times) // 2]
        res.append({"tensor": name, "weights": r * c, "ms_fwd_bwd": ms,
                    "peak_mem_GiB": torch.cuda.max_memory_allocated() / 2**30})
    tab = time_table_path(Ws, Gs, wl, a.steps)
    tot_w = sum(x["weights"] for x in res)
    d_ms = sum(x["ms_fwd_bwd"] for x in res)
    t_ms = sum(x["ms_fwd_bwd"] for x in tab)
    print(json.dumps({
        "workload": wl.name, "weights": tot_w,
        "dense": {"impl": f"torch autograd, {a.dtype} |W|x|C| map per iteration (P:39)", "ms_fwd_bwd": d_ms,
                  "weights_per_s": tot_w / (d_ms / 1e3), "peak_mem_GiB_max": max(x["peak_mem_GiB"] for x in res),
                  "per_tensor": res},
        "table_path": {"impl": "libedkm.so via edkm.Plan, one tensor per call (uniquified table, P:77)",
                       "ms_fwd_bwd": t_ms, "weights_per_s": tot_w / (t_ms / 1e3),
                       "extra_peak_mem_GiB_max": max(x["extra_peak_mem_GiB"] for x in tab), "per_tensor": tab},
        "speedup": d_ms / t_ms, "paper_table2": TABLE2}))


if __name__ == "__main__":
    main()
