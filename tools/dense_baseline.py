"""Dense-map DKM on B200 with torch autograd -- the design eDKM starts from (an
|W| x |C| attention map per iteration, kept for backward), run on the same GPU for comparison
(SURVEY.md S8(f) NEXT #4).  Not part of the product path: plain torch ops, fp32 map.

For each weight matrix of the workload it times forward (T unrolled iterations + W~) and
backward (autograd) and records the peak memory, the quantities of the paper's Table 2
(P:97-107).  Usage:  python tools/dense_baseline.py [--workload cfg2] [--steps 3]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2309_00964_b200 import synth  # noqa: E402


def dkm_dense(W, C0, tau, T):
    w = W.float().reshape(-1, 1)
    C = C0
    for _ in range(T):
        A = torch.softmax(-(w - C[None, :]) ** 2 / tau, dim=1)     # |W| x |C| map
        C = (A * w).sum(0) / A.sum(0)
    A = torch.softmax(-(w - C[None, :]) ** 2 / tau, dim=1)
    return (A @ C).reshape(W.shape)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--workload", default="cfg2")
    ap.add_argument("--steps", type=int, default=3)
    a = ap.parse_args()
    wl = synth.workload(a.workload)
    dev = torch.device("cuda")
    res = []
    for t, (name, r, c) in enumerate(wl.shapes):
        W = synth.weights(wl, t, dev).reshape(r, c).float().requires_grad_()
        G = synth.grads(wl, t, dev).reshape(r, c).float()
        C0 = torch.tensor(synth.quantile_centroids(wl.k, wl.sigma), device=dev, requires_grad=True)
        times = []
        for s in range(a.steps + 1):
            torch.cuda.reset_peak_memory_stats()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            Wt = dkm_dense(W, C0, wl.tau, wl.max_iter)
            Wt.backward(G)
            e1.record()
            torch.cuda.synchronize()
            if s:
                times.append(e0.elapsed_time(e1))
            W.grad = None
            C0.grad = None
        ms = sorted(times)[len(times) // 2]
        res.append({"tensor": name, "weights": r * c, "ms_fwd_bwd": ms,
                    "peak_mem_GiB": torch.cuda.max_memory_allocated() / 2**30,
                    "weights_per_s": r * c / (ms / 1e3)})
        print(json.dumps(res[-1]))
    tot_w = sum(x["weights"] for x in res)
    tot_ms = sum(x["ms_fwd_bwd"] for x in res)
    print(json.dumps({"workload": wl.name, "impl": "dense torch autograd (fp32 map)", "weights": tot_w,
                      "ms_fwd_bwd": tot_ms, "weights_per_s": tot_w / (tot_ms / 1e3),
                      "peak_mem_GiB_max": max(x["peak_mem_GiB"] for x in res)}))


if __name__ == "__main__":
    main()
