"""eDKM step on host-resident weights and gradients, overlapping PCIe and compute.

For callers whose W and dL/dW~ live in (pinned) host memory: tensors are split
into groups; the host->device copy of group g+1, the eDKM step of group g (all
seven kernels through the C ABI, ``edkm.Plan``) and the device->host copy of
group g-1's W~ and dW run concurrently on three CUDA streams.  DKM clustering is
per tensor, so groups are independent; with several ranks each group's counts
and gamma_T are all-reduced as in ``dist.ShardedStep``.
"""
from __future__ import annotations

import torch

from . import edkm as E


def _groups(numels, n_groups):
    total = sum(numels)
    out, cur, acc = [], [], 0
    for t, n in enumerate(numels):
        cur.append(t)
        acc += n
        if acc >= total * (len(out) + 1) / n_groups and len(out) < n_groups - 1:
            out.append(cur)
            cur = []
    if cur:
        out.append(cur)
    return out


class HostPipeline:
    def __init__(self, numels, p: E.Params, device="cuda", n_groups: int = 8, allreduce=None, buffers=None):
        """buffers: optional (W, G, W~, dW) lists of device tensors to reuse (else allocated)."""
        self.p, self.dev = p, torch.device(device)
        self.groups = _groups(list(numels), n_groups)
        self.plans = [E.Plan([numels[t] for t in g], p, self.dev) for g in self.groups]
        if buffers is None:
            buffers = [[torch.empty(n, dtype=p.wdtype, device=self.dev) for n in numels] for _ in range(4)]
        self.Wd, self.Gd, self.Wt, self.dW = (list(b) for b in buffers)
        self.s_in, self.s_c, self.s_out = (torch.cuda.Stream(self.dev) for _ in range(3))
        self.allreduce = allreduce

    def step(self, hW, hG, C0: torch.Tensor, hWt, hdW):
        """Enqueue one step; hW/hG/hWt/hdW are per-tensor host tensors (pinned for overlap).
        Returns after enqueueing; the current stream waits for the last copy-out."""
        cur = torch.cuda.current_stream(self.dev)
        self.s_in.wait_stream(cur)
        for g, (ts, plan) in enumerate(zip(self.groups, self.plans)):
            with torch.cuda.stream(self.s_in):
                for t in ts:
                    self.Wd[t].copy_(hW[t], non_blocking=True)
                    self.Gd[t].copy_(hG[t], non_blocking=True)
                ev_in = torch.cuda.Event()
                ev_in.record(self.s_in)
            self.s_c.wait_event(ev_in)
            with torch.cuda.stream(self.s_c):
                W = [self.Wd[t] for t in ts]
                G = [self.Gd[t] for t in ts]
                plan.step(W, G, C0[ts[0]:ts[-1] + 1], [self.Wt[t] for t in ts], [self.dW[t] for t in ts],
                          allreduce=self.allreduce, stream=self.s_c)
                ev_c = torch.cuda.Event()
                ev_c.record(self.s_c)
            self.s_out.wait_event(ev_c)
            with torch.cuda.stream(self.s_out):
                for t in ts:
                    hWt[t].copy_(self.Wt[t], non_blocking=True)
                    hdW[t].copy_(self.dW[t], non_blocking=True)
        cur.wait_stream(self.s_out)
        cur.wait_stream(self.s_c)
        return [pl.dC0 for pl in self.plans]
