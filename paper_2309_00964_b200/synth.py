"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds no DKM arithmetic: it only draws weights W, upstream
gradients G and initial centroids C_0 with the shapes and distributions of the
paper's workloads, so the CUDA path and the oracle
are fed identical inputs.

Workloads (BASELINE.json configs; PAPER.md P:87 LLaMA-7B bf16, P:91 3-bit):
  cfg1  one 1024x1024 bf16 N(0, 1) matrix, k=8, tau=1e-3, T=5
  cfg2  one LLaMA-7B decoder layer (q,k,v,o 4096^2; gate, up 11008x4096;
        down 4096x11008) bf16 N(0, 0.02^2), k=8, tau=1e-5, T=5
  cfg3  LLaMA-7B: 32 layers x 7 linears + embed + lm_head (32000x4096),
        226 tensors, 6,738,149,376 weights
  cfg4  cfg3 shapes in fp16, k=16 (and k=4), T=30
  cfg5  LLaMA-13B: 40 x (4 x 5120^2, 3 x 5120x13824) + 2 x 32000x5120
G ~ N(0, (1e-3)^2) in the weights' dtype (R15).  C_0 = the k quantiles
sigma * Phi^-1((j + 0.5) / k) of the generating normal law (R5).
"""
from __future__ import annotations

from dataclasses import dataclass, field
from statistics import NormalDist

import torch

LLAMA7B_LAYER = [("q_proj", 4096, 4096), ("k_proj", 4096, 4096), ("v_proj", 4096, 4096),
                 ("o_proj", 4096, 4096), ("gate_proj", 11008, 4096), ("up_proj", 11008, 4096),
                 ("down_proj", 4096, 11008)]
LLAMA13B_LAYER = [("q_proj", 5120, 5120), ("k_proj", 5120, 5120), ("v_proj", 5120, 5120),
                  ("o_proj", 5120, 5120), ("gate_proj", 13824, 5120), ("up_proj", 13824, 5120),
                  ("down_proj", 5120, 13824)]


@dataclass
class Workload:
    name: str
    shapes: list            # [(name, rows, cols)]
    wdtype: torch.dtype
    sigma: float
    bits: int
    tau: float
    max_iter: int
    eps: float = 0.0
    g_scale: float = 1e-3
    seed_base: int = 1000
    notes: str = ""
    extra: dict = field(default_factory=dict)

    @property
    def k(self) -> int:
        return 1 << self.bits

    @property
    def numel(self) -> int:
        return sum(r * c for _, r, c in self.shapes)


def llama_shapes(layers, hidden, layer_shapes, vocab=32000):
    s = [("embed_tokens", vocab, hidden)]
    for l in range(layers):
        s += [(f"layers.{l}.{n}", r, c) for n, r, c in layer_shapes]
    s.append(("lm_head", vocab, hidden))
    return s


def workload(name: str) -> Workload:
    if name == "cfg1":
        return Workload("cfg1", [("w", 1024, 1024)], torch.bfloat16, 1.0, 3, 1e-3, 5, seed_base=0)
    if name == "cfg2":
        return Workload("cfg2", [(f"layers.0.{n}", r, c) for n, r, c in LLAMA7B_LAYER], torch.bfloat16,
                        0.02, 3, 1e-5, 5)
    if name == "cfg3":
        return Workload("cfg3", llama_shapes(32, 4096, LLAMA7B_LAYER), torch.bfloat16, 0.02, 3, 1e-5, 5)
    if name == "cfg4":
        return Workload("cfg4", llama_shapes(32, 4096, LLAMA7B_LAYER), torch.float16, 0.02, 4, 1e-5, 30)
    if name == "cfg4_b2":
        return Workload("cfg4_b2", llama_shapes(32, 4096, LLAMA7B_LAYER), torch.float16, 0.02, 2, 1e-5, 30)
    if name == "cfg5":
        return Workload("cfg5", llama_shapes(40, 5120, LLAMA13B_LAYER), torch.bfloat16, 0.02, 3, 1e-5, 5)
    raise KeyError(name)


def quantile_centroids(k: int, sigma: float) -> list:
    """C_0[j] = sigma * Phi^-1((j + 0.5) / k): the k quantiles of N(0, sigma^2) (R5)."""
    nd = NormalDist(0.0, sigma)
    return [nd.inv_cdf((j + 0.5) / k) for j in range(k)]


def data_quantile_centroids(w: torch.Tensor, k: int) -> list:
    """C_0 from the data (R5's alternative for small tensors): the k quantiles of the DISTINCT
    finite values of w, C_0[j] = d[floor((j + 0.5) m / k)] with d the m sorted distinct values.
    With m >= k the k centroids are distinct weights, so no cluster starts empty (R6)."""
    x = w.detach().reshape(-1).double().cpu()
    d = torch.unique(x[torch.isfinite(x)])
    m = d.numel()
    if m == 0:
        return [0.0] * k
    return [float(d[min(m - 1, ((2 * j + 1) * m) // (2 * k))]) for j in range(k)]


def _gen(device, seed):
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    return g


def normal_tensor(n: int, sigma: float, dtype: torch.dtype, seed: int, device="cpu") -> torch.Tensor:
    """n draws of N(0, sigma^2) rounded (RNE) to dtype, from a seeded generator."""
    x = torch.randn(n, generator=_gen(device, seed), device=device, dtype=torch.float32)
    if sigma != 1.0:
        x.mul_(sigma)
    return x.to(dtype)


def weights(wl: Workload, t: int, device="cpu", n: int | None = None) -> torch.Tensor:
    _, r, c = wl.shapes[t]
    return normal_tensor(n if n is not None else r * c, wl.sigma, wl.wdtype, wl.seed_base + t, device)


def grads(wl: Workload, t: int, device="cpu", n: int | None = None, dtype=None) -> torch.Tensor:
    _, r, c = wl.shapes[t]
    return normal_tensor(n if n is not None else r * c, wl.g_scale, dtype or wl.wdtype,
                         wl.seed_base + 1000 + t, device)


HEAVY_TAILS = ("cauchy", "student_t1.2", "lognormal3", "spike")


def heavy_tailed(n: int, kind: str, scale: float, dtype: torch.dtype, seed: int) -> torch.Tensor:
    """n heavy-tailed draws x scale rounded (RNE) to dtype, from a seeded numpy generator (CPU).

    LLM gradients are heavy-tailed; these exercise B1's fixed-point buckets far from the
    Gaussian law of `grads` (Cauchy, Student-t(1.2), random-sign log-normal(3), and
    a N(0, 1) tensor with one 1e4x spike inside the first 4,096 elements)."""
    import numpy as np
    r = np.random.default_rng(seed)
    if kind == "cauchy":
        x = r.standard_cauchy(n)
    elif kind == "student_t1.2":
        x = r.standard_t(1.2, n)
    elif kind == "lognormal3":
        x = r.lognormal(0.0, 3.0, n) * np.where(r.random(n) < 0.5, -1.0, 1.0)
    elif kind == "spike":
        x = r.standard_normal(n)
        if n:
            x[min(n - 1, 100)] = 1e4
    else:
        raise KeyError(kind)
    return torch.from_numpy(x * scale).to(dtype)


def random_bits(n: int, seed: int, device="cpu") -> torch.Tensor:
    """Uniformly random 16-bit patterns as int16 (every pattern, NaN/Inf included)."""
    return torch.randint(-32768, 32768, (n,), generator=_gen(device, seed), device=device, dtype=torch.int32).to(
        torch.int16)


def gib(nbytes: float) -> float:
    return nbytes / float(1 << 30)


__all__ = ["Workload", "workload", "quantile_centroids", "normal_tensor", "weights", "grads", "random_bits",
           "heavy_tailed", "HEAVY_TAILS", "data_quantile_centroids",
           "llama_shapes", "LLAMA7B_LAYER", "LLAMA13B_LAYER"]
