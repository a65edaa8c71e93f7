"""Multi-process orchestration of the eDKM step (one process per GPU, P:79 sharding).

Every rank holds the contiguous slice [floor(r n / P), floor((r+1) n / P)) of every
tensor (the paper shards the index list over learners; here the weights
themselves are sliced, so only histograms and k-vectors move).  The path has two
real exchange steps, both all-reduces over the process group (NCCL on B200):

  1. after F1: the int32 pattern counts [nt][65536] (exact, order independent), so
     every rank runs the identical table phase (TF) -- no per-iteration exchange;
  2. after B1: the fp64 partial gamma_T [nt][k] (linear in the local buckets).

Nothing else crosses ranks: W~ and dW are produced for the local slice only, C_T
and dC_0 come out identical on every rank.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[lo, hi) of a length-n tensor held by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def shard_all(numels, rank: int, world: int):
    return [shard_range(n, rank, world) for n in numels]


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (no-op without an initialised process group of size > 1)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


class ShardedStep:
    """Runs one eDKM step over this rank's slices with the two collectives.

    `kernels` is any object with the Plan interface (uniquify, forward,
    reconstruct, backward_reduce, backward_apply, counts, gamma, dC0); on a
    B200 it is paper_2309_00964_b200.edkm.Plan.
    """

    def __init__(self, kernels, group=None, allreduce=None):
        self.k = kernels
        self.group = group
        self.allreduce = allreduce or (lambda t: allreduce_sum(t, self.group))

    def __call__(self, weights, grads, C0, outs, dW):
        self.k.uniquify(weights)
        self.allreduce(self.k.counts)                     # exchange 1: integer counts
        self.k.forward(C0)
        self.k.reconstruct(weights, outs)
        self.k.backward_reduce(weights, grads)
        self.allreduce(self.k.gamma)                      # exchange 2: gamma_T partials
        self.k.backward_apply(weights, grads, dW)
        return self.k.dC0
