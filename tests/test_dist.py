"""Multi-process (N>1) path on CPU: world size 2 over gloo (127.0.0.1).

The product orchestration (paper_2309_00964_b200.dist: contiguous slices per
rank; all-reduce of the int32 counts after F1 and of gamma_T after B1)
runs unchanged; the per-rank compute is an oracle-backed stand-in with the
Plan interface (test infrastructure only -- on a B200 it is edkm.Plan).  Each
rank's slice of W~ and dW, and the rank-identical C_T and dC_0, must match a
single-process dense oracle run on the whole tensors.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2309_00964_b200 import synth
from paper_2309_00964_b200.dist import ShardedStep, assign_tensors, shard_all, shard_range

TAU, T, K = 2e-2, 3, 4


class OracleKernels:
    """Plan-shaped stand-in computing each stage with the CPU oracle on this rank's slices."""

    def __init__(self, nt, k):
        self.nt, self.k = nt, k
        self.counts = torch.zeros((nt, 65536), dtype=torch.int32)
        self.gamma = torch.zeros((nt, k), dtype=torch.float64)
        self.dC0 = torch.zeros((nt, k), dtype=torch.float64)

    @staticmethod
    def bits(w):
        return w.view(torch.int16).numpy().view(np.uint16)

    def uniquify(self, weights):
        for t, w in enumerate(weights):
            self.counts[t] = torch.from_numpy(O.histogram(self.bits(w)).astype(np.int32))

    # page-compact count exchange (stand-ins of edkm_count_pages / _counts_pack / _counts_unpack)
    def count_pages(self):
        return (self.counts.reshape(self.nt, 256, 256) != 0).any(dim=2).to(torch.uint8)

    def pack_counts(self, pages):
        return self.counts.reshape(-1, 256)[pages.long()].clone()

    def unpack_counts(self, pages, compact):
        self.counts.reshape(-1, 256)[pages.long()] = compact

    def _uniq(self, t):
        u = np.nonzero(self.counts[t].numpy())[0]
        v = O.decode16(u.astype(np.uint16), O.BF16)
        return u, v, self.counts[t].numpy()[u].astype(np.float64)

    def forward(self, C0):
        self.traj = []
        for t in range(self.nt):
            u, v, c = self._uniq(t)
            Ct, St, _ = O.dkm_forward(v, C0[t].numpy(), TAU, T, mult=c)
            self.traj.append((Ct, St))
        return self.traj

    def reconstruct(self, weights, outs):
        for t, w in enumerate(weights):
            outs[t][:] = torch.from_numpy(O.reconstruct(O.decode16(self.bits(w), O.BF16), self.traj[t][0][-1], TAU))

    def backward_reduce(self, weights, grads):
        for t, (w, g) in enumerate(zip(weights, grads)):
            u, v, c = self._uniq(t)
            pos = np.searchsorted(u, self.bits(w))
            B = np.bincount(pos, weights=g.double().numpy(), minlength=u.size)
            Ct, St = self.traj[t]
            self.gamma[t] = torch.from_numpy(O.dkm_backward_table(v, c, B, Ct[-1:], St[:0], TAU)[2])

    def backward_apply(self, weights, grads, dW):
        for t, (w, g) in enumerate(zip(weights, grads)):
            u, v, c = self._uniq(t)
            Ct, St = self.traj[t]
            phi, psi, dC = O.dkm_backward_table(v, c, None, Ct, St, TAU, gammaT=self.gamma[t].numpy())
            pos = np.searchsorted(u, self.bits(w))
            dW[t][:] = torch.from_numpy(g.double().numpy() * phi[pos] + psi[pos])
            self.dC0[t] = torch.from_numpy(dC)


def inputs():
    sizes = [10_007, 3, 1, 65_536 + 17]  # the 1-element tensor leaves rank 0 an empty slice
    Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 700 + i) for i, n in enumerate(sizes)]
    Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 800 + i) for i, n in enumerate(sizes)]
    C0 = torch.tensor([synth.quantile_centroids(K, 1.0)] * len(sizes), dtype=torch.float64)
    return sizes, Ws, Gs, C0


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        sizes, Ws, Gs, C0 = inputs()
        rng = shard_all(sizes, rank, world)
        Wl = [w[a:b].contiguous() for w, (a, b) in zip(Ws, rng)]
        Gl = [g[a:b].contiguous() for g, (a, b) in zip(Gs, rng)]
        kern = OracleKernels(len(sizes), K)
        outs = [torch.empty(b - a, dtype=torch.float64) for a, b in rng]
        dW = [torch.empty(b - a, dtype=torch.float64) for a, b in rng]
        ShardedStep(kern)(Wl, Gl, C0, outs, dW)
        q.put((rank, [o.numpy() for o in outs], [d.numpy() for d in dW], kern.dC0.numpy(),
               [tr[0] for tr in kern.traj], kern.counts.numpy().sum(1)))
    finally:
        dist.destroy_process_group()


def _compact_worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_00964_b200.dist import exchange_counts_compact, allreduce_max, allreduce_sum
        sizes, Ws = compact_inputs()
        rng = shard_all(sizes, rank, world)
        kern = OracleKernels(len(sizes), K)
        kern.uniquify([w[a:b].contiguous() for w, (a, b) in zip(Ws, rng)])
        local_pages = int(kern.count_pages().sum())
        npages = int(exchange_counts_compact(kern, allreduce_sum, allreduce_max).numel())
        q.put((rank, kern.counts.numpy().copy(), npages, local_pages))
    finally:
        dist.destroy_process_group()


def compact_inputs():
    # rank-disjoint page sets (tensor 1: positive weights in the first half, negative in the second),
    # a tensor only one rank populates, an empty tensor, and a tiny one
    sizes = [50_000, 40_000, 0, 3, 1]
    Ws = [synth.normal_tensor(sizes[0], 0.02, torch.bfloat16, 901)]
    x = synth.normal_tensor(sizes[1], 1.0, torch.bfloat16, 902).abs()
    Ws.append(torch.cat([x[:20_000], -x[20_000:]]))
    Ws += [torch.zeros(0, dtype=torch.bfloat16), synth.normal_tensor(3, 1.0, torch.bfloat16, 903),
           torch.tensor([1e-30], dtype=torch.bfloat16)]
    return sizes, Ws


def test_world_size_2_gloo_compact_count_exchange_matches_oracle_histogram():
    """dist.exchange_counts_compact: every rank ends with the exact global counts of
    every tensor (O.histogram of the whole tensor) although only the union of the ranks' populated pages
    was summed."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_compact_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes, Ws = compact_inputs()
    for r in range(world):
        for t, w in enumerate(Ws):
            ref = O.histogram(w.view(torch.int16).numpy().view(np.uint16))
            np.testing.assert_array_equal(res[r][1][t], ref.astype(np.int32))
    assert res[0][2] == res[1][2] < len(sizes) * 256            # same union on both ranks, compact
    assert res[0][2] >= max(res[0][3], res[1][3])               # it covers each rank's own pages
    assert res[0][2] < res[0][3] + res[1][3]                    # pages shared by both are summed once


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_ranges_partition_every_tensor():
    for n in (0, 1, 2, 7, 1000, 6_738_149_376):
        for world in (1, 2, 3, 8):
            r = [shard_range(n, k, world) for k in range(world)]
            assert r[0][0] == 0 and r[-1][1] == n
            assert all(r[k][1] == r[k + 1][0] for k in range(world - 1))
            assert all(b - a in (n // world, n // world + 1) for a, b in r)
    with pytest.raises(ValueError):
        shard_range(10, 2, 2)


@pytest.mark.parametrize("cfg", ["cfg3", "cfg5", "ragged"])
def test_assign_tensors_covers_every_tensor_once_and_balances(cfg):
    """Sharding by tensor (bench.py's default at N > 1): every tensor on exactly one rank,
    deterministic, and the largest rank load within one tensor of the mean (the longest-first
    greedy's bound: a rank only receives a tensor while it is the least loaded)."""
    if cfg == "ragged":
        numels = [0, 1, 17, 5_000_000, 3, 131_072_000, 2, 45_088_768] * 5
    else:
        numels = [r * c for _, r, c in synth.workload(cfg).shapes]
    for world in (1, 2, 3, 4, 8):
        owned = assign_tensors(numels, world)
        assert owned == assign_tensors(numels, world)
        flat = sorted(t for o in owned for t in o)
        assert flat == list(range(len(numels)))
        loads = [sum(numels[t] for t in o) for o in owned]
        assert max(loads) <= sum(numels) / world + max(numels)
        if cfg == "cfg3" and world == 8:
            assert max(loads) <= 1.01 * sum(numels) / world  # LLaMA-7B at N = 8: within 1%
    with pytest.raises(ValueError):
        assign_tensors(numels, 0)


def test_world_size_2_gloo_matches_single_process_oracle():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=300)
        res[r[0]] = r
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    sizes, Ws, Gs, C0 = inputs()
    for t, n in enumerate(sizes):
        w = O.decode16(Ws[t].view(torch.int16).numpy().view(np.uint16), O.BF16)
        Ct, St, _ = O.dkm_forward(w, C0[t].numpy(), TAU, T)
        Wt = O.reconstruct(w, Ct[-1], TAU)
        dW, dC = O.dkm_backward(w, Gs[t].double().numpy(), Ct, St, TAU)
        # counts after the all-reduce are global (exact), centroids and dC_0 rank-identical
        for r in range(world):
            assert res[r][5][t] == n
            np.testing.assert_array_equal(res[r][4][t], res[0][4][t])
            np.testing.assert_array_equal(res[r][3][t], res[0][3][t])
        np.testing.assert_allclose(res[0][4][t], Ct, rtol=1e-12, atol=1e-15)
        assert np.max(np.abs(res[0][3][t] - dC)) <= 1e-10 * max(np.max(np.abs(dC)), 1e-300) + 1e-300
        got_Wt = np.concatenate([res[r][1][t] for r in range(world)])
        got_dW = np.concatenate([res[r][2][t] for r in range(world)])
        assert np.max(np.abs(got_Wt - Wt)) <= 1e-10 * np.max(np.abs(Wt)), (t, np.max(np.abs(got_Wt - Wt)))
        assert np.max(np.abs(got_dW - dW)) <= 1e-10 * np.max(np.abs(dW))


def _fd_peer(name, q):
    from paper_2309_00964_b200.dist import _recv_fd
    fd = _recv_fd(name, timeout=30)
    with os.fdopen(fd, "rb") as f:
        q.put(f.read())


def test_nvls_handle_passing_between_processes():
    """NvlsCounts' plumbing: rank 0's multicast-object file descriptor reaches the other ranks
    over an abstract local socket (SCM_RIGHTS); here a pipe's read end stands in for it."""
    import multiprocessing as mpm
    import uuid

    from paper_2309_00964_b200.dist import _send_fd
    ctx = mpm.get_context("spawn")
    q = ctx.Queue()
    name = f"edkm-test-{uuid.uuid4().hex}"
    peers = [ctx.Process(target=_fd_peer, args=(name, q)) for _ in range(2)]
    for p in peers:
        p.start()
    r, w = os.pipe()
    os.write(w, b"multicast handle")
    os.close(w)
    try:
        _send_fd(name, r, 2, timeout=30)
    finally:
        os.close(r)
    got = [q.get(timeout=30) for _ in peers]
    for p in peers:
        p.join(timeout=30)
    # both peers hold a duplicate of the same pipe: the bytes are read once in total
    assert sorted(got) == sorted([b"multicast handle", b""])
