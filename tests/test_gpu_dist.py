"""The sharded N>1 path end to end on the CUDA kernels: two processes share the one B200,
each holding a contiguous slice of every tensor, exchanging counts and gamma_T over
a gloo process group (NCCL cannot put two ranks on one device; the exchanged tensors and the
orchestration -- paper_2309_00964_b200.dist.ShardedStep driving edkm.Plan -- are the same).
The concatenated slices of W~ and dW, and the rank-identical C_T and dC_0, must match the
dense oracle on the whole tensors; counts after the all-reduce are bit-exact.
"""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle as O
from paper_2309_00964_b200 import edkm as E
from paper_2309_00964_b200 import synth
from paper_2309_00964_b200.dist import ShardedStep, allreduce_sum, shard_all  # noqa: F401

pytestmark = pytest.mark.gpu
TOL = 1e-5
# two configurations of the sharded step: a bf16 k=8 T=4 one on N(0, 1) weights, and a CFG4-like
# one (fp16 N(0, 0.02^2), k=16, tau=1e-5, T=30) with 40 tensors, so that the table phase runs
# with CFG4's cluster size (4 CTAs per tensor for fp16 when nt > 37) -- the configuration bench.py
# splits by tensor block at N > 1 (k T >= 64)
CONFIGS = {
    "bf16_k8": dict(dtype=torch.bfloat16, sigma=1.0, sizes=[200_003, 65_536 * 2 + 7, 50_000],
                    p=dict(bits=3, tau=1e-3, max_iter=4)),
    "fp16_k16_T30": dict(dtype=torch.float16, sigma=0.02, sizes=[20_011 + 37 * i for i in range(40)],
                         p=dict(bits=4, tau=1e-5, max_iter=30)),
}
SIZES = CONFIGS["bf16_k8"]["sizes"]
P_ = CONFIGS["bf16_k8"]["p"]


def _inputs(cfg):
    Ws = [synth.normal_tensor(n, cfg["sigma"], cfg["dtype"], 500 + i) for i, n in enumerate(cfg["sizes"])]
    Gs = [synth.normal_tensor(n, 1e-3, cfg["dtype"], 600 + i) for i, n in enumerate(cfg["sizes"])]
    return Ws, Gs


def _reduce_via_host(t: torch.Tensor):
    h = t.cpu()
    allreduce_sum(h)
    t.copy_(h)


def _gather_via_host(t: torch.Tensor):
    """all-gather of rank blocks (rows) through host memory (gloo)."""
    world, rank = dist.get_world_size(), dist.get_rank()
    b = t.shape[0] // world
    parts = [torch.empty_like(t[:b], device="cpu") for _ in range(world)]
    dist.all_gather(parts, t[rank * b:(rank + 1) * b].cpu())
    t.copy_(torch.cat(parts).to(t.device))


def _max_via_host(t: torch.Tensor):
    from paper_2309_00964_b200.dist import allreduce_max
    h = t.cpu()
    allreduce_max(h)
    t.copy_(h)


def _worker(rank, world, port, q, shard_table=False, cfg_name="bf16_k8"):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2309_00964_b200.dist import padded_numels
        cfg = CONFIGS[cfg_name]
        dev = torch.device("cuda", 0)
        dt = cfg["dtype"]
        p = E.Params(dt, **cfg["p"])
        Ws, Gs = _inputs(cfg)
        rng = shard_all(cfg["sizes"], rank, world)
        Wl = [w[a:b].contiguous().to(dev) for w, (a, b) in zip(Ws, rng)]
        Gl = [g[a:b].contiguous().to(dev) for g, (a, b) in zip(Gs, rng)]
        numels = [w.numel() for w in Wl]
        if shard_table:  # empty tensors pad the list to equal per-rank table-phase blocks
            numels = padded_numels(numels, world)
            Wl += [torch.empty(0, dtype=dt, device=dev)] * (len(numels) - len(Wl))
            Gl += [torch.empty(0, dtype=dt, device=dev)] * (len(numels) - len(Gl))
        C0 = torch.tensor([synth.quantile_centroids(p.k, cfg["sigma"])] * len(numels), dtype=torch.float32,
                          device=dev)
        plan = E.Plan(numels, p, dev)
        outs = [torch.empty(w.numel(), dtype=torch.float32, device=dev) for w in Wl]
        dW = [torch.empty(w.numel(), dtype=torch.float32, device=dev) for w in Wl]
        compact = shard_table == "compact"
        step = ShardedStep(plan, allreduce=_reduce_via_host, allgather=_gather_via_host, shard_table=bool(shard_table),
                           out_mode="fp32", compact_tables=compact, allreduce_max=_max_via_host)
        for _ in range(2 if compact else 1):  # twice: the second step reuses the cached page lists
            step(Wl, Gl, C0, outs, dW)
        torch.cuda.synchronize()
        q.put((rank, plan.counts.cpu().numpy(), plan.C_out.cpu().numpy(), plan.dC0.cpu().numpy(),
               [o.cpu().double().numpy() for o in outs], [d.cpu().double().numpy() for d in dW]))
    finally:
        dist.destroy_process_group()


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


@pytest.mark.parametrize("cfg_name", list(CONFIGS))
@pytest.mark.parametrize("shard_table", [False, True, "compact"])
def test_two_ranks_on_one_gpu_match_single_process_oracle(shard_table, cfg_name):
    """shard_table=True: each rank runs TF/TB for its own tensor block and the ranks all-gather
    the per-tensor results; "compact": the other tensors' layout is derived
    locally and only the owners' states, trajectories and populated table pages are exchanged.
    Results must be the same."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q, shard_table, cfg_name)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=60)
        assert pr.exitcode == 0
    cfg = CONFIGS[cfg_name]
    pp = cfg["p"]
    Ws, Gs = _inputs(cfg)
    k = 1 << pp["bits"]
    C0 = np.float32(synth.quantile_centroids(k, cfg["sigma"])).astype(np.float64)
    fmt = O.BF16 if cfg["dtype"] == torch.bfloat16 else O.FP16
    for t, n in enumerate(cfg["sizes"]):
        bits = Ws[t].view(torch.int16).numpy().view(np.uint16)
        w = O.decode16(bits, fmt)
        Ct, St, _ = O.dkm_forward(w, C0, pp["tau"], pp["max_iter"])
        Wt = O.reconstruct(w, Ct[-1], pp["tau"])
        dW, dC = O.dkm_backward(w, Gs[t].double().numpy(), Ct, St, pp["tau"])
        for r in range(world):
            assert np.array_equal(res[r][1][t], O.histogram(bits).astype(np.int32))  # global counts, exact
            assert np.array_equal(res[r][2][t], res[0][2][t])                        # C_T rank-identical
            assert np.array_equal(res[r][3][t], res[0][3][t])                        # dC_0 rank-identical
        assert np.max(np.abs(res[0][2][t] - Ct[-1])) <= TOL * np.max(np.abs(Ct[-1]))
        assert np.max(np.abs(res[0][3][t] - dC)) <= TOL * np.max(np.abs(dC))
        gWt = np.concatenate([res[r][4][t] for r in range(world)])
        gdW = np.concatenate([res[r][5][t] for r in range(world)])
        assert np.max(np.abs(gWt - Wt)) <= TOL * np.max(np.abs(Wt))
        assert np.max(np.abs(gdW - dW)) <= TOL * np.max(np.abs(dW))


def _nvls_worker(port, q, emulate):
    """World size 1 over NCCL on the one B200: the NVLS-fused F1 (multimem reductions into a
    symmetric buffer + in-kernel arrival barrier) against plain F1, over several steps (the two
    alternating count buffers and the monotonic epoch), plus one ShardedStep with it."""
    from paper_2309_00964_b200.dist import NvlsCounts, NvlsUnavailable
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=dev)
    try:
        p = E.Params(torch.bfloat16, **P_)
        try:
            nv = NvlsCounts(len(SIZES), dev, emulate=emulate)
        except NvlsUnavailable as e:
            q.put(("skip", str(e)))
            return
        plan = E.Plan(SIZES, p, dev)
        ref = E.Plan(SIZES, p, dev)
        res = []
        for step in range(5):
            Ws = [synth.normal_tensor(n, 1.0 + step, torch.bfloat16, 700 + 10 * step + i).to(dev)
                  for i, n in enumerate(SIZES)]
            if step == 3:  # an fp16-like spread: the shared-array path of F1
                Ws[0] = torch.randint(0, 65536, (SIZES[0],), dtype=torch.int32).to(torch.int16).view(torch.bfloat16).to(dev)
            got = plan.uniquify_nvls(Ws, nv).cpu().numpy()
            want = np.stack([O.histogram(w.view(torch.int16).cpu().numpy().view(np.uint16)) for w in Ws])
            res.append(bool(np.array_equal(got, want.astype(np.int32))))  # against the oracle
        Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 800 + i).to(dev) for i, n in enumerate(SIZES)]
        Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 900 + i).to(dev) for i, n in enumerate(SIZES)]
        C0 = torch.tensor([synth.quantile_centroids(p.k, 1.0)] * len(SIZES), dtype=torch.float32, device=dev)
        outs = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        dW = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        outs2 = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        dW2 = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        ShardedStep(plan, nvls=nv)(Ws, Gs, C0, outs, dW)
        ref.step(Ws, Gs, C0, outs2, dW2)
        torch.cuda.synchronize()
        same = all(torch.equal(a, b) for a, b in zip(outs + dW, outs2 + dW2)) and torch.equal(plan.dC0, ref.dC0)
        epoch = int(nv.epoch.item())
        timeout_ok = None
        if emulate:
            # a barrier that can never complete (epoch pushed ahead of every arrival counter) with
            # trap = 0: the wait gives up after the timeout and reports it instead of trapping
            E.nvls_set_timeout(0.05, trap=False)
            nv.epoch += 100
            plan.uniquify_nvls(Ws, nv)
            first, second = E.nvls_failed(), E.nvls_failed()
            E.nvls_set_timeout(20.0, trap=True)
            timeout_ok = first and not second
        q.put(("ok", res, bool(same), epoch, timeout_ok))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("emulate", [True, False])
def test_nvls_fused_counts_world1(emulate):
    """emulate=False needs a system where multicast objects can be created (skips otherwise);
    emulate=True runs the identical kernels/protocol with plain atomics on ordinary memory."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_nvls_worker, args=(free_port(), q, emulate))
    pr.start()
    out = q.get(timeout=600)
    pr.join(timeout=120)
    if out[0] == "skip":
        pytest.skip(out[1])
    _, res, same, epoch, timeout_ok = out
    assert all(res), res
    assert same
    assert epoch == 6  # five uniquify_nvls steps + the ShardedStep
    if emulate:
        assert timeout_ok  # non-trapping timeout recorded once (edkm_nvls_set_timeout / edkm_nvls_failed)


def _comm_worker(q, compact):
    """The sharded step with every collective inside libedkm.so: edkm_comm_init at
    nranks = 1 on the one B200, then ShardedStep(comm=...) -- counts summed inside edkm_uniquify (or by
    the page-compact exchange through edkm_comm_allreduce), gamma_T inside edkm_backward_reduce."""
    from paper_2309_00964_b200.dist import ShardedStep as SS
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    comm = E.Comm()
    try:
        p = E.Params(torch.bfloat16, **P_)
        Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 500 + i).to(dev) for i, n in enumerate(SIZES)]
        Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 600 + i).to(dev) for i, n in enumerate(SIZES)]
        C0 = torch.tensor([synth.quantile_centroids(p.k, 1.0)] * len(SIZES), dtype=torch.float32, device=dev)
        plan = E.Plan(SIZES, p, dev)
        outs = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        dW = [torch.empty(n, dtype=torch.float32, device=dev) for n in SIZES]
        step = SS(plan, comm=comm, compact_counts=compact)
        for _ in range(2):  # twice: the step reuses every buffer
            step(Ws, Gs, C0, outs, dW)
        torch.cuda.synchronize()
        q.put(("ok", comm.nranks, comm.nccl_version, step.pages_exchanged, plan.counts.cpu().numpy(),
               plan.C_out.cpu().numpy(), plan.dC0.cpu().numpy(), [o.cpu().double().numpy() for o in outs],
               [d.cpu().double().numpy() for d in dW]))
    except Exception as e:  # report to the parent instead of hanging it
        q.put(("err", repr(e)))
    finally:
        comm.close()


@pytest.mark.parametrize("compact", [False, True])
def test_comm_in_the_c_abi_nranks1_matches_oracle(compact):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    pr = ctx.Process(target=_comm_worker, args=(q, compact))
    pr.start()
    out = q.get(timeout=600)
    pr.join(timeout=120)
    assert out[0] == "ok", out
    _, nranks, version, npages, counts, C, dC0, outs, dWs = out
    assert nranks == 1 and version >= 22700
    k = 1 << P_["bits"]
    C0 = np.float32(synth.quantile_centroids(k, 1.0)).astype(np.float64)
    pages = 0
    for t, n in enumerate(SIZES):
        W = synth.normal_tensor(n, 1.0, torch.bfloat16, 500 + t)
        G = synth.normal_tensor(n, 1e-3, torch.bfloat16, 600 + t)
        bits = W.view(torch.int16).numpy().view(np.uint16)
        c = O.histogram(bits)
        assert np.array_equal(counts[t], c.astype(np.int32))
        pages += int(np.any(c.reshape(256, 256) != 0, axis=1).sum())
        w = O.decode16(bits, O.BF16)
        Ct, St, _ = O.dkm_forward(w, C0, P_["tau"], P_["max_iter"])
        Wt = O.reconstruct(w, Ct[-1], P_["tau"])
        dWr, dC = O.dkm_backward(w, G.double().numpy(), Ct, St, P_["tau"])
        assert np.max(np.abs(C[t] - Ct[-1])) <= TOL * np.max(np.abs(Ct[-1]))
        assert np.max(np.abs(dC0[t] - dC)) <= TOL * np.max(np.abs(dC))
        assert np.max(np.abs(outs[t] - Wt)) <= TOL * np.max(np.abs(Wt))
        assert np.max(np.abs(dWs[t] - dWr)) <= TOL * np.max(np.abs(dWr))
    assert npages == (pages if compact else None)


@pytest.mark.parametrize("nt", [1, 226, 600])
def test_page_exchange_kernels(nt):
    """edkm_count_pages / _counts_pack / _counts_unpack at up to 600 x 256 pages (more than one grid of
    the kernels) against their plain definitions: a page is populated iff any of its 256 counts is
    nonzero; pack gathers the listed pages in list order; unpack scatters them back."""
    g = torch.Generator().manual_seed(nt)
    counts = torch.zeros((nt, 65536), dtype=torch.int32)
    pages = torch.randperm(nt * 256, generator=g)[: max(1, nt * 256 // 7)]
    for pg in pages.tolist():
        counts.view(-1, 256)[pg, int(torch.randint(0, 256, (1,), generator=g))] = int(torch.randint(1, 1000, (1,),
                                                                                                    generator=g))
    d = counts.cuda()
    mask = E.count_pages(d).cpu()
    want = (counts.view(nt, 256, 256) != 0).any(dim=2).to(torch.uint8)
    assert torch.equal(mask, want)
    lst = torch.nonzero(want.reshape(-1)).reshape(-1).to(torch.int32)
    lst = lst[torch.randperm(lst.numel(), generator=g)].cuda()           # any order
    comp = torch.empty((lst.numel(), 256), dtype=torch.int32, device="cuda")
    E.counts_pack(d, lst, comp)
    assert torch.equal(comp.cpu(), counts.view(-1, 256)[lst.cpu().long()])
    out = torch.zeros_like(d)
    E.counts_unpack(comp * 3, lst, out)
    assert torch.equal(out.cpu(), counts * 3)


def _nvls2_worker(rank, world, port, q):
    """Two processes on the one B200, each F1-ing its slices with the NVLS protocol in emulate mode:
    every add and arrival goes into both ranks' count copies (the peer's mapped by CUDA IPC), so the
    arrival barrier, epochs and alternating buffers run with a real second writer."""
    from paper_2309_00964_b200.dist import NvlsCounts
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    try:
        p = E.Params(torch.bfloat16, **P_)
        nv = NvlsCounts(len(SIZES), dev, emulate=True)
        plan = E.Plan([b - a for a, b in shard_all(SIZES, rank, world)], p, dev)
        got = []
        for step in range(5):
            Ws = [synth.normal_tensor(n, 1.0 + step, torch.bfloat16, 700 + 10 * step + i) for i, n in enumerate(SIZES)]
            if step == 3:  # uniformly random bits: the shared-array path of F1 and the global atomics
                Ws[0] = synth.random_bits(SIZES[0], 55).view(torch.bfloat16)
            Wl = [w[a:b].contiguous().to(dev) for w, (a, b) in zip(Ws, shard_all(SIZES, rank, world))]
            got.append(plan.uniquify_nvls(Wl, nv).cpu().numpy().copy())
        # one full sharded step with the fused exchange (gamma through gloo)
        Ws = [synth.normal_tensor(n, 1.0, torch.bfloat16, 500 + i) for i, n in enumerate(SIZES)]
        Gs = [synth.normal_tensor(n, 1e-3, torch.bfloat16, 600 + i) for i, n in enumerate(SIZES)]
        rng = shard_all(SIZES, rank, world)
        Wl = [w[a:b].contiguous().to(dev) for w, (a, b) in zip(Ws, rng)]
        Gl = [g[a:b].contiguous().to(dev) for g, (a, b) in zip(Gs, rng)]
        C0 = torch.tensor([synth.quantile_centroids(p.k, 1.0)] * len(SIZES), dtype=torch.float32, device=dev)
        outs = [torch.empty(w.numel(), dtype=torch.float32, device=dev) for w in Wl]
        dW = [torch.empty(w.numel(), dtype=torch.float32, device=dev) for w in Wl]
        ShardedStep(plan, allreduce=_reduce_via_host, nvls=nv)(Wl, Gl, C0, outs, dW)
        torch.cuda.synchronize()
        q.put((rank, got, int(nv.epoch.item()), plan.C_out.cpu().numpy(), plan.dC0.cpu().numpy(),
               [o.cpu().double().numpy() for o in outs], [d.cpu().double().numpy() for d in dW]))
        nv.close()
    except Exception as e:
        q.put((rank, "err", repr(e)))
    finally:
        dist.destroy_process_group()


def test_nvls_protocol_two_writers_matches_oracle():
    """the fused count exchange against O.histogram (not CUDA F1), with two writers."""
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=_nvls2_worker, args=(r, world, port, q)) for r in range(world)]
    for pr in procs:
        pr.start()
    res = {}
    for _ in range(world):
        r = q.get(timeout=600)
        res[r[0]] = r
    for pr in procs:
        pr.join(timeout=120)
    for r in range(world):
        assert res[r][1] != "err", res[r]
    for step in range(5):
        Ws = [synth.normal_tensor(n, 1.0 + step, torch.bfloat16, 700 + 10 * step + i) for i, n in enumerate(SIZES)]
        if step == 3:
            Ws[0] = synth.random_bits(SIZES[0], 55).view(torch.bfloat16)
        for t, w in enumerate(Ws):
            ref = O.histogram(w.view(torch.int16).numpy().view(np.uint16)).astype(np.int32)
            for r in range(world):
                assert np.array_equal(res[r][1][step][t], ref), (step, t, r)
    for r in range(world):
        assert res[r][2] == 6  # five uniquify_nvls steps + the ShardedStep's
    k = 1 << P_["bits"]
    C0 = np.float32(synth.quantile_centroids(k, 1.0)).astype(np.float64)
    for t, n in enumerate(SIZES):
        W = synth.normal_tensor(n, 1.0, torch.bfloat16, 500 + t)
        G = synth.normal_tensor(n, 1e-3, torch.bfloat16, 600 + t)
        w = O.decode16(W.view(torch.int16).numpy().view(np.uint16), O.BF16)
        Ct, St, _ = O.dkm_forward(w, C0, P_["tau"], P_["max_iter"])
        Wt = O.reconstruct(w, Ct[-1], P_["tau"])
        dWr, dC = O.dkm_backward(w, G.double().numpy(), Ct, St, P_["tau"])
        assert np.array_equal(res[0][3][t], res[1][3][t]) and np.array_equal(res[0][4][t], res[1][4][t])
        assert np.max(np.abs(res[0][3][t] - Ct[-1])) <= TOL * np.max(np.abs(Ct[-1]))
        assert np.max(np.abs(res[0][4][t] - dC)) <= TOL * np.max(np.abs(dC))
        gWt = np.concatenate([res[r][5][t] for r in range(world)])
        gdW = np.concatenate([res[r][6][t] for r in range(world)])
        assert np.max(np.abs(gWt - Wt)) <= TOL * np.max(np.abs(Wt))
        assert np.max(np.abs(gdW - dWr)) <= TOL * np.max(np.abs(dWr))


@pytest.mark.parametrize("dtype,bits", [(torch.bfloat16, 3), (torch.float16, 4), (torch.bfloat16, 6)])
def test_forward_layout_range_matches_full_tf(dtype, bits):
    """edkm_forward_layout_range (a non-owner's view of a tensor in the compact table split) writes the
    same rows, partitions, page masses, non-finite counts and per-weight-kernel windows as the full TF,
    from the counts alone."""
    dev = torch.device("cuda")
    sizes = [300_001, 65_536 + 3, 17, 0, 1_000_000]
    p = E.Params(dtype, bits, 1e-3, 3)
    Ws = [synth.normal_tensor(n, 0.02, dtype, 40 + i).to(dev) for i, n in enumerate(sizes)]
    Ws[0][5] = float("nan")
    C0 = torch.tensor([synth.quantile_centroids(p.k, 0.02)] * len(sizes), dtype=torch.float32, device=dev)
    full, lay = E.Plan(sizes, p, dev), E.Plan(sizes, p, dev)
    for pl in (full, lay):
        pl.uniquify(Ws)
    full.forward(C0)
    lay.views()["state"].zero_()
    lay.forward_layout_range(0, len(sizes))
    torch.cuda.synchronize()
    vf, vl = full.views(), lay.views()
    st_f, st_l = vf["state"].cpu().numpy(), vl["state"].cpu().numpy()
    assert torch.equal(vf["page_cnt"].cpu(), vl["page_cnt"].cpu())
    for t in range(len(sizes)):
        # TensorState (launch.h): T @0 is the owner's; cl @4, pbase[9] @8, nrows[8] @44, win[4] @76,
        # nonfinite[8] (int64) @80 -- the first cl entries of each are defined
        st, sl = st_f[t], st_l[t]
        cl = int(st[4:8].view(np.int32)[0])
        assert cl == int(sl[4:8].view(np.int32)[0])
        pb = st[8:44].view(np.int32)
        nr = st[44:76].view(np.int32)
        assert np.array_equal(pb[:cl + 1], sl[8:44].view(np.int32)[:cl + 1])
        assert np.array_equal(nr[:cl], sl[44:76].view(np.int32)[:cl])
        assert np.array_equal(st[76:80], sl[76:80])
        assert np.array_equal(st[80:144].view(np.int64)[:cl], sl[80:144].view(np.int64)[:cl])
        rf = vf["rows"][t].cpu().view(torch.int16).numpy().view(np.uint16)
        rl = vl["rows"][t].cpu().view(torch.int16).numpy().view(np.uint16)
        for q in range(cl):
            assert np.array_equal(rf[pb[q]:pb[q] + nr[q]], rl[pb[q]:pb[q] + nr[q]])
