"""Multi-process orchestration of the eDKM step (one process per GPU, P:79 sharding).

Two ways to shard (the north star: "by tensor and by contiguous slices").  By tensor
(`assign_tensors`, bench.py's default at N > 1 while the largest tensor fits a rank's share):
every rank clusters whole tensors, which are independent problems, so nothing crosses
ranks in the data path.  By slice (below; the paper's sharding of the index list, and the
only way when one tensor outweighs a rank's share): every rank holds the contiguous slice [floor(r n / P), floor((r+1) n / P)) of every
tensor (the paper shards the index list over learners; here the weights
themselves are sliced, so only histograms and k-vectors move).  The path has two
real exchange steps, both all-reduces over the process group (NCCL on B200):

  1. after F1: the int32 pattern counts [nt][65536] (exact, order independent), so
     every rank runs the identical table phase (TF) -- no per-iteration exchange;
  2. after B1: the fp64 partial gamma_T [nt][k] (linear in the local buckets).

Nothing else crosses ranks: W~ and dW are produced for the local slice only, C_T
and dC_0 come out identical on every rank.

On NVSwitch systems with NVLS multicast, exchange 1 is fused into F1 itself
(`NvlsCounts` + edkm_uniquify_nvls): F1's shared-memory flushes are multimem
reductions into a symmetric buffer, summed by the switch into every rank's copy, and
an in-kernel arrival barrier replaces the collective.  Exchange 2 (fp64) stays an
NCCL all-reduce, whose result is bit-identical on every rank (in-switch fp64 adds
would arrive in a different order on each GPU).

Where the collectives run: with `comm` (an edkm.Comm, the NCCL communicator owned by
libedkm.so) the library does them on the step's stream -- inside
edkm_uniquify / edkm_backward_reduce, or through edkm_comm_allreduce / _allgather.
Without it, torch.distributed does (gloo in the CPU tests).

compact_counts=True exchanges only the 256-pattern pages of the counts that some rank
populated: an all-reduce (MAX) of one byte per page, the host lists
the union's pages (one device->host read of nt*256 bytes: the step's only host sync),
then the packed pages are summed (~7 MB instead of 59 MB for CFG3) and unpacked.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

NVLS_FLAGS = 1024  # edkm.h EDKM_NVLS_FLAGS


def shard_range(n: int, rank: int, world: int) -> tuple:
    """[lo, hi) of a length-n tensor held by `rank` of `world`."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    return (n * rank) // world, (n * (rank + 1)) // world


def shard_all(numels, rank: int, world: int):
    return [shard_range(n, rank, world) for n in numels]


def assign_tensors(numels, world: int):
    """Whole tensors to ranks (sharding by tensor): each tensor is an independent clustering
    problem (one C per tensor, DESIGN R12), so a rank that holds whole tensors needs no exchange at
    all -- no count or gamma all-reduce, no replicated table phase.  Longest-processing-time
    greedy: tensors by size (descending, ties by index) to the least-loaded rank (ties by rank);
    deterministic, every tensor exactly once.  Returns [rank] -> ascending list of tensor indices."""
    if world < 1:
        raise ValueError("bad world")
    load = [0] * world
    owned = [[] for _ in range(world)]
    for t in sorted(range(len(numels)), key=lambda i: (-numels[i], i)):
        r = min(range(world), key=lambda j: (load[j], j))
        owned[r].append(t)
        load[r] += numels[t]
    return [sorted(o) for o in owned]


def allreduce_sum(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place sum over ranks (no-op without an initialised process group of size > 1)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t


def allreduce_max(t: torch.Tensor, group=None) -> torch.Tensor:
    """In-place max over ranks (no-op without an initialised process group of size > 1)."""
    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


_pinned = {}


_allreduce_max = allreduce_max  # (ShardedStep's parameter of the same name shadows it)


def union_pages(mask: torch.Tensor) -> torch.Tensor:
    """Global page ids t*256 + p of the pages set in the all-reduced [nt][256] mask, ascending (int32,
    on the host: the mask's one device->host read).  Identical on every rank (the mask is).

    The read goes to a pinned buffer and the host spins on its event: a blocking stream sync that
    waited out the rest of the previous step let the thread sleep, and its wake-up left the GPU idle
    ~1.3 ms per step (bench at N=1 under torchrun: AR_counts 1.43 ms vs 0.25 ms in isolation)."""
    if not mask.is_cuda:
        return torch.nonzero(mask.reshape(-1)).reshape(-1).to(torch.int32)
    n = mask.numel()
    buf = _pinned.get("mask")
    if buf is None or buf.numel() < n:
        buf = torch.empty(max(n, 1 << 16), dtype=torch.uint8, pin_memory=True)
        _pinned["mask"] = buf
    h = buf[:n]
    h.copy_(mask.reshape(-1), non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    while not ev.query():
        pass
    return torch.nonzero(h).reshape(-1).to(torch.int32)


def exchange_counts_compact(k, allreduce_sum_fn, allreduce_max_fn):
    """Sum the ranks' counts over the union of their populated pages only.

    `k` has the Plan interface (counts, count_pages, pack_counts, unpack_counts).  Pages that no rank
    populated are zero on every rank, so after this every rank holds the exact global counts.
    Returns the union's global page ids t*256 + p (host int32, ascending)."""
    mask = k.count_pages()
    allreduce_max_fn(mask)
    host = union_pages(mask)
    pages = host.to(k.counts.device)
    compact = k.pack_counts(pages)
    allreduce_sum_fn(compact)
    k.unpack_counts(pages, compact)
    return host


def padded_numels(numels, world: int):
    """Tensor list padded with empty tensors to a multiple of `world` (the table-phase split needs
    equal per-rank tensor blocks, so that each exchanged array is one all-gather)."""
    numels = list(numels)
    return numels + [0] * ((-len(numels)) % world)


def allgather_blocks(full: torch.Tensor, group=None):
    """In-place all-gather of rank blocks: rank r's block is rows [r nt/P, (r+1) nt/P) of `full`."""
    if not (dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1):
        return full
    P, r = dist.get_world_size(group), dist.get_rank(group)
    b = full.shape[0] // P
    dist.all_gather_into_tensor(full, full[r * b:(r + 1) * b].contiguous(), group=group)
    return full


class ShardedStep:
    """Runs one eDKM step over this rank's slices with the two collectives.

    `kernels` is any object with the Plan interface (uniquify, forward,
    reconstruct, backward_reduce, backward_apply, counts, gamma, dC0); on a
    B200 it is paper_2309_00964_b200.edkm.Plan.

    compact_tables=True (with shard_table; implies the page-compact count exchange): ranks derive
    the tensors they do not own from the global counts (edkm_forward_layout_range: rows, windows)
    and exchange only the owners' C trajectories, states, C_T and the union pages of the W~ and
    (phi, psi) tables (edkm_pages_pack / _unpack) -- ~8x less than whole tables for CFG3.

    shard_table=True splits the table phase by tensor block: rank r runs
    TF and TB only for tensors [r nt/P, (r+1) nt/P) (edkm_forward_range / _backward_table_range)
    and the ranks all-gather the per-tensor results the per-weight kernels need -- after TF the
    tensor state, C trajectory, compacted rows, W~ table(s), page masses and C_T; after TB the
    (phi, psi) table and dC_0.  Otherwise (default) every rank runs the whole table phase
    (identical results, no extra exchange).  Requires plan.nt % P == 0 (dist.padded_numels).
    `out_mode` selects which W~ tables are exchanged: "16" (16-bit soft), "fp32", or "all".
    """

    def __init__(self, kernels, group=None, allreduce=None, nvls=None, shard_table=False, allgather=None,
                 out_mode="all", comm=None, compact_counts=False, compact_tables=False, allreduce_max=None):
        self.k = kernels
        self.group = group
        self.comm = comm
        if comm is not None:
            self.allreduce = allreduce or (lambda t: comm.allreduce(t))
            self.allreduce_max = allreduce_max or (lambda t: comm.allreduce(t, op=1))
            self.allgather = allgather or (lambda t: comm.allgather_blocks(t))
        else:
            self.allreduce = allreduce or (lambda t: allreduce_sum(t, self.group))
            self.allreduce_max = allreduce_max or (lambda t: _allreduce_max(t, self.group))
            self.allgather = allgather or (lambda t: allgather_blocks(t, self.group))
        self.nvls = nvls
        self.shard_table = shard_table
        self.out_mode = out_mode
        self.compact_counts = compact_counts or compact_tables
        self.compact_tables = compact_tables
        self.pages_exchanged = None  # pages summed by the last compact count exchange
        self.page_list = None        # their global ids t*256 + p (host int32), for compact_tables
        self._pg_cache = {}          # per-rank page lists of the last union

    def _block(self):
        P = dist.get_world_size(self.group) if dist.is_initialized() else 1
        r = dist.get_rank(self.group) if dist.is_initialized() else 0
        if self.k.nt % P:
            raise ValueError("shard_table needs plan.nt divisible by the world size (use dist.padded_numels)")
        b = self.k.nt // P
        return r * b, (r + 1) * b

    def __call__(self, weights, grads, C0, outs, dW):
        if self.nvls is not None:
            self.k.uniquify_nvls(weights, self.nvls)      # exchange 1 fused into F1 (NVSwitch)
        elif self.compact_counts:
            self.k.uniquify(weights)                      # exchange 1, populated pages only
            self.page_list = exchange_counts_compact(self.k, self.allreduce, self.allreduce_max)
            self.pages_exchanged = int(self.page_list.numel())
        elif self.comm is not None:
            self.k.uniquify(weights, comm=self.comm)      # exchange 1 inside edkm_uniquify
        else:
            self.k.uniquify(weights)
            self.allreduce(self.k.counts)                 # exchange 1: integer counts
        if not self.shard_table:
            self.k.forward(C0)
            self.k.reconstruct(weights, outs)
            if self.comm is not None:
                self.k.backward_reduce(weights, grads, comm=self.comm)  # exchange 2 inside the call
            else:
                self.k.backward_reduce(weights, grads)
                self.allreduce(self.k.gamma)              # exchange 2: gamma_T partials
            self.k.backward_apply(weights, grads, dW)
            return self.k.dC0
        t0, t1 = self._block()
        v = self.k.views()
        tables = {"16": ["table16"], "fp32": ["table"]}.get(self.out_mode, ["table16", "table", "idx8"])
        self.k.forward_range(t0, t1, C0)                  # TF, own tensor block
        if self.compact_tables:
            # the other tensors' layout from the global counts (identical on every rank), then only
            # the owners' C trajectories, states, C_T and the populated pages of their tables
            if t0 > 0:
                self.k.forward_layout_range(0, t0)
            if t1 < self.k.nt:
                self.k.forward_layout_range(t1, self.k.nt)
            for n in ("state", "ctraj", "C_out"):
                self.allgather(v[n])
            for n in tables:
                self._exchange_pages(n)
        else:
            for n in ["state", "ctraj", "rows", "page_cnt", "C_out"] + tables:
                self.allgather(v[n])
        self.k.reconstruct(weights, outs)
        self.k.backward_buckets(weights, grads)
        self.k.backward_gamma()
        self.allreduce(self.k.gamma)                      # exchange 2: gamma_T partials
        self.k.backward_table_range(t0, t1)               # TB, own tensor block
        if self.compact_tables:
            self._exchange_pages("phipsi")
            self.allgather(v["dC0"])
        else:
            for n in ("phipsi", "dC0"):
                self.allgather(v[n])
        self.k.backward_dw(weights, grads, dW)
        return self.k.dC0

    def _exchange_pages(self, name):
        """All-gather of the populated pages of each rank's tensor block of the per-pattern table
        `name` (a views() array): rank r packs the union pages of tensors [r b, (r+1) b) into rows
        [r m, r m + n_r) of one [P m][page bytes] buffer (m = the largest n_r), the buffer is
        all-gathered and every other rank's rows are unpacked (edkm_pages_pack / _unpack)."""
        P = dist.get_world_size(self.group) if dist.is_initialized() else 1
        r = dist.get_rank(self.group) if dist.is_initialized() else 0
        b = self.k.nt // P
        v = self.k.views()[name]
        pb = v.shape[1] // 256  # bytes per page
        hit = self._pg_cache.get("lists")
        if hit is None or not torch.equal(hit[0], self.page_list):  # per-rank lists of this step's union
            owner = self.page_list.long() // (256 * b)
            lists = [self.page_list[owner == q] for q in range(P)]
            m = max(1, max(int(x.numel()) for x in lists))
            dev = self.k.counts.device
            hit = (self.page_list.clone(), [x.to(dev) for x in lists], m)
            self._pg_cache["lists"] = hit
        _, lists, m = hit
        full = torch.empty((P * m, pb), dtype=torch.uint8, device=self.k.counts.device)
        if lists[r].numel():
            self.k.pack_pages(name, lists[r], full[r * m:r * m + lists[r].numel()])
        self.allgather(full)
        for q in range(P):
            if q != r and lists[q].numel():
                self.k.unpack_pages(name, lists[q], full[q * m:q * m + lists[q].numel()])


class NvlsUnavailable(RuntimeError):
    pass


class _CudaArray:
    """Zero-copy torch view of raw device memory (the __cuda_array_interface__ protocol)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _send_fd(name: str, fd: int, npeers: int, timeout: float = 120.0):
    import socket
    srv = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
    srv.bind("\0" + name)
    srv.listen(npeers)
    srv.settimeout(timeout)
    try:
        for _ in range(npeers):
            c, _ = srv.accept()
            with c:
                socket.send_fds(c, [b"x"], [fd])
    finally:
        srv.close()


def _recv_fd(name: str, timeout: float = 120.0) -> int:
    import socket
    import time
    t0 = time.time()
    while True:
        c = socket.socket(socket.AF_UNIX, socket.SOCK_STREAM)
        try:
            c.connect("\0" + name)
            break
        except OSError:
            c.close()
            if time.time() - t0 > timeout:
                raise
            time.sleep(0.01)
    with c:
        _, fds, _, _ = socket.recv_fds(c, 1, 1)
    return fds[0]


class NvlsCounts:
    """NVLS buffers of the fused count exchange (include/edkm.h edkm_uniquify_nvls).

    One multicast object (edkm_mc_*: driver-API plumbing in the library) holds two [nt][65536]
    int32 count buffers used on alternate steps -- the one of the next step is zeroed before
    this step's F1, so no rank can add into a copy another rank has not cleared -- and
    NVLS_FLAGS monotonic arrival counters; plus this rank's epoch.  Rank 0 creates the object
    and passes its file descriptor to the other ranks over a local socket (SCM_RIGHTS).
    Raises NvlsUnavailable when the system has no NVLS multicast.  emulate=True runs the same
    protocol -- kernels, epochs, alternating buffers -- on ordinary device memory with plain
    atomics, to test it where multicast objects cannot be created: one rank, or two ranks (e.g.
    two processes on one GPU) whose F1 adds into both ranks' copies through CUDA IPC.
    """

    def __init__(self, nt: int, device, group=None, emulate: bool = False):
        import ctypes
        import os
        import uuid

        from . import edkm as E
        L = E.lib()
        self.group = group
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        dev = torch.device(device)
        torch.cuda.set_device(dev)
        self.emulate = bool(emulate)
        self._nt = nt
        self.step_index = 0
        self.epoch = torch.zeros(1, dtype=torch.int32, device=dev)
        self.peer_delta = 0
        if self.emulate:
            # the protocol on ordinary memory: one rank, or two ranks each adding into both copies
            # (its own and the peer's, mapped by CUDA IPC) as the switch would -- a real second writer
            if self.nranks > 2:
                raise ValueError("emulate supports one or two ranks")
            self._buf = None
            cb = (max(nt, 1) * 65536 * 4 + 255) // 256 * 256
            self._emu = torch.zeros(2 * cb + NVLS_FLAGS * 4, dtype=torch.uint8, device=dev)
            self.bufs = [self._emu[o:o + cb].view(torch.int32)[:max(nt, 1) * 65536].view(max(nt, 1), 65536)
                         for o in (0, cb)]
            self.flags = self._emu[2 * cb:].view(torch.int32)
            self.mc_ptrs = [t.data_ptr() for t in self.bufs] + [self.flags.data_ptr()]
            self.current = self.bufs[0][:nt]
            self._peer = None
            if self.nranks == 2:
                h, off = (ctypes.c_uint8 * 64)(), ctypes.c_size_t(0)
                if L.edkm_ipc_handle(ctypes.c_void_p(self._emu.data_ptr()), h, ctypes.byref(off)) != 0:
                    raise NvlsUnavailable(f"edkm_ipc_handle: {L.edkm_mc_last_error().decode()}")
                objs = [None, None]
                dist.all_gather_object(objs, (bytes(h), off.value), group=group)
                ph, poff = objs[1 - rank]
                base = ctypes.c_void_p()
                hb = (ctypes.c_uint8 * 64).from_buffer_copy(ph)
                if L.edkm_ipc_open(hb, ctypes.byref(base)) != 0:
                    raise NvlsUnavailable(f"edkm_ipc_open: {L.edkm_mc_last_error().decode()}")
                self._peer = base
                self.peer_delta = base.value + poff - self._emu.data_ptr()
                torch.cuda.synchronize(dev)
                dist.barrier(group)
            return
        self._dev = dev
        sup = ctypes.c_int(0)
        self._agree(L.edkm_mc_supported(ctypes.byref(sup)) == 0 and bool(sup.value),
                    "no NVLS multicast support on this system")
        self.nt = max(nt, 1)
        cbytes = (self.nt * 65536 * 4 + 255) // 256 * 256
        need = 2 * cbytes + NVLS_FLAGS * 4
        buf = ctypes.c_void_p()
        fd = ctypes.c_int(-1)
        name = None
        err = ""
        if rank == 0:
            rc = L.edkm_mc_create(ctypes.c_size_t(need), self.nranks, int(self.nranks > 1), ctypes.byref(fd),
                                  ctypes.byref(buf))
            if rc != 0:
                err = L.edkm_mc_last_error().decode()
            name = f"edkm-nvls-{os.getpid()}-{uuid.uuid4().hex}"
        info = [name, int(L.edkm_mc_bytes(buf)) if buf.value else 0, err]
        if self.nranks > 1:
            dist.broadcast_object_list(info, src=0, group=group)
        name, size, err = info
        if not size:
            raise NvlsUnavailable(f"multicast object creation failed: {err}")  # identical on every rank
        self._buf = buf
        ok, why = True, ""
        if self.nranks > 1:  # rank 0's descriptor to the others (every failure is agreed on below)
            try:
                if rank == 0:
                    _send_fd(name, fd.value, self.nranks - 1)
                else:
                    rfd = _recv_fd(name)
                    rc = L.edkm_mc_import(rfd, ctypes.c_size_t(size), ctypes.byref(buf))
                    os.close(rfd)
                    ok, why = rc == 0, f"multicast import failed: {L.edkm_mc_last_error().decode()}"
            except OSError as e:
                ok, why = False, f"descriptor hand-off failed: {e}"
            finally:
                if rank == 0:
                    os.close(fd.value)
        self._agree(ok, why or "descriptor hand-off failed on another rank")
        rc = L.edkm_mc_add_device(buf)
        self._agree(rc == 0, f"cuMulticastAddDevice failed: {L.edkm_mc_last_error().decode()}")
        loc, mc = ctypes.c_void_p(), ctypes.c_void_p()
        rc = L.edkm_mc_bind(buf, ctypes.byref(loc), ctypes.byref(mc))
        self._agree(rc == 0, f"multicast bind failed: {L.edkm_mc_last_error().decode()}")
        self.local, self.mcbase = loc.value, mc.value
        self.offs = [0, cbytes, 2 * cbytes]
        self.bufs = [torch.as_tensor(_CudaArray(self.local + o, (self.nt, 65536), "<i4"), device=dev)
                     for o in self.offs[:2]]
        self.flags = torch.as_tensor(_CudaArray(self.local + self.offs[2], (NVLS_FLAGS,), "<i4"), device=dev)
        self.mc_ptrs = [self.mcbase + o for o in self.offs]
        for t in self.bufs + [self.flags]:
            t.zero_()
        self.current = self.bufs[0][:nt]
        torch.cuda.synchronize(dev)
        if self.nranks > 1:
            dist.barrier(group)

    def _agree(self, ok: bool, why: str):
        """All ranks learn whether every rank succeeded (MIN all-reduce) and raise together:
        a rank that gave up alone would leave the others in a collective."""
        if self.nranks > 1:
            backend = dist.get_backend(self.group)
            t = torch.tensor([1.0 if ok else 0.0], device=self._dev if backend == "nccl" else "cpu")
            dist.all_reduce(t, op=dist.ReduceOp.MIN, group=self.group)
            all_ok = bool(t.item() == 1.0)
        else:
            all_ok = ok
        if not all_ok:
            if getattr(self, "_buf", None) is not None and self._buf.value:
                from . import edkm as E
                E.lib().edkm_mc_destroy(self._buf)
                self._buf = None
            raise NvlsUnavailable(why if not ok else "failed on another rank")

    def next_step(self, stream=None):
        """C struct for this step's call; zeroes the next step's buffer on `stream` first."""
        from . import edkm as E
        s = self.step_index
        self.step_index += 1
        cur, nxt = s % 2, (s + 1) % 2
        with torch.cuda.stream(stream or torch.cuda.current_stream()):
            self.bufs[nxt].zero_()
        self.current = self.bufs[cur][:self._nt]
        return E._Nvls(self.mc_ptrs[cur], self.mc_ptrs[2], self.flags.data_ptr(), self.epoch.data_ptr(), self.nranks,
                       int(self.emulate), self.peer_delta)

    def close(self):
        from . import edkm as E
        if getattr(self, "_peer", None) is not None:
            torch.cuda.synchronize()
            if self.nranks > 1:
                dist.barrier(self.group)  # the peer's last adds into our copy are done
            E.lib().edkm_ipc_close(self._peer)
            self._peer = None
        if getattr(self, "_buf", None) is not None and self._buf.value:
            torch.cuda.synchronize()
            self.bufs = self.flags = self.current = None
            E.lib().edkm_mc_destroy(self._buf)
            self._buf = None
