"""Thin Python binding of libedkm.so (include/edkm.h) -- argument marshalling only.

Every step of the eDKM hot path runs in the CUDA kernels behind the C ABI; this
module turns torch tensors into raw device pointers and the current CUDA stream
into a ``cudaStream_t``.  There is no CPU fallback: if libedkm.so is missing or
a call fails, an exception is raised.

Entry points (same names as the C ABI; PAPER.md = /root/reference/PAPER.md):
  uniquify          F1: counts per 16-bit pattern (Fig. 3)
  forward           TF: unrolled DKM iterations on the attention table
  reconstruct       F2: W~ = table[bits(w)] / hard palettisation (Fig. 1)
  backward_reduce   B1 + gamma_T partial   (= backward_buckets + backward_gamma)
  backward_apply    TB + B2: dC_0 and dW   (= backward_table + backward_dw)
  backward          both (single process)
``Plan`` owns the per-step buffers (counts, saved, ws, ...) so a training step
allocates nothing; ``EDKMFunction`` wraps one tensor as a torch.autograd.Function.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
# EDKM_LIB selects another build of the same library (A/B measurements of kernel variants)
LIB_PATH = os.environ.get("EDKM_LIB") or os.path.join(_HERE, "libedkm.so")

BF16, FP16, FP32, U8, I32, FP64 = 0, 1, 2, 3, 4, 5
SOFT, HARD_VALUE, HARD_INDEX = 0, 1, 2
SUM, MAX = 0, 1
PATTERNS = 65536

_DT = {torch.bfloat16: BF16, torch.float16: FP16, torch.float32: FP32, torch.uint8: U8, torch.int32: I32,
       torch.float64: FP64}


class EDKMError(RuntimeError):
    pass


class _Tensor(ctypes.Structure):
    _fields_ = [("w", ctypes.c_void_p), ("n", ctypes.c_int64)]


class _Nvls(ctypes.Structure):
    _fields_ = [("counts_mc", ctypes.c_void_p), ("flags_mc", ctypes.c_void_p), ("flags", ctypes.c_void_p),
                ("epoch", ctypes.c_void_p), ("nranks", ctypes.c_int), ("emulate", ctypes.c_int),
                ("peer_delta", ctypes.c_int64)]


NVLS_FLAGS = 1024


class _Params(ctypes.Structure):
    _fields_ = [("wdtype", ctypes.c_int), ("bits", ctypes.c_int), ("tau", ctypes.c_double),
                ("max_iter", ctypes.c_int), ("eps", ctypes.c_double)]


_lib = None


def lib():
    """Load libedkm.so (raises if it has not been built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise EDKMError(f"{LIB_PATH} not found: run `python -m paper_2309_00964_b200.build` "
                            "(or __graft_entry__.build()) first")
        L = ctypes.CDLL(LIB_PATH)
        P, i32, i64 = ctypes.c_void_p, ctypes.c_int, ctypes.c_int64
        pp = ctypes.POINTER(_Params)
        sig = {
            "edkm_saved_bytes": ([i32, pp], ctypes.c_size_t),
            "edkm_workspace_bytes": ([i32, pp], ctypes.c_size_t),
            "edkm_uniquify": ([P, i32, i32, P, P, P], i32),
            "edkm_uniquify_nvls": ([P, i32, i32, ctypes.POINTER(_Nvls), P], i32),
            "edkm_nvls_set_timeout": ([ctypes.c_double, i32], i32),
            "edkm_nvls_failed": ([P], i32),
            "edkm_forward": ([P, i32, pp, P, P, P, P, P], i32),
            "edkm_forward_range": ([P, i32, i32, i32, pp, P, P, P, P, P], i32),
            "edkm_backward_table_range": ([i32, i32, i32, pp, P, P, P, P, P, P], i32),
            "edkm_layout": ([i32, pp, P, P], i32),
            "edkm_reconstruct": ([P, i32, pp, P, P, P, i32, i32, P, P], i32),
            "edkm_backward_reduce": ([P, i32, pp, P, i32, P, P, P, P, P, P], i32),
            "edkm_backward_apply": ([P, i32, pp, P, i32, P, P, P, P, P, i32, P, P], i32),
            "edkm_backward": ([P, i32, pp, P, i32, P, P, P, P, i32, P, P], i32),
            "edkm_backward_buckets": ([P, i32, pp, P, i32, P, P, P], i32),
            "edkm_backward_gamma": ([i32, pp, P, P, P, P, P], i32),
            "edkm_backward_table": ([i32, pp, P, P, P, P, P, P], i32),
            "edkm_backward_dw": ([P, i32, pp, P, i32, P, P, P, i32, P], i32),
            "edkm_read_status": ([P, i32, pp, P, P, P], i32),
            "edkm_last_launch_count": ([], i32),
            "edkm_mc_supported": ([P], i32),
            "edkm_mc_create": ([ctypes.c_size_t, i32, i32, P, P], i32),
            "edkm_mc_import": ([i32, ctypes.c_size_t, P], i32),
            "edkm_mc_bytes": ([P], ctypes.c_size_t),
            "edkm_mc_add_device": ([P], i32),
            "edkm_mc_bind": ([P, P, P], i32),
            "edkm_mc_destroy": ([P], i32),
            "edkm_mc_last_error": ([], ctypes.c_char_p),
            "edkm_ipc_handle": ([P, P, P], i32),
            "edkm_ipc_open": ([P, P], i32),
            "edkm_ipc_close": ([P], i32),
            "edkm_set_max_ctas": ([i32], i32),
            "edkm_comm_unique_id": ([P], i32),
            "edkm_comm_init": ([P, P, i32, i32], i32),
            "edkm_comm_destroy": ([P], i32),
            "edkm_comm_info": ([P, P, P, P], i32),
            "edkm_comm_allreduce": ([P, P, ctypes.c_size_t, i32, i32, P], i32),
            "edkm_comm_allgather": ([P, P, P, ctypes.c_size_t, P], i32),
            "edkm_count_pages": ([P, i32, P, P], i32),
            "edkm_counts_pack": ([P, i32, P, i32, P, P], i32),
            "edkm_counts_unpack": ([P, P, i32, i32, P, P], i32),
            "edkm_pages_pack": ([P, i32, i32, P, i32, P, P], i32),
            "edkm_pages_unpack": ([P, i32, P, i32, i32, P, P], i32),
            "edkm_forward_layout_range": ([P, i32, i32, i32, pp, P, P, P], i32),
            "edkm_status_string": ([i32], ctypes.c_char_p),
            "edkm_last_error": ([], ctypes.c_char_p),
        }
        for name, (args, res) in sig.items():
            f = getattr(L, name)
            f.argtypes, f.restype = args, res
        _lib = L
    return _lib


def exported_symbols() -> list:
    return ["edkm_saved_bytes", "edkm_workspace_bytes", "edkm_uniquify", "edkm_uniquify_nvls", "edkm_nvls_set_timeout",
            "edkm_nvls_failed", "edkm_forward", "edkm_forward_range",
            "edkm_backward_table_range", "edkm_layout", "edkm_reconstruct",
            "edkm_backward_reduce", "edkm_backward_apply", "edkm_backward", "edkm_backward_buckets",
            "edkm_backward_gamma", "edkm_backward_table", "edkm_backward_dw", "edkm_read_status",
            "edkm_last_launch_count", "edkm_set_max_ctas", "edkm_status_string", "edkm_last_error",
            "edkm_mc_supported", "edkm_mc_create", "edkm_mc_import", "edkm_mc_bytes", "edkm_mc_add_device",
            "edkm_mc_bind", "edkm_mc_destroy", "edkm_mc_last_error", "edkm_comm_unique_id", "edkm_comm_init",
            "edkm_comm_destroy", "edkm_comm_info", "edkm_comm_allreduce", "edkm_comm_allgather", "edkm_count_pages",
            "edkm_counts_pack", "edkm_counts_unpack", "edkm_ipc_handle", "edkm_ipc_open", "edkm_ipc_close",
            "edkm_pages_pack", "edkm_pages_unpack", "edkm_forward_layout_range"]


def _check(rc: int, what: str):
    if rc != 0:
        L = lib()
        raise EDKMError(f"{what}: {L.edkm_status_string(rc).decode()} -- {L.edkm_last_error().decode()}")


def last_launch_count() -> int:
    return lib().edkm_last_launch_count()


def set_max_ctas(ctas: int) -> int:
    """Cap the streaming kernels' grid for later calls on this thread (0 = SM count); returns the old cap."""
    return lib().edkm_set_max_ctas(int(ctas))


def nvls_set_timeout(seconds: float, trap: bool = True):
    """Arrival-barrier timeout of later NVLS uniquify calls (edkm_nvls_set_timeout)."""
    _check(lib().edkm_nvls_set_timeout(ctypes.c_double(seconds), int(bool(trap))), "edkm_nvls_set_timeout")


def nvls_failed() -> bool:
    """True if a non-trapping NVLS arrival wait timed out since the last call (clears the flag; syncs)."""
    f = ctypes.c_int(0)
    _check(lib().edkm_nvls_failed(ctypes.byref(f)), "edkm_nvls_failed")
    return bool(f.value)


@dataclass(frozen=True)
class Params:
    """DKM hyper-parameters (P:31 LUT of k = 2^bits centroids; tau, iterations per DESIGN R3/R4)."""
    wdtype: torch.dtype = torch.bfloat16
    bits: int = 3
    tau: float = 1e-3
    max_iter: int = 5
    eps: float = 0.0

    @property
    def k(self) -> int:
        return 1 << self.bits

    def c(self) -> _Params:
        if self.wdtype not in (torch.bfloat16, torch.float16):
            raise EDKMError("weights must be bfloat16 or float16")
        return _Params(_DT[self.wdtype], self.bits, float(self.tau), int(self.max_iter), float(self.eps))


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr()) if t is not None else None


def _flat(t: torch.Tensor) -> torch.Tensor:
    if not t.is_cuda:
        raise EDKMError("tensors must be CUDA tensors (no CPU fallback)")
    if not t.is_contiguous():
        raise EDKMError("tensors must be contiguous")
    return t.reshape(-1)


def _tensor_array(ws):
    arr = (_Tensor * max(len(ws), 1))()
    for i, w in enumerate(ws):
        arr[i].w = w.data_ptr() if w.numel() else None
        arr[i].n = w.numel()
    return arr


def _ptr_array(ts):
    arr = (ctypes.c_void_p * max(len(ts), 1))()
    for i, t in enumerate(ts):
        arr[i] = t.data_ptr() if t.numel() else None
    return arr


def _comm(comm):
    return None if comm is None else comm.handle


class Comm:
    """The library's NCCL communicator of the learners (edkm_comm): one per rank, on the current
    CUDA device.  Rank 0 draws the NCCL unique id (edkm_comm_unique_id) and the id reaches the other
    ranks through `torch.distributed` (the only thing it is used for); edkm_comm_init then builds the
    communicator inside the library, and the library's own calls (uniquify / backward_reduce with
    comm=, allreduce, allgather) run the collectives on the caller's stream."""

    def __init__(self, group=None):
        import torch.distributed as dist
        self.rank = dist.get_rank(group) if dist.is_initialized() else 0
        self.nranks = dist.get_world_size(group) if dist.is_initialized() else 1
        uid = (ctypes.c_uint8 * 128)()
        if self.rank == 0:
            _check(lib().edkm_comm_unique_id(uid), "edkm_comm_unique_id")
        if self.nranks > 1:
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=dist.get_global_rank(group, 0) if group is not None else 0,
                                       group=group)
            ctypes.memmove(uid, obj[0], 128)
        h = ctypes.c_void_p()
        _check(lib().edkm_comm_init(ctypes.byref(h), uid, self.rank, self.nranks), "edkm_comm_init")
        self.handle = h
        r, n, v = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _check(lib().edkm_comm_info(h, ctypes.byref(r), ctypes.byref(n), ctypes.byref(v)), "edkm_comm_info")
        self.nccl_version = v.value
        if (r.value, n.value) != (self.rank, self.nranks):
            raise EDKMError(f"edkm_comm rank/nranks {r.value}/{n.value} != {self.rank}/{self.nranks}")

    def allreduce(self, t: torch.Tensor, op: int = SUM, stream=None) -> torch.Tensor:
        """In-place all-reduce (SUM or MAX) of a contiguous CUDA tensor (int32, fp64, fp32 or uint8)."""
        t = _flat(t)
        _check(lib().edkm_comm_allreduce(self.handle, _ptr(t), t.numel(), _DT[t.dtype], op, _stream(stream)),
               "edkm_comm_allreduce")
        return t

    def allgather_blocks(self, full: torch.Tensor, stream=None) -> torch.Tensor:
        """In place: rank r's block is rows [r n/P, (r+1) n/P) of `full`; afterwards every rank has all."""
        if full.shape[0] % self.nranks:
            raise EDKMError("allgather_blocks: rows not divisible by the number of ranks")
        b = full.shape[0] // self.nranks
        nb = full[0:b].numel() * full.element_size()
        if not full.is_contiguous():
            raise EDKMError("allgather_blocks needs a contiguous tensor")
        send = ctypes.c_void_p(full.data_ptr() + self.rank * nb)
        _check(lib().edkm_comm_allgather(self.handle, send, _ptr(full), nb, _stream(stream)), "edkm_comm_allgather")
        return full

    def close(self):
        if getattr(self, "handle", None) is not None and self.handle.value:
            torch.cuda.synchronize()
            _check(lib().edkm_comm_destroy(self.handle), "edkm_comm_destroy")
            self.handle = None


def count_pages(counts: torch.Tensor, mask: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """uint8 [nt][256]: 1 where a 256-pattern page of counts has a nonzero entry (edkm_count_pages)."""
    nt = counts.shape[0]
    mask = torch.empty((nt, 256), dtype=torch.uint8, device=counts.device) if mask is None else mask
    _check(lib().edkm_count_pages(_ptr(counts), nt, _ptr(mask), _stream(stream)), "edkm_count_pages")
    return mask


def counts_pack(counts: torch.Tensor, pages: torch.Tensor, compact: torch.Tensor, stream=None):
    """compact[i] = page pages[i] of counts (edkm_counts_pack); pages: int32 global page ids t*256 + p."""
    _check(lib().edkm_counts_pack(_ptr(counts), counts.shape[0], _ptr(pages), pages.numel(), _ptr(compact),
                                  _stream(stream)), "edkm_counts_pack")
    return compact


def counts_unpack(compact: torch.Tensor, pages: torch.Tensor, counts: torch.Tensor, stream=None):
    """page pages[i] of counts = compact[i] (edkm_counts_unpack)."""
    _check(lib().edkm_counts_unpack(_ptr(compact), _ptr(pages), pages.numel(), counts.shape[0], _ptr(counts),
                                    _stream(stream)), "edkm_counts_unpack")
    return counts


def saved_bytes(nt: int, p: Params) -> int:
    return lib().edkm_saved_bytes(nt, ctypes.byref(p.c()))


def workspace_bytes(nt: int, p: Params) -> int:
    return lib().edkm_workspace_bytes(nt, ctypes.byref(p.c()))


# ----------------------------------------------------------------------------- functional API
def uniquify(weights, p: Params, counts: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    ws = [_flat(w) for w in weights]
    for w in ws:
        if w.dtype != p.wdtype:
            raise EDKMError("all weights must have the params' dtype")
    if counts is None:
        counts = torch.empty((len(ws), PATTERNS), dtype=torch.int32, device=ws[0].device if ws else "cuda")
    _check(lib().edkm_uniquify(_tensor_array(ws), len(ws), _DT[p.wdtype], _ptr(counts), None, _stream(stream)),
           "edkm_uniquify")
    return counts


def forward(counts: torch.Tensor, C0: torch.Tensor, p: Params, saved=None, C_out=None, table=None, stream=None):
    nt = counts.shape[0]
    dev = counts.device
    C0 = C0.to(device=dev, dtype=torch.float32).contiguous()
    if C0.shape != (nt, p.k):
        raise EDKMError(f"C0 must have shape ({nt}, {p.k})")
    if saved is None:
        saved = torch.empty(saved_bytes(nt, p), dtype=torch.uint8, device=dev)
    C_out = torch.empty((nt, p.k), dtype=torch.float32, device=dev) if C_out is None else C_out
    table = torch.empty((nt, PATTERNS), dtype=torch.float32, device=dev) if table is None else table
    _check(lib().edkm_forward(_ptr(counts), nt, ctypes.byref(p.c()), _ptr(C0), _ptr(C_out), _ptr(table),
                              _ptr(saved), _stream(stream)), "edkm_forward")
    return C_out, table, saved


def reconstruct(weights, p: Params, table, C_out, saved, mode: int = SOFT, out_dtype: torch.dtype | None = None,
                outs=None, stream=None):
    ws = [_flat(w) for w in weights]
    if out_dtype is None:
        out_dtype = torch.uint8 if mode == HARD_INDEX else p.wdtype
    if outs is None:
        outs = [torch.empty_like(w, dtype=out_dtype) for w in ws]
    _check(lib().edkm_reconstruct(_tensor_array(ws), len(ws), ctypes.byref(p.c()), _ptr(table), _ptr(C_out),
                                  _ptr(saved), mode, _DT[out_dtype], _ptr_array([o.reshape(-1) for o in outs]),
                                  _stream(stream)), "edkm_reconstruct")
    return outs


def backward_reduce(weights, grads, p: Params, counts, saved, ws_buf, gamma=None, stream=None):
    ws = [_flat(w) for w in weights]
    gs = [_flat(g) for g in grads]
    gdt = _DT[gs[0].dtype] if gs else _DT[p.wdtype]
    gamma = torch.empty((len(ws), p.k), dtype=torch.float64, device=counts.device) if gamma is None else gamma
    _check(lib().edkm_backward_reduce(_tensor_array(ws), len(ws), ctypes.byref(p.c()), _ptr_array(gs), gdt,
                                      _ptr(counts), _ptr(saved), _ptr(ws_buf), _ptr(gamma), None, _stream(stream)),
           "edkm_backward_reduce")
    return gamma


def backward_apply(weights, grads, p: Params, counts, saved, ws_buf, gamma, dW=None, dw_dtype=None, dC0=None,
                   stream=None):
    ws = [_flat(w) for w in weights]
    gs = [_flat(g) for g in grads]
    gdt = _DT[gs[0].dtype] if gs else _DT[p.wdtype]
    dw_dtype = dw_dtype or p.wdtype
    dW = [torch.empty_like(w, dtype=dw_dtype) for w in ws] if dW is None else dW
    dC0 = torch.empty((len(ws), p.k), dtype=torch.float32, device=counts.device) if dC0 is None else dC0
    _check(lib().edkm_backward_apply(_tensor_array(ws), len(ws), ctypes.byref(p.c()), _ptr_array(gs), gdt,
                                     _ptr(counts), _ptr(saved), _ptr(ws_buf), _ptr(gamma),
                                     _ptr_array([d.reshape(-1) for d in dW]), _DT[dw_dtype], _ptr(dC0),
                                     _stream(stream)), "edkm_backward_apply")
    return dW, dC0


def backward(weights, grads, p: Params, counts, saved, ws_buf=None, dW=None, dw_dtype=None, dC0=None, stream=None):
    ws = [_flat(w) for w in weights]
    gs = [_flat(g) for g in grads]
    gdt = _DT[gs[0].dtype] if gs else _DT[p.wdtype]
    dw_dtype = dw_dtype or p.wdtype
    if ws_buf is None:
        ws_buf = torch.empty(workspace_bytes(len(ws), p), dtype=torch.uint8, device=counts.device)
    dW = [torch.empty_like(w, dtype=dw_dtype) for w in ws] if dW is None else dW
    dC0 = torch.empty((len(ws), p.k), dtype=torch.float32, device=counts.device) if dC0 is None else dC0
    _check(lib().edkm_backward(_tensor_array(ws), len(ws), ctypes.byref(p.c()), _ptr_array(gs), gdt, _ptr(counts),
                               _ptr(saved), _ptr(ws_buf), _ptr_array([d.reshape(-1) for d in dW]), _DT[dw_dtype],
                               _ptr(dC0), _stream(stream)), "edkm_backward")
    return dW, dC0


def read_status(saved, nt: int, p: Params, stream=None):
    """(nonfinite weights per tensor, iterations run per tensor); synchronises the stream."""
    nf = (ctypes.c_int64 * max(nt, 1))()
    it = (ctypes.c_int32 * max(nt, 1))()
    _check(lib().edkm_read_status(_ptr(saved), nt, ctypes.byref(p.c()), nf, it, _stream(stream)), "edkm_read_status")
    return list(nf)[:nt], list(it)[:nt]


# ----------------------------------------------------------------------------- reusable step plan
class Plan:
    """Buffers of one eDKM step over a fixed list of tensors (no allocation per step).

    A step is: uniquify -> [all-reduce counts] -> forward -> reconstruct ->
    backward_reduce -> [all-reduce gamma] -> backward_apply.  The bracketed
    collectives are the caller's (paper_2309_00964_b200.dist); single-process
    callers skip them.
    """

    def __init__(self, numels, p: Params, device="cuda"):
        self.p = p
        self.nt = len(numels)
        self.numels = list(numels)
        dev = torch.device(device)
        self.counts = torch.empty((self.nt, PATTERNS), dtype=torch.int32, device=dev)
        self.C_out = torch.empty((self.nt, p.k), dtype=torch.float32, device=dev)
        self.table = torch.empty((self.nt, PATTERNS), dtype=torch.float32, device=dev)
        self.saved = torch.empty(saved_bytes(self.nt, p), dtype=torch.uint8, device=dev)
        self.ws = torch.empty(workspace_bytes(self.nt, p), dtype=torch.uint8, device=dev)
        self.gamma = torch.empty((self.nt, p.k), dtype=torch.float64, device=dev)
        self.dC0 = torch.empty((self.nt, p.k), dtype=torch.float32, device=dev)
        self._cache = {}

    def _n(self, tensors, what):
        """Every list a Plan call passes to the C ABI holds exactly nt tensors of the planned sizes:
        a shorter list would make the library read past the host array."""
        if len(tensors) != self.nt:
            raise EDKMError(f"{what}: {len(tensors)} tensors, the plan has {self.nt}")
        for t, n in zip(tensors, self.numels):
            if t.numel() != n:
                raise EDKMError(f"{what}: a tensor of {t.numel()} elements where the plan has {n}")

    def _arr(self, key, tensors, maker):
        ptrs = tuple(t.data_ptr() for t in tensors)
        hit = self._cache.get(key)
        if hit is None or hit[0] != ptrs:
            hit = (ptrs, maker([_flat(t) for t in tensors]))
            self._cache[key] = hit
        return hit[1]

    def uniquify(self, weights, stream=None, comm=None):
        """F1; with `comm` (a Comm) the counts are summed over the ranks inside the call."""
        self._n(weights, "weights")
        _check(lib().edkm_uniquify(self._arr("w", weights, _tensor_array), self.nt, _DT[self.p.wdtype],
                                   _ptr(self.counts), _comm(comm), _stream(stream)), "edkm_uniquify")
        return self.counts

    def uniquify_nvls(self, weights, nvls, stream=None):
        """F1 with the cross-rank count sum done in the NVSwitch (edkm_uniquify_nvls); `nvls` is a
        dist.NvlsCounts.  Leaves self.counts = this step's local view of the global counts."""
        self._n(weights, "weights")
        x = nvls.next_step(stream)
        _check(lib().edkm_uniquify_nvls(self._arr("w", weights, _tensor_array), self.nt, _DT[self.p.wdtype],
                                        ctypes.byref(x), _stream(stream)), "edkm_uniquify_nvls")
        self.counts = nvls.current
        return self.counts

    # the page-compact count exchange (include/edkm.h; dist.ShardedStep(compact_counts=True))
    def count_pages(self, stream=None):
        """uint8 [nt][256]: pages of this rank's counts with a nonzero entry (edkm_count_pages)."""
        if getattr(self, "_mask", None) is None:
            self._mask = torch.empty((max(self.nt, 1), 256), dtype=torch.uint8, device=self.counts.device)
        return count_pages(self.counts, self._mask[:self.nt], stream)

    def pack_counts(self, pages: torch.Tensor, stream=None) -> torch.Tensor:
        """int32 [len(pages)][256]: the listed pages of the counts, in list order (edkm_counts_pack)."""
        if getattr(self, "_compact", None) is None:
            self._compact = torch.empty((max(self.nt, 1) * 256, 256), dtype=torch.int32, device=self.counts.device)
        return counts_pack(self.counts, pages, self._compact[:pages.numel()], stream)

    def unpack_counts(self, pages: torch.Tensor, compact: torch.Tensor, stream=None):
        """The listed pages of the counts = compact (edkm_counts_unpack)."""
        return counts_unpack(compact, pages, self.counts, stream)

    def forward(self, C0, stream=None):
        _check(lib().edkm_forward(_ptr(self.counts), self.nt, ctypes.byref(self.p.c()), _ptr(C0), _ptr(self.C_out),
                                  _ptr(self.table), _ptr(self.saved), _stream(stream)), "edkm_forward")
        return self.C_out

    def forward_range(self, t0, t1, C0, stream=None):
        """TF for tensors [t0, t1) only (edkm_forward_range)."""
        _check(lib().edkm_forward_range(_ptr(self.counts), self.nt, t0, t1, ctypes.byref(self.p.c()), _ptr(C0),
                                        _ptr(self.C_out), _ptr(self.table), _ptr(self.saved), _stream(stream)),
               "edkm_forward_range")
        return self.C_out

    def forward_layout_range(self, t0, t1, stream=None):
        """TF's layout part only for tensors [t0, t1) (edkm_forward_layout_range)."""
        _check(lib().edkm_forward_layout_range(_ptr(self.counts), self.nt, t0, t1, ctypes.byref(self.p.c()),
                                               _ptr(self.table), _ptr(self.saved), _stream(stream)),
               "edkm_forward_layout_range")

    def pack_pages(self, name, pages: torch.Tensor, out: torch.Tensor, stream=None):
        """The listed pages of the per-pattern table `name` (a views() array) into `out` (edkm_pages_pack)."""
        v = self.views()[name]
        es = v.shape[1] // 65536
        _check(lib().edkm_pages_pack(_ptr(v), es, self.nt, _ptr(pages), pages.numel(), _ptr(out), _stream(stream)),
               "edkm_pages_pack")
        return out

    def unpack_pages(self, name, pages: torch.Tensor, src: torch.Tensor, stream=None):
        """The listed pages of the per-pattern table `name` = src (edkm_pages_unpack)."""
        v = self.views()[name]
        es = v.shape[1] // 65536
        _check(lib().edkm_pages_unpack(_ptr(src), es, _ptr(pages), pages.numel(), self.nt, _ptr(v), _stream(stream)),
               "edkm_pages_unpack")

    def backward_table_range(self, t0, t1, stream=None):
        """TB for tensors [t0, t1) only (edkm_backward_table_range)."""
        _check(lib().edkm_backward_table_range(self.nt, t0, t1, ctypes.byref(self.p.c()), _ptr(self.counts),
                                               _ptr(self.saved), _ptr(self.ws), _ptr(self.gamma), _ptr(self.dC0),
                                               _stream(stream)), "edkm_backward_table_range")
        return self.dC0

    SAVED_ARRAYS = ("state", "ctraj", "straj", "rows", "table16", "idx8", "page_cnt")
    WS_ARRAYS = ("B", "psi", "phipsi", "gamma")

    def views(self):
        """uint8 views [nt][bytes per tensor] of every per-tensor array of `saved` and `ws` (edkm_layout),
        plus the C_out / table / dC0 buffers: the blocks ranks exchange when they split the table phase."""
        if getattr(self, "_views", None) is None:
            so = (ctypes.c_size_t * 8)()
            wo = (ctypes.c_size_t * 5)()
            _check(lib().edkm_layout(self.nt, ctypes.byref(self.p.c()), so, wo), "edkm_layout")
            nt = max(self.nt, 1)
            v = {}
            sizes = {"state": 144, "ctraj": (self.p.max_iter + 1) * self.p.k * 8,
                     "straj": max(self.p.max_iter, 1) * self.p.k * 8, "rows": PATTERNS * 2, "table16": PATTERNS * 2,
                     "idx8": PATTERNS, "page_cnt": 256 * 8}
            for i, name in enumerate(self.SAVED_ARRAYS):
                v[name] = self.saved[so[i]:so[i] + nt * sizes[name]].view(nt, sizes[name])
            wsz = {"B": PATTERNS * 8, "psi": PATTERNS * 8, "phipsi": PATTERNS * 8, "gamma": self.p.k * 8}
            for i, name in enumerate(self.WS_ARRAYS):
                v[name] = self.ws[wo[i]:wo[i] + nt * wsz[name]].view(nt, wsz[name])
            for name in ("C_out", "table", "dC0"):
                t = getattr(self, name)
                v[name] = t.view(torch.uint8).view(nt, -1)
            self._views = v
        return self._views

    def reconstruct(self, weights, outs, mode=SOFT, stream=None):
        self._n(weights, "weights")
        self._n(outs, "outs")
        odt = _DT[outs[0].dtype] if outs else _DT[self.p.wdtype]
        _check(lib().edkm_reconstruct(self._arr("w", weights, _tensor_array), self.nt, ctypes.byref(self.p.c()),
                                      _ptr(self.table), _ptr(self.C_out), _ptr(self.saved), mode, odt,
                                      self._arr(("o", mode), outs, _ptr_array), _stream(stream)), "edkm_reconstruct")
        return outs

    def backward_reduce(self, weights, grads, stream=None, comm=None):
        """B1 + TGAMMA; with `comm` gamma_T is summed over the ranks inside the call."""
        self._n(weights, "weights")
        self._n(grads, "grads")
        gdt = _DT[grads[0].dtype] if grads else _DT[self.p.wdtype]
        _check(lib().edkm_backward_reduce(self._arr("w", weights, _tensor_array), self.nt, ctypes.byref(self.p.c()),
                                          self._arr("g", grads, _ptr_array), gdt, _ptr(self.counts),
                                          _ptr(self.saved), _ptr(self.ws), _ptr(self.gamma), _comm(comm),
                                          _stream(stream)), "edkm_backward_reduce")
        return self.gamma

    # the four backward kernels individually (B1, TGAMMA, TB, B2)
    def backward_buckets(self, weights, grads, stream=None):
        self._n(weights, "weights")
        self._n(grads, "grads")
        gdt = _DT[grads[0].dtype] if grads else _DT[self.p.wdtype]
        _check(lib().edkm_backward_buckets(self._arr("w", weights, _tensor_array), self.nt, ctypes.byref(self.p.c()),
                                           self._arr("g", grads, _ptr_array), gdt, _ptr(self.saved), _ptr(self.ws),
                                           _stream(stream)), "edkm_backward_buckets")

    def backward_gamma(self, stream=None):
        _check(lib().edkm_backward_gamma(self.nt, ctypes.byref(self.p.c()), _ptr(self.counts), _ptr(self.saved),
                                         _ptr(self.ws), _ptr(self.gamma), _stream(stream)), "edkm_backward_gamma")
        return self.gamma

    def backward_table(self, stream=None):
        _check(lib().edkm_backward_table(self.nt, ctypes.byref(self.p.c()), _ptr(self.counts), _ptr(self.saved),
                                         _ptr(self.ws), _ptr(self.gamma), _ptr(self.dC0), _stream(stream)),
               "edkm_backward_table")
        return self.dC0

    def backward_dw(self, weights, grads, dW, stream=None):
        self._n(weights, "weights")
        self._n(grads, "grads")
        self._n(dW, "dW")
        gdt = _DT[grads[0].dtype] if grads else _DT[self.p.wdtype]
        ddt = _DT[dW[0].dtype] if dW else _DT[self.p.wdtype]
        _check(lib().edkm_backward_dw(self._arr("w", weights, _tensor_array), self.nt, ctypes.byref(self.p.c()),
                                      self._arr("g", grads, _ptr_array), gdt, _ptr(self.saved), _ptr(self.ws),
                                      self._arr("dw", dW, _ptr_array), ddt, _stream(stream)), "edkm_backward_dw")
        return dW

    def backward_apply(self, weights, grads, dW, stream=None):
        self._n(weights, "weights")
        self._n(grads, "grads")
        self._n(dW, "dW")
        gdt = _DT[grads[0].dtype] if grads else _DT[self.p.wdtype]
        ddt = _DT[dW[0].dtype] if dW else _DT[self.p.wdtype]
        _check(lib().edkm_backward_apply(self._arr("w", weights, _tensor_array), self.nt, ctypes.byref(self.p.c()),
                                         self._arr("g", grads, _ptr_array), gdt, _ptr(self.counts), _ptr(self.saved),
                                         _ptr(self.ws), _ptr(self.gamma), self._arr("dw", dW, _ptr_array), ddt,
                                         _ptr(self.dC0), _stream(stream)), "edkm_backward_apply")
        return self.dC0

    def step(self, weights, grads, C0, outs, dW, allreduce=None, stream=None):
        """One full fwd+bwd over all tensors.  `allreduce(tensor)` sums in place over ranks."""
        self.uniquify(weights, stream)
        if allreduce is not None:
            allreduce(self.counts)
        self.forward(C0, stream)
        self.reconstruct(weights, outs, SOFT, stream)
        self.backward_reduce(weights, grads, stream)
        if allreduce is not None:
            allreduce(self.gamma)
        self.backward_apply(weights, grads, dW, stream)
        return self.dC0

    def graph(self, weights, grads, C0, outs, dW, allreduce=None):
        """Capture one `step` over these buffers into a CUDA graph and return it (a
        torch.cuda.CUDAGraph): `replay()` re-runs the whole step -- memsets, the seven kernels and
        the collectives, if any -- with no per-launch host work.  Each replay reads whatever the
        captured input tensors (weights, grads, C0) hold and writes the captured outputs."""
        side = torch.cuda.Stream(self.counts.device)
        side.wait_stream(torch.cuda.current_stream(self.counts.device))
        with torch.cuda.stream(side):  # one eager step first: kernel attributes, cached pointer arrays
            self.step(weights, grads, C0, outs, dW, allreduce)
        torch.cuda.current_stream(self.counts.device).wait_stream(side)
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            self.step(weights, grads, C0, outs, dW, allreduce)
        return g


# ----------------------------------------------------------------------------- autograd wrapper
class EDKMFunction(torch.autograd.Function):
    """W~ = DKM(W, C0) for one weight tensor on this device (differentiable in W and C0).

    The attention table never materialises per weight: forward saves only the
    O(T k) trajectory and the per-pattern tables, backward runs TB + B2.
    """

    @staticmethod
    def forward(ctx, W, C0, p: Params):
        w = W.detach().contiguous()
        counts = uniquify([w], p)
        C_out, table, saved = forward(counts, C0.detach().reshape(1, -1), p)
        (Wt,) = reconstruct([w], p, table, C_out, saved, SOFT, W.dtype)
        ctx.p = p
        ctx.C0_shape, ctx.C0_dtype = C0.shape, C0.dtype  # dC0 is returned in C0's shape and dtype
        ctx.save_for_backward(w, counts, saved)
        return Wt.view_as(W)

    @staticmethod
    def backward(ctx, G):
        w, counts, saved = ctx.saved_tensors
        g = G.contiguous()
        if g.dtype not in (ctx.p.wdtype, torch.float32):
            g = g.float()
        (dW,), dC0 = backward([w], [g], ctx.p, counts, saved, dw_dtype=w.dtype)
        return dW.view_as(w), dC0.reshape(ctx.C0_shape).to(ctx.C0_dtype), None


def edkm(W: torch.Tensor, C0: torch.Tensor, bits: int = 3, tau: float = 1e-3, max_iter: int = 5, eps: float = 0.0):
    """Differentiable soft-clustered weight W~ (Fig. 1) computed by the CUDA path."""
    return EDKMFunction.apply(W, C0, Params(W.dtype, bits, tau, max_iter, eps))
