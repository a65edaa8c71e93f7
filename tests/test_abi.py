"""CPU-side checks of the C ABI boundary: libedkm.so builds, loads without a GPU,
exports every entry point include/edkm.h declares, and rejects bad arguments
before launching anything (include/edkm.h "Conventions")."""
import ctypes
import os
import re

import pytest

from paper_2309_00964_b200 import build as B
from paper_2309_00964_b200 import edkm as E

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    B.build()
    return E.lib()


def declared_functions():
    h = open(os.path.join(ROOT, "include", "edkm.h")).read()
    h = re.sub(r"/\*.*?\*/", "", h, flags=re.S)
    return sorted(set(re.findall(r"\b(edkm_[a-z_]+)\s*\(", h)))


def test_header_declares_the_north_star_calls():
    names = declared_functions()
    for n in ("edkm_uniquify", "edkm_forward", "edkm_backward", "edkm_reconstruct"):
        assert n in names


def test_every_declared_symbol_is_exported(L):
    for n in declared_functions():
        assert hasattr(L, n), n
    assert sorted(E.exported_symbols()) == declared_functions()


def test_bad_arguments_return_errors_without_launch(L):
    p = E.Params()
    cp = ctypes.byref(p.c())
    assert L.edkm_uniquify(None, -1, 0, None, None, None) == 1
    assert L.edkm_uniquify(None, 1, 0, None, None, None) == 1           # NULL tensors
    assert L.edkm_uniquify(None, 0, 7, None, None, None) == 2           # bad dtype
    t = (E._Tensor * 1)()
    t[0].w, t[0].n = None, 5
    assert L.edkm_uniquify(t, 1, 0, ctypes.c_void_p(16), None, None) == 1   # n > 0 with NULL data
    t[0].w, t[0].n = 3, 5
    assert L.edkm_uniquify(t, 1, 0, ctypes.c_void_p(16), None, None) == 1   # odd address
    for bad in (E._Params(0, 3, -1.0, 5, 0.0), E._Params(0, 3, float("nan"), 5, 0.0), E._Params(0, 3, 1.0, -1, 0.0),
                E._Params(0, 3, 1.0, 5, -1.0), E._Params(0, 3, float("inf"), 5, 0.0)):
        assert L.edkm_forward(ctypes.c_void_p(16), 1, ctypes.byref(bad), ctypes.c_void_p(16), ctypes.c_void_p(16),
                              ctypes.c_void_p(16), ctypes.c_void_p(16), None) == 1
    assert L.edkm_forward(ctypes.c_void_p(16), 1, ctypes.byref(E._Params(0, 9, 1.0, 5, 0.0)), None, None, None, None,
                          None) == 4                              # bits > 8: unsupported
    assert L.edkm_forward(ctypes.c_void_p(16), 1, ctypes.byref(E._Params(0, 0, 1.0, 5, 0.0)), None, None, None, None,
                          None) == 4                              # bits < 1
    assert L.edkm_forward(ctypes.c_void_p(16), 1, ctypes.byref(E._Params(2, 3, 1.0, 5, 0.0)), None, None, None, None,
                          None) == 2                              # fp32 weights
    assert L.edkm_forward(None, 1, cp, None, None, None, None, None) == 1
    assert L.edkm_saved_bytes(-1, cp) == 0 and L.edkm_saved_bytes(3, cp) > 0
    assert L.edkm_workspace_bytes(226, cp) >= 226 * 65536 * 24
    assert L.edkm_last_error()
    assert L.edkm_status_string(0) == b"EDKM_OK"


def test_comm_and_exchange_arguments(L):
    """the communicator behind the ABI and the page-compact exchange reject bad arguments
    synchronously (nothing launched, no NCCL call), and EDKM_E_NCCL exists."""
    h = ctypes.c_void_p(1)
    assert L.edkm_comm_init(None, None, 0, 1) == 1
    uid = (ctypes.c_uint8 * 128)()
    assert L.edkm_comm_init(ctypes.byref(h), uid, 1, 1) == 1 and h.value is None   # rank outside [0, nranks)
    assert L.edkm_comm_init(ctypes.byref(h), uid, 0, 0) == 1                       # nranks < 1
    assert L.edkm_comm_unique_id(None) in (1, 5)
    assert L.edkm_comm_destroy(None) == 0
    assert L.edkm_comm_allreduce(None, None, 0, E.I32, E.SUM, None) == 1
    assert L.edkm_comm_allgather(None, None, None, 0, None) == 1
    assert L.edkm_count_pages(None, -1, None, None) == 1
    assert L.edkm_count_pages(None, 0, None, None) == 0
    assert L.edkm_count_pages(None, 2, None, None) == 1
    assert L.edkm_counts_pack(None, 1, None, 257, None, None) == 1                 # npages > 256 nt
    assert L.edkm_counts_pack(None, 1, None, 0, None, None) == 0
    assert L.edkm_counts_unpack(None, None, 3, 1, None, None) == 1
    assert L.edkm_status_string(5).startswith(b"EDKM_E_NCCL")
    assert L.edkm_pages_pack(None, 3, 1, None, 1, None, None) == 1                 # esize not 1/2/4/8
    assert L.edkm_pages_pack(None, 8, 1, None, 0, None, None) == 0
    assert L.edkm_pages_unpack(None, 2, None, 300, 1, None, None) == 1             # npages > 256 nt
    assert L.edkm_pages_pack(ctypes.c_void_p(8), 2, 1, ctypes.c_void_p(16), 1, ctypes.c_void_p(16), None) == 1  # misaligned
    p = E.Params()
    assert L.edkm_forward_layout_range(None, 2, 1, 3, ctypes.byref(p.c()), None, None, None) == 1  # range outside
    assert L.edkm_forward_layout_range(None, 2, 1, 1, ctypes.byref(p.c()), None, None, None) == 0  # empty range
    assert L.edkm_ipc_handle(None, None, None) == 1
    assert L.edkm_ipc_close(None) == 0


def test_empty_calls_are_noops(L):
    p = E.Params()
    cp = ctypes.byref(p.c())
    assert L.edkm_uniquify(None, 0, 0, None, None, None) == 0
    assert L.edkm_forward(None, 0, cp, None, None, None, None, None) == 0
    assert L.edkm_backward(None, 0, cp, None, 0, None, None, None, None, 0, None, None) == 0


def test_product_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_2309_00964_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                src = open(os.path.join(dirpath, f)).read()
                assert not re.search(r"(import\s+oracle|from\s+oracle|liboracle|edkm_oracle|oracle_dkm)", src), f


def test_pipeline_groups_cover_tensors_in_order():
    from paper_2309_00964_b200.pipeline import _groups
    for numels, g in (([5, 1, 1, 1, 10, 3], 3), ([1] * 10, 4), ([100], 8), ([0, 0, 5], 2)):
        gs = _groups(numels, g)
        assert sum(gs, []) == list(range(len(numels)))
        assert 1 <= len(gs) <= g and all(gs)


def test_range_layout_and_nvls_entry_points_check_arguments(L):
    """Tensor-range table phase, layout query and the NVLS-fused F1 reject bad arguments before
    any CUDA call (include/edkm.h conventions)."""
    p = E.Params()
    cp = ctypes.byref(p.c())
    one = ctypes.c_void_p(16)
    # ranges outside [0, nt] or reversed
    for t0, t1 in ((-1, 2), (2, 1), (0, 5)):
        assert L.edkm_forward_range(one, 4, t0, t1, cp, one, one, one, one, None) == 1
        assert L.edkm_backward_table_range(4, t0, t1, cp, one, one, one, one, one, None) == 1
    # empty range: nothing to do
    assert L.edkm_forward_range(one, 4, 2, 2, cp, one, one, one, one, None) == 0
    assert L.edkm_backward_table_range(4, 3, 3, cp, one, one, one, one, one, None) == 0
    # layout: offsets increase, the totals match the size queries, arrays hold nt entries each
    so = (ctypes.c_size_t * 8)()
    wo = (ctypes.c_size_t * 5)()
    nt = 7
    assert L.edkm_layout(nt, cp, so, wo) == 0
    assert list(so) == sorted(so) and so[7] == L.edkm_saved_bytes(nt, cp)
    assert list(wo) == sorted(wo) and wo[4] == L.edkm_workspace_bytes(nt, cp)
    assert so[4] - so[3] >= nt * 65536 * 2 and so[7] - so[6] >= nt * 256 * 8   # rows, page_cnt
    assert wo[3] - wo[2] >= nt * 65536 * 8                                        # (phi, psi)
    assert L.edkm_layout(-1, cp, so, wo) == 1
    # NVLS F1: missing buffers, bad rank count, emulation with several ranks
    x = E._Nvls(16, 16, 16, 16, 1, 0)
    assert L.edkm_uniquify_nvls(None, 0, 0, None, None) == 1
    assert L.edkm_uniquify_nvls(None, 0, 5, ctypes.byref(x), None) == 2
    assert L.edkm_uniquify_nvls(None, 0, 0, ctypes.byref(E._Nvls(0, 16, 16, 16, 1, 0)), None) == 1
    assert L.edkm_uniquify_nvls(None, 0, 0, ctypes.byref(E._Nvls(16, 16, 16, 16, 0, 0)), None) == 1
    assert L.edkm_uniquify_nvls(None, 0, 0, ctypes.byref(E._Nvls(16, 16, 16, 16, 2, 1)), None) == 1
    # multicast plumbing
    assert L.edkm_mc_create(0, 1, 0, None, None) == 1
    assert L.edkm_mc_import(-1, 1 << 21, None) == 1
    assert L.edkm_mc_add_device(None) == 1
    assert L.edkm_mc_bytes(None) == 0
    assert L.edkm_mc_destroy(None) == 0
    assert L.edkm_set_max_ctas(0) == 0 and L.edkm_set_max_ctas(3) == 0 and L.edkm_set_max_ctas(0) == 3
