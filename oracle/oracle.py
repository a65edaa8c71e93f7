"""Python front of the CPU oracle (oracle/edkm_oracle.c) -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / ``--impl
reference`` legs may import this module.  The product package
(paper_2309_00964_b200/) never imports it, and the two share no code: this file
marshals numpy arrays into liboracle.so, a plain dense fp64 C implementation of
DKM written from the paper (see the header of edkm_oracle.c for the passage
each function follows and the pins in tests/test_oracle.py).

Functions follow PAPER.md and DESIGN.md readings:
  histogram      P:77, Fig. 3 -- counts per 16-bit pattern
  decode16       P:77 -- exact value of each bf16/fp16 pattern
  attention      north star / R1 -- softmax(-(w-c)^2/tau) rows
  dkm_forward    R2-R6 -- unrolled soft k-means, dense or with multiplicities
  reconstruct    Fig. 1, R2 -- W~ = A(C_T) . C_T
  dkm_backward   R3, R6 -- dense chain rule to dW and dC_0
  dkm_backward_table  P:77 table form -- (phi, psi) per pattern, dC_0
  hard_assign    P:31, R9 -- nearest centroid, lowest index on ties

The eps > 0 stopping decision (R4) is pinned against textbook Lloyd k-means
in exact rational arithmetic (tests/test_oracle.py::test_eps_stop_pinned_to_lloyd).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "edkm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None

BF16, FP16 = 0, 1


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (-O2, no fast-math: IEEE fp64 throughout)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        cmd = ["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math", "-ffp-contract=off",
               "-pthread", "-o", _LIB, _SRC, "-lm"]
        subprocess.run(cmd, check=True)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(build())
        P = ctypes.c_void_p
        i64, i32, f64 = ctypes.c_int64, ctypes.c_int, ctypes.c_double
        _lib.oracle_decode16.argtypes = [P, i64, i32, P]
        _lib.oracle_decode16.restype = i32
        _lib.oracle_histogram.argtypes = [P, i64, P]
        _lib.oracle_histogram.restype = None
        _lib.oracle_attention.argtypes = [P, i64, P, i32, f64, P]
        _lib.oracle_attention.restype = None
        _lib.oracle_dkm_forward.argtypes = [P, P, i64, i32, P, f64, i32, f64, i32, P, P, P]
        _lib.oracle_dkm_forward.restype = i32
        _lib.oracle_reconstruct.argtypes = [P, i64, P, i32, f64, P]
        _lib.oracle_reconstruct.restype = None
        _lib.oracle_hard_assign.argtypes = [P, i64, P, i32, P]
        _lib.oracle_hard_assign.restype = None
        _lib.oracle_dkm_backward.argtypes = [P, P, i64, i32, f64, i32, P, P, i32, P, P]
        _lib.oracle_dkm_backward.restype = i32
        _lib.oracle_dkm_backward_table.argtypes = [P, P, P, i64, i32, f64, i32, P, P, P, P, P, P]
        _lib.oracle_dkm_backward_table.restype = i32
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def decode16(bits, dtype: int) -> np.ndarray:
    """Exact fp64 value of each 16-bit pattern (dtype BF16=0 / FP16=1)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16)
    out = np.empty(b.size, np.float64)
    if _load().oracle_decode16(_p(b), b.size, dtype, _p(out)) != 0:
        raise ValueError("bad dtype")
    return out.reshape(b.shape)


def histogram(bits) -> np.ndarray:
    """counts[u] = #{i : bits_i == u}, int64[65536] (Fig. 3)."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).ravel()
    c = np.zeros(65536, np.int64)
    _load().oracle_histogram(_p(b), b.size, _p(c))
    return c


def attention(w, C, tau: float) -> np.ndarray:
    """Dense attention map A[i, j] (n x k)."""
    w, C = _f64(w).ravel(), _f64(C)
    A = np.empty((w.size, C.size), np.float64)
    _load().oracle_attention(_p(w), w.size, _p(C), C.size, tau, _p(A))
    return A


def dkm_forward(w, C0, tau: float, max_iter: int, eps: float = 0.0, mult=None, nthreads: int = 0):
    """Returns (C_traj[T+1, k], S_traj[T, k], T)."""
    w, C0 = _f64(w).ravel(), _f64(C0)
    k = C0.size
    m = None if mult is None else _f64(mult).ravel()
    if m is not None and m.size != w.size:
        raise ValueError("mult size")
    Ct = np.zeros((max_iter + 1) * k, np.float64)
    St = np.zeros(max(max_iter, 1) * k, np.float64)
    T = ctypes.c_int(0)
    rc = _load().oracle_dkm_forward(_p(w), None if m is None else _p(m), w.size, k, _p(C0), float(tau),
                                    int(max_iter), float(eps), int(nthreads), _p(Ct), _p(St), ctypes.byref(T))
    if rc != 0:
        raise ValueError("oracle_dkm_forward: bad arguments")
    T = T.value
    return Ct.reshape(-1, k)[: T + 1].copy(), St.reshape(-1, k)[:T].copy(), T


def reconstruct(w, C, tau: float) -> np.ndarray:
    """W~_i = sum_j A(w_i, C)[j] C[j] (reading R2: pass C = C_T)."""
    w, C = _f64(w), _f64(C)
    out = np.empty(w.size, np.float64)
    _load().oracle_reconstruct(_p(w.ravel()), w.size, _p(C), C.size, float(tau), _p(out))
    return out.reshape(w.shape)


def hard_assign(w, C_f32) -> np.ndarray:
    """argmin_j (w - C[j])^2 in fp64 from the fp32 table C, lowest j on ties."""
    w = _f64(w)
    C = np.ascontiguousarray(C_f32, dtype=np.float32)
    idx = np.empty(w.size, np.int32)
    _load().oracle_hard_assign(_p(w.ravel()), w.size, _p(C), C.size, _p(idx))
    return idx.reshape(w.shape)


def dkm_backward(w, G, C_traj, S_traj, tau: float, nthreads: int = 0):
    """Dense backward. Returns (dW[n], dC0[k])."""
    w, G = _f64(w).ravel(), _f64(G).ravel()
    Ct, St = _f64(C_traj), _f64(S_traj)
    T, k = Ct.shape[0] - 1, Ct.shape[1]
    St = St if St.size else np.zeros((1, k))
    dW = np.empty(w.size, np.float64)
    dC = np.empty(k, np.float64)
    rc = _load().oracle_dkm_backward(_p(w), _p(G), w.size, k, float(tau), T, _p(Ct), _p(np.ascontiguousarray(St)),
                                     int(nthreads), _p(dW), _p(dC))
    if rc != 0:
        raise ValueError("oracle_dkm_backward: bad arguments")
    return dW, dC


def dkm_backward_table(v, cnt, B, C_traj, S_traj, tau: float, gammaT=None):
    """Attention-table backward on unique values v with counts cnt and bucket sums
    B[u] = sum_{i in u} G_i.  Returns (phi[m], psi[m], dC0[k]); dW_i = G_i phi + psi.
    If gammaT is given (e.g. summed over learners) it replaces sum_u B[u] f_T(u, .)
    and B may be None.  With T = 0 the returned dC0 is gamma_T itself."""
    v, cnt = _f64(v).ravel(), _f64(cnt).ravel()
    B = None if B is None else _f64(B).ravel()
    g = None if gammaT is None else _f64(gammaT).ravel()
    Ct, St = _f64(C_traj), _f64(S_traj)
    T, k = Ct.shape[0] - 1, Ct.shape[1]
    St = St if St.size else np.zeros((1, k))
    phi, psi, dC = np.empty(v.size), np.empty(v.size), np.empty(k)
    rc = _load().oracle_dkm_backward_table(_p(v), _p(cnt), None if B is None else _p(B), v.size, k, float(tau), T,
                                           _p(Ct), _p(np.ascontiguousarray(St)), None if g is None else _p(g),
                                           _p(phi), _p(psi), _p(dC))
    if rc != 0:
        raise ValueError("oracle_dkm_backward_table: bad arguments")
    return phi, psi, dC
