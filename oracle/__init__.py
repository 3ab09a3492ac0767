"""CPU oracle for sparse CP-ALS — TEST INFRASTRUCTURE, NOT PRODUCT CODE.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package.  The product path
(``paper_1812_05961_b200``) never imports it and shares no code with it.

This is a ctypes wrapper over ``oracle/oracle.cpp`` (plain C++17 + OpenMP, fp64);
see that file's header for the paper passage each function follows.  Parity of
each function is pinned in ``tests/test_oracle_pins.py``.  Parity unpinned: the
multi-iteration ALS trajectory on random data beyond the per-step pins (SURVEY.md
§8(c) last row).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.cpp")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

OK, BADINPUT, SINGULAR, EMPTY = 0, -1, -3, -6


def build(force: bool = False) -> str:
    """Compile liboracle.so (g++ -O2 -fopenmp).  Cheap; rebuilt when stale."""
    if (not force and os.path.exists(_LIB)
            and os.path.getmtime(_LIB) >= os.path.getmtime(_SRC)):
        return _LIB
    tmp = _LIB + ".tmp.%d" % os.getpid()
    cmd = ["g++", "-std=c++17", "-O2", "-fopenmp", "-fPIC", "-shared",
           "-ffp-contract=off", _SRC, "-o", tmp]
    subprocess.check_call(cmd)
    os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_LIB)
            u64, i32, f64 = C.c_uint64, C.c_int, C.c_double
            P = C.c_void_p
            L.oracle_splitmix64_raw.restype = u64
            L.oracle_splitmix64_raw.argtypes = [u64, u64]
            L.oracle_u01.restype = f64
            L.oracle_u01.argtypes = [u64, u64]
            L.oracle_init_factors.argtypes = [i32, P, i32, u64, P]
            L.oracle_validate.argtypes = [i32, P, u64, P]
            L.oracle_norm_sq.restype = f64
            L.oracle_norm_sq.argtypes = [u64, P]
            L.oracle_gram.argtypes = [u64, i32, P, P]
            L.oracle_hadamard_except.argtypes = [i32, i32, P, i32, P]
            L.oracle_group_by_mode.argtypes = [u64, P, u64, P, P]
            L.oracle_mttkrp.argtypes = [i32, P, u64, P, P, i32, i32, P, P]
            L.oracle_cholesky_solve.argtypes = [i32, P, u64, P, P]
            L.oracle_normalize.argtypes = [u64, i32, P, i32, P]
            L.oracle_fit.restype = f64
            L.oracle_fit.argtypes = [i32, i32, P, P, u64, P, P, f64]
            L.oracle_cpd_als.argtypes = [i32, P, u64, P, P, i32, i32, f64, u64, P, P, P, P,
                                         P, P, P]
            L.oracle_csf_perm.argtypes = [i32, P, i32, P]
            L.oracle_csf_build.restype = P
            L.oracle_csf_build.argtypes = [i32, P, u64, P, P, i32]
            L.oracle_csf_perm_of.argtypes = [P, P]
            L.oracle_csf_nodes.restype = u64
            L.oracle_csf_nodes.argtypes = [P, i32]
            L.oracle_csf_copy.argtypes = [P, i32, P, P]
            L.oracle_csf_vals.argtypes = [P, P]
            L.oracle_csf_free.argtypes = [P]
            L.oracle_partition.argtypes = [P, u64, i32, P]
            L.oracle_csf_alloc.argtypes = [i32, P, i32, P, P, P, P]
            L.oracle_num_threads.restype = i32
            L.oracle_set_threads.argtypes = [i32]
            _lib = L
    return _lib


def _p(a):
    return a.ctypes.data_as(C.c_void_p)


def _ptrs(arrs, ctype=C.c_void_p):
    return (ctype * len(arrs))(*[a.ctypes.data for a in arrs])


def _dims(dims):
    return np.ascontiguousarray(np.asarray(dims, dtype=np.uint64))


def _ind(ind):
    return [np.ascontiguousarray(np.asarray(a, dtype=np.uint32)) for a in ind]


class OracleError(RuntimeError):
    def __init__(self, code):
        super().__init__(f"oracle status {code}")
        self.code = code


# ----------------------------------------------------------------------- C-2
def splitmix64_raw(seed: int, k: int) -> int:
    return int(lib().oracle_splitmix64_raw(seed, k))


def u01(seed: int, k: int) -> float:
    return float(lib().oracle_u01(seed, k))


def init_factors(dims, R, seed):
    out = [np.empty((int(d), R)) for d in dims]
    lib().oracle_init_factors(len(dims), _p(_dims(dims)), R, seed, _ptrs(out))
    return out


def set_threads(t: int) -> None:
    lib().oracle_set_threads(int(t))


def num_threads() -> int:
    return int(lib().oracle_num_threads())


# ---------------------------------------------------------------- C-1, C-3
def validate(dims, ind) -> int:
    ind = _ind(ind)
    nnz = ind[0].shape[0]
    return int(lib().oracle_validate(len(dims), _p(_dims(dims)), nnz, _ptrs(ind)))


def norm_sq(vals) -> float:
    v = np.ascontiguousarray(vals, dtype=np.float64)
    return float(lib().oracle_norm_sq(v.shape[0], _p(v)))


# ---------------------------------------------------------------- C-4 .. C-10
def gram(A):
    A = np.ascontiguousarray(A, dtype=np.float64)
    G = np.empty((A.shape[1], A.shape[1]))
    lib().oracle_gram(A.shape[0], A.shape[1], _p(A), _p(G))
    return G


def hadamard_except(grams, n):
    gs = [np.ascontiguousarray(g, dtype=np.float64) for g in grams]
    R = gs[0].shape[0]
    V = np.empty((R, R))
    lib().oracle_hadamard_except(len(gs), R, _ptrs(gs), n, _p(V))
    return V


def mttkrp(dims, ind, vals, factors, mode):
    """M = X_(mode) (KRP of the other factors) by definition (C-6).  ld = R."""
    ind = _ind(ind)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    fs = [np.ascontiguousarray(f, dtype=np.float64) for f in factors]
    R = fs[0].shape[1]
    M = np.empty((int(dims[mode]), R))
    st = lib().oracle_mttkrp(len(dims), _p(_dims(dims)), v.shape[0], _ptrs(ind), _p(v), mode, R,
                             _ptrs(fs), _p(M))
    if st:
        raise OracleError(st)
    return M


def cholesky_solve(V, M):
    V = np.ascontiguousarray(V, dtype=np.float64)
    M = np.ascontiguousarray(M, dtype=np.float64)
    X = np.empty_like(M)
    st = lib().oracle_cholesky_solve(V.shape[0], _p(V), M.shape[0], _p(M), _p(X))
    if st:
        raise OracleError(st)
    return X


def normalize(A, which):
    """which: 0 = 2-norm (iteration 1), 1 = max-norm (later).  Returns (A', lambda)."""
    A = np.array(A, dtype=np.float64, copy=True, order="C")
    lam = np.empty(A.shape[1])
    lib().oracle_normalize(A.shape[0], A.shape[1], _p(A), which, _p(lam))
    return A, lam


def fit(grams, lam, M_last, A_last, normx_sq):
    gs = [np.ascontiguousarray(g, dtype=np.float64) for g in grams]
    lam = np.ascontiguousarray(lam, dtype=np.float64)
    M_last = np.ascontiguousarray(M_last, dtype=np.float64)
    A_last = np.ascontiguousarray(A_last, dtype=np.float64)
    return float(lib().oracle_fit(len(gs), lam.shape[0], _ptrs(gs), _p(lam), A_last.shape[0],
                                  _p(M_last), _p(A_last), float(normx_sq)))


def cpd_als(dims, ind, vals, rank, max_iters, tol=0.0, seed=0, init=None, timings=False):
    """Full CP-ALS (C-1..C-12).  Returns dict(factors, lam, fit, iters, fit_history[, timings])."""
    ind = _ind(ind)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    N = len(dims)
    A = [np.empty((int(d), rank)) for d in dims]
    lam = np.empty(rank)
    hist = np.zeros(max_iters)
    iters = C.c_int(0)
    fitv = C.c_double(0.0)
    tm = np.zeros(7)
    init_p = None
    if init is not None:
        init = [np.ascontiguousarray(a, dtype=np.float64) for a in init]
        init_p = _ptrs(init)
    st = lib().oracle_cpd_als(N, _p(_dims(dims)), v.shape[0], _ptrs(ind), _p(v), rank,
                              max_iters, float(tol), seed, init_p, _ptrs(A), _p(lam), _p(hist),
                              C.byref(iters), C.byref(fitv), _p(tm))
    if st:
        raise OracleError(st)
    out = dict(factors=A, lam=lam, fit=fitv.value, iters=iters.value,
               fit_history=hist[:iters.value].copy())
    if timings:
        out["timings"] = dict(zip(["mttkrp", "sort", "mat_ata", "mat_norm", "cpd_fit",
                                   "inverse", "loop"], tm.tolist()))
    return out


# ---------------------------------------------------------------------- C-13
def csf_perm(dims, root):
    perm = np.zeros(len(dims), dtype=np.int32)
    lib().oracle_csf_perm(len(dims), _p(_dims(dims)), root, _p(perm))
    return perm


def csf_build(dims, ind, vals, root):
    """Returns dict(perm, ids=[...N levels], ptr=[...N-1 levels], vals)."""
    ind = _ind(ind)
    v = np.ascontiguousarray(vals, dtype=np.float64)
    N = len(dims)
    L = lib()
    h = L.oracle_csf_build(N, _p(_dims(dims)), v.shape[0], _ptrs(ind), _p(v), root)
    try:
        perm = np.zeros(N, dtype=np.int32)
        L.oracle_csf_perm_of(h, _p(perm))
        ids, ptr = [], []
        for l in range(N):
            n = int(L.oracle_csf_nodes(h, l))
            a = np.empty(n, dtype=np.uint32)
            b = np.empty(n + 1, dtype=np.uint32) if l < N - 1 else None
            L.oracle_csf_copy(h, l, _p(a), _p(b) if b is not None else None)
            ids.append(a)
            if b is not None:
                ptr.append(b)
        vv = np.empty(v.shape[0])
        L.oracle_csf_vals(h, _p(vv))
    finally:
        L.oracle_csf_free(h)
    return dict(perm=perm, ids=ids, ptr=ptr, vals=vv)


# ---------------------------------------------------------------------- C-15
def csf_alloc(dims, policy):
    """CSF allocation policy (0 ALL, 1 ONE, 2 TWO).
    Returns dict(roots=[...], mode_csf=[...N], mode_level=[...N])."""
    N = len(dims)
    n = C.c_int(0)
    roots = np.zeros(N, dtype=np.int32)
    mc = np.zeros(N, dtype=np.int32)
    ml = np.zeros(N, dtype=np.int32)
    st = lib().oracle_csf_alloc(N, _p(_dims(dims)), int(policy), C.byref(n), _p(roots), _p(mc),
                                _p(ml))
    if st:
        raise OracleError(st)
    return dict(roots=roots[: n.value].tolist(), mode_csf=mc.tolist(), mode_level=ml.tolist())


# ---------------------------------------------------------------------- C-14
def partition(weights, G):
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    b = np.zeros(G + 1, dtype=np.uint64)
    lib().oracle_partition(_p(w), w.shape[0], G, _p(b))
    return b.astype(np.int64)
