"""paper_1812_05961_b200 — B200-native sparse CP-ALS hot path (arXiv 1812.05961).

Thin ctypes binding of ``libsplatt_b200.so`` (C ABI: ``include/splatt_b200.h``).
Argument marshalling only: every step of the method (CSF build, MTTKRP, Gram,
Hadamard, Cholesky solve, normalisation, fit) runs in the library's sm_100a CUDA
kernels.  There is no CPU fallback: if the shared library is missing or no CUDA
device is present, calls raise.

    ctx = Context()                                   # device 0, torch's current stream
    csf = csf_build(ind, vals, dims, ctx=ctx)         # splatt_csf_build
    M = mttkrp(csf, mode, factors, ctx=ctx)           # splatt_mttkrp
    res = cpd_als(ind, vals, dims, rank=35, max_iters=20, tol=0.0, seed=2)   # splatt_cpd_als
"""
from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

__all__ = ["lib", "Context", "Loopback", "Csf", "csf_build", "mttkrp", "cpd_als", "cpd_als_csf",
           "partition",
           "Tensor", "read_tns", "write_tns", "coo_stats",
           "SplattError", "SingularError", "EmptyTensorError", "STATUS", "padded_ld",
           "CSF_ALL", "CSF_ONE", "CSF_TWO", "POLICIES", "LEAF_TILING_AUTO"]

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SPLATT_B200_LIB") or os.path.join(_HERE, "libsplatt_b200.so")
MAX_NMODES = 8
MAX_RANK = 128
CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy

CSF_ALL, CSF_ONE, CSF_TWO = 0, 1, 2  # SPLATT_CSF_* (include/splatt_b200.h)
POLICIES = {"all": CSF_ALL, "one": CSF_ONE, "two": CSF_TWO}
LEAF_TILING_AUTO = -1.0  # SPLATT_LEAF_TILING_AUTO

STATUS = {0: "OK", -1: "BADINPUT", -2: "NOMEM", -3: "SINGULAR", -4: "CUDA", -5: "NCCL",
          -6: "EMPTY", -7: "UNSUPPORTED"}


class SplattError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"splatt {STATUS.get(code, code)}: {msg}")
        self.code = code


class SingularError(SplattError, ArithmeticError):
    pass


class EmptyTensorError(SplattError, ValueError):
    pass


class BadInputError(SplattError, ValueError):
    pass


class Coo(C.Structure):
    _fields_ = [("nmodes", C.c_int32), ("nnz", C.c_uint64), ("dims", C.c_uint64 * MAX_NMODES),
                ("ind", C.c_void_p * MAX_NMODES), ("vals", C.c_void_p)]


class Kruskal(C.Structure):
    _fields_ = [("factors", C.c_void_p * MAX_NMODES), ("lambda_", C.c_void_p),
                ("fit", C.c_double), ("iters", C.c_int32), ("fit_history", C.c_void_p)]


class Stats(C.Structure):
    _fields_ = [("t_mttkrp", C.c_double), ("t_build", C.c_double), ("t_ata", C.c_double),
                ("t_norm", C.c_double), ("t_fit", C.c_double), ("t_inverse", C.c_double),
                ("t_comm", C.c_double), ("t_loop", C.c_double),
                ("mttkrp_alg_bytes", C.c_double), ("mttkrp_launches", C.c_uint64),
                ("kernel_launches", C.c_uint64),
                ("csf_nodes", (C.c_uint64 * MAX_NMODES) * MAX_NMODES),
                ("iters", C.c_int32), ("nranks", C.c_int32), ("t_call", C.c_double),
                ("t_host_sync", C.c_double), ("host_syncs", C.c_int32),
                ("t_aux_inverse", C.c_double), ("t_aux_fit", C.c_double),
                ("mttkrp_min_bytes", C.c_double),
                ("exchange", C.c_int32)]

    def to_dict(self, nmodes=None):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "csf_nodes"}
        n = nmodes or MAX_NMODES
        d["csf_nodes"] = [[int(self.csf_nodes[i][l]) for l in range(n)] for i in range(n)]
        return d


class TensorStats(C.Structure):
    _fields_ = [("nmodes", C.c_int32), ("nnz", C.c_uint64), ("dims", C.c_uint64 * MAX_NMODES),
                ("density", C.c_double), ("nonempty_slices", C.c_uint64 * MAX_NMODES),
                ("max_slice_nnz", C.c_uint64 * MAX_NMODES)]

    def to_dict(self):
        n = self.nmodes
        return dict(nmodes=n, nnz=int(self.nnz), dims=[int(x) for x in self.dims[:n]],
                    density=float(self.density),
                    nonempty_slices=[int(x) for x in self.nonempty_slices[:n]],
                    max_slice_nnz=[int(x) for x in self.max_slice_nnz[:n]])


_lib = None
_lib_lock = threading.Lock()


def lib():
    """Load libsplatt_b200.so (built in-tree by ``paper_1812_05961_b200.build``)."""
    global _lib
    with _lib_lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1812_05961_b200.build`"
                                  " (no CPU fallback exists)")
            L = C.CDLL(LIB_PATH, mode=C.RTLD_GLOBAL)
            P, i32, u64, f64 = C.c_void_p, C.c_int32, C.c_uint64, C.c_double
            st = C.c_int
            sig = {
                "splatt_version": (C.c_char_p, []),
                "splatt_ctx_create": (st, [C.POINTER(P), C.c_int, P]),
                "splatt_ctx_destroy": (None, [P]),
                "splatt_ctx_sync": (st, [P]),
                "splatt_last_error": (C.c_char_p, [P]),
                "splatt_comm_unique_id": (st, [P]),
                "splatt_ctx_set_comm": (st, [P, P, C.c_int, C.c_int]),
                "splatt_loopback_create": (st, [i32, C.POINTER(P)]),
                "splatt_ctx_set_comm_loopback": (st, [P, P, i32]),
                "splatt_loopback_destroy": (None, [P]),
                "splatt_partition": (st, [P, u64, i32, P]),
                "splatt_partition_nnz": (st, [P, u64, i32, i32, P, P, P, P]),
                "splatt_ctx_set_partition": (st, [P, i32]),
                "splatt_ctx_set_exchange": (st, [P, i32]),
                "splatt_ctx_set_leaf_tiling": (st, [P, f64]),
                "splatt_ctx_set_deterministic": (st, [P, i32]),
                "splatt_csf_build": (st, [P, C.POINTER(Coo), i32, P, i32, C.POINTER(P)]),
                "splatt_csf_info": (st, [P, i32, C.POINTER(i32), P, P]),
                "splatt_csf_export": (st, [P, i32, i32, P, P, P]),
                "splatt_csf_free": (None, [P]),
                "splatt_mttkrp": (st, [P, P, i32, P, i32, i32, P]),
                "splatt_mttkrp_csf": (st, [P, P, i32, i32, P, i32, i32, P]),
                "splatt_csf_dispatch": (st, [P, i32, C.POINTER(i32), C.POINTER(i32),
                                             C.POINTER(i32)]),
                "splatt_cpd_als": (st, [P, C.POINTER(Coo), i32, i32, f64, u64, C.POINTER(Kruskal)]),
                "splatt_cpd_als_ex": (st, [P, C.POINTER(Coo), i32, i32, f64, u64, P, i32,
                                           C.POINTER(Kruskal), C.POINTER(Stats)]),
                "splatt_cpd_als_csf": (st, [P, P, i32, i32, f64, u64, P, C.POINTER(Kruskal),
                                            C.POINTER(Stats)]),
                "splatt_tns_read": (st, [C.c_char_p, C.POINTER(P)]),
                "splatt_tensor_coo": (st, [P, C.POINTER(Coo)]),
                "splatt_tensor_free": (None, [P]),
                "splatt_tensor_error": (C.c_char_p, []),
                "splatt_tns_write": (st, [C.c_char_p, C.POINTER(Coo)]),
                "splatt_coo_stats": (st, [C.POINTER(Coo), C.POINTER(TensorStats)]),
            }
            for name, (res, args) in sig.items():
                fn = getattr(L, name)
                fn.restype = res
                fn.argtypes = args
            _lib = L
    return _lib


def _raise(code, ctx_ptr=None):
    if code == 0:
        return
    msg = lib().splatt_last_error(ctx_ptr)
    msg = msg.decode() if msg else ""
    cls = {-1: BadInputError, -3: SingularError, -6: EmptyTensorError}.get(code, SplattError)
    raise cls(code, msg)


def padded_ld(rank: int) -> int:
    return (rank + 3) // 4 * 4


def _ptr(x):
    """Raw address of a torch tensor or numpy array (no copy; caller keeps it alive)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        return x.ctypes.data
    return x.data_ptr()


class Context:
    """splatt_ctx: a device, a stream (torch's current stream by default), a comm."""

    def __init__(self, device: int = 0, stream=None):
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("no CUDA device: the B200 path has no CPU fallback")
        self.device = int(device)
        if stream is None:
            stream = torch.cuda.current_stream(self.device)
        self.stream = stream
        handle = stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)
        if handle == 0:  # torch's default stream is the legacy default stream
            handle = CUDA_STREAM_LEGACY
        p = C.c_void_p()
        _raise(lib().splatt_ctx_create(C.byref(p), self.device, C.c_void_p(handle)))
        self._p = p
        self.nranks, self.rank = 1, 0

    @property
    def ptr(self):
        return self._p

    def sync(self):
        _raise(lib().splatt_ctx_sync(self._p), self._p)

    def set_comm(self, group=None, single=False):
        """Create the NCCL communicator of this rank from a torch.distributed group, or
        (single=True, no process group needed) a one-rank NCCL communicator that runs the
        sharded path on this GPU alone."""
        if single:
            buf = (C.c_char * 128)()
            _raise(lib().splatt_comm_unique_id(buf))
            _raise(lib().splatt_ctx_set_comm(self._p, buf, 1, 0), self._p)
            self.nranks, self.rank = 1, 0
            return
        import torch.distributed as dist
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        buf = (C.c_char * 128)()
        if rank == 0:
            _raise(lib().splatt_comm_unique_id(buf))
        obj = [bytes(buf)]
        dist.broadcast_object_list(obj, src=0, group=group)
        raw = (C.c_char * 128).from_buffer_copy(obj[0])
        _raise(lib().splatt_ctx_set_comm(self._p, raw, world, rank), self._p)
        self.nranks, self.rank = world, rank

    def set_partition(self, mode: str = "auto"):
        """How a sharded context splits each mode: "slices" (P1, whole root slices, the
        C-14 cut), "nnz" (P2, equal nonzero ranges, split slices exchanged) or "auto"
        (per mode, P2 where P1's imbalance is large; the default)."""
        _raise(lib().splatt_ctx_set_partition(self._p, {"slices": 0, "nnz": 1, "auto": 2}[mode]),
               self._p)

    def set_exchange(self, mode: str = "collective"):
        """How a sharded context shares solved factor rows: "collective" (NCCL all-gather
        after the solve; the default) or "peer" (the solve kernel stores its rows straight
        into the peers' factor matrices over NVLink; <= 8 ranks of one node)."""
        _raise(lib().splatt_ctx_set_exchange(self._p, {"collective": 0, "peer": 1}[mode]),
               self._p)

    def set_deterministic(self, on: bool = True):
        """Bitwise-reproducible ROOT MTTKRP (fixed-order chunk-seam sums instead of atomics)."""
        _raise(lib().splatt_ctx_set_deterministic(self._p, 1 if on else 0), self._p)

    def set_leaf_tiling(self, l2_fraction=0.5):
        """ROOT-MTTKRP leaf tiling for leaf factors above l2_fraction x L2: a fraction > 0
        (always), 0 (off) or "auto" (the default: half-L2 tiles in ALS runs of >= 10
        iterations)."""
        f = LEAF_TILING_AUTO if l2_fraction == "auto" else float(l2_fraction)
        _raise(lib().splatt_ctx_set_leaf_tiling(self._p, f), self._p)

    def set_comm_loopback(self, group: "Loopback", rank: int):
        """Join an in-process loopback group as logical rank `rank` (testing the sharded
        path on one device; the context must own a non-default stream)."""
        _raise(lib().splatt_ctx_set_comm_loopback(self._p, group._p, rank), self._p)
        self.nranks, self.rank = group.nranks, rank

    def close(self):
        if getattr(self, "_p", None):
            lib().splatt_ctx_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class Loopback:
    """splatt_loopback: a group of in-process logical ranks on one device."""

    def __init__(self, nranks: int):
        p = C.c_void_p()
        _raise(lib().splatt_loopback_create(int(nranks), C.byref(p)))
        self._p = p
        self.nranks = int(nranks)

    def close(self):
        if getattr(self, "_p", None):
            lib().splatt_loopback_destroy(self._p)
            self._p = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx = {}


def default_context(device: int = 0) -> Context:
    if device not in _default_ctx:
        _default_ctx[device] = Context(device)
    return _default_ctx[device]


def _make_coo(ind, vals, dims):
    N = len(dims)
    if N != len(ind):
        raise ValueError("len(ind) must equal len(dims)")
    if N < 1 or N > MAX_NMODES:
        raise ValueError("nmodes must be in [3, 8]")
    coo = Coo()
    coo.nmodes = N
    coo.nnz = int(vals.shape[0])
    for m in range(N):
        coo.dims[m] = int(dims[m])
        if int(ind[m].shape[0]) != coo.nnz:
            raise ValueError("every ind[m] must have nnz entries")
        coo.ind[m] = _ptr(ind[m])
    coo.vals = _ptr(vals)
    return coo


def _as_u32(a):
    if isinstance(a, np.ndarray):
        if a.dtype == np.int32 and a.flags.c_contiguous:
            return a.view(np.uint32)  # same bits, no copy (keeps pinned buffers pinned)
        if a.dtype != np.uint32:
            # narrowing a wider (or signed) integer type must not wrap out-of-range values
            # into valid-looking indices that would bypass the library's BADINPUT check
            if not np.issubdtype(a.dtype, np.integer):
                raise TypeError("index arrays must have an integer dtype")
            if a.size and (int(a.min()) < 0 or int(a.max()) >= (1 << 32)):
                raise ValueError("index values must lie in [0, 2^32)")
        return np.ascontiguousarray(a, dtype=np.uint32)
    import torch
    if a.dtype == torch.int32 or a.dtype == torch.uint32:
        return a.contiguous()
    raise TypeError("index tensors must be uint32/int32 (uint32 semantics)")


def _as_f64(a):
    if isinstance(a, np.ndarray):
        return np.ascontiguousarray(a, dtype=np.float64)
    import torch
    if a.dtype != torch.float64:
        raise TypeError("values must be float64")
    return a.contiguous()


class Csf:
    """Handle to a device-resident CSF set (splatt_csf)."""

    def __init__(self, p, ctx, dims):
        self._p = p
        self.ctx = ctx
        self.dims = tuple(int(d) for d in dims)

    @property
    def ncsf(self) -> int:
        n = C.c_int32()
        _raise(lib().splatt_csf_dispatch(self._p, 0, C.byref(n), None, None), self.ctx.ptr)
        return n.value

    def dispatch(self, mode: int):
        """(which CSF, level) the policy assigns to `mode` (level 0 ROOT, N-1 LEAF)."""
        w, l = C.c_int32(), C.c_int32()
        _raise(lib().splatt_csf_dispatch(self._p, mode, None, C.byref(w), C.byref(l)),
               self.ctx.ptr)
        return w.value, l.value

    def info(self, which: int):
        n = C.c_int32()
        perm = np.zeros(MAX_NMODES, dtype=np.int32)
        nodes = np.zeros(MAX_NMODES, dtype=np.uint64)
        _raise(lib().splatt_csf_info(self._p, which, C.byref(n), perm.ctypes.data, nodes.ctypes.data),
               self.ctx.ptr)
        return perm[: n.value].tolist(), nodes[: n.value].astype(np.int64).tolist()

    def export(self, which: int):
        """All levels of CSF `which` as host numpy arrays: dict(perm, ids, ptr, vals)."""
        perm, nodes = self.info(which)
        N = len(perm)
        ids, ptr = [], []
        vals = np.empty(nodes[N - 1], dtype=np.float64)
        for l in range(N):
            a = np.empty(nodes[l], dtype=np.uint32)
            b = np.empty(nodes[l] + 1, dtype=np.uint32) if l < N - 1 else None
            _raise(lib().splatt_csf_export(self._p, which, l, a.ctypes.data,
                                           b.ctypes.data if b is not None else None,
                                           vals.ctypes.data if l == N - 1 else None), self.ctx.ptr)
            ids.append(a)
            if b is not None:
                ptr.append(b)
        return dict(perm=perm, ids=ids, ptr=ptr, vals=vals)

    def free(self):
        if getattr(self, "_p", None):
            lib().splatt_csf_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _policy(policy) -> int:
    return POLICIES[policy.lower()] if isinstance(policy, str) else int(policy)


def csf_build(ind, vals, dims, ctx: Context | None = None, policy=CSF_ALL) -> Csf:
    """splatt_csf_build under `policy` (CSF_ALL / CSF_ONE / CSF_TWO or "all"/"one"/"two").
    ind/vals host or device."""
    policy = _policy(policy)
    ctx = ctx or default_context()
    ind = [_as_u32(a) for a in ind]
    vals = _as_f64(vals)
    coo = _make_coo(ind, vals, dims)
    d = (C.c_uint64 * MAX_NMODES)(*[int(x) for x in dims])
    p = C.c_void_p()
    _raise(lib().splatt_csf_build(ctx.ptr, C.byref(coo), len(dims), d, policy, C.byref(p)), ctx.ptr)
    return Csf(p, ctx, dims)


def mttkrp(csf: Csf, mode: int, factors, out=None, rank: int | None = None,
           which: int | None = None):
    """splatt_mttkrp (or splatt_mttkrp_csf on CSF `which`).  factors: list of N float64
    CUDA tensors (I_m x ld, row-major); factors[mode] may be None.  Returns out
    (I_mode x ld)."""
    import torch
    ctx = csf.ctx
    N = len(csf.dims)
    if not 0 <= mode < N or len(factors) != N:
        raise ValueError("mode out of range or len(factors) != nmodes")
    ref = next(f for m, f in enumerate(factors) if m != mode and f is not None)
    ld = int(ref.stride(0))
    R = int(rank if rank is not None else ref.shape[1])
    # the C call reads every factor as dims[m] x ld and writes out as dims[mode] x ld
    for m, f in enumerate(factors):
        if m == mode:
            continue
        if f is None or not isinstance(f, torch.Tensor) or not f.is_cuda or f.dtype != torch.float64:
            raise TypeError(f"factors[{m}] must be a float64 CUDA tensor")
        if f.dim() != 2 or f.shape[0] != csf.dims[m] or f.stride(1) != 1 or f.stride(0) != ld \
                or f.shape[1] < R:
            raise ValueError(f"factors[{m}] must be dims[{m}] x >= rank, row stride {ld}")
    if out is None:
        out = torch.empty((csf.dims[mode], ld), dtype=torch.float64, device=ref.device)
    elif (not out.is_cuda or out.dtype != torch.float64 or out.dim() != 2 or out.stride(1) != 1
          or out.stride(0) != ld or out.shape[0] != csf.dims[mode]):
        raise ValueError(f"out must be a float64 CUDA tensor dims[mode] x ld with row stride {ld}")
    arr = (C.c_void_p * len(factors))(*[(_ptr(f) if f is not None and m != mode else None)
                                        for m, f in enumerate(factors)])
    if which is None:
        code = lib().splatt_mttkrp(ctx.ptr, csf._p, mode, arr, R, int(out.stride(0)), _ptr(out))
    else:
        code = lib().splatt_mttkrp_csf(ctx.ptr, csf._p, int(which), mode, arr, R,
                                       int(out.stride(0)), _ptr(out))
    _raise(code, ctx.ptr)
    return out


def _check_out_buffer(b, shape, ctx):
    """A caller-supplied cpd_als output: the C side writes rank*8-byte rows with pitch
    rank*8 into it, so it must be float64, C-contiguous, of exactly `shape`, and (CUDA
    tensors) on the context's device."""
    if isinstance(b, np.ndarray):
        if b.dtype != np.float64 or not b.flags.c_contiguous or tuple(b.shape) != shape:
            raise ValueError(f"out buffers must be C-contiguous float64 arrays of shape {shape}")
        return
    import torch
    if not isinstance(b, torch.Tensor):
        raise TypeError("out buffers must be numpy arrays or torch tensors")
    if b.dtype != torch.float64 or not b.is_contiguous() or tuple(b.shape) != shape:
        raise ValueError(f"out buffers must be contiguous float64 tensors of shape {shape}")
    if b.is_cuda and b.device.index != ctx.device:
        raise ValueError(f"out tensor on {b.device}, context on cuda:{ctx.device}")


def _als_call(dims, rank, max_iters, init, ctx, out_device, stats, out, call):
    """Output buffers, initial factors and result dict shared by cpd_als / cpd_als_csf;
    `call(kr, init_arr, st)` performs the C call and returns its status."""
    import torch
    N = len(dims)
    if out is not None:  # caller buffers (host — e.g. pinned — or device), ld = rank
        fac, lam = list(out["factors"]), out["lam"]
        if len(fac) != N:
            raise ValueError("out['factors'] must hold one buffer per mode")
        for f, d in zip(fac + [lam], list(dims) + [None]):
            _check_out_buffer(f, (int(d), rank) if d is not None else (rank,), ctx)
    elif out_device:
        fac = [torch.empty((int(d), rank), dtype=torch.float64, device=f"cuda:{ctx.device}")
               for d in dims]
        lam = torch.empty(rank, dtype=torch.float64, device=f"cuda:{ctx.device}")
    else:
        fac = [np.empty((int(d), rank)) for d in dims]
        lam = np.empty(rank)
    hist = np.zeros(max(1, max_iters))
    kr = Kruskal()
    for m in range(N):
        kr.factors[m] = _ptr(fac[m])
    kr.lambda_ = _ptr(lam)
    kr.fit_history = hist.ctypes.data
    init_arr = None
    if init is not None:
        init = [np.ascontiguousarray(a, dtype=np.float64) if isinstance(a, np.ndarray)
                else a.contiguous() for a in init]
        if len(init) != N or any(tuple(a.shape) != (int(d), rank) for a, d in zip(init, dims)):
            raise ValueError("init factors must be N arrays of shape (I_n, rank)")
        if any(not isinstance(a, np.ndarray) and a.dtype != torch.float64 for a in init):
            raise TypeError("init factors must be float64")
        init_arr = (C.c_void_p * N)(*[_ptr(a) for a in init])
    st = Stats() if stats else None
    _raise(call(kr, init_arr, st), ctx.ptr)
    res = dict(factors=fac, lam=lam, fit=kr.fit, iters=kr.iters,
               fit_history=hist[: kr.iters].copy())
    if st is not None:
        res["stats"] = st.to_dict(N)
    return res


def cpd_als(ind, vals, dims, rank: int, max_iters: int, tol: float = 0.0, seed: int = 0,
            init=None, ctx: Context | None = None, out_device: bool = True, stats: bool = False,
            out=None, policy=CSF_ALL):
    """splatt_cpd_als(_ex).  Returns dict(factors, lam, fit, iters, fit_history[, stats]).

    ind/vals may be host (numpy / CPU tensors) or CUDA tensors; outputs are CUDA
    tensors if out_device else numpy arrays."""
    ctx = ctx or default_context()
    ind = [_as_u32(a) if not (hasattr(a, "is_cuda") and not a.is_cuda) else _as_u32(a.numpy())
           for a in ind]
    vals = _as_f64(vals.numpy() if hasattr(vals, "is_cuda") and not vals.is_cuda else vals)
    coo = _make_coo(ind, vals, dims)

    def call(kr, init_arr, st):
        return lib().splatt_cpd_als_ex(ctx.ptr, C.byref(coo), rank, max_iters, float(tol),
                                       int(seed), init_arr, _policy(policy), C.byref(kr),
                                       C.byref(st) if st else None)
    return _als_call(dims, rank, max_iters, init, ctx, out_device, stats, out, call)


def cpd_als_csf(csf: Csf, rank: int, max_iters: int, tol: float = 0.0, seed: int = 0,
                init=None, out_device: bool = True, stats: bool = False, out=None):
    """splatt_cpd_als_csf: CP-ALS on a prebuilt CSF set (no build / validation per call)."""
    ctx = csf.ctx

    def call(kr, init_arr, st):
        return lib().splatt_cpd_als_csf(ctx.ptr, csf._p, rank, max_iters, float(tol), int(seed),
                                        init_arr, C.byref(kr), C.byref(st) if st else None)
    return _als_call(csf.dims, rank, max_iters, init, ctx, out_device, stats, out, call)


def partition(weights, G: int):
    """splatt_partition (host-only, C-14): optimal contiguous split of slice weights."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    b = np.zeros(G + 1, dtype=np.uint64)
    _raise(lib().splatt_partition(w.ctypes.data if w.size else None, w.shape[0], G, b.ctypes.data))
    return b.astype(np.int64)


class Tensor:
    """A host COO parsed by the library's .tns reader (splatt_tns_read).  ind[m] / vals are
    zero-copy numpy views of library memory (alive as long as this object)."""

    def __init__(self, path: str):
        p = C.c_void_p()
        code = lib().splatt_tns_read(os.fsencode(path), C.byref(p))
        if code != 0:
            msg = lib().splatt_tensor_error()
            cls = {-1: BadInputError}.get(code, SplattError)
            raise cls(code, (msg.decode() if msg else "") + f" ({path})")
        self._p = p
        coo = Coo()
        _raise(lib().splatt_tensor_coo(p, C.byref(coo)))
        self.nmodes = int(coo.nmodes)
        self.nnz = int(coo.nnz)
        self.dims = tuple(int(coo.dims[m]) for m in range(self.nmodes))
        self.ind = [np.ctypeslib.as_array(C.cast(coo.ind[m], C.POINTER(C.c_uint32)),
                                          shape=(self.nnz,)) for m in range(self.nmodes)]
        self.vals = np.ctypeslib.as_array(C.cast(coo.vals, C.POINTER(C.c_double)),
                                          shape=(self.nnz,))

    def stats(self) -> dict:
        return coo_stats(self.ind, self.vals, self.dims)

    def free(self):
        if getattr(self, "_p", None):
            self.ind, self.vals = [], None
            lib().splatt_tensor_free(self._p)
            self._p = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def read_tns(path: str) -> Tensor:
    """splatt_tns_read: parse a FROSTT .tns file (host, multi-threaded)."""
    return Tensor(path)


def _host_coo(ind, vals, dims):
    ind = [np.ascontiguousarray(np.asarray(a), dtype=np.uint32) for a in ind]
    vals = np.ascontiguousarray(np.asarray(vals), dtype=np.float64)
    coo = Coo()
    coo.nmodes = len(dims)
    coo.nnz = int(vals.shape[0])
    for m, d in enumerate(dims):
        coo.dims[m] = int(d)
        coo.ind[m] = ind[m].ctypes.data
    coo.vals = vals.ctypes.data
    return coo, (ind, vals)


def write_tns(path: str, ind, vals, dims) -> None:
    """splatt_tns_write: host COO -> .tns (1-based, shortest round-trip values)."""
    coo, keep = _host_coo(ind, vals, dims)
    code = lib().splatt_tns_write(os.fsencode(path), C.byref(coo))
    if code != 0:
        msg = lib().splatt_tensor_error()
        raise SplattError(code, msg.decode() if msg else "")
    del keep


def coo_stats(ind, vals, dims) -> dict:
    """splatt_coo_stats: Table I statistics of a host COO."""
    coo, keep = _host_coo(ind, vals, dims)
    out = TensorStats()
    _raise(lib().splatt_coo_stats(C.byref(coo), C.byref(out)))
    del keep
    return out.to_dict()


class NnzShare(C.Structure):
    _fields_ = [("full_lo", C.c_uint64), ("full_hi", C.c_uint64), ("npart", C.c_int32),
                ("part_slice", C.c_uint64 * 2), ("part_begin", C.c_uint64 * 2),
                ("part_end", C.c_uint64 * 2)]


def partition_nnz(weights, G: int, rank: int):
    """splatt_partition_nnz (host-only, P2): dict(row_bounds, split, full, parts)."""
    w = np.ascontiguousarray(np.asarray(weights, dtype=np.uint64))
    rb = np.zeros(G + 1, dtype=np.uint64)
    sp = np.zeros(max(1, G - 1), dtype=np.uint64)
    ns = C.c_uint64()
    sh = NnzShare()
    _raise(lib().splatt_partition_nnz(w.ctypes.data if w.size else None, w.shape[0], G, rank,
                                      rb.ctypes.data, sp.ctypes.data, C.byref(ns), C.byref(sh)))
    parts = [(int(sh.part_slice[q]), int(sh.part_begin[q]), int(sh.part_end[q]))
             for q in range(sh.npart)]
    return dict(row_bounds=rb.astype(np.int64).tolist(), split=sp[: ns.value].astype(np.int64).tolist(),
                full=(int(sh.full_lo), int(sh.full_hi)), parts=parts)


def version() -> str:
    return lib().splatt_version().decode()
