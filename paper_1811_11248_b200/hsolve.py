"""Thin ctypes binding of libhsolve (include/hsolve.h) — argument marshalling only.

Every function keeps the C name.  Host arrays are numpy; device arrays may be
torch CUDA tensors (their data_ptr() is passed with on_device=1).  A non-OK status
raises HSError carrying the status and hs_last_error().  There is no CPU fallback:
loading fails loudly when libhsolve.so is missing, and factor/apply/pcg need a GPU.
"""
from __future__ import annotations

import ctypes as C
import os

import weakref

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhsolve.so")

HS_OK = 0
STATUS = ["HS_OK", "HS_E_INVALID_ARG", "HS_E_DIM", "HS_E_NOT_SYMMETRIC", "HS_E_NOT_SPD", "HS_E_COLUMN_SPLIT",
          "HS_E_PRECOND_NOT_POSITIVE", "HS_E_NOT_CONVERGED", "HS_E_OOM", "HS_E_CUDA", "HS_E_NCCL",
          "HS_E_NO_DEVICE", "HS_E_UNSUPPORTED", "HS_E_INTERNAL"]
for _i, _s in enumerate(STATUS):
    globals()[_s] = _i

# hs_analysis_export keys
(HS_EXP_PERM, HS_EXP_LEAF_OFF, HS_EXP_H_PTR, HS_EXP_H_IDX, HS_EXP_W_PTR, HS_EXP_W_IDX, HS_EXP_BATCH_PTR,
 HS_EXP_BATCH_IDX, HS_EXP_INTERIOR, HS_EXP_F_PTR, HS_EXP_F_IDX, HS_EXP_NPHASE1, HS_EXP_HTOP_PTR,
 HS_EXP_HTOP_IDX, HS_EXP_FS_PTR, HS_EXP_FS_IDX) = range(16)
# hs_dist_plan_export keys
HS_DEXP_OWNER, HS_DEXP_RECV_PTR, HS_DEXP_RECV, HS_DEXP_HELD_PTR, HS_DEXP_HELD = range(5)
# hs_factor_export keys
HS_FEXP_RANKS, HS_FEXP_LIVE0, HS_FEXP_PIV_PTR, HS_FEXP_PIV, HS_FEXP_TOP, HS_FEXP_KN, HS_FEXP_KW = range(7)

# every symbol include/hsolve.h declares
SYMBOLS = ["hs_create", "hs_nccl_unique_id", "hs_loopback_world_create", "hs_loopback_world_destroy",
           "hs_create_loopback", "hs_set_stream", "hs_destroy", "hs_last_error", "hs_status_string", "hs_analyze",
           "hs_analysis_get_info", "hs_analysis_export", "hs_dist_plan_export", "hs_analysis_destroy", "hs_factor_create",
           "hs_factor_get_stats", "hs_factor_export", "hs_factor_export_cluster", "hs_factor_destroy", "hs_apply", "hs_gmres",
           "hs_pcg", "hs_spmv", "hs_launch_count"]
HS_CEXP_SHAPE, HS_CEXP_G, HS_CEXP_V, HS_CEXP_TAU, HS_CEXP_B = range(5)


class HSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS[status] if 0 <= status < len(STATUS) else status}: {msg}")
        self.status = status


class hs_analyze_opts(C.Structure):
    _fields_ = [("leaf_size", C.c_int32), ("leaf_columns", C.c_int32), ("top_log2", C.c_int32),
                ("nsub_log2", C.c_int32), ("coarse_fill", C.c_int32)]


class hs_factor_opts(C.Structure):
    _fields_ = [("eps", C.c_double), ("eps_relative", C.c_int32), ("dc", C.c_int32),
                ("values_on_device", C.c_int32), ("reserved", C.c_int32)]


class hs_analysis_info(C.Structure):
    _fields_ = [("n", C.c_int64), ("depth", C.c_int32), ("L_top", C.c_int32), ("nsub_log2", C.c_int32),
                ("top_log2", C.c_int32)]


class hs_factor_stats_t(C.Structure):
    _fields_ = [("t_factor_s", C.c_double), ("flops", C.c_double), ("factor_bytes", C.c_double),
                ("n_top", C.c_int64), ("n_levels", C.c_int32), ("n_batches", C.c_int32), ("max_m", C.c_int32),
                ("max_rank", C.c_int32), ("t_phase_s", C.c_double * 8), ("flops_phase", C.c_double * 8),
                ("t_level_s", C.c_double * 32), ("flops_level", C.c_double * 32)]

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_}
        for k in ("t_phase_s", "flops_phase"):
            d[k] = list(getattr(self, k))
        for k in ("t_level_s", "flops_level"):
            d[k] = list(getattr(self, k))[:self.n_levels]
        return d


class hs_pcg_report(C.Structure):
    _fields_ = [("iters", C.c_int32), ("converged", C.c_int32), ("relres", C.c_double), ("relres_true", C.c_double),
                ("t_pcg_s", C.c_double), ("t_apply_s", C.c_double), ("t_spmv_s", C.c_double),
                ("history", C.POINTER(C.c_double)), ("history_cap", C.c_int32), ("history_len", C.c_int32)]

    def __init__(self, cap=1024):
        super().__init__()
        self._hist = (C.c_double * cap)()
        self.history = C.cast(self._hist, C.POINTER(C.c_double))
        self.history_cap = cap

    def as_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k not in ("history", "history_cap", "history_len")}
        d["history"] = list(self._hist[:self.history_len])
        return d


_lib = None
_exiting = False


def _at_exit():
    # Handles, analyses and factors are not released during interpreter shutdown: the
    # CUDA runtime may already be torn down and object finalisation order is arbitrary.
    global _exiting
    _exiting = True


import atexit  # noqa: E402
atexit.register(_at_exit)


def lib():
    """Load libhsolve.so (built by paper_1811_11248_b200.build); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_1811_11248_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64, dp = C.c_void_p, C.c_int32, C.c_int64, C.c_double
        L.hs_create.argtypes = [C.POINTER(vp), C.c_int, C.c_int, C.c_int, vp]
        L.hs_set_stream.argtypes = [vp, vp]
        L.hs_nccl_unique_id.argtypes = [vp]
        L.hs_loopback_world_create.argtypes = [i32, C.POINTER(vp)]
        L.hs_loopback_world_destroy.argtypes = [vp]
        L.hs_loopback_world_destroy.restype = None
        L.hs_create_loopback.argtypes = [C.POINTER(vp), C.c_int, vp, i32]
        L.hs_destroy.argtypes = [vp]
        L.hs_destroy.restype = None
        L.hs_last_error.argtypes = [vp]
        L.hs_last_error.restype = C.c_char_p
        L.hs_status_string.argtypes = [C.c_int]
        L.hs_status_string.restype = C.c_char_p
        L.hs_analyze.argtypes = [vp, i64, vp, vp, vp, i32, vp, C.POINTER(hs_analyze_opts), C.POINTER(vp)]
        L.hs_analysis_get_info.argtypes = [vp, C.POINTER(hs_analysis_info)]
        L.hs_analysis_export.argtypes = [vp, i32, i32, vp, i64, C.POINTER(i64)]
        L.hs_dist_plan_export.argtypes = [vp, i32, i32, i32, i32, vp, i64, C.POINTER(i64)]
        L.hs_analysis_destroy.argtypes = [vp]
        L.hs_analysis_destroy.restype = None
        L.hs_factor_create.argtypes = [vp, vp, vp, C.POINTER(hs_factor_opts), C.POINTER(vp)]
        L.hs_factor_get_stats.argtypes = [vp, C.POINTER(hs_factor_stats_t)]
        L.hs_factor_export.argtypes = [vp, i32, i32, vp, i64, C.POINTER(i64)]
        L.hs_factor_export_cluster.argtypes = [vp, i32, i32, i32, vp, i64, C.POINTER(i64)]
        L.hs_factor_destroy.argtypes = [vp]
        L.hs_factor_destroy.restype = None
        L.hs_apply.argtypes = [vp, vp, vp, i32]
        L.hs_pcg.argtypes = [vp, vp, vp, dp, i32, i32, C.POINTER(hs_pcg_report)]
        L.hs_gmres.argtypes = [vp, vp, vp, dp, i32, i32, i32, C.POINTER(hs_pcg_report)]
        L.hs_spmv.argtypes = [vp, vp, vp, i32]
        L.hs_launch_count.argtypes = []
        L.hs_launch_count.restype = i64
        for s in SYMBOLS:
            if s not in ("hs_destroy", "hs_analysis_destroy", "hs_factor_destroy", "hs_last_error",
                         "hs_loopback_world_destroy",
                         "hs_status_string", "hs_launch_count"):
                getattr(L, s).restype = C.c_int
        _lib = L
    return _lib


def _check(st, h=None):
    if st != HS_OK:
        msg = lib().hs_last_error(h)
        raise HSError(st, msg.decode() if msg else "")


def _ptr(a):
    """(pointer, on_device) for a numpy array or a torch CUDA tensor."""
    if a is None:
        return None, 0
    if hasattr(a, "data_ptr") and hasattr(a, "is_cuda"):
        return C.c_void_p(a.data_ptr()), int(bool(a.is_cuda))
    return C.c_void_p(a.ctypes.data), 0


def _is_cuda(a):
    return hasattr(a, "is_cuda") and a.is_cuda


def _dev_ready(*tensors):
    """Device inputs may still be being written by torch's current stream, which is not the
    library's stream: wait for it before the C call reads them (the C calls synchronise their
    own stream before returning, so device outputs are complete when they return)."""
    import torch
    for t in tensors:
        if _is_cuda(t):
            torch.cuda.current_stream(t.device).synchronize()
            return


def _check_dev_vec(t, n, name):
    import torch
    if t.dtype != torch.float64 or not t.is_contiguous() or t.numel() != n:
        raise HSError(HS_E_DIM, f"{name}: need a contiguous float64 CUDA tensor of {n} elements "
                                f"(got {t.dtype}, {tuple(t.shape)}, contiguous={t.is_contiguous()})")


def _host_vec(a, n, name, out=False):
    """A float64 C-contiguous host vector of n entries: inputs are converted, a caller-given
    output must already be one (the library writes n doubles into it)."""
    if out:
        if not (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.flags.c_contiguous and a.size == n
                and a.flags.writeable):
            raise HSError(HS_E_DIM, f"{name}: need a writable C-contiguous float64 array of {n} entries")
        return a
    a = np.ascontiguousarray(a, dtype=np.float64)
    if a.size != n:
        raise HSError(HS_E_DIM, f"{name}: {a.size} entries, the factor has {n}")
    return a


class Handle:
    def __init__(self, ptr):
        self.ptr = ptr
        self._factors = weakref.WeakSet()   # a factor must go before its handle (its memory is the handle's)

    def close(self):
        """Destroy the handle now (its factors first): its cached device memory goes back to the driver."""
        if self.ptr and _lib is not None and not _exiting:
            for f in list(self._factors):   # garbage-collected cycles finalize in any order
                f._destroy()
            _lib.hs_destroy(self.ptr)
        self.ptr = None

    def __del__(self):
        self.close()


class Analysis:
    def __init__(self, ptr, keep):
        self.ptr = ptr
        self._keep = keep

    def __del__(self):
        if self.ptr and _lib is not None and not _exiting:
            _lib.hs_analysis_destroy(self.ptr)
            self.ptr = None


class Factor:
    def __init__(self, ptr, handle, analysis, n):
        self.ptr = ptr
        self.handle = handle       # keep alive
        self.analysis = analysis
        self.n = n
        handle._factors.add(self)

    def _destroy(self):
        if self.ptr and _lib is not None and not _exiting and self.handle.ptr:
            _lib.hs_factor_destroy(self.ptr)
        self.ptr = None

    def __del__(self):
        self._destroy()


def hs_nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    _check(lib().hs_nccl_unique_id(buf))
    return buf.raw


class LoopbackWorld:
    """Test harness: `world` ranks as host threads on one device (hs_create_loopback)."""

    def __init__(self, world: int):
        self.ptr = C.c_void_p()
        _check(lib().hs_loopback_world_create(world, C.byref(self.ptr)))
        self.world = world

    def __del__(self):
        if getattr(self, "ptr", None) and self.ptr.value and _lib is not None:
            _lib.hs_loopback_world_destroy(self.ptr)
            self.ptr = C.c_void_p()


def hs_create_loopback(device: int, world: LoopbackWorld, rank: int) -> Handle:
    h = C.c_void_p()
    _check(lib().hs_create_loopback(C.byref(h), device, world.ptr, rank))
    return Handle(h)


def hs_create(device: int = 0, world_size: int = 1, rank: int = 0, nccl_unique_id: bytes | None = None) -> Handle:
    h = C.c_void_p()
    uid = C.create_string_buffer(nccl_unique_id, 128) if nccl_unique_id is not None else None
    _check(lib().hs_create(C.byref(h), device, world_size, rank, uid))
    return Handle(h)


def hs_set_stream(h: Handle, stream_ptr: int | None):
    _check(lib().hs_set_stream(h.ptr, C.c_void_p(stream_ptr) if stream_ptr else None), h.ptr)


def hs_analyze(h: Handle | None, n, rowptr, colind, coords=None, column_id=None, leaf_size=64, leaf_columns=0,
               top_log2=3, nsub_log2=3, coarse_fill=0) -> Analysis:
    rowptr = np.ascontiguousarray(rowptr, dtype=np.int64)
    colind = np.ascontiguousarray(colind, dtype=np.int32)
    cd = 0
    if coords is not None:
        coords = np.ascontiguousarray(coords, dtype=np.float64).reshape(n, -1)
        cd = coords.shape[1]
    if column_id is not None:
        column_id = np.ascontiguousarray(column_id, dtype=np.int32)
    opt = hs_analyze_opts(leaf_size, leaf_columns, top_log2, nsub_log2, coarse_fill)
    a = C.c_void_p()
    hp = h.ptr if h is not None else None
    _check(lib().hs_analyze(hp, int(n), rowptr.ctypes.data, colind.ctypes.data,
                            coords.ctypes.data if coords is not None else None, cd,
                            column_id.ctypes.data if column_id is not None else None, C.byref(opt), C.byref(a)), hp)
    return Analysis(a, (rowptr, colind))


def hs_analysis_get_info(a: Analysis) -> dict:
    info = hs_analysis_info()
    _check(lib().hs_analysis_get_info(a.ptr, C.byref(info)))
    return {k: getattr(info, k) for k, _ in info._fields_}


def hs_dist_plan_export(a: Analysis, world: int, rank: int, key: int, level: int = 0) -> np.ndarray:
    n = C.c_int64()
    _check(lib().hs_dist_plan_export(a.ptr, world, rank, key, level, None, 0, C.byref(n)))
    out = np.empty(n.value, dtype=np.int64)
    _check(lib().hs_dist_plan_export(a.ptr, world, rank, key, level, out.ctypes.data, n.value, C.byref(n)))
    return out


def hs_analysis_export(a: Analysis, key: int, level: int = 0) -> np.ndarray:
    n = C.c_int64()
    _check(lib().hs_analysis_export(a.ptr, key, level, None, 0, C.byref(n)))
    out = np.zeros(max(n.value, 1), dtype=np.int64)
    _check(lib().hs_analysis_export(a.ptr, key, level, out.ctypes.data, n.value, C.byref(n)))
    return out[:n.value]


def hs_factor_create(h: Handle, a: Analysis, values, eps=1e-2, eps_relative=1, dc=1) -> Factor:
    """values: numpy (host) or a torch CUDA float64 tensor (device-resident CSR values)."""
    nnz = int(a._keep[0][-1])
    if _is_cuda(values):
        _check_dev_vec(values, nnz, "values")
        _dev_ready(values)
        vp, on_dev = _ptr(values)
    else:
        values = _host_vec(values, nnz, "values")
        vp, on_dev = C.c_void_p(values.ctypes.data), 0
    opt = hs_factor_opts(eps, eps_relative, dc, on_dev, 0)
    f = C.c_void_p()
    _check(lib().hs_factor_create(h.ptr, a.ptr, vp, C.byref(opt), C.byref(f)), h.ptr)
    info = hs_analysis_get_info(a)
    return Factor(f, h, a, info["n"])


def hs_launch_count() -> int:
    return int(lib().hs_launch_count())


def hs_factor_get_stats(f: Factor) -> dict:
    st = hs_factor_stats_t()
    _check(lib().hs_factor_get_stats(f.ptr, C.byref(st)), f.handle.ptr)
    return st.as_dict()


def hs_factor_export(f: Factor, key: int, level: int = 0) -> np.ndarray:
    n = C.c_int64()
    _check(lib().hs_factor_export(f.ptr, key, level, None, 0, C.byref(n)), f.handle.ptr)
    out = np.zeros(max(n.value, 1), dtype=np.int64)
    _check(lib().hs_factor_export(f.ptr, key, level, out.ctypes.data, n.value, C.byref(n)), f.handle.ptr)
    return out[:n.value]


def hs_factor_export_cluster(f: Factor, key: int, level: int, cluster: int) -> np.ndarray:
    n = C.c_int64()
    _check(lib().hs_factor_export_cluster(f.ptr, key, level, cluster, None, 0, C.byref(n)), f.handle.ptr)
    out = np.zeros(max(n.value, 1), dtype=np.float64)
    _check(lib().hs_factor_export_cluster(f.ptr, key, level, cluster, out.ctypes.data, n.value, C.byref(n)),
           f.handle.ptr)
    return out[:n.value]


def cluster_record(f: Factor, level: int, cluster: int) -> dict:
    """G, V, tau, B of one eliminated cluster (debug / per-cluster parity aid)."""
    m, r, kw, kn, ldB = (int(x) for x in hs_factor_export_cluster(f, HS_CEXP_SHAPE, level, cluster))
    return {"m": m, "r": r, "kw": kw, "kn": kn,
            "G": hs_factor_export_cluster(f, HS_CEXP_G, level, cluster).reshape(m, m),
            "V": hs_factor_export_cluster(f, HS_CEXP_V, level, cluster).reshape(r, m).T,
            "tau": hs_factor_export_cluster(f, HS_CEXP_TAU, level, cluster),
            "B": hs_factor_export_cluster(f, HS_CEXP_B, level, cluster).reshape(m, ldB)}


def _dev_io(f, b, x):
    _check_dev_vec(b, f.n, "b")
    x = b.new_empty(b.shape) if x is None else x
    if not _is_cuda(x) or x.device != b.device:
        raise HSError(HS_E_DIM, "x: need a CUDA tensor on b's device")
    _check_dev_vec(x, f.n, "x")
    _dev_ready(b)
    return x


def _host_io(f, b, x):
    b = _host_vec(b, f.n, "b")
    x = np.empty_like(b) if x is None else _host_vec(x, f.n, "x", out=True)
    return b, x


def hs_apply(f: Factor, b, x=None):
    """x = M^{-1} b.  numpy in -> numpy out; torch CUDA tensor in -> written into x (a tensor)."""
    if _is_cuda(b):
        x = _dev_io(f, b, x)
        _check(lib().hs_apply(f.ptr, _ptr(b)[0], _ptr(x)[0], 1), f.handle.ptr)
        return x
    b, x = _host_io(f, b, x)
    _check(lib().hs_apply(f.ptr, b.ctypes.data, x.ctypes.data, 0), f.handle.ptr)
    return x


def hs_spmv(f: Factor, x):
    if _is_cuda(x):
        y = _dev_io(f, x, None)
        _check(lib().hs_spmv(f.ptr, _ptr(x)[0], _ptr(y)[0], 1), f.handle.ptr)
        return y
    x, y = _host_io(f, x, None)
    _check(lib().hs_spmv(f.ptr, x.ctypes.data, y.ctypes.data, 0), f.handle.ptr)
    return y


def hs_pcg(f: Factor, b, tol=1e-8, maxit=1000, x=None, raise_not_converged=True):
    """PCG with M = the factor.  Returns (x, report dict)."""
    rep = hs_pcg_report()
    if _is_cuda(b):
        x = _dev_io(f, b, x)
        st = lib().hs_pcg(f.ptr, _ptr(b)[0], _ptr(x)[0], tol, maxit, 1, C.byref(rep))
    else:
        b, x = _host_io(f, b, x)
        st = lib().hs_pcg(f.ptr, b.ctypes.data, x.ctypes.data, tol, maxit, 0, C.byref(rep))
    if st == HS_E_NOT_CONVERGED and not raise_not_converged:
        return x, rep.as_dict()
    _check(st, f.handle.ptr)
    return x, rep.as_dict()


def hs_gmres(f: Factor, b, tol=1e-12, restart=200, maxit=1000, x=None, raise_not_converged=True):
    """Right-preconditioned GMRES(restart) with M = the factor.  Returns (x, report)."""
    rep = hs_pcg_report()
    if _is_cuda(b):
        x = _dev_io(f, b, x)
        st = lib().hs_gmres(f.ptr, _ptr(b)[0], _ptr(x)[0], tol, restart, maxit, 1, C.byref(rep))
    else:
        b, x = _host_io(f, b, x)
        st = lib().hs_gmres(f.ptr, b.ctypes.data, x.ctypes.data, tol, restart, maxit, 0, C.byref(rep))
    if st == HS_E_NOT_CONVERGED and not raise_not_converged:
        return x, rep.as_dict()
    _check(st, f.handle.ptr)
    return x, rep.as_dict()
