"""ctypes binding of the in-tree CUDA library ``libddblas.so`` (include/ddblas.h).

There is no CPU fallback: if the library is missing or cannot load, every
call raises.  Build it with ``python -c "import __graft_entry__ as g; g.build()"``
or ``make -C paper_2109_13406_b200/csrc``.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# DDBLAS_LIB points at an alternative build (kernel experiments); default in-tree
LIB_PATH = os.environ.get("DDBLAS_LIB") or os.path.join(HERE, "libddblas.so")

MODES = {"exact": 0, "fast": 1, "reference": 2, "twosum": 3}

_dp = ctypes.c_void_p
_i64 = ctypes.c_int64
_d = ctypes.c_double
_c = ctypes.c_char

EXPORTS = ("ddb_rgemm", "ddb_rsyrk", "ddb_rgemm_host", "ddb_rsyrk_host",
           "ddb_rgemm_validate", "ddb_rsyrk_validate", "ddb_last_error",
           "ddb_version", "ddb_launch_count", "ddb_last_route", "ddb_fp64_peak_probe",
           "ddb_dgemm", "ddb_dsyrk", "ddb_dgemm_host", "ddb_dsyrk_host",
           "ddb_cgemm", "ddb_cgemm_host", "ddb_zgemm", "ddb_zgemm_host",
           "ddb_rpotrf", "ddb_rpotrf_host", "ddb_rpotrf_validate",
           "ddb_rtrsm", "ddb_rtrsm_host", "ddb_rtrsm_validate",
           "ddb_rgetrf", "ddb_rgetrf_host", "ddb_rgetrf_validate",
           "ddb_rgetrs", "ddb_rgetrs_host", "ddb_rgetrs_validate",
           "ddb_rgemm_mgpu", "ddb_rsyrk_mgpu",
           "ddb_dtrsm", "ddb_dtrsm_host", "ddb_dgetrf", "ddb_dgetrf_host",
           "ddb_dgetrs", "ddb_dgetrs_host", "ddb_dpotrf", "ddb_dpotrf_host",
           "ddb_cross_terms", "ddb_abs_bound", "ddb_host_register", "ddb_host_unregister")

_lib = None


class LibraryMissing(RuntimeError):
    pass


def load():
    """Load libddblas.so (once).  Raises LibraryMissing if it is not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise LibraryMissing(
            f"{LIB_PATH} is not built: the dd kernels exist only as CUDA code "
            "(run __graft_entry__.build()); there is no CPU fallback")
    L = ctypes.CDLL(LIB_PATH)
    gemm_args = [_c, _c, _i64, _i64, _i64, _d, _d, _dp, _dp, _i64, _dp, _dp, _i64,
                 _d, _d, _dp, _dp, _i64, ctypes.c_int, _dp]
    syrk_args = [_c, _c, _i64, _i64, _d, _d, _dp, _dp, _i64, _d, _d, _dp, _dp, _i64,
                 ctypes.c_int, _dp]
    for name, args in (("ddb_rgemm", gemm_args), ("ddb_rgemm_host", gemm_args),
                       ("ddb_rsyrk", syrk_args), ("ddb_rsyrk_host", syrk_args)):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = args
    dgemm_args = [_c, _c, _i64, _i64, _i64, _d, _dp, _i64, _dp, _i64, _d, _dp, _i64, _dp]
    dsyrk_args = [_c, _c, _i64, _i64, _d, _dp, _i64, _d, _dp, _i64, _dp]
    for name, args in (("ddb_dgemm", dgemm_args), ("ddb_dgemm_host", dgemm_args),
                       ("ddb_dsyrk", dsyrk_args), ("ddb_dsyrk_host", dsyrk_args)):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = args
    cg = [_c, _c, _i64, _i64, _i64, _dp, _dp, _i64, _dp, _i64, _dp, _dp, _i64, ctypes.c_int, _dp]
    zg = [_c, _c, _i64, _i64, _i64, _dp, _dp, _i64, _dp, _i64, _dp, _dp, _i64, _dp]
    for name, args in (("ddb_cgemm", cg), ("ddb_cgemm_host", cg), ("ddb_zgemm", zg),
                       ("ddb_zgemm_host", zg)):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = args
    po = [_c, _i64, _dp, _dp, _i64, _i64, ctypes.c_int, _dp, ctypes.POINTER(ctypes.c_int)]
    for name in ("ddb_rpotrf", "ddb_rpotrf_host"):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = po
    tr = [_c, _c, _c, _c, _i64, _i64, _d, _d, _dp, _dp, _i64, _dp, _dp, _i64, ctypes.c_int, _dp]
    for name in ("ddb_rtrsm", "ddb_rtrsm_host"):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = tr
    L.ddb_rtrsm_validate.restype = ctypes.c_int
    L.ddb_rtrsm_validate.argtypes = [_c, _c, _c, _c] + [_i64] * 4
    lu = [_i64, _i64, _dp, _dp, _i64, ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int),
          ctypes.c_int, _dp]
    for name in ("ddb_rgetrf", "ddb_rgetrf_host"):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = lu
    rs = [_c, _i64, _i64, _dp, _dp, _i64, ctypes.POINTER(ctypes.c_int64), _dp, _dp, _i64,
          ctypes.c_int, _dp]
    for name in ("ddb_rgetrs", "ddb_rgetrs_host"):
        f = getattr(L, name)
        f.restype = ctypes.c_int
        f.argtypes = rs
    L.ddb_rgetrs_validate.restype = ctypes.c_int
    L.ddb_rgetrs_validate.argtypes = [_c] + [_i64] * 4
    i64p, ip_ = ctypes.POINTER(ctypes.c_int64), ctypes.POINTER(ctypes.c_int)
    f64sig = {
        "ddb_dtrsm": [_c, _c, _c, _c, _i64, _i64, _d, _dp, _i64, _dp, _i64, _dp],
        "ddb_dgetrf": [_i64, _i64, _dp, _i64, i64p, ip_, _dp],
        "ddb_dgetrs": [_c, _i64, _i64, _dp, _i64, i64p, _dp, _i64, _dp],
        "ddb_dpotrf": [_c, _i64, _dp, _i64, _i64, _dp, ip_],
    }
    for name, args in f64sig.items():
        for nm in (name, name + "_host"):
            f = getattr(L, nm)
            f.restype = ctypes.c_int
            f.argtypes = args
    L.ddb_rgetrf_validate.restype = ctypes.c_int
    L.ddb_rgetrf_validate.argtypes = [_i64, _i64, _i64]
    L.ddb_rpotrf_validate.restype = ctypes.c_int
    L.ddb_rpotrf_validate.argtypes = [_c, _i64, _i64]
    ip = ctypes.POINTER(ctypes.c_int)
    L.ddb_rgemm_mgpu.restype = ctypes.c_int
    L.ddb_rgemm_mgpu.argtypes = gemm_args[:-1] + [ctypes.c_int, ip]
    L.ddb_rsyrk_mgpu.restype = ctypes.c_int
    L.ddb_rsyrk_mgpu.argtypes = syrk_args[:-1] + [ctypes.c_int, ip]
    L.ddb_rgemm_validate.restype = ctypes.c_int
    L.ddb_rgemm_validate.argtypes = [_c, _c] + [_i64] * 6
    L.ddb_rsyrk_validate.restype = ctypes.c_int
    L.ddb_rsyrk_validate.argtypes = [_c, _c] + [_i64] * 4
    L.ddb_last_error.restype = ctypes.c_char_p
    L.ddb_last_error.argtypes = []
    L.ddb_version.restype = ctypes.c_int
    L.ddb_launch_count.restype = ctypes.c_longlong
    L.ddb_last_route.restype = ctypes.c_int
    L.ddb_fp64_peak_probe.restype = ctypes.c_double
    L.ddb_fp64_peak_probe.argtypes = [_dp]
    L.ddb_host_register.restype = ctypes.c_int
    L.ddb_host_register.argtypes = [_dp, _i64]
    L.ddb_host_unregister.restype = ctypes.c_int
    L.ddb_host_unregister.argtypes = [_dp]
    L.ddb_abs_bound.restype = ctypes.c_int
    L.ddb_abs_bound.argtypes = [_c, _c, _i64, _i64, _i64, _dp, _i64, _dp, _i64, _dp, _dp, _dp,
                                _dp, _dp, _dp]
    L.ddb_cross_terms.restype = ctypes.c_int
    L.ddb_cross_terms.argtypes = [_i64, _i64, _i64, _dp, _dp, _i64, _dp, _dp, _i64, _dp,
                                  ctypes.c_int, _dp]
    _lib = L
    return L


def last_error():
    return load().ddb_last_error().decode(errors="replace")


def launch_count():
    return int(load().ddb_launch_count())


def last_route():
    return int(load().ddb_last_route())


def fp64_peak_probe(stream=None):
    """Measured FP64 FLOP/s of the current device (DFMA burn, FMA = 2)."""
    if stream is None:
        import torch
        stream = torch.cuda.current_stream().cuda_stream
    v = load().ddb_fp64_peak_probe(stream)
    if v <= 0:
        raise RuntimeError(f"fp64 peak probe failed: {last_error()}")
    return v
