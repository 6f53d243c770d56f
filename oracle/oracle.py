"""ctypes front end of the C oracle (``dd_oracle.c``) -- TEST INFRASTRUCTURE ONLY.

See ``oracle/__init__.py`` for who may import this.  Operands are numpy
float64 planes in the reference's column-major flat layout: element (i, j)
of a matrix with leading dimension ``ld`` lives at ``i + j*ld``
(``/root/reference/pkg/src/mpkit/mpblas/matrix.py:1-7``).
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libdd_oracle.so")
_lib = None

_dp = ctypes.POINTER(ctypes.c_double)
_i64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    src = os.path.join(_HERE, "dd_oracle.c")
    if force or not os.path.exists(_LIB_PATH) or \
            os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.run(["make", "-s", "-C", _HERE], check=True)
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = ctypes.CDLL(_LIB_PATH)
        L.oracle_rgemm.restype = ctypes.c_int
        L.oracle_rgemm.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64, _i64,
                                   ctypes.c_double, ctypes.c_double,
                                   _dp, _dp, _i64, _dp, _dp, _i64,
                                   ctypes.c_double, ctypes.c_double,
                                   _dp, _dp, _i64, ctypes.c_int]
        L.oracle_rsyrk.restype = ctypes.c_int
        L.oracle_rsyrk.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64,
                                   ctypes.c_double, ctypes.c_double,
                                   _dp, _dp, _i64,
                                   ctypes.c_double, ctypes.c_double,
                                   _dp, _dp, _i64, ctypes.c_int]
        for name in ("oracle_add2", "oracle_mul2"):
            f = getattr(L, name)
            f.restype = None
            f.argtypes = [ctypes.c_double] * 4 + [_dp]
        L.oracle_two_prod.restype = None
        L.oracle_two_prod.argtypes = [ctypes.c_double, ctypes.c_double, _dp]
        L.oracle_dgemm.restype = ctypes.c_int
        L.oracle_dgemm.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64, _i64, ctypes.c_double,
                                   _dp, _i64, _dp, _i64, ctypes.c_double, _dp, _i64]
        L.oracle_dsyrk.restype = ctypes.c_int
        L.oracle_dsyrk.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64, ctypes.c_double,
                                   _dp, _i64, ctypes.c_double, _dp, _i64]
        L.oracle_cgemm.restype = ctypes.c_int
        L.oracle_cgemm.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64, _i64, ctypes.c_void_p,
                                   ctypes.c_void_p, _i64, ctypes.c_void_p, _i64, ctypes.c_void_p,
                                   ctypes.c_void_p, _i64]
        L.oracle_zgemm.restype = ctypes.c_int
        L.oracle_zgemm.argtypes = [ctypes.c_char, ctypes.c_char, _i64, _i64, _i64, ctypes.c_void_p,
                                   ctypes.c_void_p, _i64, ctypes.c_void_p, _i64, ctypes.c_void_p,
                                   ctypes.c_void_p, _i64]
        L.oracle_max_threads.restype = ctypes.c_int
        L.oracle_rpotrf.restype = ctypes.c_int
        L.oracle_rpotrf.argtypes = [ctypes.c_char, _i64, _dp, _dp, _i64,
                                    ctypes.POINTER(ctypes.c_int64)]
        L.oracle_potrf_validate.restype = ctypes.c_int
        L.oracle_potrf_validate.argtypes = [ctypes.c_char, _i64, _i64]
        L.oracle_rtrsm.restype = ctypes.c_int
        L.oracle_rtrsm.argtypes = [ctypes.c_char] * 4 + [_i64, _i64, ctypes.c_double, ctypes.c_double,
                                                         _dp, _dp, _i64, _dp, _dp, _i64]
        L.oracle_trsm_validate.restype = ctypes.c_int
        L.oracle_trsm_validate.argtypes = [ctypes.c_char] * 4 + [_i64] * 4
        L.oracle_rgetrf.restype = ctypes.c_int
        L.oracle_rgetrf.argtypes = [_i64, _i64, _dp, _dp, _i64, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.oracle_getrf_validate.restype = ctypes.c_int
        L.oracle_getrf_validate.argtypes = [_i64, _i64, _i64]
        L.oracle_rgetrs.restype = ctypes.c_int
        L.oracle_rgetrs.argtypes = [ctypes.c_char, _i64, _i64, _dp, _dp, _i64,
                                    ctypes.POINTER(ctypes.c_int64), _i64, _dp, _dp, _i64]
        L.oracle_getrs_validate.restype = ctypes.c_int
        L.oracle_getrs_validate.argtypes = [ctypes.c_char] + [_i64] * 4
        dp1 = _dp
        L.oracle_dpotrf.restype = ctypes.c_int
        L.oracle_dpotrf.argtypes = [ctypes.c_char, _i64, dp1, _i64, ctypes.POINTER(ctypes.c_int64)]
        L.oracle_dtrsm.restype = ctypes.c_int
        L.oracle_dtrsm.argtypes = [ctypes.c_char] * 4 + [_i64, _i64, ctypes.c_double, dp1, _i64,
                                                         dp1, _i64]
        L.oracle_dgetrf.restype = ctypes.c_int
        L.oracle_dgetrf.argtypes = [_i64, _i64, dp1, _i64, ctypes.POINTER(ctypes.c_int64),
                                    ctypes.POINTER(ctypes.c_int64)]
        L.oracle_dgetrs.restype = ctypes.c_int
        L.oracle_dgetrs.argtypes = [ctypes.c_char, _i64, _i64, dp1, _i64,
                                    ctypes.POINTER(ctypes.c_int64), _i64, dp1, _i64]
        L.oracle_div2.restype = None
        L.oracle_div2.argtypes = [ctypes.c_double] * 4 + [_dp]
        L.oracle_sqrt2.restype = None
        L.oracle_sqrt2.argtypes = [ctypes.c_double] * 2 + [_dp]
        L.oracle_gemm_validate.restype = ctypes.c_int
        L.oracle_gemm_validate.argtypes = [ctypes.c_char, ctypes.c_char] + [_i64] * 6
        L.oracle_syrk_validate.restype = ctypes.c_int
        L.oracle_syrk_validate.argtypes = [ctypes.c_char, ctypes.c_char] + [_i64] * 4
        _lib = L
    return _lib


def _ptr(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def _flag(c):
    return c.encode() if isinstance(c, str) else bytes([c])


def rgemm(transa, transb, m, n, k, alpha, a_hi, a_lo, lda, b_hi, b_lo, ldb,
          beta, c_hi, c_lo, ldc, threads=0):
    """In-place C <- alpha*op(A)*op(B) + beta*C with the reference's rounding.

    ``alpha``/``beta`` are (hi, lo) pairs.  Returns 0 or the reference
    argument index of the first invalid argument."""
    return lib().oracle_rgemm(_flag(transa), _flag(transb), m, n, k,
                              float(alpha[0]), float(alpha[1]),
                              _ptr(a_hi), _ptr(a_lo), lda, _ptr(b_hi), _ptr(b_lo), ldb,
                              float(beta[0]), float(beta[1]),
                              _ptr(c_hi), _ptr(c_lo), ldc, int(threads))


def rsyrk(uplo, trans, n, k, alpha, a_hi, a_lo, lda, beta, c_hi, c_lo, ldc,
          threads=0):
    return lib().oracle_rsyrk(_flag(uplo), _flag(trans), n, k,
                              float(alpha[0]), float(alpha[1]),
                              _ptr(a_hi), _ptr(a_lo), lda,
                              float(beta[0]), float(beta[1]),
                              _ptr(c_hi), _ptr(c_lo), ldc, int(threads))


def dgemm(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
    """binary64 Rgemm with the reference's order (F64 backend)."""
    return lib().oracle_dgemm(_flag(transa), _flag(transb), m, n, k, float(alpha), _ptr(a), lda,
                              _ptr(b), ldb, float(beta), _ptr(c), ldc)


def dsyrk(uplo, trans, n, k, alpha, a, lda, beta, c, ldc):
    return lib().oracle_dsyrk(_flag(uplo), _flag(trans), n, k, float(alpha), _ptr(a), lda,
                              float(beta), _ptr(c), ldc)


def cgemm(transa, transb, m, n, k, alpha4, a4, lda, b4, ldb, beta4, c4, ldc):
    """'cdd' Cgemm; a4/b4/c4 = four float64 planes, alpha4/beta4 four doubles."""
    keep = []

    def arr(vals):
        x = (ctypes.c_double * 4)(*vals)
        keep.append(x)
        return ctypes.cast(x, ctypes.c_void_p)

    def ptrs(planes):
        x = (ctypes.c_void_p * 4)(*(p.ctypes.data for p in planes))
        keep.append(x)
        return ctypes.cast(x, ctypes.c_void_p)
    return lib().oracle_cgemm(_flag(transa), _flag(transb), m, n, k, arr(alpha4), ptrs(a4), lda,
                              ptrs(b4), ldb, arr(beta4), ptrs(c4), ldc)


def zgemm(transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc):
    """'c64' Cgemm on complex128 arrays."""
    al = (ctypes.c_double * 2)(alpha.real, alpha.imag)
    be = (ctypes.c_double * 2)(beta.real, beta.imag)
    return lib().oracle_zgemm(_flag(transa), _flag(transb), m, n, k,
                              ctypes.cast(al, ctypes.c_void_p), a.ctypes.data, lda, b.ctypes.data,
                              ldb, ctypes.cast(be, ctypes.c_void_p), c.ctypes.data, ldc)


def rpotrf(uplo, n, a_hi, a_lo, lda):
    """In-place unblocked dd Cholesky in the reference's order
    (mplapack/chol.py:21-65).  Returns (rc, info): rc = reference argument
    index of an invalid argument, else 0; info as chol.py returns it."""
    info = ctypes.c_int64(0)
    rc = lib().oracle_rpotrf(_flag(uplo), n, _ptr(a_hi), _ptr(a_lo), lda, ctypes.byref(info))
    return rc, int(info.value)


def rtrsm(side, uplo, transa, diag, m, n, alpha, a_hi, a_lo, lda, b_hi, b_lo, ldb):
    """In-place dd triangular solve in the reference's order
    (mpblas/level23.py:288-380); alpha = (hi, lo).  Returns the reference
    argument index of an invalid argument, else 0."""
    return lib().oracle_rtrsm(_flag(side), _flag(uplo), _flag(transa), _flag(diag), m, n,
                              float(alpha[0]), float(alpha[1]), _ptr(a_hi), _ptr(a_lo), lda,
                              _ptr(b_hi), _ptr(b_lo), ldb)


def rgetrf(m, n, a_hi, a_lo, lda):
    """In-place dd LU with partial pivoting (mplapack/lu.py:74-114).
    Returns (rc, ipiv list (1-based), info)."""
    mn = max(0, min(m, n))
    ipiv = (ctypes.c_int64 * max(1, mn))()
    info = ctypes.c_int64(0)
    rc = lib().oracle_rgetrf(m, n, _ptr(a_hi), _ptr(a_lo), lda, ipiv, ctypes.byref(info))
    return rc, [int(ipiv[i]) for i in range(mn)], int(info.value)


def rgetrs(trans, n, nrhs, a_hi, a_lo, lda, ipiv, b_hi, b_lo, ldb):
    """In-place solve with an Rgetrf factorization (mplapack/lu.py:117-145)."""
    arr = (ctypes.c_int64 * max(1, len(ipiv)))(*ipiv)
    return lib().oracle_rgetrs(_flag(trans), n, nrhs, _ptr(a_hi), _ptr(a_lo), lda, arr, len(ipiv),
                               _ptr(b_hi), _ptr(b_lo), ldb)


def dpotrf(uplo, n, a, lda):
    """binary64 Rpotrf (F64 backend); returns (rc, info)."""
    info = ctypes.c_int64(0)
    rc = lib().oracle_dpotrf(_flag(uplo), n, _ptr(a), lda, ctypes.byref(info))
    return rc, int(info.value)


def dtrsm(side, uplo, transa, diag, m, n, alpha, a, lda, b, ldb):
    return lib().oracle_dtrsm(_flag(side), _flag(uplo), _flag(transa), _flag(diag), m, n,
                              float(alpha), _ptr(a), lda, _ptr(b), ldb)


def dgetrf(m, n, a, lda):
    mn = max(0, min(m, n))
    ipiv = (ctypes.c_int64 * max(1, mn))()
    info = ctypes.c_int64(0)
    rc = lib().oracle_dgetrf(m, n, _ptr(a), lda, ipiv, ctypes.byref(info))
    return rc, [int(ipiv[i]) for i in range(mn)], int(info.value)


def dgetrs(trans, n, nrhs, a, lda, ipiv, b, ldb):
    arr = (ctypes.c_int64 * max(1, len(ipiv)))(*ipiv)
    return lib().oracle_dgetrs(_flag(trans), n, nrhs, _ptr(a), lda, arr, len(ipiv), _ptr(b), ldb)


def div2(x, y):
    out = np.zeros(2)
    lib().oracle_div2(x[0], x[1], y[0], y[1], _ptr(out))
    return float(out[0]), float(out[1])


def sqrt2(x):
    out = np.zeros(2)
    lib().oracle_sqrt2(x[0], x[1], _ptr(out))
    return float(out[0]), float(out[1])


def add2(x, y):
    out = np.zeros(2)
    lib().oracle_add2(x[0], x[1], y[0], y[1], _ptr(out))
    return float(out[0]), float(out[1])


def mul2(x, y):
    out = np.zeros(2)
    lib().oracle_mul2(x[0], x[1], y[0], y[1], _ptr(out))
    return float(out[0]), float(out[1])


def two_prod(a, b):
    out = np.zeros(2)
    lib().oracle_two_prod(a, b, _ptr(out))
    return float(out[0]), float(out[1])


def max_threads():
    return lib().oracle_max_threads()
