"""Drop-in ``Rgemm`` / ``Rsyrk`` over dd (hi, lo) planes, computed on the B200.

Same call surface, defaults, validation order, error types / indices and
early exits as the reference (``/root/reference/pkg/src/mpkit/mpblas/``):

  Rgemm(transa, transb, m, n, k, alpha, a, lda=None, b=None, ldb=None,
        beta=1.0, c=None, ldc=None)                          level23.py:180-198
  Rsyrk(uplo, trans, n, k, alpha, a, lda=None, beta=1.0, c=None, ldc=None)
                                                             level23.py:226-270

plus one keyword, ``mode``:

  "fast"   (default; env ``DDBLAS_MODE`` overrides) certified-anchor dd
           accumulation on the FP64 pipe, componentwise error
           <= c*k*2**-104*(|alpha| sum|a*b| + |beta||c|), c = 4 -- the
           north-star tolerance -- for every input: elements whose row /
           column exponent spreads are too wide for the certified bound
           (and calls with k > 2**17) take the TwoSum accumulation, elements
           whose op(A) row / op(B) column holds an inf / nan / out-of-window
           value take the reference-semantics kernel.  Not bitwise equal to
           the reference: of the reference's own pins it keeps the integer
           instance (test_acceptance.py:121-139) but not the Hilbert n = 2
           residual of exactly (2**-106, 0) (test_acceptance.py:298-305),
           which it meets only to the dd bound (tests/test_gpu_pins.py)
  "twosum" the same bound with TwoSum accumulation (no bound GEMM; slower)
  "exact"  bit-identical to the reference's result (every reference pin);
           the mode to select (``mode="exact"`` or DDBLAS_MODE=exact) when a
           drop-in must reproduce the reference bit for bit
  "reference"  the one-thread-per-element checked kernel (debugging)

C is updated in place; A and B are read only; nothing is returned.
Precision 'f64' (the reference's binary64 Matrix, one plane) runs the same
routines over the reference's F64 backend bit for bit (``mode`` is ignored).
Operands are either all ``DeviceMatrix`` (planes resident in HBM; the call is
asynchronous on torch's current stream) or all host matrices (numpy planes:
``HostMatrix`` or the reference's own ``mpkit`` Matrix; the call stages
through device memory and returns after C is back on the host).  The complex
precisions raise NotImplementedError -- there is no CPU fallback.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

from . import _lib
from .matrix import (BlasError, check_storage, dd_is_one, dd_truthy, is_device, require,
                     same_precision, to_c64, to_cdd, to_dd)

__all__ = ["Rgemm", "Rsyrk", "Rtrsm", "Cgemm", "BlasError", "default_mode"]


def default_mode():
    return os.environ.get("DDBLAS_MODE", "fast")


def _flag(routine, value, allowed, index):
    """level23.py:23-26."""
    ok = isinstance(value, str) and len(value) == 1 and value.upper() in allowed
    require(routine, ok, index)
    return value.upper()


def _ld_of(mat, ld):
    return mat.ld if ld is None else ld


def _mode_code(mode):
    mode = default_mode() if mode is None else mode
    try:
        return _lib.MODES[mode]
    except KeyError:
        raise ValueError(f"unknown mode {mode!r}; expected one of {sorted(_lib.MODES)}") from None


def _raise_rc(routine, rc):
    if rc > 0:
        raise BlasError(routine, rc)
    if rc < 0:
        raise RuntimeError(f"{routine}: CUDA failure ({rc}): {_lib.last_error()}")


def _precision_gate(routine, tag):
    if tag not in ("dd", "f64"):
        raise NotImplementedError(
            f"{routine}: precision {tag!r} is not on the B200 path (only 'dd' and 'f64')")


def _scalar(tag, v):
    """``_scalar_for`` (matrix.py:29-37): DDouble for dd, float() for f64."""
    if tag == "f64":
        f = float(v)
        return f, 0.0
    return to_dd(v)


class _HostPlanes:
    """Contiguous float64 views of a host store; writes back on ``commit``."""

    def __init__(self, store, nplanes=2, dtype=np.float64):
        self.src = store
        self.planes = [p if (isinstance(p, np.ndarray) and p.dtype == dtype
                             and p.flags.c_contiguous)
                       else np.ascontiguousarray(p, dtype=dtype) for p in store[:nplanes]]

    def ptr(self, i):
        return self.planes[i].ctypes.data

    def commit(self):
        for dst, src in zip(self.src[:len(self.planes)], self.planes):
            if dst is not src:
                dst[...] = src


def _dev_ptr(mat, i):
    return mat.store[i].data_ptr()


def _placement(routine, *mats):
    kinds = {is_device(m) for m in mats}
    if len(kinds) > 1:
        raise ValueError(f"{routine}: operands must all be device or all be host matrices")
    if kinds.pop():
        devs = {m.store[0].device for m in mats}
        if len(devs) > 1:
            raise ValueError(f"{routine}: operands on different devices {sorted(map(str, devs))}")
        return devs.pop()
    return None


def Rgemm(transa, transb, m, n, k, alpha, a, lda=None, b=None, ldb=None,
          beta=1.0, c=None, ldc=None, *, mode=None, _check_storage=True):
    """C <- alpha*op(A)*op(B) + beta*C on the B200 (level23.py:180-198).

    (``_check_storage=False`` is for sub-matrix views made by parallel.py,
    whose storage ends before ``ld*ncol``; the kernels never touch it.)"""
    routine = "Rgemm"
    tag = same_precision(routine, a, b, c)
    if tag in ("cdd", "c64"):   # the reference's Rgemm runs any backend (level23.py:180-198)
        return _complex_gemm(routine, transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c,
                             ldc, mode)
    _precision_gate(routine, tag)
    lda, ldb, ldc = _ld_of(a, lda), _ld_of(b, ldb), _ld_of(c, ldc)
    transa = _flag(routine, transa, ("N", "T", "C"), 1)
    transb = _flag(routine, transb, ("N", "T", "C"), 2)
    require(routine, m >= 0, 3)
    require(routine, n >= 0, 4)
    require(routine, k >= 0, 5)
    nrowa, ncola = (m, k) if transa == "N" else (k, m)
    nrowb, ncolb = (k, n) if transb == "N" else (n, k)
    require(routine, lda >= max(1, nrowa), 8)
    require(routine, ldb >= max(1, nrowb), 10)
    require(routine, ldc >= max(1, m), 13)
    al = _scalar(tag, alpha)
    be = _scalar(tag, beta)
    code = _mode_code(mode)
    if m == 0 or n == 0 or ((not dd_truthy(al) or k == 0) and dd_is_one(be)):
        return
    if _check_storage:
        check_storage(a, nrowa, ncola, lda)
        check_storage(b, nrowb, ncolb, ldb)
        check_storage(c, m, n, ldc)
    L = _lib.load()
    dev = _placement(routine, a, b, c)
    if tag == "f64":
        head = (transa.encode(), transb.encode(), m, n, k, al[0])
        if dev is not None:
            import torch
            with torch.cuda.device(dev):
                stream = torch.cuda.current_stream(dev).cuda_stream
                rc = L.ddb_dgemm(*head, _dev_ptr(a, 0), lda, _dev_ptr(b, 0), ldb, be[0],
                                 _dev_ptr(c, 0), ldc, stream)
            _raise_rc(routine, rc)
            return
        ha, hb, hc = _HostPlanes(a.store, 1), _HostPlanes(b.store, 1), _HostPlanes(c.store, 1)
        rc = L.ddb_dgemm_host(*head, ha.ptr(0), lda, hb.ptr(0), ldb, be[0], hc.ptr(0), ldc, None)
        _raise_rc(routine, rc)
        hc.commit()
        return
    args_head = (transa.encode(), transb.encode(), m, n, k, al[0], al[1])
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            rc = L.ddb_rgemm(*args_head, _dev_ptr(a, 0), _dev_ptr(a, 1), lda,
                             _dev_ptr(b, 0), _dev_ptr(b, 1), ldb, be[0], be[1],
                             _dev_ptr(c, 0), _dev_ptr(c, 1), ldc, code, stream)
        _raise_rc(routine, rc)
        return
    ha, hb, hc = _HostPlanes(a.store), _HostPlanes(b.store), _HostPlanes(c.store)
    rc = L.ddb_rgemm_host(*args_head, ha.ptr(0), ha.ptr(1), lda, hb.ptr(0), hb.ptr(1), ldb,
                          be[0], be[1], hc.ptr(0), hc.ptr(1), ldc, code, None)
    _raise_rc(routine, rc)
    hc.commit()


def Rsyrk(uplo, trans, n, k, alpha, a, lda=None, beta=1.0, c=None, ldc=None, *, mode=None,
          _check_storage=True):
    """C <- alpha*A*A^T + beta*C (trans='N') or alpha*A^T*A + beta*C on the
    uplo triangle only (level23.py:226-270)."""
    routine = "Rsyrk"
    tag = same_precision(routine, a, c)
    _precision_gate(routine, tag)
    lda, ldc = _ld_of(a, lda), _ld_of(c, ldc)
    uplo = _flag(routine, uplo, ("U", "L"), 1)
    trans = _flag(routine, trans, ("N", "T", "C"), 2)
    require(routine, n >= 0, 3)
    require(routine, k >= 0, 4)
    nrowa, ncola = (n, k) if trans == "N" else (k, n)
    require(routine, lda >= max(1, nrowa), 7)
    require(routine, ldc >= max(1, n), 10)
    al = _scalar(tag, alpha)
    be = _scalar(tag, beta)
    code = _mode_code(mode)
    if n == 0 or ((not dd_truthy(al) or k == 0) and dd_is_one(be)):
        return
    if _check_storage:
        check_storage(c, n, n, ldc)
        if dd_truthy(al):
            check_storage(a, nrowa, ncola, lda)   # A viewed only when alpha != 0 (:250-260)
    L = _lib.load()
    dev = _placement(routine, a, c)
    if tag == "f64":
        head = (uplo.encode(), trans.encode(), n, k, al[0])
        if dev is not None:
            import torch
            with torch.cuda.device(dev):
                stream = torch.cuda.current_stream(dev).cuda_stream
                rc = L.ddb_dsyrk(*head, _dev_ptr(a, 0), lda, be[0], _dev_ptr(c, 0), ldc, stream)
            _raise_rc(routine, rc)
            return
        ha, hc = _HostPlanes(a.store, 1), _HostPlanes(c.store, 1)
        rc = L.ddb_dsyrk_host(*head, ha.ptr(0), lda, be[0], hc.ptr(0), ldc, None)
        _raise_rc(routine, rc)
        hc.commit()
        return
    args_head = (uplo.encode(), trans.encode(), n, k, al[0], al[1])
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            rc = L.ddb_rsyrk(*args_head, _dev_ptr(a, 0), _dev_ptr(a, 1), lda, be[0], be[1],
                             _dev_ptr(c, 0), _dev_ptr(c, 1), ldc, code, stream)
        _raise_rc(routine, rc)
        return
    ha, hc = _HostPlanes(a.store), _HostPlanes(c.store)
    rc = L.ddb_rsyrk_host(*args_head, ha.ptr(0), ha.ptr(1), lda, be[0], be[1],
                          hc.ptr(0), hc.ptr(1), ldc, code, None)
    _raise_rc(routine, rc)
    hc.commit()


def Rtrsm(side, uplo, transa, diag, m, n, alpha, a, lda=None, b=None, ldb=None, *,
          mode=None):
    """Solve op(A)*X = alpha*B (side 'L') or X*op(A) = alpha*B ('R') in place
    in B on the B200 (level23.py:288-380; checks :292-304).  mode "exact" /
    "reference": bit-identical to the reference; "fast" / "twosum": blocked
    with fast-mode GEMM updates (dd accuracy, not bit-identical)."""
    routine = "Rtrsm"
    tag = same_precision(routine, a, b)
    _precision_gate(routine, tag)
    f64 = tag == "f64"
    lda, ldb = _ld_of(a, lda), _ld_of(b, ldb)
    side = _flag(routine, side, ("L", "R"), 1)
    uplo = _flag(routine, uplo, ("U", "L"), 2)
    transa = _flag(routine, transa, ("N", "T", "C"), 3)
    diag = _flag(routine, diag, ("U", "N"), 4)
    require(routine, m >= 0, 5)
    require(routine, n >= 0, 6)
    nrowa = m if side == "L" else n
    require(routine, lda >= max(1, nrowa), 9)
    require(routine, ldb >= max(1, m), 11)
    al = _scalar(tag, alpha)
    code = _mode_code(mode)
    if m == 0 or n == 0:
        return
    check_storage(a, nrowa, nrowa, lda)
    check_storage(b, m, n, ldb)
    L = _lib.load()
    dev = _placement(routine, a, b)
    flags = (side.encode(), uplo.encode(), transa.encode(), diag.encode(), m, n)
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            if f64:
                rc = L.ddb_dtrsm(*flags, al[0], _dev_ptr(a, 0), lda, _dev_ptr(b, 0), ldb, stream)
            else:
                rc = L.ddb_rtrsm(*flags, al[0], al[1], _dev_ptr(a, 0), _dev_ptr(a, 1), lda,
                                 _dev_ptr(b, 0), _dev_ptr(b, 1), ldb, code, stream)
        _raise_rc(routine, rc)
        return
    np_ = 1 if f64 else 2
    ha, hb = _HostPlanes(a.store, np_), _HostPlanes(b.store, np_)
    if f64:
        rc = L.ddb_dtrsm_host(*flags, al[0], ha.ptr(0), lda, hb.ptr(0), ldb, None)
    else:
        rc = L.ddb_rtrsm_host(*flags, al[0], al[1], ha.ptr(0), ha.ptr(1), lda, hb.ptr(0),
                              hb.ptr(1), ldb, code, None)
    _raise_rc(routine, rc)
    hb.commit()


def Cgemm(transa, transb, m, n, k, alpha, a, lda=None, b=None, ldb=None,
          beta=1.0, c=None, ldc=None, *, mode=None):
    """Complex GEMM, 'C' flags conjugate (level23.py:201-221).

    'cdd' (complex double-double, four planes) and 'c64' (complex128).
    Reference quirks kept: a DDComplex has no truth value, so for 'cdd' the
    alpha == 0 shortcut never fires and beta == 0 multiplies C."""
    routine = "Cgemm"
    tag = same_precision(routine, a, b, c)
    if tag not in ("cdd", "c64"):
        if tag in ("dd", "f64"):
            raise ValueError("Cgemm requires complex matrices")
        raise NotImplementedError(f"{routine}: precision {tag!r} is not on the B200 path")
    return _complex_gemm(routine, transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc,
                         mode)


def _complex_gemm(routine, transa, transb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, mode):
    tag = a.precision
    lda, ldb, ldc = _ld_of(a, lda), _ld_of(b, ldb), _ld_of(c, ldc)
    transa = _flag(routine, transa, ("N", "T", "C"), 1)
    transb = _flag(routine, transb, ("N", "T", "C"), 2)
    require(routine, m >= 0, 3)
    require(routine, n >= 0, 4)
    require(routine, k >= 0, 5)
    nrowa, ncola = (m, k) if transa == "N" else (k, m)
    nrowb, ncolb = (k, n) if transb == "N" else (n, k)
    require(routine, lda >= max(1, nrowa), 8)
    require(routine, ldb >= max(1, nrowb), 10)
    require(routine, ldc >= max(1, m), 13)
    if tag == "cdd":
        al, be = to_cdd(alpha), to_cdd(beta)
        alpha_zero = False                       # DDComplex is always truthy
        beta_one = be[0] == 1.0 and be[1] == 0.0 and be[2] == 0.0 and be[3] == 0.0
    else:
        al, be = to_c64(alpha), to_c64(beta)
        alpha_zero = al == 0
        beta_one = be == 1
    code = _mode_code(mode)
    if m == 0 or n == 0 or ((alpha_zero or k == 0) and beta_one):
        return
    check_storage(a, nrowa, ncola, lda)
    check_storage(b, nrowb, ncolb, ldb)
    check_storage(c, m, n, ldc)
    L = _lib.load()
    dev = _placement(routine, a, b, c)
    fl = (transa.encode(), transb.encode(), m, n, k)
    if tag == "c64":
        av = ctypes.cast((ctypes.c_double * 2)(al.real, al.imag), ctypes.c_void_p)
        bv = ctypes.cast((ctypes.c_double * 2)(be.real, be.imag), ctypes.c_void_p)
        if dev is not None:
            import torch
            with torch.cuda.device(dev):
                stream = torch.cuda.current_stream(dev).cuda_stream
                rc = L.ddb_zgemm(*fl, av, _dev_ptr(a, 0), lda, _dev_ptr(b, 0), ldb, bv,
                                 _dev_ptr(c, 0), ldc, stream)
            _raise_rc(routine, rc)
            return
        ha, hb, hc = (_HostPlanes(x.store, 1, np.complex128) for x in (a, b, c))
        rc = L.ddb_zgemm_host(*fl, av, ha.ptr(0), lda, hb.ptr(0), ldb, bv, hc.ptr(0), ldc, None)
        _raise_rc(routine, rc)
        hc.commit()
        return
    keep = [(ctypes.c_double * 4)(*al), (ctypes.c_double * 4)(*be)]
    av, bv = (ctypes.cast(x, ctypes.c_void_p) for x in keep)

    def P4(*ptrs):
        arr = (ctypes.c_void_p * 4)(*ptrs)
        keep.append(arr)
        return ctypes.cast(arr, ctypes.c_void_p)
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            rc = L.ddb_cgemm(*fl, av, P4(*(_dev_ptr(a, i) for i in range(4))), lda,
                             P4(*(_dev_ptr(b, i) for i in range(4))), ldb, bv,
                             P4(*(_dev_ptr(c, i) for i in range(4))), ldc, code, stream)
        _raise_rc(routine, rc)
        return
    ha, hb, hc = (_HostPlanes(x.store, 4) for x in (a, b, c))
    rc = L.ddb_cgemm_host(*fl, av, P4(*(ha.ptr(i) for i in range(4))), lda,
                          P4(*(hb.ptr(i) for i in range(4))), ldb, bv,
                          P4(*(hc.ptr(i) for i in range(4))), ldc, code, None)
    _raise_rc(routine, rc)
    hc.commit()
