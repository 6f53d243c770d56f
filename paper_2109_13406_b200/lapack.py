"""Drop-in ``Rpotrf`` / ``Rgetrf`` (dd Cholesky, LU) on the B200.

The O(n^3) work runs as GPU ``Rsyrk`` / ``Rgemm`` trailing updates.

Same call surface, validation order, BlasError indices and return value as
the reference (``/root/reference/pkg/src/mpkit/mplapack/chol.py:21-65``):

  info = Rpotrf(uplo, n, a, lda=None)

A = L*L^T (uplo 'L') or U^T*U ('U') in place on that triangle; info = 0, or
j + 1 for the first pivot that is NaN or <= 0, whose value is left in A(j, j)
with the later entries as the reference leaves them.  Keywords:

  mode  "exact": bit-identical to the reference (operands inside the safe
        window), blocked, the trailing updates are exact-mode Rsyrk calls;
        "fast" (default, env DDBLAS_MODE) / "twosum": the same blocked
        algorithm with those modes' Rsyrk -- residual within the reference's
        testkit threshold (testkit.residual_chol < 30); "reference": the
        trailing updates on the checked one-thread-per-element kernel.
  nb    outer block width = the trailing updates' depth (default 256, env
        DDB_POTRF_NB); the inner (diagonal-block) width is min(nb, 64).

``a`` is a dd ``DeviceMatrix`` (asynchronous up to the final info read) or a
host matrix (``HostMatrix`` / the reference's Matrix; staged through HBM).
binary64 ('f64') matrices run the same algorithms in the F64 backend's IEEE
arithmetic, bit-identical to the reference (``mode`` does not apply).  Other
precisions raise NotImplementedError; there is no CPU fallback.
"""

from __future__ import annotations

import ctypes

from . import _lib
from .matrix import check_storage, require
from .mpblas import _HostPlanes, _dev_ptr, _mode_code, _placement, _raise_rc

__all__ = ["Rpotrf", "Rgetrf", "Rgetrs", "PivotVector"]


def _precision(routine, *mats):
    """True for the reference's binary64 Matrix ('f64'), False for 'dd'."""
    tags = {m.precision for m in mats}
    if len(tags) > 1:
        raise ValueError(f"{routine}: mixed precisions {sorted(tags)}")
    tag = tags.pop()
    if tag not in ("dd", "f64"):
        raise NotImplementedError(
            f"{routine}: precision {tag!r} is not on the B200 path (only 'dd' and 'f64')")
    return tag == "f64"


class PivotVector:
    """1-based row interchange record (mplapack/lu.py:17-41): row k was
    swapped with ipiv[k-1]."""

    def __init__(self, ipiv=()):
        self.ipiv = [int(p) for p in ipiv]

    def __len__(self):
        return len(self.ipiv)

    def __getitem__(self, k):
        return self.ipiv[k]

    def __iter__(self):
        return iter(self.ipiv)

    def __eq__(self, other):
        other = list(other) if not isinstance(other, PivotVector) else other.ipiv
        return self.ipiv == other

    def __repr__(self):
        return f"PivotVector({self.ipiv})"


def Rgetrf(m, n, a, lda=None, *, mode=None):
    """A = P*L*U in place (mplapack/lu.py:74-114); returns (PivotVector, info).

    info = k > 0 flags an exactly zero pivot U(k, k); the factorization still
    completes.  mode "exact" / "reference": bit-identical to the reference;
    "fast" / "twosum": the trailing updates in that mode (the pivot order can
    then differ where two candidates agree to ~2**-100)."""
    routine = "Rgetrf"
    lda = a.ld if lda is None else lda
    require(routine, m >= 0, 1)                                     # lu.py:83-85
    require(routine, n >= 0, 2)
    require(routine, lda >= max(1, m), 4)
    if m == 0 or n == 0:                                            # lu.py:86-87
        return PivotVector(), 0
    f64 = _precision(routine, a)
    code = _mode_code(mode)
    check_storage(a, m, n, lda)
    L = _lib.load()
    mn = min(m, n)
    ipiv = (ctypes.c_int64 * mn)()
    info = ctypes.c_int(0)
    dev = _placement(routine, a)
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            if f64:
                rc = L.ddb_dgetrf(m, n, _dev_ptr(a, 0), lda, ipiv, ctypes.byref(info), stream)
            else:
                rc = L.ddb_rgetrf(m, n, _dev_ptr(a, 0), _dev_ptr(a, 1), lda, ipiv,
                                  ctypes.byref(info), code, stream)
        _raise_rc(routine, rc)
    else:
        ha = _HostPlanes(a.store, 1 if f64 else 2)
        if f64:
            rc = L.ddb_dgetrf_host(m, n, ha.ptr(0), lda, ipiv, ctypes.byref(info), None)
        else:
            rc = L.ddb_rgetrf_host(m, n, ha.ptr(0), ha.ptr(1), lda, ipiv, ctypes.byref(info),
                                   code, None)
        _raise_rc(routine, rc)
        ha.commit()
    return PivotVector(ipiv[:]), int(info.value)


def Rpotrf(uplo, n, a, lda=None, *, mode=None, nb=0):
    routine = "Rpotrf"
    lda = a.ld if lda is None else lda
    ok = isinstance(uplo, str) and uplo.upper() in ("U", "L")     # chol.py:24-26
    require(routine, ok, 1)
    uplo = uplo.upper()
    require(routine, n >= 0, 2)                                     # chol.py:28
    require(routine, lda >= max(1, n), 4)                           # chol.py:29
    if n == 0:                                                      # chol.py:30-31
        return 0
    f64 = _precision(routine, a)
    code = _mode_code(mode)
    check_storage(a, n, n, lda)
    L = _lib.load()
    info = ctypes.c_int(0)
    dev = _placement(routine, a)
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            if f64:
                rc = L.ddb_dpotrf(uplo.encode(), n, _dev_ptr(a, 0), lda, int(nb), stream,
                                  ctypes.byref(info))
            else:
                rc = L.ddb_rpotrf(uplo.encode(), n, _dev_ptr(a, 0), _dev_ptr(a, 1), lda, int(nb),
                                  code, stream, ctypes.byref(info))
        _raise_rc(routine, rc)
        return int(info.value)
    ha = _HostPlanes(a.store, 1 if f64 else 2)
    if f64:
        rc = L.ddb_dpotrf_host(uplo.encode(), n, ha.ptr(0), lda, int(nb), None, ctypes.byref(info))
    else:
        rc = L.ddb_rpotrf_host(uplo.encode(), n, ha.ptr(0), ha.ptr(1), lda, int(nb), code, None,
                               ctypes.byref(info))
    _raise_rc(routine, rc)
    ha.commit()
    return int(info.value)


def Rgetrs(trans, n, nrhs, a, lda=None, ipiv=None, b=None, ldb=None, *, mode=None):
    """Solve op(A)*X = B in place in B from an Rgetrf factorization
    (mplapack/lu.py:117-145); returns 0.  mode as for Rtrsm."""
    routine = "Rgetrs"
    lda = a.ld if lda is None else lda
    ldb = b.ld if (b is not None and ldb is None) else ldb
    ok = isinstance(trans, str) and trans.upper() in ("N", "T", "C")   # lu.py:123-125
    require(routine, ok, 1)
    trans = trans.upper()
    require(routine, n >= 0, 2)
    require(routine, nrhs >= 0, 3)
    require(routine, lda >= max(1, n), 5)
    require(routine, ldb is not None and ldb >= max(1, n), 8)
    if n == 0 or nrhs == 0:                                         # lu.py:130-131
        return 0
    f64 = _precision(routine, a, b)
    code = _mode_code(mode)
    check_storage(b, n, nrhs, ldb)
    piv = (ctypes.c_int64 * n)(*[int(p) for p in list(ipiv)[:n]])
    L = _lib.load()
    dev = _placement(routine, a, b)
    if dev is not None:
        import torch
        with torch.cuda.device(dev):
            stream = torch.cuda.current_stream(dev).cuda_stream
            if f64:
                rc = L.ddb_dgetrs(trans.encode(), n, nrhs, _dev_ptr(a, 0), lda, piv,
                                  _dev_ptr(b, 0), ldb, stream)
            else:
                rc = L.ddb_rgetrs(trans.encode(), n, nrhs, _dev_ptr(a, 0), _dev_ptr(a, 1), lda,
                                  piv, _dev_ptr(b, 0), _dev_ptr(b, 1), ldb, code, stream)
        _raise_rc(routine, rc)
        return 0
    np_ = 1 if f64 else 2
    ha, hb = _HostPlanes(a.store, np_), _HostPlanes(b.store, np_)
    if f64:
        rc = L.ddb_dgetrs_host(trans.encode(), n, nrhs, ha.ptr(0), lda, piv, hb.ptr(0), ldb, None)
    else:
        rc = L.ddb_rgetrs_host(trans.encode(), n, nrhs, ha.ptr(0), ha.ptr(1), lda, piv,
                               hb.ptr(0), hb.ptr(1), ldb, code, None)
    _raise_rc(routine, rc)
    hb.commit()
    return 0
