"""Containers, scalar coercion and argument errors of the drop-in surface.

Mirrors the parts of the reference the dd Rgemm / Rsyrk path touches:

* ``BlasError``           mpkit/mpblas/matrix.py:18-26 (message and attributes)
* ``same_precision``      mpkit/mpblas/matrix.py:235-239
* ``to_dd``               the ``_scalar_for('dd', v)`` -> ``DDouble(v)`` coercion
                          of alpha / beta (matrix.py:29-37, ddarith.py:192-214,
                          decimal strings: ddarith.py:504-532)
* ``HostMatrix``          the reference ``Matrix`` layout: column-major, element
                          (i, j) at ``i + j*ld``, dd store = (hi, lo) float64
                          planes (matrix.py:100-195, elem.py DDBackend)
* ``DeviceMatrix``        the same layout with the planes resident in HBM as
                          torch CUDA tensors (no host staging per call)

Any object with ``m, n, ld, precision, store`` attributes is accepted by
``Rgemm`` / ``Rsyrk`` -- in particular the reference's own ``mpkit`` Matrix.
"""

from __future__ import annotations

import math
import re
from fractions import Fraction

import numpy as np


class BlasError(ValueError):
    """Invalid argument, reported with the reference argument index."""

    def __init__(self, routine, index):
        self.routine = routine
        self.index = index
        super().__init__(
            f"on entry to {routine} parameter number {index} "
            "had an illegal value")


def require(routine, cond, index):
    if not cond:
        raise BlasError(routine, index)


def same_precision(routine, *objs):
    tags = {o.precision for o in objs}
    if len(tags) > 1:
        raise ValueError(f"{routine}: mixed precisions {sorted(tags)}")
    return tags.pop()


# --------------------------------------------------------------------------
# dd scalars (alpha, beta)

_DECIMAL_RE = re.compile(
    r"^\s*([+-]?)(?:(\d+)(?:\.(\d*))?|\.(\d+))(?:[eE]([+-]?\d+))?\s*$")


def _two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def _norm(hi, lo):
    s, e = _two_sum(hi, lo)
    return (s, e) if math.isfinite(s) else (s, 0.0)


def _round_fraction(v):
    try:
        hi = float(v)
    except OverflowError:
        return (math.inf if v > 0 else -math.inf), 0.0
    if math.isinf(hi):
        return hi, 0.0
    return _norm(hi, float(v - Fraction(hi)))


def _parse_decimal(s):
    m = _DECIMAL_RE.match(s)
    if not m:
        raise ValueError(f"not a decimal number: {s!r}")
    sign, ip, fp1, fp2, ex = m.groups()
    frac = (fp1 if fp1 is not None else fp2) or ""
    v = Fraction(int((ip or "") + frac), 1) * Fraction(10) ** (int(ex or 0) - len(frac))
    return _round_fraction(-v if sign == "-" else v)


def to_dd(value):
    """Coerce alpha / beta exactly as ``DDouble(value)`` does; returns (hi, lo)."""
    if hasattr(value, "hi") and hasattr(value, "lo") and not isinstance(value, (int, float, str)):
        return float(value.hi), float(value.lo)
    if isinstance(value, str):
        return _parse_decimal(value)
    if isinstance(value, float):
        return float(value), 0.0
    if isinstance(value, int):
        try:
            hi = float(value)
        except OverflowError:
            return (math.inf if value > 0 else -math.inf), 0.0
        if math.isfinite(hi):
            return _norm(hi, float(value - int(hi)))
        return hi, 0.0
    raise TypeError(f"cannot make DDouble from {type(value).__name__}")


def to_cdd(value):
    """``_scalar_for('cdd', v)`` (matrix.py:36-37): DDComplex(value) as
    (re_hi, re_lo, im_hi, im_lo)."""
    if hasattr(value, "re") and hasattr(value, "im"):
        return to_dd(value.re) + to_dd(value.im)
    if isinstance(value, complex):
        return to_dd(value.real) + to_dd(value.imag)
    return to_dd(value) + (0.0, 0.0)


def to_c64(value):
    """``_scalar_for('c64', v)``: complex(value)."""
    return complex(value)


def dd_truthy(v):
    """``DDouble.__bool__`` (ddarith.py:290-291)."""
    return v[0] != 0.0 or v[1] != 0.0


def dd_is_one(v):
    """``DDouble == 1`` via ``_cmp2`` (ddarith.py:166-176)."""
    return v[0] == 1.0 and v[1] == 0.0


# --------------------------------------------------------------------------
# containers

PRECISIONS = {"dd": 2, "f64": 1, "cdd": 4, "c64": 1}   # planes per matrix (c64: complex128)


def _planes(precision):
    try:
        return PRECISIONS[precision]
    except KeyError:
        raise NotImplementedError(
            f"precision {precision!r} is not on the B200 path") from None


def _plane_dtype(precision):
    return np.complex128 if precision == "c64" else np.float64


class HostMatrix:
    """m x n dd matrix in host memory, column-major (hi, lo) numpy planes.

    Same attributes as the reference ``mpkit.mpblas.Matrix`` for the dd
    precision (``m, n, ld, precision, store``)."""

    def __init__(self, m, n, precision="dd", ld=None, pinned=False):
        if m < 0 or n < 0:
            raise ValueError("matrix dimensions must be >= 0")
        ld = max(1, m) if ld is None else ld
        if ld < max(1, m):
            raise ValueError("leading dimension too small")
        planes = _planes(precision)
        self.m, self.n, self.ld, self.precision = m, n, ld, precision
        size = ld * n
        if pinned:
            import torch
            tdt = torch.complex128 if precision == "c64" else torch.float64
            self.store = tuple(torch.zeros(size, dtype=tdt, pin_memory=True).numpy()
                               for _ in range(planes))
        else:
            self.store = tuple(np.zeros(size, dtype=_plane_dtype(precision)) for _ in range(planes))

    @classmethod
    def from_planes(cls, m, n, hi, lo=None, ld=None):
        """dd from (hi, lo); binary64 ('f64') when lo is None."""
        a = cls(0, 0, "dd" if lo is not None else "f64")
        a.m, a.n = m, n
        a.ld = max(1, m) if ld is None else ld
        a.store = tuple(np.ascontiguousarray(p, dtype=np.float64)
                        for p in ((hi, lo) if lo is not None else (hi,)))
        return a

    def to_device(self, device=None):
        return DeviceMatrix.from_host(self, device)

    def __repr__(self):
        return f"HostMatrix({self.m}x{self.n}, ld={self.ld}, precision={self.precision!r})"


class SharedHostMatrix(HostMatrix):
    """HostMatrix whose planes live in POSIX shared memory, so that every
    process of a one-process-per-GPU job maps the same host buffer and copies
    its own part over its own PCIe link (parallel.rgemm_host_shared).

    The creator (``create=True``) allocates; the others attach by ``name``.
    ``pin()`` page-locks this process's mapping through the library
    (``ddb_host_register``) so the host entry points copy by DMA."""

    def __init__(self, m, n, precision="dd", ld=None, name=None, create=False):
        from multiprocessing import shared_memory
        ld = max(1, m) if ld is None else ld
        if ld < max(1, m) or m < 0 or n < 0:
            raise ValueError("bad shared matrix shape")
        self.m, self.n, self.ld, self.precision = m, n, ld, precision
        planes = _planes(precision)
        dt = np.dtype(_plane_dtype(precision))
        self._plane_bytes = ld * n * dt.itemsize
        nbytes = max(1, planes * self._plane_bytes)
        self._shm = shared_memory.SharedMemory(name=name, create=create, size=nbytes)
        self.name = self._shm.name
        self._owner = create
        self._pinned = False
        self.store = tuple(np.ndarray((ld * n,), dtype=dt, buffer=self._shm.buf,
                                      offset=i * self._plane_bytes) for i in range(planes))

    def pin(self):
        from . import _lib
        if not self._pinned and self._plane_bytes:
            rc = _lib.load().ddb_host_register(self.store[0].ctypes.data,
                                               len(self.store) * self._plane_bytes)
            if rc != 0:
                raise RuntimeError(f"ddb_host_register: {_lib.last_error()}")
            self._pinned = True
        return self

    def close(self):
        """Unpin, unmap, and (creator) unlink the shared segment."""
        if self._pinned:
            from . import _lib
            _lib.load().ddb_host_unregister(self.store[0].ctypes.data)
            self._pinned = False
        self.store = ()
        self._shm.close()
        if self._owner:
            self._shm.unlink()


class DeviceMatrix:
    """m x n dd matrix resident in HBM: ``store = (hi, lo)`` torch float64
    CUDA tensors of length ``ld*n`` in the reference's column-major layout."""

    def __init__(self, m, n, precision="dd", ld=None, device=None, store=None):
        import torch
        if m < 0 or n < 0:
            raise ValueError("matrix dimensions must be >= 0")
        ld = max(1, m) if ld is None else ld
        if ld < max(1, m):
            raise ValueError("leading dimension too small")
        planes = _planes(precision)
        self.m, self.n, self.ld, self.precision = m, n, ld, precision
        if store is None:
            dev = torch.device("cuda" if device is None else device)
            tdt = torch.complex128 if precision == "c64" else torch.float64
            store = tuple(torch.zeros(ld * n, dtype=tdt, device=dev) for _ in range(planes))
        self.store = store

    @classmethod
    def from_host(cls, mat, device=None):
        import torch
        dev = torch.device("cuda" if device is None else device)
        planes = _planes(mat.precision)
        store = tuple(torch.as_tensor(np.ascontiguousarray(p, dtype=_plane_dtype(mat.precision)))
                      .to(dev) for p in mat.store[:planes])
        return cls(mat.m, mat.n, mat.precision, mat.ld, store=store)

    @property
    def device(self):
        return self.store[0].device

    def to_host(self):
        planes = [p.cpu().numpy() for p in self.store]
        return HostMatrix.from_planes(self.m, self.n, planes[0],
                                      planes[1] if len(planes) > 1 else None, self.ld)

    def copy(self):
        return DeviceMatrix(self.m, self.n, self.precision, self.ld,
                            store=tuple(p.clone() for p in self.store))

    def packed(self):
        """This matrix with a tight leading dimension (ld = max(1, m)): self
        when it already is, else a packed copy of the m x n values."""
        if self.ld == max(1, self.m):
            return self
        store = tuple(p[:self.ld * self.n].view(self.n, self.ld)[:, :self.m].contiguous().view(-1)
                      if self.n else p[:0].clone() for p in self.store)
        return DeviceMatrix(self.m, self.n, self.precision, max(1, self.m), store=store)

    def __repr__(self):
        return (f"DeviceMatrix({self.m}x{self.n}, ld={self.ld}, precision={self.precision!r}, "
                f"device={self.device})")


def is_device(mat):
    try:
        import torch
    except ImportError:
        return False
    return isinstance(mat.store[0], torch.Tensor) and mat.store[0].is_cuda


def storage_len(mat):
    s = mat.store[0]
    return int(s.shape[0])


def check_storage(mat, nrow, ncol, ld):
    """``Matrix.view2d``'s length rule (matrix.py:140-155)."""
    need = ld * ncol
    if storage_len(mat) < need:
        raise ValueError(
            f"storage of length {storage_len(mat)} too short for "
            f"{nrow}x{ncol} with ld={ld}")
