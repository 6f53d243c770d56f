"""B200-native double-double Rgemm / Rsyrk (arXiv 2109.13406 / MPLAPACK path).

Drop-in for ``mpkit.mpblas.Rgemm`` / ``Rsyrk`` over dd (hi, lo) planes; the
compute runs in hand-written sm_100a kernels (``csrc/``) behind the C ABI in
``include/ddblas.h``.
"""

from .matrix import BlasError, DeviceMatrix, HostMatrix, to_dd
from .lapack import PivotVector, Rgetrf, Rgetrs, Rpotrf
from .mpblas import Cgemm, Rgemm, Rsyrk, Rtrsm, default_mode

__all__ = ["Rgemm", "Rsyrk", "Rtrsm", "Cgemm", "Rpotrf", "Rgetrf", "Rgetrs", "PivotVector", "BlasError", "DeviceMatrix", "HostMatrix", "to_dd",
           "default_mode", "flop_count"]


def flop_count(routine, n, k=None, m=None):
    """dd flops as the reference bench counts them (mpkit/bench.py:51-70;
    m and k default to n): Rgemm 2mnk, Rsyrk n^2*k + n*k = n(n+1)k,
    Rgetrf 2n^3/3, Rpotrf n^3/3."""
    m = n if m is None else m
    k = n if k is None else k
    if routine == "Rgemm":
        return 2.0 * m * n * k
    if routine == "Rsyrk":
        return float(n * n * k + n * k)
    if routine == "Rpotrf":
        return n ** 3 / 3.0
    if routine == "Rgetrf":
        return 2.0 * n ** 3 / 3.0
    raise ValueError(f"unknown routine {routine!r}")
