"""Exact values of sampled entries of alpha*op(A)*op(B) + beta*C -- TEST INFRASTRUCTURE ONLY.

Every dd word is a binary64 number, so a dd value is an exact dyadic
rational.  Scaling all words by a common 2**S turns them into Python ints;
the dot products are then exact big-int sums, and alpha / beta / C are
applied exactly with ``fractions.Fraction``.  This is the "exact rational"
oracle of the reference's own tests (pkg/tests/test_mpblas.py:399-418), made
fast enough for k = 65536 by staying in integer arithmetic.  ``mp_check``
cross-checks a few entries with mpmath at 240 bits, as the reference's
acceptance test does (test_acceptance.py:361-415).

The error bound of the north star:
    |C_gpu - C_exact| <= c * k * 2**-104 * (|alpha| * sum_l |a_il * b_lj| + |beta| * |c_ij|)
"""

from __future__ import annotations

import math
from fractions import Fraction

import numpy as np

U2 = Fraction(1, 2 ** 104)


def _scaled_ints(x, S):
    """Exact int(x * 2**S) for a float64 array (requires x*2**S integral)."""
    m, e = np.frexp(np.asarray(x, dtype=np.float64))
    mi = (m * 2.0 ** 53).astype(np.int64)          # exact: |m| < 1
    sh = (e.astype(np.int64) - 53 + S)
    out = []
    for a, s in zip(mi.tolist(), sh.tolist()):
        if a == 0:
            out.append(0)
        elif s >= 0:
            out.append(a << s)
        else:
            if a % (1 << -s):
                raise ValueError("scale too small for exact conversion")
            out.append(a >> -s)
    return out


def _min_exp(*arrays):
    lo = 0
    for x in arrays:
        x = np.asarray(x, dtype=np.float64)
        nz = x[x != 0]
        if nz.size:
            _, e = np.frexp(nz)
            lo = min(lo, int(e.min()))
    return lo


def _op_rows(trans, hi, lo, ld, rows, k):
    """Rows ``rows`` of op(X) (length-k vectors of hi and lo), X column-major."""
    out_h, out_l = [], []
    for i in rows:
        if trans == "N":
            idx = i + np.arange(k) * ld
        else:
            idx = i * ld + np.arange(k)
        out_h.append(hi[idx])
        out_l.append(lo[idx])
    return np.array(out_h).reshape(len(rows), k), np.array(out_l).reshape(len(rows), k)


def exact_entries(transa, transb, k, alpha, a_hi, a_lo, lda, b_hi, b_lo, ldb,
                  beta, c_hi, c_lo, ldc, I, J):
    """Return (exact Fractions, scale floats) for entries (I[x], J[y]).

    ``scale[x][y] = |alpha| * sum_l |a_il b_lj| + |beta| * |c_ij|`` (float64,
    relative error ~1e-15, fine for a bound)."""
    ta, tb = transa.upper(), transb.upper()
    ta = "N" if ta == "N" else "T"
    tb = "N" if tb == "N" else "T"
    Ah, Al = _op_rows(ta, a_hi, a_lo, lda, I, k)
    # column j of op(B) == row j of op(B)^T
    Bh, Bl = _op_rows("T" if tb == "N" else "N", b_hi, b_lo, ldb, J, k)
    S = 60 - _min_exp(Ah, Al, Bh, Bl)
    A_int = [[h + l for h, l in zip(_scaled_ints(Ah[x], S), _scaled_ints(Al[x], S))]
             for x in range(len(I))]
    B_int = [[h + l for h, l in zip(_scaled_ints(Bh[y], S), _scaled_ints(Bl[y], S))]
             for y in range(len(J))]
    absA = np.abs(Ah + Al)
    absB = np.abs(Bh + Bl)
    al = Fraction(alpha[0]) + Fraction(alpha[1])
    be = Fraction(beta[0]) + Fraction(beta[1])
    den = 1 << (2 * S)
    vals, scales = [], []
    for x, i in enumerate(I):
        row_v, row_s = [], []
        ai = A_int[x]
        for y, j in enumerate(J):
            bj = B_int[y]
            dot = sum(p * q for p, q in zip(ai, bj))
            v = al * Fraction(dot, den)
            cij = 0
            if be != 0:   # beta == 0 never reads C (it may hold NaN: level23.py:163-169)
                cij = Fraction(float(c_hi[i + j * ldc])) + Fraction(float(c_lo[i + j * ldc]))
                v += be * cij
            row_v.append(v)
            s = abs(float(al)) * float(np.dot(absA[x], absB[y]))
            if be != 0:
                s += abs(float(be)) * abs(float(cij))
            row_s.append(s)
        vals.append(row_v)
        scales.append(row_s)
    return vals, scales


def error_ratios(got_hi, got_lo, ldc, I, J, vals, scales, k, c=4.0):
    """max over entries of |got - exact| / (c * k * 2**-104 * scale)."""
    worst = 0.0
    for x, i in enumerate(I):
        for y, j in enumerate(J):
            g = Fraction(float(got_hi[i + j * ldc])) + Fraction(float(got_lo[i + j * ldc]))
            err = abs(g - vals[x][y])
            bound = Fraction(c) * max(k, 1) * U2 * Fraction(scales[x][y])
            if bound == 0:
                r = 0.0 if err == 0 else math.inf
            else:
                r = float(err / bound)
            worst = max(worst, r)
    return worst


def mp_check(value_fraction, hi, lo, prec=240):
    """|hi + lo - value| computed by mpmath at ``prec`` bits (cross-check)."""
    import mpmath
    with mpmath.workprec(prec):
        v = mpmath.mpf(value_fraction.numerator) / mpmath.mpf(value_fraction.denominator)
        return abs(mpmath.mpf(hi) + mpmath.mpf(lo) - v)
