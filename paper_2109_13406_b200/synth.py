"""Seeded synthetic dd operands (host numpy planes).

Recipe of SURVEY.md section 8(d): per matrix a generator seeded with
``SeedSequence([seed, tag, rows, cols])`` (the pattern of the reference's
``testkit._rng``, ``/root/reference/pkg/src/mpkit/testkit.py:64-67``),
``hi ~ U(-1, 1)``, ``lo = hi * U(-1, 1) * 2**-53``, then TwoSum-normalised so
the pair is a genuine double-double with a non-zero tail (the style of the
reference's ``random_dd`` test helper, ``pkg/tests/test_ddarith.py:55-58``).

Tags: A=1, B=2, C=3.
"""

from __future__ import annotations

import numpy as np

TAG_A, TAG_B, TAG_C = 1, 2, 3


def two_sum(a, b):
    s = a + b
    bb = s - a
    return s, (a - (s - bb)) + (b - bb)


def random_dd(rows: int, cols: int, ld: int | None = None, seed: int = 0,
              tag: int = TAG_A):
    """Return ``(hi, lo)`` flat float64 planes of length ``ld*cols``.

    Padding rows (``ld > rows``) are filled from the same stream, so a padded
    matrix exercises "the kernel must not read or write the padding"."""
    ld = max(1, rows) if ld is None else ld
    g = np.random.default_rng(np.random.SeedSequence([seed, tag, rows, cols]))
    size = ld * cols
    hi = g.uniform(-1.0, 1.0, size)
    lo = hi * g.uniform(-1.0, 1.0, size) * 2.0 ** -53
    with np.errstate(all="ignore"):
        hi, lo = two_sum(hi, lo)
    return np.ascontiguousarray(hi), np.ascontiguousarray(lo)
