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


def spd_dd(n: int, ld: int | None = None, seed: int = 0, scale: float = 1.0):
    """Symmetric positive definite dd test matrix for Rpotrf: the triangle
    either factorization reads is ``random_dd`` (tag 4) with ``n + 1 + U(-1, 1)``
    on the diagonal (strictly diagonally dominant), a non-zero dd tail on
    every entry, times ``scale`` (a power of two, exact).  Both triangles
    are filled, as the symmetric matrix they define."""
    ld = max(1, n) if ld is None else ld
    hi, lo = random_dd(n, n, ld, seed, 4)
    g = np.random.default_rng(np.random.SeedSequence([seed, 5, n, n]))
    dh = n + 1.0 + g.uniform(-1.0, 1.0, n)
    dl = dh * g.uniform(-1.0, 1.0, n) * 2.0 ** -55
    dh, dl = two_sum(dh, dl)
    idx = np.arange(n)
    for i in range(n):          # mirror the lower triangle into the upper
        hi[i + idx[i + 1:] * ld] = hi[idx[i + 1:] + i * ld]
        lo[i + idx[i + 1:] * ld] = lo[idx[i + 1:] + i * ld]
    hi[idx + idx * ld] = dh
    lo[idx + idx * ld] = dl
    return hi * scale, lo * scale


# --------------------------------------------------------------------------
# Counter-based dd operands: element (i, j) is a pure function of
# (seed, tag, i, j) (splitmix64), so a 16 GiB matrix can be generated on the
# GPU while any sampled entries are reproduced on the host for checking.

_M64 = (1 << 64) - 1


def _splitmix_np(x):
    import numpy as np
    x = (x + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(_M64)
    x = ((x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(_M64)
    x = ((x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(_M64)
    return x ^ (x >> np.uint64(31))


def hashed_entries(seed, tag, ii, jj):
    """(hi, lo) float64 arrays of entries (ii[x], jj[x]) -- host reference."""
    import numpy as np
    ii = np.asarray(ii, dtype=np.uint64)
    jj = np.asarray(jj, dtype=np.uint64)
    with np.errstate(over="ignore"):
        key = (np.uint64(seed) * np.uint64(1000003) + np.uint64(tag)) * np.uint64(0x100000001B3)
        base = _splitmix_np((ii << np.uint64(32)) ^ jj ^ key)
        u1 = _splitmix_np(base)
        u2 = _splitmix_np(u1)
    hi = (u1 >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0      # [-1, 1)
    lo = hi * ((u2 >> np.uint64(11)).astype(np.float64) * 2.0 ** -52 - 1.0) * 2.0 ** -53
    with np.errstate(all="ignore"):
        return two_sum(hi, lo)


def hashed_dd_device(rows, cols, seed, tag, device, chunk_cols=256):
    """(hi, lo) torch CUDA planes (ld = rows) with the same values as
    ``hashed_entries``; generated column-chunk by column-chunk on the GPU."""
    import torch

    def u64(v):   # reinterpret an unsigned 64-bit constant as int64
        return v - (1 << 64) if v >= 1 << 63 else v

    def lsr(x, s):   # logical shift right on int64 tensors
        return (x >> s) & ((1 << (64 - s)) - 1)

    def splitmix(x):
        x = x + u64(0x9E3779B97F4A7C15)
        x = (x ^ lsr(x, 30)) * u64(0xBF58476D1CE4E5B9)
        x = (x ^ lsr(x, 27)) * u64(0x94D049BB133111EB)
        return x ^ lsr(x, 31)

    key_py = ((seed * 1000003 + tag) * 0x100000001B3) & _M64
    key = u64(key_py)
    hi = torch.empty(rows * cols, dtype=torch.float64, device=device)
    lo = torch.empty(rows * cols, dtype=torch.float64, device=device)
    ii = torch.arange(rows, dtype=torch.int64, device=device)
    for c0 in range(0, cols, chunk_cols):
        c1 = min(cols, c0 + chunk_cols)
        jj = torch.arange(c0, c1, dtype=torch.int64, device=device)
        x = ((ii[:, None] << 32) ^ jj[None, :]) ^ key          # rows x chunk (i fastest below)
        u1 = splitmix(splitmix(x))
        u2 = splitmix(u1)
        h = lsr(u1, 11).to(torch.float64) * 2.0 ** -52 - 1.0
        l = h * (lsr(u2, 11).to(torch.float64) * 2.0 ** -52 - 1.0) * 2.0 ** -53
        s = h + l
        bb = s - h
        e = (h - (s - bb)) + (l - bb)
        hi[c0 * rows:c1 * rows] = s.t().reshape(-1)
        lo[c0 * rows:c1 * rows] = e.t().reshape(-1)
    return hi, lo
