"""GPU: randomised adversarial inputs for the fast modes -- many shapes, trans
pairs, exponent ranges and special values at once, every sampled element
checked against exact rationals (c = 4 bound) or, where an unsafe word routes
it, bit for bit against mode='reference'.

Each trial draws: m, n in [1, 300], k in [1, 3000] (some deep enough for the
split algorithm and split-K), transa / transb, per-row and per-column scales
2^U(-s/2, s/2) with s up to 150 (so some rows / columns exceed the certified
bound's spread limit and take the TwoSum fallback, others do not), random
zero entries, signs, normalised dd tails, alpha / beta with dd tails, and in
a quarter of the trials a few NaN / inf / 2^+-400 words."""

import numpy as np
import pytest

from oracle import exact
from paper_2109_13406_b200 import DeviceMatrix, Rgemm, _lib
from paper_2109_13406_b200.synth import two_sum

pytestmark = pytest.mark.gpu


def dev(rows, cols, planes):
    import torch
    return DeviceMatrix(rows, cols, "dd", max(1, rows),
                        store=tuple(torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in planes))


def _mat(g, rows, cols, s):
    x = g.uniform(1.0, 2.0, (rows, cols)) * np.where(g.random((rows, cols)) < 0.5, -1.0, 1.0)
    # |exponent| <= 1.125 s <= 169: inside the safe window (2^-300, 2^301)
    x *= 2.0 ** np.round(g.uniform(-s / 2, s / 2, (rows, 1)))
    x *= 2.0 ** np.round(g.uniform(-s / 2, s / 2, (1, cols)))
    x *= 2.0 ** np.round(g.uniform(-s / 8, s / 8, (rows, cols)))
    x[g.random((rows, cols)) < 0.1] = 0.0
    hi = x.reshape(-1, order="F")
    lo = hi * g.uniform(-1, 1, hi.shape) * 2.0 ** -53
    return [np.ascontiguousarray(p) for p in two_sum(hi, lo)]


@pytest.mark.parametrize("trial", range(120))
def test_fast_mode_fuzz(trial):
    g = np.random.default_rng(1000 + trial)
    m, n = int(g.integers(1, 300)), int(g.integers(1, 300))
    k = int(g.choice([1, 2, 7, 64, 300, 1100, 3000]))
    ta, tb = g.choice(["N", "T"]), g.choice(["N", "T"])
    s = float(g.choice([0, 10, 40, 80, 150]))
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A, B, C = _mat(g, nra, nca, s), _mat(g, nrb, ncb, s), _mat(g, m, n, 5)
    bad_rows, bad_cols = set(), set()
    if trial % 4 == 3:       # a few unsafe words: route only their rows / columns
        for _ in range(3):
            v = float(g.choice([np.nan, np.inf, 2.0 ** 400, 2.0 ** -400]))
            if g.random() < 0.5:
                i, l = int(g.integers(0, m)), int(g.integers(0, k))
                A[0][(i + l * nra) if ta == "N" else (l + i * nra)] = v
                A[1][(i + l * nra) if ta == "N" else (l + i * nra)] = 0.0
                bad_rows.add(i)
            else:
                l, j = int(g.integers(0, k)), int(g.integers(0, n))
                B[0][(l + j * nrb) if tb == "N" else (j + l * nrb)] = v
                B[1][(l + j * nrb) if tb == "N" else (j + l * nrb)] = 0.0
                bad_cols.add(j)
    alpha = (1.5, 2.0 ** -60) if trial % 2 else (-0.75, 0.0)
    beta = (0.5, -2.0 ** -58) if trial % 3 else (0.0, 0.0)
    outs = {}
    for mode in ("fast", "reference"):
        if mode == "reference" and not (bad_rows or bad_cols):
            continue
        c = dev(m, n, C)
        with np.errstate(all="ignore"):
            Rgemm(ta, tb, m, n, k, _S(alpha), dev(nra, nca, A), nra, dev(nrb, ncb, B), nrb,
                  _S(beta), c, m, mode=mode)
        outs[mode] = (c.store[0].cpu().numpy(), c.store[1].cpu().numpy())
    gh, gl = outs["fast"]
    I = sorted(set(int(x) for x in g.integers(0, m, 6)) | bad_rows)
    J = sorted(set(int(x) for x in g.integers(0, n, 6)) | bad_cols)
    good_I = [i for i in I if i not in bad_rows]
    good_J = [j for j in J if j not in bad_cols]
    if good_I and good_J:
        vals, scales = exact.exact_entries(ta, tb, k, alpha, A[0], A[1], nra, B[0], B[1], nrb,
                                           beta, C[0], C[1], m, good_I, good_J)
        assert exact.error_ratios(gh, gl, m, good_I, good_J, vals, scales, k) <= 1.0
    if bad_rows or bad_cols:
        rh, rl = outs["reference"]
        for i in range(m):
            for j in range(n):
                if i in bad_rows or j in bad_cols:
                    x = i + j * m
                    assert (np.array(gh[x]).view(np.uint64) == np.array(rh[x]).view(np.uint64) or
                            (np.isnan(gh[x]) and np.isnan(rh[x]))), (i, j)
                    assert (np.array(gl[x]).view(np.uint64) == np.array(rl[x]).view(np.uint64) or
                            (np.isnan(gl[x]) and np.isnan(rl[x]))), (i, j)


class _S:
    """A dd scalar (hi, lo) the package coerces like DDouble."""

    def __init__(self, v):
        self.hi, self.lo = v
