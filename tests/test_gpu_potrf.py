"""GPU parity of the blocked Rpotrf (mplapack/chol.py:21-65).

exact mode: bit-identical to the reference's golden outputs (and to the C
oracle at larger sizes) for every block width -- the blocking only regroups
the reference's per-element operation sequence; info and the failing
pivot's value too.  fast / twosum: the reference's own acceptance metric,
testkit.residual_chol  ||F F^T - A||_inf / (n ||A||_inf eps_dd) < 30
(testkit.py:473-486, THRESHOLD testkit.py:32), with the factor product
formed by the (parity-tested) exact GPU Rgemm."""

import os

import numpy as np
import pytest

from oracle import golden, oracle
from paper_2109_13406_b200 import DeviceMatrix, HostMatrix, Rgemm, Rpotrf
from paper_2109_13406_b200.synth import spd_dd

pytestmark = pytest.mark.gpu

EPS_DD = float.fromhex("0x1.ffffffffffff9p-105")   # machine_params("dd").eps
THRESHOLD = 30.0

PCASES = [c for c in golden.load_cases() if c[0]["routine"] == "Rpotrf" and c[0].get("precision") != "f64"]


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | both_nan))


def dev(n, ld, hi, lo):
    import torch
    return DeviceMatrix(n, n, "dd", ld, store=(torch.from_numpy(np.ascontiguousarray(hi)).cuda(),
                                               torch.from_numpy(np.ascontiguousarray(lo)).cuda()))


def run(uplo, n, ld, hi, lo, mode, nb=0, on_device=True):
    if on_device:
        a = dev(n, ld, hi, lo)
        with np.errstate(all="ignore"):
            info = Rpotrf(uplo, n, a, ld, mode=mode, nb=nb)
        return info, a.store[0].cpu().numpy(), a.store[1].cpu().numpy()
    a = HostMatrix.from_planes(n, n, hi.copy(), lo.copy(), ld)
    with np.errstate(all="ignore"):
        info = Rpotrf(uplo, n, a, ld, mode=mode, nb=nb)
    return info, a.store[0], a.store[1]


def residual_ratio(uplo, n, ld, a_hi, a_lo, f_hi, f_lo):
    """testkit.residual_chol on the GPU: F = the uplo triangle of the
    factor; R = F F^T - A ('L') or F^T F - A ('U') by exact-mode Rgemm."""
    import torch
    idx = np.arange(n)
    keep = (idx[:, None] >= idx[None, :]) if uplo.upper() == "L" else (idx[:, None] <= idx[None, :])
    fh = np.zeros((n, n))
    fl = np.zeros((n, n))
    Fh = f_hi[: ld * n].reshape(n, ld)[:, :n].T       # (row, col)
    Fl = f_lo[: ld * n].reshape(n, ld)[:, :n].T
    fh[keep], fl[keep] = Fh[keep], Fl[keep]
    Ah = a_hi[: ld * n].reshape(n, ld)[:, :n].T
    Al = a_lo[: ld * n].reshape(n, ld)[:, :n].T
    col = lambda M: np.ascontiguousarray(M.T.reshape(-1))
    F = dev(n, n, col(fh), col(fl))
    R = dev(n, n, col(Ah), col(Al))
    ta, tb = ("N", "T") if uplo.upper() == "L" else ("T", "N")
    Rgemm(ta, tb, n, n, n, 1.0, F, n, F, n, -1.0, R, n, mode="exact")
    rh = R.store[0].cpu().numpy().reshape(n, n).T
    rnorm = np.abs(rh).sum(axis=1).max()
    anorm = np.abs(Ah).sum(axis=1).max()
    return float(rnorm / (max(1, n) * anorm * EPS_DD))


@pytest.mark.parametrize("nb", [0, 16, 5, 40])
@pytest.mark.parametrize("mode", ["exact", "reference"])
@pytest.mark.parametrize("idx", range(len(PCASES)))
def test_rpotrf_golden_bitwise(idx, mode, nb):
    case, arr, out_hi, out_lo = PCASES[idx]
    info, gh, gl = run(case["uplo"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], mode, nb)
    assert info == case["info"], case
    assert bits_equal(gh, out_hi), case
    assert bits_equal(gl, out_lo), case


@pytest.mark.parametrize("idx", range(0, len(PCASES), 3))
def test_rpotrf_golden_host_path(idx):
    case, arr, out_hi, out_lo = PCASES[idx]
    info, gh, gl = run(case["uplo"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], "exact", 16,
                       on_device=False)
    assert info == case["info"]
    assert bits_equal(gh, out_hi) and bits_equal(gl, out_lo), case


@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("idx", range(len(PCASES)))
def test_rpotrf_golden_fast_modes(idx, mode):
    """Same info; on success the reference's residual test passes.  (On
    failure the factor's first columns agree to dd accuracy, not bits.)"""
    case, arr, out_hi, out_lo = PCASES[idx]
    info, gh, gl = run(case["uplo"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], mode, 16)
    assert info == case["info"], case
    sp = case.get("special")
    if info == 0 and sp not in ("scale_huge", "scale_tiny", "lo_only") and case["n"] > 1:
        r = residual_ratio(case["uplo"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], gh, gl)
        assert r < THRESHOLD, (case, r)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("n,nb", [(700, 0), (1000, 100), (900, 48), (650, 130), (1100, 600),
                                  (1300, 520)])
def test_rpotrf_exact_matches_oracle(uplo, n, nb):
    """Multi-block sizes, default and odd block widths: bitwise vs the C
    oracle (the reference's order, pinned by the golden tests)."""
    ld = n + 3
    hi, lo = spd_dd(n, ld, seed=77 + n)
    info, gh, gl = run(uplo, n, ld, hi, lo, "exact", nb)
    oh, ol = hi.copy(), lo.copy()
    rc, oinfo = oracle.rpotrf(uplo, n, oh, ol, ld)
    assert rc == 0 and info == oinfo == 0
    assert bits_equal(gh, oh) and bits_equal(gl, ol)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("nb", [0, 100])
def test_rpotrf_out_of_window_rows_exact_matches_oracle(uplo, nb):
    """D A D with a few 2^+-350 scales: factor entries far outside the safe
    window in some rows / columns, so the row-recurrence kernel's warps, the
    window mask of its factor block and the diagonal kernel's check-free
    updates all take their checked fallbacks -- still bitwise vs the oracle."""
    n = 700
    ld = n + 1
    hi, lo = spd_dd(n, ld, seed=91)
    d = np.ones(n)
    for i, e in ((5, 350), (300, 350), (450, -350), (650, -350), (257, 320)):
        d[i] = 2.0 ** e
    for c in range(n):
        sl = slice(c * ld, c * ld + n)
        hi[sl] *= d * d[c]        # exact: powers of two
        lo[sl] *= d * d[c]
    info, gh, gl = run(uplo, n, ld, hi, lo, "exact", nb)
    oh, ol = hi.copy(), lo.copy()
    rc, oinfo = oracle.rpotrf(uplo, n, oh, ol, ld)
    assert rc == 0 and info == oinfo == 0
    assert bits_equal(gh, oh) and bits_equal(gl, ol)


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("nb", [64, 300])
def test_rpotrf_late_failure_restores_trailing(uplo, nb):
    """A failing pivot deep in a multi-block run: info, A(j,j) and every
    entry the reference leaves untouched match the oracle bit for bit."""
    n, ld = 600, 600
    hi, lo = spd_dd(n, ld, seed=5)
    j = 517
    hi[j + j * ld], lo[j + j * ld] = -3.0, 0.0
    oh, ol = hi.copy(), lo.copy()
    rc, oinfo = oracle.rpotrf(uplo, n, oh, ol, ld)
    assert oinfo == j + 1
    for mode in ("exact", "fast"):
        info, gh, gl = run(uplo, n, ld, hi, lo, mode, nb)
        assert info == j + 1
        if mode == "exact":
            assert bits_equal(gh, oh) and bits_equal(gl, ol)
        else:   # the untouched part is restored exactly
            r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
            untouched = (c > j) & (r >= c) if uplo == "L" else (r > j) & (r <= c)
            flat = (r + c * ld)[untouched]
            assert bits_equal(gh[flat], hi[flat]) and bits_equal(gl[flat], lo[flat])


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("mode", ["fast", "twosum"])
def test_rpotrf_default_blocking_large_n_residual(uplo, mode):
    """n = 6400: the fast modes' default outer width 384 (three block levels:
    256- and 128-column middle panels, the lean lookahead kernel late in the
    factorization, TwoSum accumulation in the row kernels and the diagonal
    kernel's Newton pivots) -- inside the reference's acceptance residual."""
    n = 6400
    hi, lo = spd_dd(n, n, seed=23)
    info, gh, gl = run(uplo, n, n, hi, lo, mode)
    assert info == 0
    r = residual_ratio(uplo, n, n, hi, lo, gh, gl)
    assert r < THRESHOLD, r


@pytest.mark.parametrize("uplo", ["L", "U"])
@pytest.mark.parametrize("mode", ["fast", "twosum", "exact"])
@pytest.mark.parametrize("n", [2500, 4500])
def test_rpotrf_large_residual(uplo, mode, n):
    hi, lo = spd_dd(n, n, seed=11)
    info, gh, gl = run(uplo, n, n, hi, lo, mode)
    assert info == 0
    r = residual_ratio(uplo, n, n, hi, lo, gh, gl)
    assert r < THRESHOLD, r


def test_rpotrf_other_triangle_untouched():
    n, ld = 300, 301
    hi, lo = spd_dd(n, ld, seed=3)
    for uplo in ("L", "U"):
        _, gh, gl = run(uplo, n, ld, hi, lo, "fast", 64)
        r, c = np.meshgrid(np.arange(n), np.arange(n), indexing="ij")
        other = (r < c) if uplo == "L" else (r > c)
        flat = (r + c * ld)[other]
        pad = np.arange(n)[None, :] * ld + n       # padding rows
        assert bits_equal(gh[flat], hi[flat]) and bits_equal(gl[flat], lo[flat])
        assert bits_equal(gh[pad.ravel()[:-1]], hi[pad.ravel()[:-1]])
