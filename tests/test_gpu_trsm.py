"""GPU parity of Rtrsm (mpblas/level23.py:288-380).

exact / reference modes: bit-identical to the reference's golden outputs
and, at sizes with many blocks, to the C oracle (pinned by those goldens),
for every side x uplo x transa x diag.  fast / twosum: within a dd-level
tolerance of the exact solution (the triangular systems are diagonally
dominant, so the solution error is a small multiple of the rounding)."""

import numpy as np
import pytest

from oracle import golden, oracle
from paper_2109_13406_b200 import DeviceMatrix, HostMatrix, Rtrsm
from paper_2109_13406_b200.synth import random_dd

pytestmark = pytest.mark.gpu

TCASES = [c for c in golden.load_cases() if c[0]["routine"] == "Rtrsm" and c[0].get("precision") != "f64"]


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | both_nan))


def dev(m, n, ld, hi, lo):
    import torch
    return DeviceMatrix(m, n, "dd", ld, store=(torch.from_numpy(np.ascontiguousarray(hi)).cuda(),
                                               torch.from_numpy(np.ascontiguousarray(lo)).cuda()))


class _S:
    def __init__(self, v):
        self.hi, self.lo = v


def run(case, arr, mode, on_device=True):
    m, n = case["m"], case["n"]
    na = m if case["side"].upper() == "L" else n
    if on_device:
        a = dev(na, na, case["lda"], arr["A_hi"], arr["A_lo"])
        b = dev(m, n, case["ldb"], arr["B_hi"], arr["B_lo"])
    else:
        a = HostMatrix.from_planes(na, na, arr["A_hi"].copy(), arr["A_lo"].copy(), case["lda"])
        b = HostMatrix.from_planes(m, n, arr["B_hi"].copy(), arr["B_lo"].copy(), case["ldb"])
    with np.errstate(all="ignore"):
        Rtrsm(case["side"], case["uplo"], case["transa"], case["diag"], m, n,
              _S(case["alpha_v"]), a, case["lda"], b, case["ldb"], mode=mode)
    if on_device:
        return b.store[0].cpu().numpy(), b.store[1].cpu().numpy()
    return b.store[0], b.store[1]


@pytest.mark.parametrize("mode", ["exact", "reference"])
@pytest.mark.parametrize("idx", range(len(TCASES)))
def test_rtrsm_golden_bitwise(idx, mode):
    case, arr, out_hi, out_lo = TCASES[idx]
    gh, gl = run(case, arr, mode)
    assert bits_equal(gh, out_hi), case
    assert bits_equal(gl, out_lo), case


@pytest.mark.parametrize("idx", range(0, len(TCASES), 4))
def test_rtrsm_golden_host_path(idx):
    case, arr, out_hi, out_lo = TCASES[idx]
    gh, gl = run(case, arr, "exact", on_device=False)
    assert bits_equal(gh, out_hi) and bits_equal(gl, out_lo), case


def _case(side, uplo, ta, diag, m, n, seed, alpha=(1.5, 1.5 * 2.0 ** -60), damp=False):
    na = m if side == "L" else n
    lda, ldb = na + 1, m + 2
    ah, al = random_dd(na, na, lda, seed, 1)
    if damp:   # off-diagonal row sums < 1 < diagonal: a well-conditioned system
        f = 2.0 ** -int(np.ceil(np.log2(na)))
        ah *= f
        al *= f
    idx = np.arange(na)
    ah[idx + idx * lda] += 4.0
    bh, bl = random_dd(m, n, ldb, seed, 2)
    case = dict(side=side, uplo=uplo, transa=ta, diag=diag, m=m, n=n, lda=lda, ldb=ldb,
                alpha_v=list(alpha))
    return case, dict(A_hi=ah, A_lo=al, B_hi=bh, B_lo=bl)


BRANCHES = [(s, u, t, d) for s in "LR" for u in "UL" for t in "NT" for d in "NU"]


@pytest.mark.parametrize("side,uplo,ta,diag", BRANCHES)
def test_rtrsm_exact_matches_oracle_multiblock(side, uplo, ta, diag):
    """p = 200 (four 64-blocks, ragged last), both alpha kinds."""
    for alpha in ((1.5, 1.5 * 2.0 ** -60), (1.0, 0.0)):
        m, n = (200, 37) if side == "L" else (37, 200)
        case, arr = _case(side, uplo, ta, diag, m, n, seed=hash((side, uplo, ta, diag)) % 1000,
                          alpha=alpha)
        gh, gl = run(case, arr, "exact")
        oh, ol = arr["B_hi"].copy(), arr["B_lo"].copy()
        rc = oracle.rtrsm(side, uplo, ta, diag, m, n, alpha, arr["A_hi"], arr["A_lo"],
                          case["lda"], oh, ol, case["ldb"])
        assert rc == 0
        assert bits_equal(gh, oh) and bits_equal(gl, ol), (case, alpha)


@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("side,uplo,ta,diag", BRANCHES)
def test_rtrsm_fast_modes_close_to_exact(side, uplo, ta, diag, mode):
    m, n = (300, 41) if side == "L" else (41, 300)
    case, arr = _case(side, uplo, ta, diag, m, n, seed=7, damp=True)
    gh, gl = run(case, arr, mode)
    oh, ol = arr["B_hi"].copy(), arr["B_lo"].copy()
    oracle.rtrsm(side, uplo, ta, diag, m, n, case["alpha_v"], arr["A_hi"], arr["A_lo"],
                 case["lda"], oh, ol, case["ldb"])
    ldb = case["ldb"]
    sel = (np.arange(m)[:, None] + np.arange(n)[None, :] * ldb).ravel()
    diff = (gh[sel] - oh[sel]) + (gl[sel] - ol[sel])
    scale = np.abs(oh[sel]).max()
    assert np.abs(diff).max() <= 1e-28 * scale, np.abs(diff).max() / scale
