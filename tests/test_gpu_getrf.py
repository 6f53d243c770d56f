"""GPU parity of the blocked Rgetrf (mplapack/lu.py:74-114).

exact / reference modes: factors, pivot vector and info bit-identical to
the reference's golden outputs (pivot ties, a zero column, sub-safmin
pivots, NaN, tall and wide shapes) and to the C oracle at multi-panel
sizes.  fast / twosum: the same pivots on random matrices and factors
within a dd-level tolerance of the exact ones."""

import numpy as np
import pytest

from oracle import golden, oracle
from paper_2109_13406_b200 import DeviceMatrix, HostMatrix, Rgetrf
from paper_2109_13406_b200.synth import random_dd

pytestmark = pytest.mark.gpu

LCASES = [c for c in golden.load_cases() if c[0]["routine"] == "Rgetrf" and c[0].get("precision") != "f64"]


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | both_nan))


def run(m, n, ld, hi, lo, mode, on_device=True):
    if on_device:
        import torch
        a = DeviceMatrix(m, n, "dd", ld, store=(torch.from_numpy(np.ascontiguousarray(hi)).cuda(),
                                                 torch.from_numpy(np.ascontiguousarray(lo)).cuda()))
    else:
        a = HostMatrix.from_planes(m, n, hi.copy(), lo.copy(), ld)
    with np.errstate(all="ignore"):
        ipiv, info = Rgetrf(m, n, a, ld, mode=mode)
    if on_device:
        return list(ipiv), info, a.store[0].cpu().numpy(), a.store[1].cpu().numpy()
    return list(ipiv), info, a.store[0], a.store[1]


@pytest.mark.parametrize("mode", ["exact", "reference"])
@pytest.mark.parametrize("idx", range(len(LCASES)))
def test_rgetrf_golden_bitwise(idx, mode):
    case, arr, out_hi, out_lo = LCASES[idx]
    ipiv, info, gh, gl = run(case["m"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], mode)
    assert ipiv == case["ipiv"] and info == case["info"], case
    assert bits_equal(gh, out_hi), case
    assert bits_equal(gl, out_lo), case


@pytest.mark.parametrize("idx", range(0, len(LCASES), 3))
def test_rgetrf_golden_host_path(idx):
    case, arr, out_hi, out_lo = LCASES[idx]
    ipiv, info, gh, gl = run(case["m"], case["n"], case["lda"], arr["A_hi"], arr["A_lo"], "exact",
                             on_device=False)
    assert ipiv == case["ipiv"] and info == case["info"]
    assert bits_equal(gh, out_hi) and bits_equal(gl, out_lo), case


def _inputs(m, n, ld, seed, special=None):
    hi, lo = random_dd(m, n, ld, seed, 1)
    if special == "ties":
        g = np.random.default_rng(seed)
        hi[:] = g.integers(-3, 4, hi.size).astype(np.float64)
        lo[:] = np.where(hi != 0.0, g.choice([-1.0, 0.0, 1.0], hi.size) * 2.0 ** -60, 0.0)
    elif special == "zero_col":
        hi[70 * ld: 70 * ld + m] = 0.0
        lo[70 * ld: 70 * ld + m] = 0.0
    return hi, lo


@pytest.mark.parametrize("m,n,special", [(300, 300, None), (400, 150, None), (150, 400, None),
                                         (257, 257, "ties"), (200, 200, "zero_col"),
                                         (130, 129, None)])
def test_rgetrf_exact_matches_oracle_multipanel(m, n, special):
    ld = m + 1
    hi, lo = _inputs(m, n, ld, seed=m * 7 + n, special=special)
    ipiv, info, gh, gl = run(m, n, ld, hi, lo, "exact")
    oh, ol = hi.copy(), lo.copy()
    rc, oipiv, oinfo = oracle.rgetrf(m, n, oh, ol, ld)
    assert rc == 0
    assert ipiv == oipiv and info == oinfo
    assert bits_equal(gh, oh) and bits_equal(gl, ol)


def test_rgetrf_out_of_window_rows_exact_matches_oracle():
    """Rows / columns scaled by 2^+-350: the panel's check-free updates and
    the U12 kernel's window mask fall back to the checked forms on them --
    still bitwise vs the oracle across several 256-column blocks."""
    m = n = 600
    ld = m + 1
    hi, lo = _inputs(m, n, ld, seed=99)
    rs = np.ones(m)
    cs = np.ones(n)
    for i, e in ((3, 350), (290, -350), (411, 330)):
        rs[i] = 2.0 ** e
    for j, e in ((7, -340), (300, 350), (520, -300)):
        cs[j] = 2.0 ** e
    for c in range(n):
        sl = slice(c * ld, c * ld + m)
        hi[sl] *= rs * cs[c]       # exact: powers of two
        lo[sl] *= rs * cs[c]
    ipiv, info, gh, gl = run(m, n, ld, hi, lo, "exact")
    oh, ol = hi.copy(), lo.copy()
    rc, oipiv, oinfo = oracle.rgetrf(m, n, oh, ol, ld)
    assert rc == 0
    assert ipiv == oipiv and info == oinfo
    assert bits_equal(gh, oh) and bits_equal(gl, ol)


@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("m,n", [(320, 320), (500, 200), (200, 500), (1600, 1600)])
def test_rgetrf_fast_modes_close_to_exact(m, n, mode):
    ld = m
    hi, lo = _inputs(m, n, ld, seed=3)
    ipiv, info, gh, gl = run(m, n, ld, hi, lo, mode)
    oh, ol = hi.copy(), lo.copy()
    _, oipiv, oinfo = oracle.rgetrf(m, n, oh, ol, ld)
    assert ipiv == oipiv and info == oinfo == 0
    diff = (gh - oh) + (gl - ol)
    scale = np.abs(oh).max()
    assert np.abs(diff).max() <= 1e-26 * scale, np.abs(diff).max() / scale


SCASES = [c for c in golden.load_cases() if c[0]["routine"] == "Rgetrs" and c[0].get("precision") != "f64"]


@pytest.mark.parametrize("mode", ["exact", "reference"])
@pytest.mark.parametrize("idx", range(len(SCASES)))
def test_rgetrs_golden_bitwise(idx, mode):
    """Rgetrf + Rgetrs on the GPU (lu.py:74-145) against the reference's output."""
    import torch
    from paper_2109_13406_b200 import Rgetrs
    case, arr, out_hi, out_lo = SCASES[idx]
    n, nrhs = case["n"], case["nrhs"]
    a = DeviceMatrix(n, n, "dd", case["lda"], store=(torch.from_numpy(arr["A_hi"].copy()).cuda(),
                                                      torch.from_numpy(arr["A_lo"].copy()).cuda()))
    ipiv, info = Rgetrf(n, n, a, case["lda"], mode=mode)
    assert list(ipiv) == case["ipiv"]
    b = DeviceMatrix(n, max(nrhs, 1), "dd", case["ldb"],
                     store=(torch.from_numpy(arr["B_hi"].copy()).cuda(),
                            torch.from_numpy(arr["B_lo"].copy()).cuda()))
    assert Rgetrs(case["trans"], n, nrhs, a, case["lda"], ipiv, b, case["ldb"], mode=mode) == 0
    assert bits_equal(b.store[0].cpu().numpy(), out_hi), case
    assert bits_equal(b.store[1].cpu().numpy(), out_lo), case


@pytest.mark.parametrize("trans", ["N", "T"])
def test_rgetrs_exact_matches_oracle_multiblock(trans):
    import torch
    from paper_2109_13406_b200 import Rgetrs
    n, nrhs = 260, 17
    ah, al = random_dd(n, n, n, 9, 1)
    bh, bl = random_dd(n, nrhs, n, 9, 2)
    a = DeviceMatrix(n, n, "dd", n, store=(torch.from_numpy(ah.copy()).cuda(),
                                           torch.from_numpy(al.copy()).cuda()))
    ipiv, _ = Rgetrf(n, n, a, n, mode="exact")
    b = DeviceMatrix(n, nrhs, "dd", n, store=(torch.from_numpy(bh.copy()).cuda(),
                                              torch.from_numpy(bl.copy()).cuda()))
    Rgetrs(trans, n, nrhs, a, n, ipiv, b, n, mode="exact")
    oh, ol = ah.copy(), al.copy()
    _, oipiv, _ = oracle.rgetrf(n, n, oh, ol, n)
    xh, xl = bh.copy(), bl.copy()
    assert oracle.rgetrs(trans, n, nrhs, oh, ol, n, oipiv, xh, xl, n) == 0
    assert bits_equal(b.store[0].cpu().numpy(), xh) and bits_equal(b.store[1].cpu().numpy(), xl)


def test_rgetrf_tall_panel_global_fallback():
    """m = 30000 rows: more than the shared-memory panel kernel stages per CTA
    (192 x 148), so the panel runs in the global-memory kernel; bitwise vs
    the oracle."""
    m, n = 30000, 70
    hi, lo = random_dd(m, n, m, 12, 1)
    ipiv, info, gh, gl = run(m, n, m, hi, lo, "exact")
    oh, ol = hi.copy(), lo.copy()
    _, oipiv, oinfo = oracle.rgetrf(m, n, oh, ol, m)
    assert ipiv == oipiv and info == oinfo
    assert bits_equal(gh, oh) and bits_equal(gl, ol)


def test_block_widths_from_env_bitwise():
    """DDB_GETRF_NB / DDB_TRSM_NB (read once per process): ragged outer
    blocks (100 = 64 + 36 inner) stay bit-identical to the oracle."""
    import os
    import subprocess
    import sys
    code = r'''
import numpy as np, torch, sys
sys.path.insert(0, ".")
from oracle import oracle
from paper_2109_13406_b200 import DeviceMatrix, Rgetrf, Rtrsm
from paper_2109_13406_b200.synth import random_dd
n = 333
hi, lo = random_dd(n, n, n, 5, 1)
a = DeviceMatrix(n, n, "dd", n, store=(torch.from_numpy(hi.copy()).cuda(), torch.from_numpy(lo.copy()).cuda()))
ipiv, info = Rgetrf(n, n, a, n, mode="exact")
oh, ol = hi.copy(), lo.copy()
_, oipiv, _ = oracle.rgetrf(n, n, oh, ol, n)
assert list(ipiv) == oipiv
assert np.array_equal(a.store[0].cpu().numpy(), oh) and np.array_equal(a.store[1].cpu().numpy(), ol)
bh, bl = random_dd(n, 9, n, 5, 2)
b = DeviceMatrix(n, 9, "dd", n, store=(torch.from_numpy(bh.copy()).cuda(), torch.from_numpy(bl.copy()).cuda()))
Rtrsm("L", "U", "N", "N", n, 9, 1.5, a, n, b, n, mode="exact")
xh, xl = bh.copy(), bl.copy()
assert oracle.rtrsm("L", "U", "N", "N", n, 9, (1.5, 0.0), oh, ol, n, xh, xl, n) == 0
assert np.array_equal(b.store[0].cpu().numpy(), xh) and np.array_equal(b.store[1].cpu().numpy(), xl)
print("ok")
'''
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, DDB_GETRF_NB="100", DDB_TRSM_NB="100")
    out = subprocess.run([sys.executable, "-c", code], cwd=repo, env=env, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
