"""GPU parity of the LAPACK consumers on the reference's binary64 Matrix
('f64', the F64 backend): Rpotrf / Rtrsm / Rgetrf / Rgetrs bit-identical to
the reference's golden outputs and, at multi-block sizes, to the C oracle."""

import numpy as np
import pytest

from oracle import golden, oracle
from paper_2109_13406_b200 import DeviceMatrix, HostMatrix, Rgetrf, Rgetrs, Rpotrf, Rtrsm
from paper_2109_13406_b200.synth import random_dd, spd_dd

pytestmark = pytest.mark.gpu

FCASES = [c for c in golden.load_cases()
          if c[0]["routine"] in ("Rpotrf", "Rtrsm", "Rgetrf", "Rgetrs")
          and c[0].get("precision") == "f64"]


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | both_nan))


def mat(rows, cols, ld, x, on_device):
    if on_device:
        import torch
        return DeviceMatrix(rows, cols, "f64", ld,
                            store=(torch.from_numpy(np.ascontiguousarray(x).copy()).cuda(),))
    return HostMatrix.from_planes(rows, cols, x.copy(), None, ld)


def plane(m, on_device):
    return m.store[0].cpu().numpy() if on_device else m.store[0]


def run_case(case, arr, on_device, nb=0):
    r = case["routine"]
    with np.errstate(all="ignore"):
        if r == "Rpotrf":
            a = mat(case["n"], case["n"], case["lda"], arr["A_hi"], on_device)
            info = Rpotrf(case["uplo"], case["n"], a, case["lda"], nb=nb)
            return plane(a, on_device), {"info": info}
        if r == "Rtrsm":
            m, n = case["m"], case["n"]
            na = m if case["side"].upper() == "L" else n
            a = mat(na, na, case["lda"], arr["A_hi"], on_device)
            b = mat(m, n, case["ldb"], arr["B_hi"], on_device)
            Rtrsm(case["side"], case["uplo"], case["transa"], case["diag"], m, n,
                  case["alpha_v"][0], a, case["lda"], b, case["ldb"])
            return plane(b, on_device), {}
        if r == "Rgetrf":
            a = mat(case["m"], case["n"], case["lda"], arr["A_hi"], on_device)
            ipiv, info = Rgetrf(case["m"], case["n"], a, case["lda"])
            return plane(a, on_device), {"ipiv": list(ipiv), "info": info}
        n, nrhs = case["n"], case["nrhs"]
        a = mat(n, n, case["lda"], arr["A_hi"], on_device)
        ipiv, _ = Rgetrf(n, n, a, case["lda"])
        b = mat(n, nrhs, case["ldb"], arr["B_hi"], on_device)
        Rgetrs(case["trans"], n, nrhs, a, case["lda"], ipiv, b, case["ldb"])
        return plane(b, on_device), {"ipiv": list(ipiv)}


@pytest.mark.parametrize("on_device", [True, False])
@pytest.mark.parametrize("idx", range(len(FCASES)))
def test_lapack_f64_golden_bitwise(idx, on_device):
    case, arr, out_hi, _ = FCASES[idx]
    got, meta = run_case(case, arr, on_device, nb=16)
    for key, val in meta.items():
        assert val == case[key], (case, key)
    assert bits_equal(got, out_hi), case


@pytest.mark.parametrize("uplo", ["L", "U"])
def test_dpotrf_multiblock_vs_oracle(uplo):
    n, ld = 650, 651
    hi, _ = spd_dd(n, ld, seed=21)
    a = mat(n, n, ld, hi, True)
    info = Rpotrf(uplo, n, a, ld)
    oh = hi.copy()
    rc, oinfo = oracle.dpotrf(uplo, n, oh, ld)
    assert rc == 0 and info == oinfo == 0
    assert bits_equal(plane(a, True), oh)


@pytest.mark.parametrize("m,n", [(400, 400), (500, 230), (230, 500)])
def test_dgetrf_dgetrs_multiblock_vs_oracle(m, n):
    hi, _ = random_dd(m, n, m, 22, 1)
    a = mat(m, n, m, hi, True)
    ipiv, info = Rgetrf(m, n, a, m)
    oh = hi.copy()
    _, oipiv, oinfo = oracle.dgetrf(m, n, oh, m)
    assert list(ipiv) == oipiv and info == oinfo
    assert bits_equal(plane(a, True), oh)
    if m == n:
        for trans in ("N", "T"):
            bh, _ = random_dd(n, 7, n, 23, 2)
            b = mat(n, 7, n, bh, True)
            Rgetrs(trans, n, 7, a, n, ipiv, b, n)
            ob = bh.copy()
            assert oracle.dgetrs(trans, n, 7, oh, n, oipiv, ob, n) == 0
            assert bits_equal(plane(b, True), ob)


@pytest.mark.parametrize("side,uplo,ta", [(s, u, t) for s in "LR" for u in "UL" for t in "NT"])
def test_dtrsm_multiblock_vs_oracle(side, uplo, ta):
    m, n = (300, 31) if side == "L" else (31, 300)
    na = m if side == "L" else n
    ah, _ = random_dd(na, na, na, 24, 1)
    ah[:: na + 1] += 4.0
    bh, _ = random_dd(m, n, m, 24, 2)
    a, b = mat(na, na, na, ah, True), mat(m, n, m, bh, True)
    Rtrsm(side, uplo, ta, "N", m, n, 1.5, a, na, b, m)
    ob = bh.copy()
    assert oracle.dtrsm(side, uplo, ta, "N", m, n, 1.5, ah, na, ob, m) == 0
    assert bits_equal(plane(b, True), ob)
