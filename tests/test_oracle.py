"""The C oracle is pinned against the reference's own outputs (tests/golden)."""

import numpy as np
import pytest

from oracle import golden, oracle


def bits_equal(a, b):
    """Bitwise equality, NaN payload-insensitive, -0.0 != +0.0."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    same = a.view(np.uint64) == b.view(np.uint64)
    return bool(np.all(same | both_nan))


ALL = list(golden.load_cases())
CASES = [c for c in ALL if c[0]["routine"] in ("Rgemm", "Rsyrk")]
PCASES = [c for c in ALL if c[0]["routine"] == "Rpotrf" and c[0].get("precision") != "f64"]
TCASES = [c for c in ALL if c[0]["routine"] == "Rtrsm" and c[0].get("precision") != "f64"]
LCASES = [c for c in ALL if c[0]["routine"] == "Rgetrf" and c[0].get("precision") != "f64"]
SCASES = [c for c in ALL if c[0]["routine"] == "Rgetrs" and c[0].get("precision") != "f64"]
FCASES = [c for c in ALL if c[0]["routine"] in ("Rpotrf", "Rtrsm", "Rgetrf", "Rgetrs")
          and c[0].get("precision") == "f64"]
CCASES = [c for c in ALL if c[0]["routine"] == "Cgemm"]


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_oracle_matches_reference_bitwise(idx):
    case, arr, out_hi, out_lo = CASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"], "input regeneration drifted"
    if case.get("precision") == "f64":
        ch = arr["C_hi"].copy()
        with np.errstate(all="ignore"):
            if case["routine"] == "Rgemm":
                rc = oracle.dgemm(case["transa"], case["transb"], case["m"], case["n"], case["k"],
                                  case["alpha_v"][0], arr["A_hi"], case["lda"], arr["B_hi"],
                                  case["ldb"], case["beta_v"][0], ch, case["ldc"])
            else:
                rc = oracle.dsyrk(case["uplo"], case["trans"], case["n"], case["k"],
                                  case["alpha_v"][0], arr["A_hi"], case["lda"],
                                  case["beta_v"][0], ch, case["ldc"])
        assert rc == 0
        assert bits_equal(ch, out_hi), case
        return
    ch, cl = arr["C_hi"].copy(), arr["C_lo"].copy()
    with np.errstate(all="ignore"):
        if case["routine"] == "Rgemm":
            rc = oracle.rgemm(case["transa"], case["transb"], case["m"], case["n"], case["k"],
                              case["alpha_v"], arr["A_hi"], arr["A_lo"], case["lda"],
                              arr["B_hi"], arr["B_lo"], case["ldb"], case["beta_v"],
                              ch, cl, case["ldc"], threads=2)
        else:
            rc = oracle.rsyrk(case["uplo"], case["trans"], case["n"], case["k"],
                              case["alpha_v"], arr["A_hi"], arr["A_lo"], case["lda"],
                              case["beta_v"], ch, cl, case["ldc"], threads=2)
    assert rc == 0
    assert bits_equal(ch, out_hi), case
    assert bits_equal(cl, out_lo), case


def test_oracle_scalar_efts_match_reference():
    v = golden.load_eft()
    for i in range(len(v["xh"])):
        x = (v["xh"][i], v["xl"][i])
        y = (v["yh"][i], v["yl"][i])
        assert bits_equal(oracle.add2(x, y), (v["add_h"][i], v["add_l"][i])), i
        assert bits_equal(oracle.mul2(x, y), (v["mul_h"][i], v["mul_l"][i])), i
        assert bits_equal(oracle.two_prod(x[0], y[0]), (v["tp_p"][i], v["tp_e"][i])), i


def test_oracle_known_answer_integer_instance():
    """cli.py:160-186 / test_acceptance.py:121-139: exact at dd, lo == 0."""
    A = np.array([[1, 8, 3], [0, 10, 8], [9, -5, -1]], float)
    B = np.array([[9, 8, 3], [3, -11, 0], [-8, 6, 1]], float)
    C = np.array([[3, 3, 0], [8, 4, 8], [6, 1, -2]], float)
    col = lambda M: np.ascontiguousarray(M.T.reshape(-1))
    ch, cl = col(C), np.zeros(9)
    rc = oracle.rgemm("N", "N", 3, 3, 3, (3.0, 0.0), col(A), np.zeros(9), 3,
                      col(B), np.zeros(9), 3, (-2.0, 0.0), ch, cl, 3)
    assert rc == 0
    expect = np.array([[21, -192, 18], [-118, -194, 8], [210, 361, 82]], float)
    assert np.array_equal(ch.reshape(3, 3).T, expect)
    assert np.all(cl == 0.0)


@pytest.mark.parametrize("args,idx", [
    (("X", "N", 1, 1, 1, 1, 1, 1), 1), (("N", "Q", 1, 1, 1, 1, 1, 1), 2),
    (("N", "N", -1, 1, 1, 1, 1, 1), 3), (("N", "N", 1, -1, 1, 1, 1, 1), 4),
    (("N", "N", 1, 1, -1, 1, 1, 1), 5), (("N", "N", 4, 1, 1, 3, 4, 4), 8),
    (("N", "N", 1, 1, 4, 1, 3, 1), 10), (("N", "N", 4, 1, 1, 4, 1, 3), 13),
    (("T", "N", 4, 1, 2, 1, 2, 4), 8),
])
def test_oracle_validation_indices(args, idx):
    ta, tb, m, n, k, lda, ldb, ldc = args
    assert oracle.lib().oracle_gemm_validate(ta.encode(), tb.encode(), m, n, k, lda, ldb, ldc) == idx


@pytest.mark.parametrize("idx", range(len(CCASES)))
def test_oracle_cgemm_matches_reference_bitwise(idx):
    case, arr, outs, _ = CCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    al = complex(*case["alpha_v"])
    be = complex(*case["beta_v"])
    with np.errstate(all="ignore"):
        if case["precision"] == "cdd":
            from paper_2109_13406_b200.matrix import to_cdd
            a4 = [np.ascontiguousarray(arr[f"A_{p}"]) for p in ("rh", "rl", "ih", "il")]
            b4 = [np.ascontiguousarray(arr[f"B_{p}"]) for p in ("rh", "rl", "ih", "il")]
            c4 = [arr[f"C_{p}"].copy() for p in ("rh", "rl", "ih", "il")]
            alv = to_cdd(al if case["alpha"] != "zr" else case["alpha_v"][0])
            rc = oracle.cgemm(case["transa"], case["transb"], case["m"], case["n"], case["k"],
                              alv, a4, case["lda"], b4, case["ldb"], to_cdd(be), c4, case["ldc"])
            got = c4
        else:
            c = arr["C_z"].copy()
            rc = oracle.zgemm(case["transa"], case["transb"], case["m"], case["n"], case["k"],
                              al, np.ascontiguousarray(arr["A_z"]), case["lda"],
                              np.ascontiguousarray(arr["B_z"]), case["ldb"], be, c, case["ldc"])
            got = [c]
    assert rc == 0
    for g_, o_ in zip(got, outs):
        g_, o_ = np.asarray(g_), np.asarray(o_)
        if g_.dtype.kind == "c":
            assert bits_equal(g_.real.copy(), o_.real.copy()) and bits_equal(g_.imag.copy(), o_.imag.copy()), case
        else:
            assert bits_equal(g_, o_), case


@pytest.mark.parametrize("idx", range(len(PCASES)))
def test_oracle_rpotrf_matches_reference_bitwise(idx):
    """mplapack/chol.py:21-65 restated in C, against the reference's own output."""
    case, arr, out_hi, out_lo = PCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    ah, al = arr["A_hi"].copy(), arr["A_lo"].copy()
    with np.errstate(all="ignore"):
        rc, info = oracle.rpotrf(case["uplo"], case["n"], ah, al, case["lda"])
    assert rc == 0
    assert info == case["info"], case
    assert bits_equal(ah, out_hi), case
    assert bits_equal(al, out_lo), case


def test_oracle_scalar_div_sqrt_match_reference():
    """ddarith._div2 / _sqrt2 (the pivots of Rpotrf) through the oracle."""
    v = golden.load_eft()
    for i in range(len(v["xh"])):
        x = (v["xh"][i], v["xl"][i])
        y = (v["yh"][i], v["yl"][i])
        assert bits_equal(oracle.div2(x, y), (v["div_h"][i], v["div_l"][i])), i
        assert bits_equal(oracle.sqrt2((v["sq_in_h"][i], v["sq_in_l"][i])),
                          (v["sq_h"][i], v["sq_l"][i])), i


@pytest.mark.parametrize("args,idx", [(("X", 3, 3), 1), (("U", -1, 1), 2), (("L", 4, 3), 4),
                                      (("l", 0, 1), 0), (("u", 1, 1), 0), (("L", 0, 0), 4)])
def test_oracle_potrf_validation_indices(args, idx):
    uplo, n, lda = args
    assert oracle.lib().oracle_potrf_validate(uplo.encode(), n, lda) == idx


@pytest.mark.parametrize("idx", range(len(TCASES)))
def test_oracle_rtrsm_matches_reference_bitwise(idx):
    """mpblas/level23.py:288-380 restated in C, against the reference's output."""
    case, arr, out_hi, out_lo = TCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    bh, bl = arr["B_hi"].copy(), arr["B_lo"].copy()
    with np.errstate(all="ignore"):
        rc = oracle.rtrsm(case["side"], case["uplo"], case["transa"], case["diag"], case["m"],
                          case["n"], case["alpha_v"], arr["A_hi"], arr["A_lo"], case["lda"],
                          bh, bl, case["ldb"])
    assert rc == 0
    assert bits_equal(bh, out_hi), case
    assert bits_equal(bl, out_lo), case


@pytest.mark.parametrize("idx", range(len(LCASES)))
def test_oracle_rgetrf_matches_reference_bitwise(idx):
    """mplapack/lu.py:74-114 restated in C: factors, ipiv and info."""
    case, arr, out_hi, out_lo = LCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    ah, al = arr["A_hi"].copy(), arr["A_lo"].copy()
    with np.errstate(all="ignore"):
        rc, ipiv, info = oracle.rgetrf(case["m"], case["n"], ah, al, case["lda"])
    assert rc == 0
    assert ipiv == case["ipiv"] and info == case["info"], case
    assert bits_equal(ah, out_hi), case
    assert bits_equal(al, out_lo), case


@pytest.mark.parametrize("args,idx", [
    (("X", "U", "N", "N", 2, 2, 2, 2), 1), (("L", "X", "N", "N", 2, 2, 2, 2), 2),
    (("L", "U", "X", "N", 2, 2, 2, 2), 3), (("L", "U", "N", "X", 2, 2, 2, 2), 4),
    (("L", "U", "N", "N", -1, 2, 2, 2), 5), (("L", "U", "N", "N", 2, -1, 2, 2), 6),
    (("L", "U", "N", "N", 3, 2, 2, 3), 9), (("R", "U", "N", "N", 2, 3, 2, 2), 9),
    (("L", "U", "N", "N", 3, 2, 3, 2), 11), (("r", "l", "c", "u", 2, 3, 3, 2), 0)])
def test_oracle_trsm_validation_indices(args, idx):
    s, u, t, d, m, n, lda, ldb = args
    assert oracle.lib().oracle_trsm_validate(s.encode(), u.encode(), t.encode(), d.encode(), m, n,
                                             lda, ldb) == idx


@pytest.mark.parametrize("args,idx", [((-1, 2, 2), 1), ((2, -1, 2), 2), ((3, 2, 2), 4),
                                      ((0, 0, 0), 4), ((0, 0, 1), 0)])
def test_oracle_getrf_validation_indices(args, idx):
    assert oracle.lib().oracle_getrf_validate(*args) == idx


@pytest.mark.parametrize("idx", range(len(SCASES)))
def test_oracle_rgetrs_matches_reference_bitwise(idx):
    """mplapack/lu.py:117-145 (after the oracle's Rgetrf) against the reference."""
    case, arr, out_hi, out_lo = SCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    n, nrhs = case["n"], case["nrhs"]
    ah, al = arr["A_hi"].copy(), arr["A_lo"].copy()
    rc, ipiv, info = oracle.rgetrf(n, n, ah, al, case["lda"])
    assert rc == 0 and ipiv == case["ipiv"]
    bh, bl = arr["B_hi"].copy(), arr["B_lo"].copy()
    assert oracle.rgetrs(case["trans"], n, nrhs, ah, al, case["lda"], ipiv, bh, bl,
                         case["ldb"]) == 0
    assert bits_equal(bh, out_hi) and bits_equal(bl, out_lo), case


@pytest.mark.parametrize("idx", range(len(FCASES)))
def test_oracle_lapack_f64_matches_reference_bitwise(idx):
    """Rpotrf / Rtrsm / Rgetrf / Rgetrs on the F64 backend, restated in C."""
    case, arr, out_hi, _ = FCASES[idx]
    assert golden.input_digest(arr) == case["input_sha256"]
    r = case["routine"]
    with np.errstate(all="ignore"):
        if r == "Rpotrf":
            a = arr["A_hi"].copy()
            rc, info = oracle.dpotrf(case["uplo"], case["n"], a, case["lda"])
            assert rc == 0 and info == case["info"]
            got = a
        elif r == "Rtrsm":
            got = arr["B_hi"].copy()
            assert oracle.dtrsm(case["side"], case["uplo"], case["transa"], case["diag"],
                                case["m"], case["n"], case["alpha_v"][0], arr["A_hi"],
                                case["lda"], got, case["ldb"]) == 0
        elif r == "Rgetrf":
            got = arr["A_hi"].copy()
            rc, ipiv, info = oracle.dgetrf(case["m"], case["n"], got, case["lda"])
            assert rc == 0 and ipiv == case["ipiv"] and info == case["info"]
        else:
            a = arr["A_hi"].copy()
            _, ipiv, _ = oracle.dgetrf(case["n"], case["n"], a, case["lda"])
            assert ipiv == case["ipiv"]
            got = arr["B_hi"].copy()
            assert oracle.dgetrs(case["trans"], case["n"], case["nrhs"], a, case["lda"], ipiv,
                                 got, case["ldb"]) == 0
    assert bits_equal(got, out_hi), case


def test_oracle_reproduces_the_reference_pins():
    """The C oracle against the pins generated by running the reference
    (oracle/gen_pins.py): integer instance, Hilbert n = 2 product, and the
    thread-count-invariance operands."""
    import os
    pins = np.load(os.path.join(os.path.dirname(__file__), "golden", "pins.npz"))
    for pre, (m, n, k, al, be) in {"int": (3, 3, 3, 3.0, -2.0), "tc": (8, 8, 8, 0.75, -0.5)}.items():
        ch, cl = pins[pre + "_c_hi"].copy(), pins[pre + "_c_lo"].copy()
        assert oracle.rgemm("N", "N", m, n, k, (al, 0.0), pins[pre + "_a_hi"], pins[pre + "_a_lo"],
                            m, pins[pre + "_b_hi"], pins[pre + "_b_lo"], k, (be, 0.0), ch, cl,
                            m) == 0
        assert np.array_equal(ch.view(np.uint64), pins[pre + "_out_hi"].view(np.uint64))
        assert np.array_equal(cl.view(np.uint64), pins[pre + "_out_lo"].view(np.uint64))
    ch, cl = np.zeros(4), np.zeros(4)
    assert oracle.rgemm("N", "N", 2, 2, 2, (1.0, 0.0), pins["hil_inv_hi"], pins["hil_inv_lo"], 2,
                        pins["hil_a_hi"], pins["hil_a_lo"], 2, (0.0, 0.0), ch, cl, 2) == 0
    assert np.array_equal(ch.view(np.uint64), pins["hil_prod_hi"].view(np.uint64))
    assert np.array_equal(cl.view(np.uint64), pins["hil_prod_lo"].view(np.uint64))
