"""CPU tests of the drop-in boundary: argument validation, error types and
messages, scalar coercion, early exits, and the C ABI exports.  These mirror
the reference's own checks (pkg/tests/test_mpblas.py:542-614)."""

import ctypes
import math
import re
import subprocess

import numpy as np
import pytest

from paper_2109_13406_b200 import (BlasError, HostMatrix, Rgemm, Rsyrk, _lib, flop_count,
                                   to_dd)


def mats(m, n, k):
    return HostMatrix(m, k), HostMatrix(k, n), HostMatrix(m, n)


GEMM_BAD = [
    (("X", "N", 2, 2, 2), {}, 1), (("N", "nn", 2, 2, 2), {}, 2), ((1, "N", 2, 2, 2), {}, 1),
    (("N", "N", -1, 2, 2), {}, 3), (("N", "N", 2, -1, 2), {}, 4), (("N", "N", 2, 2, -1), {}, 5),
    (("N", "N", 2, 2, 2), {"lda": 1}, 8), (("N", "N", 2, 2, 2), {"ldb": 1}, 10),
    (("N", "N", 2, 2, 2), {"ldc": 1}, 13), (("T", "N", 2, 2, 3), {"lda": 2}, 8),
    (("N", "T", 2, 3, 2), {"ldb": 2}, 10),
]


@pytest.mark.parametrize("args,lds,idx", GEMM_BAD)
def test_rgemm_blas_error_indices(args, lds, idx):
    ta, tb, m, n, k = args
    a, b, c = HostMatrix(4, 4), HostMatrix(4, 4), HostMatrix(4, 4)
    with pytest.raises(BlasError) as e:
        Rgemm(ta, tb, m, n, k, 1.0, a, lds.get("lda", 4), b, lds.get("ldb", 4), 0.0, c,
              lds.get("ldc", 4))
    assert e.value.index == idx and e.value.routine == "Rgemm"
    assert str(e.value) == f"on entry to Rgemm parameter number {idx} had an illegal value"
    assert isinstance(e.value, ValueError)


SYRK_BAD = [(("X", "N", 2, 2), {}, 1), (("U", "Q", 2, 2), {}, 2), (("U", "N", -1, 2), {}, 3),
            (("U", "N", 2, -1), {}, 4), (("U", "N", 3, 2), {"lda": 2}, 7),
            (("U", "T", 2, 3), {"lda": 2}, 7), (("L", "N", 3, 2), {"ldc": 2}, 10)]


@pytest.mark.parametrize("args,lds,idx", SYRK_BAD)
def test_rsyrk_blas_error_indices(args, lds, idx):
    up, tr, n, k = args
    a, c = HostMatrix(4, 4), HostMatrix(4, 4)
    with pytest.raises(BlasError) as e:
        Rsyrk(up, tr, n, k, 1.0, a, lds.get("lda", 4), 0.0, c, lds.get("ldc", 4))
    assert e.value.index == idx


def test_validation_matches_c_abi():
    """The Python checks and ddb_*_validate agree on every GEMM_BAD case."""
    try:
        L = _lib.load()
    except _lib.LibraryMissing:
        pytest.skip("libddblas.so not built")
    for (ta, tb, m, n, k), lds, idx in GEMM_BAD:
        if not isinstance(ta, str) or len(tb) != 1:
            continue
        rc = L.ddb_rgemm_validate(ta.encode(), tb.encode(), m, n, k, lds.get("lda", 4),
                                  lds.get("ldb", 4), lds.get("ldc", 4))
        assert rc == idx
    for (up, tr, n, k), lds, idx in SYRK_BAD:
        rc = L.ddb_rsyrk_validate(up.encode(), tr.encode(), n, k, lds.get("lda", 4),
                                  lds.get("ldc", 4))
        assert rc == idx


def test_mixed_precision_is_value_error_before_blas_error():
    a = HostMatrix(2, 2)
    b = HostMatrix(2, 2)
    b.precision = "f64"
    with pytest.raises(ValueError, match="mixed precisions"):
        Rgemm("X", "N", 2, 2, 2, 1.0, a, 2, b, 2, 0.0, a, 2)


def test_unknown_precision_is_not_silently_run_on_cpu():
    a = HostMatrix(2, 2)
    a.precision = "qd"
    with pytest.raises(NotImplementedError):
        Rgemm("N", "N", 2, 2, 2, 1.0, a, 2, a, 2, 0.0, a, 2)
    with pytest.raises(NotImplementedError):
        HostMatrix(2, 2, "qd")


def test_cgemm_rejects_real_matrices():
    """level23.py:207-208."""
    from paper_2109_13406_b200 import Cgemm
    a = HostMatrix(2, 2)
    with pytest.raises(ValueError, match="requires complex"):
        Cgemm("N", "N", 2, 2, 2, 1.0, a, 2, a, 2, 0.0, a, 2)


def test_f64_without_gpu_fails_loudly():
    """binary64 goes to the GPU too; with no device the call raises."""
    import os
    a = HostMatrix(2, 2, "f64")
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libddblas.so not built")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    with pytest.raises(RuntimeError):
        Rgemm("N", "N", 2, 2, 2, 1.0, a, 2, a, 2, 0.0, a, 2)


def test_bad_scalar_type_is_type_error():
    a, b, c = mats(2, 2, 2)
    with pytest.raises(TypeError):
        Rgemm("N", "N", 2, 2, 2, [1.0], a, 2, b, 2, 0.0, c, 2)
    with pytest.raises(TypeError):
        Rsyrk("U", "N", 2, 2, 1.0, a, 2, np.int64(1), c, 2)


def test_short_storage_is_value_error():
    a, b, c = mats(3, 3, 3)
    with pytest.raises(ValueError, match="too short"):
        Rgemm("N", "N", 3, 3, 3, 1.0, a, 5, b, 3, 0.0, c, 3)


def test_early_exits_touch_nothing():
    """level23.py:191-192: no device work at all (so no GPU is needed)."""
    a, b, c = mats(3, 3, 3)
    c.store[0][:] = 7.0
    Rgemm("N", "N", 0, 3, 3, 1.0, a, 3, b, 3, 0.0, c, 3)
    Rgemm("N", "N", 3, 3, 3, 0.0, a, 3, b, 3, 1.0, c, 3)
    Rgemm("N", "N", 3, 3, 0, 2.0, a, 3, b, 3, "1", c, 3)
    Rsyrk("U", "N", 3, 0, 1.0, a, 3, 1, c, 3)
    assert np.all(c.store[0] == 7.0)


def test_scalar_coercion_matches_ddouble():
    assert to_dd(1.5) == (1.5, 0.0)
    assert to_dd(True) == (1.0, 0.0)
    big = 2 ** 60 + 1
    hi, lo = to_dd(big)
    assert hi == float(2 ** 60) and lo == 1.0
    hi, lo = to_dd("0.1")
    from fractions import Fraction
    err = abs(Fraction(hi) + Fraction(lo) - Fraction(1, 10))
    assert err < Fraction(1, 2 ** 110)
    assert to_dd(10 ** 400) == (math.inf, 0.0)

    class D:
        hi, lo = 2.0, 2.0 ** -60
    assert to_dd(D()) == (2.0, 2.0 ** -60)
    with pytest.raises(ValueError):
        to_dd("1.2.3")


def test_flop_count_matches_reference_bench():
    """pkg/tests/test_bench.py:21-31."""
    assert flop_count("Rgemm", 4) == 128.0
    assert flop_count("Rgemm", 3, k=5, m=2) == 60.0
    assert flop_count("Rsyrk", 4, k=3) == 60.0
    assert flop_count("Rpotrf", 3) == 9.0
    assert flop_count("Rgetrf", 3) == 18.0


def test_library_exports_every_header_symbol():
    """Every function include/ddblas.h declares is exported by libddblas.so."""
    import os
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    header = open(os.path.join(repo, "include", "ddblas.h")).read()
    declared = set(re.findall(r"^\w[\w\s\*]*?\b(ddb_\w+)\s*\(", header, re.M))
    assert declared == set(_lib.EXPORTS)
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libddblas.so not built")
    L = ctypes.CDLL(_lib.LIB_PATH)
    for name in declared:
        assert hasattr(L, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True).stdout
    for name in declared:
        assert re.search(rf"\bT {name}$", out, re.M), name
    assert _lib.load().ddb_version() == 130


POTRF_BAD = [(("X", 2), {}, 1), (("UU", 2), {}, 1), ((3, 2), {}, 1), (("U", -1), {}, 2),
             (("L", 3), {"lda": 2}, 4), (("L", 0), {"lda": 0}, 4)]


@pytest.mark.parametrize("args,lds,idx", POTRF_BAD)
def test_rpotrf_blas_error_indices(args, lds, idx):
    """mplapack/chol.py:21-29 (validation order uplo, n, lda)."""
    from paper_2109_13406_b200 import Rpotrf
    up, n = args
    a = HostMatrix(4, 4)
    with pytest.raises(BlasError) as e:
        Rpotrf(up, n, a, lds.get("lda", 4))
    assert e.value.index == idx and e.value.routine == "Rpotrf"
    try:
        L = _lib.load()
    except _lib.LibraryMissing:
        return
    if isinstance(up, str) and len(up) == 1:
        assert L.ddb_rpotrf_validate(up.encode(), n, lds.get("lda", 4)) == idx


def test_rpotrf_early_exit_and_precision_gate():
    from paper_2109_13406_b200 import Rpotrf
    a = HostMatrix(3, 3)
    a.store[0][:] = 7.0
    assert Rpotrf("L", 0, a) == 0            # chol.py:30-31, no device work
    assert Rpotrf("U", 0, a, 1) == 0
    assert np.all(a.store[0] == 7.0)
    b = HostMatrix(3, 3, "f64")
    b.precision = "qd"
    with pytest.raises(NotImplementedError):
        Rpotrf("L", 3, b)


def test_rpotrf_without_gpu_fails_loudly():
    import os
    from paper_2109_13406_b200 import Rpotrf
    if not os.path.exists(_lib.LIB_PATH):
        pytest.skip("libddblas.so not built")
    try:
        import torch
        if torch.cuda.is_available():
            pytest.skip("a GPU is present")
    except ImportError:
        pass
    a = HostMatrix(2, 2)
    a.store[0][[0, 3]] = 2.0
    with pytest.raises(RuntimeError):
        Rpotrf("L", 2, a)


TRSM_BAD = [(("X", "U", "N", "N", 2, 2), {}, 1), (("L", "X", "N", "N", 2, 2), {}, 2),
            (("L", "U", "X", "N", 2, 2), {}, 3), (("L", "U", "N", "X", 2, 2), {}, 4),
            (("L", "U", "N", "N", -1, 2), {}, 5), (("L", "U", "N", "N", 2, -1), {}, 6),
            (("L", "U", "N", "N", 3, 2), {"lda": 2}, 9), (("R", "U", "N", "N", 2, 3), {"lda": 2}, 9),
            (("L", "U", "N", "N", 3, 2), {"ldb": 2}, 11)]


@pytest.mark.parametrize("args,lds,idx", TRSM_BAD)
def test_rtrsm_blas_error_indices(args, lds, idx):
    """level23.py:290-304, and the C ABI's validate agrees."""
    from paper_2109_13406_b200 import Rtrsm
    sd, up, tr, dg, m, n = args
    a, b = HostMatrix(4, 4), HostMatrix(4, 4)
    with pytest.raises(BlasError) as e:
        Rtrsm(sd, up, tr, dg, m, n, 1.0, a, lds.get("lda", 4), b, lds.get("ldb", 4))
    assert e.value.index == idx and e.value.routine == "Rtrsm"
    try:
        L = _lib.load()
    except _lib.LibraryMissing:
        return
    assert L.ddb_rtrsm_validate(sd.encode(), up.encode(), tr.encode(), dg.encode(), m, n,
                                lds.get("lda", 4), lds.get("ldb", 4)) == idx


def test_rtrsm_early_exit_and_precision_gate():
    from paper_2109_13406_b200 import Rtrsm
    a, b = HostMatrix(3, 3), HostMatrix(3, 3)
    b.store[0][:] = 7.0
    Rtrsm("L", "U", "N", "N", 0, 3, 2.0, a, 3, b, 3)          # level23.py:306-307
    Rtrsm("R", "L", "T", "U", 3, 0, 2.0, a, 3, b, 3)
    assert np.all(b.store[0] == 7.0)
    c = HostMatrix(3, 3, "f64")
    with pytest.raises(ValueError, match="mixed precisions"):
        Rtrsm("L", "U", "N", "N", 3, 3, 1.0, a, 3, c, 3)
    q = HostMatrix(3, 3)
    q.precision = "qd"
    with pytest.raises(NotImplementedError):
        Rtrsm("L", "U", "N", "N", 3, 3, 1.0, q, 3, q, 3)


@pytest.mark.parametrize("args,idx", [((-1, 2, 2), 1), ((2, -1, 2), 2), ((3, 2, 2), 4),
                                      ((0, 0, 0), 4)])
def test_rgetrf_blas_error_indices(args, idx):
    """mplapack/lu.py:82-85 (m, n, lda), and the C ABI's validate agrees."""
    from paper_2109_13406_b200 import Rgetrf
    m, n, lda = args
    with pytest.raises(BlasError) as e:
        Rgetrf(m, n, HostMatrix(4, 4), lda)
    assert e.value.index == idx and e.value.routine == "Rgetrf"
    try:
        L = _lib.load()
    except _lib.LibraryMissing:
        return
    assert L.ddb_rgetrf_validate(m, n, lda) == idx


def test_rgetrf_early_exit_and_precision_gate():
    from paper_2109_13406_b200 import PivotVector, Rgetrf
    a = HostMatrix(3, 3)
    ipiv, info = Rgetrf(0, 3, a, 3)
    assert ipiv == [] and info == 0 and isinstance(ipiv, PivotVector)
    assert Rgetrf(3, 0, a) == (PivotVector(), 0)
    q = HostMatrix(3, 3)
    q.precision = "qd"
    with pytest.raises(NotImplementedError):
        Rgetrf(3, 3, q)


@pytest.mark.parametrize("args,lds,idx", [(("X", 2, 1), {}, 1), (("N", -1, 1), {}, 2),
                                          (("N", 2, -1), {}, 3), (("N", 3, 1), {"lda": 2}, 5),
                                          (("T", 3, 1), {"ldb": 2}, 8)])
def test_rgetrs_blas_error_indices(args, lds, idx):
    """mplapack/lu.py:117-129, and the C ABI's validate agrees."""
    from paper_2109_13406_b200 import Rgetrs
    tr, n, nrhs = args
    with pytest.raises(BlasError) as e:
        Rgetrs(tr, n, nrhs, HostMatrix(4, 4), lds.get("lda", 4), [1, 2, 3, 4], HostMatrix(4, 4),
               lds.get("ldb", 4))
    assert e.value.index == idx and e.value.routine == "Rgetrs"
    try:
        L = _lib.load()
    except _lib.LibraryMissing:
        return
    assert L.ddb_rgetrs_validate(tr.encode(), n, nrhs, lds.get("lda", 4), lds.get("ldb", 4)) == idx


def test_rgetrs_missing_b_is_index_8_and_early_exit():
    from paper_2109_13406_b200 import Rgetrs
    with pytest.raises(BlasError) as e:
        Rgetrs("N", 2, 1, HostMatrix(2, 2), 2, [1, 2], None, None)
    assert e.value.index == 8
    b = HostMatrix(3, 1)
    b.store[0][:] = 5.0
    assert Rgetrs("N", 3, 0, HostMatrix(3, 3), 3, [1, 2, 3], b, 3) == 0
    assert np.all(b.store[0] == 5.0)
