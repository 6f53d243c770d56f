"""Generate tests/golden/pins.npz: the reference's own known-answer pins for
the Rgemm path, produced by RUNNING the reference (TEST INFRASTRUCTURE ONLY).

    python oracle/gen_pins.py          # in the build container (/root/reference present)

* integer instance (test_acceptance.py:121-139, cli.py:160-186): alpha = 3,
  beta = -2, A, B, C small integer matrices; want [[21,-192,18],...], lo == 0.
* Hilbert n = 2 residual (test_acceptance.py:298-305): the reference inverts
  the dd Hilbert matrix (testkit.hilbert_infnorm_study -> Rgetrf + Rgetri),
  then _mm(ainv, a) = Rgemm('N','N', alpha 1, beta 0) and
  ||_mm(ainv, a) - I||_inf is exactly (2^-106, 0).  Stored: H, Hinv (dd
  planes, as the reference computed them), the reference's Rgemm product and
  the residual.
* thread-count invariance (test_mpblas.py:661-681): n = 8 random dd operands
  (the reference's rand_rows with random.Random(503)), alpha 0.75, beta -0.5,
  and the reference's Rgemm / Rgemm_par(t in 1,2,3,4,8) result -- all bitwise
  equal, which the generator asserts.
"""

from __future__ import annotations

import os
import random
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
OUT = os.path.join(os.path.dirname(HERE), "tests", "golden", "pins.npz")


def planes(mat):
    return np.asarray(mat.store[0], dtype=np.float64).copy(), \
        np.asarray(mat.store[1], dtype=np.float64).copy()


def main():
    sys.path.insert(0, REF)
    sys.path.insert(0, os.path.join(os.path.dirname(REF), "tests"))
    from mpkit.mpblas import Matrix, Rgemm
    from mpkit.mpblas.parallel import Rgemm_par
    from mpkit import testkit
    out = {}
    # 1. integer instance
    rows_a = [[1, 8, 3], [0, 10, 8], [9, -5, -1]]
    rows_b = [[9, 8, 3], [3, -11, 0], [-8, 6, 1]]
    rows_c = [[3, 3, 0], [8, 4, 8], [6, 1, -2]]
    a = Matrix.from_rows(rows_a, "dd")
    b = Matrix.from_rows(rows_b, "dd")
    c = Matrix.from_rows(rows_c, "dd")
    for name, m in (("int_a", a), ("int_b", b), ("int_c", c)):
        out[name + "_hi"], out[name + "_lo"] = planes(m)
    Rgemm("N", "N", 3, 3, 3, 3.0, a, a.ld, b, b.ld, -2.0, c, c.ld)
    out["int_out_hi"], out["int_out_lo"] = planes(c)
    want = np.array([[21, -192, 18], [-118, -194, 8], [210, 361, 82]], dtype=np.float64)
    assert np.array_equal(out["int_out_hi"].reshape(3, 3).T, want)
    assert not out["int_out_lo"].any()
    # 2. Hilbert n = 2 through the study's own inversion
    n = 2
    h = testkit.gen_matrix(testkit.MatrixGenSpec("hilbert", n, n), "dd")
    lu = h.copy()
    from mpkit.mplapack import Rgetrf as getrf, Rgetri as getri
    from mpkit.mplapack.workspace import workspace_query
    from mpkit.mpblas.matrix import Vector
    ipiv, info = getrf(n, n, lu)
    assert info == 0
    lwork = workspace_query("Rgetri", n)
    assert getri(n, lu, lu.ld, ipiv, Vector(lwork, "dd"), lwork) == 0
    out["hil_a_hi"], out["hil_a_lo"] = planes(h)
    out["hil_inv_hi"], out["hil_inv_lo"] = planes(lu)
    prod = testkit._mm(lu, h)
    out["hil_prod_hi"], out["hil_prod_lo"] = planes(prod)
    res = testkit.left_residual_infnorm(h, lu)
    out["hil_residual"] = np.array([res.hi, res.lo])
    assert res.hi == 2.0 ** -106 and res.lo == 0.0
    assert dict(testkit.hilbert_infnorm_study(2, "dd"))[2].hi == res.hi
    # 3. thread-count invariance (rand_rows of test_mpblas.py)
    from test_mpblas import rand_rows
    rng = random.Random(503)
    n = 8
    ad, bd, cd = rand_rows(rng, n, n), rand_rows(rng, n, n), rand_rows(rng, n, n)
    A, B, C = (Matrix.from_rows(x, "dd") for x in (ad, bd, cd))
    for name, m in (("tc_a", A), ("tc_b", B), ("tc_c", C)):
        out[name + "_hi"], out[name + "_lo"] = planes(m)
    Rgemm("N", "N", n, n, n, 0.75, A, n, B, n, -0.5, C, n)
    out["tc_out_hi"], out["tc_out_lo"] = planes(C)
    for t in (1, 2, 3, 4, 8):
        c2 = Matrix.from_rows(cd, "dd")
        Rgemm_par("N", "N", n, n, n, 0.75, Matrix.from_rows(ad, "dd"), n,
                  Matrix.from_rows(bd, "dd"), n, -0.5, c2, n, t=t)
        h2, l2 = planes(c2)
        assert np.array_equal(h2.view(np.uint64), out["tc_out_hi"].view(np.uint64))
        assert np.array_equal(l2.view(np.uint64), out["tc_out_lo"].view(np.uint64))
    np.savez_compressed(OUT, **out)
    print("wrote", OUT, sorted(out))


if __name__ == "__main__":
    main()
