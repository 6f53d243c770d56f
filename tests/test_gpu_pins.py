"""GPU: the reference's own known-answer pins for the Rgemm path, run through
the package API on the B200 (fixtures made by running the reference itself:
oracle/gen_pins.py -> tests/golden/pins.npz).

* integer instance (test_acceptance.py:121-139, cli.py:160-186): exact in
  EVERY mode -- all products and sums are small integers;
* Hilbert n = 2 (test_acceptance.py:298-305): _mm(ainv, a) of the reference's
  own inverse; exact mode reproduces the reference's product bit for bit, so
  ||_mm(ainv, a) - I||_inf is exactly (2^-106, 0) as pinned; the fast modes
  stay inside the dd bound of the exact product (they are not bitwise);
* thread-count invariance (test_mpblas.py:661-681): the reference's n = 8
  operands through ddb_rgemm_mgpu with 1, 2, 3, 4 and 8 slabs (one GPU, the
  device id repeated) are bitwise equal to the reference's Rgemm.
"""

import ctypes
import os
from fractions import Fraction

import numpy as np
import pytest

from oracle import exact
from paper_2109_13406_b200 import DeviceMatrix, Rgemm, _lib

pytestmark = pytest.mark.gpu

PINS = np.load(os.path.join(os.path.dirname(__file__), "golden", "pins.npz"))


def dev(rows, cols, name):
    import torch
    return DeviceMatrix(rows, cols, "dd", rows, store=(
        torch.from_numpy(PINS[name + "_hi"].copy()).cuda(),
        torch.from_numpy(PINS[name + "_lo"].copy()).cuda()))


def bits(t):
    return t.cpu().numpy().view(np.uint64)


@pytest.mark.parametrize("mode", ["exact", "fast", "twosum", "reference"])
def test_integer_instance_exact_in_every_mode(mode):
    a, b, c = dev(3, 3, "int_a"), dev(3, 3, "int_b"), dev(3, 3, "int_c")
    Rgemm("N", "N", 3, 3, 3, 3.0, a, 3, b, 3, -2.0, c, 3, mode=mode)
    assert np.array_equal(bits(c.store[0]), PINS["int_out_hi"].view(np.uint64))
    assert np.array_equal(bits(c.store[1]), PINS["int_out_lo"].view(np.uint64))
    want = np.array([[21, -192, 18], [-118, -194, 8], [210, 361, 82]], dtype=np.float64)
    assert np.array_equal(c.store[0].cpu().numpy().reshape(3, 3).T, want)
    assert not c.store[1].cpu().numpy().any()


def _residual_exact(ph, pl):
    """||P - I||_inf of the 2 x 2 product, in exact rationals."""
    P = [[Fraction(ph[i + 2 * j]) + Fraction(pl[i + 2 * j]) for j in range(2)] for i in range(2)]
    return max(sum(abs(P[i][j] - (1 if i == j else 0)) for j in range(2)) for i in range(2))


@pytest.mark.parametrize("mode", ["exact", "reference", "fast", "twosum"])
def test_hilbert_n2_residual(mode):
    import torch
    inv, h = dev(2, 2, "hil_inv"), dev(2, 2, "hil_a")
    c = DeviceMatrix(2, 2, "dd", 2, store=(torch.zeros(4, dtype=torch.float64).cuda(),
                                           torch.zeros(4, dtype=torch.float64).cuda()))
    Rgemm("N", "N", 2, 2, 2, 1.0, inv, 2, h, 2, 0.0, c, 2, mode=mode)   # testkit._mm
    ph, pl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    if mode in ("exact", "reference"):
        assert np.array_equal(ph.view(np.uint64), PINS["hil_prod_hi"].view(np.uint64))
        assert np.array_equal(pl.view(np.uint64), PINS["hil_prod_lo"].view(np.uint64))
        assert _residual_exact(ph, pl) == Fraction(2) ** -106      # the pinned (2^-106, 0)
        assert tuple(PINS["hil_residual"]) == (2.0 ** -106, 0.0)
    else:
        vals, scales = exact.exact_entries("N", "N", 2, (1.0, 0.0), PINS["hil_inv_hi"],
                                           PINS["hil_inv_lo"], 2, PINS["hil_a_hi"],
                                           PINS["hil_a_lo"], 2, (0.0, 0.0), ph, pl, 2,
                                           [0, 1], [0, 1])
        assert exact.error_ratios(ph, pl, 2, [0, 1], [0, 1], vals, scales, 2) <= 1.0
        assert _residual_exact(ph, pl) < Fraction(2) ** -100


@pytest.mark.parametrize("t", [1, 2, 3, 4, 8])
def test_thread_count_invariance_through_mgpu(t):
    """The reference's Rgemm_par(t) result == its Rgemm result bit for bit;
    ddb_rgemm_mgpu with t slabs must reproduce that same result."""
    import torch
    n = 8
    a, b, c = dev(n, n, "tc_a"), dev(n, n, "tc_b"), dev(n, n, "tc_c")
    devs = (ctypes.c_int * t)(*([0] * t))
    rc = _lib.load().ddb_rgemm_mgpu(b"N", b"N", n, n, n, 0.75, 0.0,
                                    a.store[0].data_ptr(), a.store[1].data_ptr(), n,
                                    b.store[0].data_ptr(), b.store[1].data_ptr(), n, -0.5, 0.0,
                                    c.store[0].data_ptr(), c.store[1].data_ptr(), n,
                                    _lib.MODES["exact"], t, devs)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert np.array_equal(bits(c.store[0]), PINS["tc_out_hi"].view(np.uint64))
    assert np.array_equal(bits(c.store[1]), PINS["tc_out_lo"].view(np.uint64))
