"""GPU: the fast mode's building blocks in isolation, through the C ABI's
diagnostic entry points.

* ddb_cross_terms -- the hand-written DMMA kernel (dd_cross.cu) for the split
  algorithm's X = A_lo B_hi + A_hi B_lo, checked against a plain binary64
  torch reference with the recursive-summation bound both sides satisfy:
  |X - X_ref| <= 2 * (2k u) * (|A_lo||B_hi| + |A_hi||B_lo|), u = 2^-53.
"""

import ctypes

import numpy as np
import pytest

from paper_2109_13406_b200 import _lib

pytestmark = pytest.mark.gpu

U = 2.0 ** -53


def _ptr(t):
    return ctypes.c_void_p(t.data_ptr())


def _planes(rows, cols, ld, seed, scale=1.0):
    import torch
    g = torch.Generator(device="cuda").manual_seed(seed)
    hi = (torch.rand(ld * cols, device="cuda", dtype=torch.float64, generator=g) * 2 - 1) * scale
    lo = hi * (torch.rand(ld * cols, device="cuda", dtype=torch.float64, generator=g) * 2 - 1) * U
    return hi, lo


def _mat(p, rows, cols, ld):
    return p.view(cols, ld)[:, :rows].T     # column-major view (rows x cols)


def _cross(m, n, k, lda, ldb, tri=0, seed=1):
    import torch
    ah, al = _planes(m, k, lda, seed)
    bh, bl = _planes(k, n, ldb, seed + 1)
    x = torch.full((m * n,), float("nan"), device="cuda", dtype=torch.float64)
    stream = torch.cuda.current_stream().cuda_stream
    rc = _lib.load().ddb_cross_terms(m, n, k, _ptr(ah), _ptr(al), lda, _ptr(bh), _ptr(bl), ldb,
                                     _ptr(x), tri, ctypes.c_void_p(stream))
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    A_h, A_l = _mat(ah, m, k, lda), _mat(al, m, k, lda)
    B_h, B_l = _mat(bh, k, n, ldb), _mat(bl, k, n, ldb)
    ref = A_l @ B_h + A_h @ B_l
    scale = A_l.abs() @ B_h.abs() + A_h.abs() @ B_l.abs()
    got = x.view(n, m).T
    return got, ref, scale


@pytest.mark.parametrize("m,n,k", [(128, 128, 16), (256, 384, 1000), (200, 130, 77),
                                   (1, 1, 1), (129, 257, 3), (1000, 64, 4096)])
def test_cross_terms_match_binary64_reference(m, n, k):
    import torch
    lda, ldb = m + (m & 1), k + (k & 1)          # even leading dimensions (TMA)
    got, ref, scale = _cross(m, n, k, lda, ldb)
    assert torch.isfinite(got).all()
    err = (got - ref).abs()
    assert bool((err <= 4 * k * U * scale + 1e-300).all()), float((err / scale).max())


@pytest.mark.parametrize("tri", [1, 2])
def test_cross_terms_triangle_tiles(tri):
    import torch
    m = n = 300
    got, ref, scale = _cross(m, n, 64, m, 64, tri=tri)
    i = torch.arange(m, device="cuda")[:, None]
    j = torch.arange(n, device="cuda")[None, :]
    inside = (i <= j) if tri == 1 else (i >= j)
    err = (got - ref).abs()
    assert bool((err[inside] <= 4 * 64 * U * scale[inside]).all())


def test_cross_terms_rejects_odd_leading_dimension():
    import torch
    ah, al = _planes(5, 8, 5, 3)
    x = torch.zeros(25, device="cuda", dtype=torch.float64)
    rc = _lib.load().ddb_cross_terms(5, 5, 8, _ptr(ah), _ptr(al), 5, _ptr(ah), _ptr(al), 8,
                                     _ptr(x), 0, None)
    assert rc == -1


# ---- the certified magnitude bound (tcgen05 kernel) -------------------------

def _bound(ta, tb, m, n, k, seed, spread=0.0, positive=False):
    import torch
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    g = torch.Generator(device="cuda").manual_seed(seed)
    def mk(r, c):
        x = torch.rand(r * c, device="cuda", dtype=torch.float64, generator=g)
        if not positive:
            x = x * 2 - 1
        if spread:
            x = x * torch.exp2(-(spread * torch.rand(r * c, device="cuda", dtype=torch.float64,
                                                      generator=g)).round())
        return x
    a, b = mk(nra, nca), mk(nrb, ncb)
    kp = (k + 7) // 8 * 8
    re = torch.zeros(m, device="cuda", dtype=torch.int32)
    ce = torch.zeros(n, device="cuda", dtype=torch.int32)
    s = torch.full((m * n,), float("nan"), device="cuda", dtype=torch.float32)
    abf = torch.zeros(m * kp, device="cuda", dtype=torch.bfloat16)
    bbf = torch.zeros(n * kp, device="cuda", dtype=torch.bfloat16)
    rc = _lib.load().ddb_abs_bound(ta.encode(), tb.encode(), m, n, k, _ptr(a), nra, _ptr(b), nrb,
                                   _ptr(re), _ptr(ce), _ptr(s), _ptr(abf), _ptr(bbf), None)
    assert rc == 0, _lib.last_error()
    A = _mat(a, nra, nca, nra)
    A = A if ta == "N" else A.T                     # op(A): m x k
    B = _mat(b, nrb, ncb, nrb)
    B = B if tb == "N" else B.T                     # op(B): k x n
    Af = abf.view(m, kp)[:, :k].double()
    Bf = bbf.view(n, kp)[:, :k].double()
    return A, B, re, ce, Af, Bf, s.view(n, m).T.double()


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (300, 200, 1000), (1, 1, 1), (129, 65, 7),
                                   (256, 384, 4096)])
def test_bound_operands_round_up_and_gemm_is_certified(ta, tb, m, n, k):
    import torch
    A, B, re, ce, Af, Bf, S = _bound(ta, tb, m, n, k, 7 + m + k)
    # every converted magnitude >= |hi| * 2^(1022 - e) (rounded up), and tight
    sa = A.abs() * torch.exp2(1022.0 - re.double())[:, None]
    sb = B.abs() * torch.exp2(1022.0 - ce.double())[None, :]
    assert bool((Af >= sa).all()) and bool((Bf.T >= sb).all())
    assert bool((Af <= sa * (1 + 2.0 ** -7) + 2.0 ** -133).all())
    assert bool((sa < 1).all()) and bool((sb < 1).all())
    exact = Af @ Bf.T          # exact in binary64 up to ~k 2^-53
    fac = 1 + k * 2.0 ** -21
    assert bool((S * fac >= exact * (1 - 2.0 ** -50)).all())
    assert bool((S <= exact * (1 + k * 2.0 ** -22) + 1e-30).all())


@pytest.mark.parametrize("k", [8192, 65536])
def test_bound_deep_nonnegative_accumulation(k):
    """All-positive magnitudes at depth k: the fp32 accumulation error must
    stay inside the (1 + k 2^-21) factor the anchor relies on."""
    A, B, re, ce, Af, Bf, S = _bound("N", "N", 256, 256, k, 3, positive=True)
    exact = Af @ Bf.T
    ratio = (S / exact)
    assert float(ratio.min()) * (1 + k * 2.0 ** -21) >= 1.0, float(ratio.min())
    assert float(ratio.max()) <= 1 + k * 2.0 ** -22


def test_bound_with_spread_magnitudes():
    A, B, re, ce, Af, Bf, S = _bound("N", "N", 200, 160, 300, 5, spread=60.0)
    exact = Af @ Bf.T
    assert bool((S * (1 + 300 * 2.0 ** -21) + 300 * 2.0 ** -120 >= exact).all())


@pytest.mark.parametrize("m,n,k", [(129, 257, 3), (1000, 64, 4096), (200, 130, 77)])
def test_cross_and_bound_stay_inside_their_outputs(m, n, k):
    """Guard zones after the m x n outputs of both diagnostics stay untouched
    (the kernels' ragged-edge masks; split-K scratch is separate)."""
    import torch
    lda, ldb = m + (m & 1), k + (k & 1)
    ah, al = _planes(m, k, lda, 9)
    bh, bl = _planes(k, n, ldb, 10)
    guard = 4096
    x = torch.full((m * n + guard,), 12345.0, device="cuda", dtype=torch.float64)
    rc = _lib.load().ddb_cross_terms(m, n, k, _ptr(ah), _ptr(al), lda, _ptr(bh), _ptr(bl), ldb,
                                     _ptr(x), 0, None)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert bool((x[m * n:] == 12345.0).all()) and bool(torch.isfinite(x[:m * n]).all())
    s = torch.full((m * n + guard,), 7.0, device="cuda", dtype=torch.float32)
    re = torch.zeros(m + 64, device="cuda", dtype=torch.int32)
    ce = torch.zeros(n + 64, device="cuda", dtype=torch.int32)
    rc = _lib.load().ddb_abs_bound(b"N", b"N", m, n, k, _ptr(ah), lda, _ptr(bh), ldb, _ptr(re),
                                   _ptr(ce), _ptr(s), None, None, None)
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert bool((s[m * n:] == 7.0).all()) and bool((s[:m * n] >= 0).all())
    assert bool((re[m:] == 0).all()) and bool((ce[n:] == 0).all())
