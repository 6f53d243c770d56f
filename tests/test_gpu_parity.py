"""GPU parity: the CUDA path (through the package API and the C ABI) against
the reference's golden outputs, the bit-exact C oracle and the exact-rational
checker.  All tests need a B200."""

import os

import numpy as np
import pytest

from oracle import exact, golden, oracle
from paper_2109_13406_b200 import DeviceMatrix, HostMatrix, Rgemm, Rsyrk, _lib
from paper_2109_13406_b200.synth import random_dd

pytestmark = pytest.mark.gpu

os.environ.setdefault("DDB_DEBUG_SYNC", "1")


def bits_equal(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    both_nan = np.isnan(a) & np.isnan(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | both_nan))


def dev(m, n, ld, planes):
    import torch
    mat = DeviceMatrix(m, n, "dd", ld,
                       store=tuple(torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in planes))
    return mat


def host(m, n, ld, planes):
    return HostMatrix.from_planes(m, n, planes[0].copy(), planes[1].copy(), ld)


ALL_CASES = list(golden.load_cases())
CASES = [c for c in ALL_CASES if c[0]["routine"] in ("Rgemm", "Rsyrk")]
CCASES = [c for c in ALL_CASES if c[0]["routine"] == "Cgemm"]


def dev64(m, n, ld, hi):
    import torch
    return DeviceMatrix(m, n, "f64", ld, store=(torch.from_numpy(np.ascontiguousarray(hi)).cuda(),))


def host64(m, n, ld, hi):
    return HostMatrix.from_planes(m, n, hi.copy(), None, ld)


def _unsafe(h, l, canon):
    """The prescan's per-word test (dd_prescan.cu): outside the safe window,
    or (fast modes) not a normalised dd."""
    h = np.asarray(h, dtype=np.float64)
    l = np.asarray(l, dtype=np.float64)
    with np.errstate(all="ignore"):
        ah, al = np.abs(h), np.abs(l)
        bad = ((h != 0) & (ah < 2.0 ** -300)) | ~(ah < 2.0 ** 301) | ~(al < 2.0 ** 301)
        if canon:
            bad |= al > ah * 2.0 ** -53
    return bad


def routed_elements(case, arr, canon):
    """(i, j) of C whose op(A) row or op(B) column holds an unsafe word: the
    elements the per-element routing sends to the reference kernel."""
    def rows_of(trans, hi, lo, ld, nrow_op, k):
        bad = set()
        for r in range(nrow_op):
            idx = (r + np.arange(k) * ld) if trans == "N" else (r * ld + np.arange(k))
            if np.any(_unsafe(hi[idx], lo[idx], canon)):
                bad.add(r)
        return bad
    if case["routine"] == "Rgemm":
        m, n, k = case["m"], case["n"], case["k"]
        ta, tb = case["transa"].upper(), case["transb"].upper()
        ra = rows_of("N" if ta == "N" else "T", arr["A_hi"], arr["A_lo"], case["lda"], m, k)
        cb = rows_of("T" if tb == "N" else "N", arr["B_hi"], arr["B_lo"], case["ldb"], n, k)
    else:
        n = m = case["n"]
        k = case["k"]
        tr = case["trans"].upper()
        ra = rows_of("N" if tr == "N" else "T", arr["A_hi"], arr["A_lo"], case["lda"], n, k)
        cb = ra
    return {(i, j) for i in range(m) for j in range(n) if i in ra or j in cb}


def _run_case(case, arr, mode, on_device=True):
    if case.get("precision") == "f64":
        return _run_case_f64(case, arr, on_device)
    mk = dev if on_device else host
    if case["routine"] == "Rgemm":
        ta, tb = case["transa"].upper(), case["transb"].upper()
        m, n, k = case["m"], case["n"], case["k"]
        nra, nca = (m, k) if ta == "N" else (k, m)
        nrb, ncb = (k, n) if tb == "N" else (n, k)
        a = mk(nra, nca, case["lda"], (arr["A_hi"], arr["A_lo"]))
        b = mk(nrb, ncb, case["ldb"], (arr["B_hi"], arr["B_lo"]))
        c = mk(m, n, case["ldc"], (arr["C_hi"], arr["C_lo"]))
        with np.errstate(all="ignore"):
            Rgemm(case["transa"], case["transb"], m, n, k, _Scalar(case["alpha_v"]),
                  a, case["lda"], b, case["ldb"],
                  _Scalar(case["beta_v"]), c, case["ldc"], mode=mode)
    else:
        n, k = case["n"], case["k"]
        nra, nca = (n, k) if case["trans"].upper() == "N" else (k, n)
        a = mk(nra, nca, case["lda"], (arr["A_hi"], arr["A_lo"]))
        c = mk(n, n, case["ldc"], (arr["C_hi"], arr["C_lo"]))
        with np.errstate(all="ignore"):
            Rsyrk(case["uplo"], case["trans"], n, k, _Scalar(case["alpha_v"]), a, case["lda"],
                  _Scalar(case["beta_v"]), c, case["ldc"], mode=mode)
    if on_device:
        return c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    return c.store[0], c.store[1]


def _run_case_f64(case, arr, on_device):
    mk = dev64 if on_device else host64
    al, be = case["alpha_v"][0], case["beta_v"][0]
    if case["routine"] == "Rgemm":
        ta, tb = case["transa"].upper(), case["transb"].upper()
        m, n, k = case["m"], case["n"], case["k"]
        nra, nca = (m, k) if ta == "N" else (k, m)
        nrb, ncb = (k, n) if tb == "N" else (n, k)
        a = mk(nra, nca, case["lda"], arr["A_hi"])
        b = mk(nrb, ncb, case["ldb"], arr["B_hi"])
        c = mk(m, n, case["ldc"], arr["C_hi"])
        with np.errstate(all="ignore"):
            Rgemm(case["transa"], case["transb"], m, n, k, al, a, case["lda"], b, case["ldb"],
                  be, c, case["ldc"])
    else:
        n, k = case["n"], case["k"]
        nra, nca = (n, k) if case["trans"].upper() == "N" else (k, n)
        a = mk(nra, nca, case["lda"], arr["A_hi"])
        c = mk(n, n, case["ldc"], arr["C_hi"])
        with np.errstate(all="ignore"):
            Rsyrk(case["uplo"], case["trans"], n, k, al, a, case["lda"], be, c, case["ldc"])
    h = c.store[0].cpu().numpy() if on_device else c.store[0]
    return h, np.zeros(0)


class _Scalar:
    """A DDouble-like (hi, lo) scalar, as the reference's DDouble."""

    def __init__(self, v):
        self.hi, self.lo = float(v[0]), float(v[1])


@pytest.mark.parametrize("mode", ["exact", "reference"])
@pytest.mark.parametrize("idx", range(len(CASES)))
def test_golden_bitwise(idx, mode):
    case, arr, out_hi, out_lo = CASES[idx]
    got_h, got_l = _run_case(case, arr, mode)
    assert bits_equal(got_h, out_hi), case
    assert bits_equal(got_l, out_lo), case


@pytest.mark.parametrize("idx", range(len(CASES)))
def test_golden_fast_within_bound(idx):
    case, arr, out_hi, out_lo = CASES[idx]
    got_h, got_l = _run_case(case, arr, "fast")
    if case.get("precision") == "f64":     # binary64: bit-exact in every mode
        assert bits_equal(got_h, out_hi), case
        return
    routed = set()
    if case.get("special") in ("inf_a", "huge", "tiny"):
        # the elements whose op(A) row / op(B) column holds a word outside the
        # safe window are routed to the reference-semantics kernel, so even
        # fast mode reproduces the reference bit for bit there; the others
        # stay on the fast path (nan_c_beta0 and mixed_scale stay inside the
        # window everywhere)
        routed = routed_elements(case, arr, canon=True)
        assert routed
        ldc = case["ldc"]
        idx = np.array([i + j * ldc for i, j in routed])
        assert bits_equal(got_h[idx], out_hi[idx]) and bits_equal(got_l[idx], out_lo[idx]), case
    # entries outside the written region are untouched
    if case["routine"] == "Rgemm":
        m, n, k, ldc = case["m"], case["n"], case["k"], case["ldc"]
        written = np.zeros(len(out_hi), bool)
        for j in range(n):
            written[j * ldc: j * ldc + m] = True
        ta, tb = case["transa"], case["transb"]
        I, J = list(range(m)), list(range(n))
        vals, scales = exact.exact_entries(ta, tb, k, case["alpha_v"], arr["A_hi"], arr["A_lo"],
                                           case["lda"], arr["B_hi"], arr["B_lo"], case["ldb"],
                                           case["beta_v"], arr["C_hi"], arr["C_lo"], ldc, I, J)
    else:
        n, k, ldc = case["n"], case["k"], case["ldc"]
        up = case["uplo"].upper() == "U"
        written = np.zeros(len(out_hi), bool)
        for j in range(n):
            for i in range(n):
                if (i <= j) if up else (i >= j):
                    written[i + j * ldc] = True
        tr = case["trans"].upper()
        ta, tb = ("N", "T") if tr == "N" else ("T", "N")
        I, J = list(range(n)), list(range(n))
        vals, scales = exact.exact_entries(ta, tb, k, case["alpha_v"], arr["A_hi"], arr["A_lo"],
                                           case["lda"], arr["A_hi"], arr["A_lo"], case["lda"],
                                           case["beta_v"], arr["C_hi"], arr["C_lo"], ldc, I, J)
        # mask the other triangle out of the comparison
        for x in range(n):
            for y in range(n):
                if not ((x <= y) if up else (x >= y)):
                    vals[x][y] = None
    assert bits_equal(got_h[~written], out_hi[~written])
    assert bits_equal(got_l[~written], out_lo[~written])
    worst = 0.0
    for x, i in enumerate(I):
        for y, j in enumerate(J):
            if vals[x][y] is None or (i, j) in routed:
                continue
            r = exact.error_ratios(got_h, got_l, ldc, [i], [j], [[vals[x][y]]], [[scales[x][y]]],
                                   max(k, 1))
            worst = max(worst, r)
    assert worst <= 1.0, (case, worst)


@pytest.mark.parametrize("idx", [i for i, c in enumerate(CASES) if c[0].get("precision") == "f64"][:6])
def test_f64_host_path_bitwise(idx):
    case, arr, out_hi, _ = CASES[idx]
    got, _ = _run_case(case, arr, "exact", on_device=False)
    assert bits_equal(got, out_hi), case


@pytest.mark.parametrize("mode", ["exact", "fast"])
def test_host_path_matches_device_path(mode):
    case, arr, out_hi, out_lo = next(c for c in CASES if c[0]["routine"] == "Rgemm"
                                     and c[0]["m"] > 100)
    dh, dl = _run_case(case, arr, mode, on_device=True)
    hh, hl = _run_case(case, arr, mode, on_device=False)
    assert bits_equal(dh, hh) and bits_equal(dl, hl)


def test_tiled_route_taken_for_in_window_inputs():
    case, arr, _, _ = next(c for c in CASES if c[0]["routine"] == "Rgemm"
                           and c[0]["m"] > 100)
    _run_case(case, arr, "exact")
    assert _lib.last_route() == 0
    _run_case(case, arr, "fast")
    assert _lib.last_route() == 1
    special = next(c for c in CASES if c[0].get("special") == "huge")
    _run_case(special[0], special[1], "fast")
    assert _lib.last_route() == 2


@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("where", ["A", "B"])
@pytest.mark.parametrize("kind", ["hi_zero", "lo_big"])
def test_non_normalised_operands_take_reference_route(mode, where, kind):
    """A hand-made dd with |lo| > 2^-53 |hi| (hi = 0, lo != 0, or lo of the
    order of hi) is outside the fast algorithms' error analysis: the
    elements of its op(A) row / op(B) column are routed to the
    reference-semantics kernel and match mode='reference' bit for bit."""
    m, n, k = 96, 80, 70
    A = [x.copy() for x in random_dd(m, k, m, 31, 1)]
    B = [x.copy() for x in random_dd(k, n, k, 31, 2)]
    C = random_dd(m, n, m, 31, 3)
    X = A if where == "A" else B
    if kind == "hi_zero":
        X[0][5], X[1][5] = 0.0, 1e-3
    else:
        X[1][7] = 0.75 * X[0][7]
    outs = []
    for md in (mode, "reference"):
        a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
        Rgemm("N", "N", m, n, k, _Scalar((1.5, 0.0)), a, m, b, k, _Scalar((0.5, 0.0)), c, m,
              mode=md)
        outs.append((c.store[0].cpu().numpy(), c.store[1].cpu().numpy()))
        if md == mode:
            assert _lib.last_route() == 2
    # the poisoned word sits in op(A) row (idx % m) or op(B) column (idx // k)
    sel = np.zeros((m, n), bool)
    if where == "A":
        sel[(5 if kind == "hi_zero" else 7) % m, :] = True
    else:
        sel[:, (5 if kind == "hi_zero" else 7) // k] = True
    flat = sel.T.reshape(-1)
    assert bits_equal(outs[0][0][flat], outs[1][0][flat])
    assert bits_equal(outs[0][1][flat], outs[1][1][flat])
    assert np.all(np.isfinite(outs[0][0][~flat]))


# ---- larger shapes against the C oracle (bitwise, exact mode) -------------

SHAPES = [(300, 260, 200, 3, 1, 5), (129, 65, 17, 0, 0, 0), (1, 1, 1, 0, 0, 0),
          (257, 3, 33, 1, 1, 1), (5, 200, 300, 2, 0, 3)]


@pytest.mark.parametrize("shape", SHAPES)
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("N", "T"), ("T", "N"), ("T", "T")])
def test_rgemm_exact_vs_oracle(shape, ta, tb):
    m, n, k, pa, pb, pc = shape
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    lda, ldb, ldc = nra + pa, nrb + pb, m + pc
    A = random_dd(nra, nca, lda, 7, 1)
    B = random_dd(nrb, ncb, ldb, 7, 2)
    C = random_dd(m, n, ldc, 7, 3)
    alpha, beta = (1.5, 1.5 * 2 ** -60), (0.5, 2 ** -58)
    ch, cl = C[0].copy(), C[1].copy()
    assert oracle.rgemm(ta, tb, m, n, k, alpha, A[0], A[1], lda, B[0], B[1], ldb, beta,
                        ch, cl, ldc) == 0
    a, b, c = dev(nra, nca, lda, A), dev(nrb, ncb, ldb, B), dev(m, n, ldc, C)
    Rgemm(ta, tb, m, n, k, _Scalar(alpha), a, lda, b, ldb, _Scalar(beta), c, ldc, mode="exact")
    assert _lib.last_route() == 0
    assert bits_equal(c.store[0].cpu().numpy(), ch)
    assert bits_equal(c.store[1].cpu().numpy(), cl)


@pytest.mark.parametrize("uplo", ["U", "L"])
@pytest.mark.parametrize("trans", ["N", "T"])
@pytest.mark.parametrize("n,k", [(300, 150), (130, 7), (64, 64)])
def test_rsyrk_exact_vs_oracle(uplo, trans, n, k):
    nra, nca = (n, k) if trans == "N" else (k, n)
    lda, ldc = nra + 1, n + 2
    A = random_dd(nra, nca, lda, 9, 1)
    C = random_dd(n, n, ldc, 9, 3)
    alpha, beta = (1.5, 0.0), (0.5, 2 ** -58)
    ch, cl = C[0].copy(), C[1].copy()
    assert oracle.rsyrk(uplo, trans, n, k, alpha, A[0], A[1], lda, beta, ch, cl, ldc) == 0
    a, c = dev(nra, nca, lda, A), dev(n, n, ldc, C)
    Rsyrk(uplo, trans, n, k, _Scalar(alpha), a, lda, _Scalar(beta), c, ldc, mode="exact")
    assert bits_equal(c.store[0].cpu().numpy(), ch)
    assert bits_equal(c.store[1].cpu().numpy(), cl)


# ---- fast mode accuracy at depth ------------------------------------------

@pytest.mark.parametrize("m,n,k", [(64, 64, 4096), (32, 48, 65536), (200, 130, 1000)])
def test_fast_mode_error_bound_deep_k(m, n, k):
    A = random_dd(m, k, m, 11, 1)
    B = random_dd(k, n, k, 11, 2)
    C = random_dd(m, n, m, 11, 3)
    alpha, beta = (1.5, 0.0), (0.5, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, _Scalar(alpha), a, m, b, k, _Scalar(beta), c, m, mode="fast")
    assert _lib.last_route() == 1
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    I = list(range(0, m, max(1, m // 8)))[:8]
    J = list(range(0, n, max(1, n // 8)))[:8]
    vals, scales = exact.exact_entries("N", "N", k, alpha, A[0], A[1], m, B[0], B[1], k,
                                       beta, C[0], C[1], m, I, J)
    worst = exact.error_ratios(gh, gl, m, I, J, vals, scales, k)
    assert worst < 0.25, worst   # cert: ~1e-3 of the bound, twosum ~1e-5


# ---- fast modes on adversarial magnitude patterns --------------------------

def _pattern(kind, m, n, k, seed):
    A = [x.copy() for x in random_dd(m, k, m, seed, 1)]
    B = [x.copy() for x in random_dd(k, n, k, seed, 2)]
    g = np.random.default_rng(seed)
    if kind == "disjoint" and k > 1:   # big A entries at l = 0, big B entries at l = 1
        A[0][:m] *= 2.0 ** 40
        A[1][:m] *= 2.0 ** 40
        B[0][1::k] *= 2.0 ** 40
        B[1][1::k] *= 2.0 ** 40
    elif kind == "graded":      # magnitudes decay along k
        scale = 2.0 ** (-np.arange(k) / 4.0)
        A[0] = (A[0].reshape(k, m) * scale[:, None]).reshape(-1)
        A[1] = (A[1].reshape(k, m) * scale[:, None]).reshape(-1)
    elif kind == "rows":        # wildly different row / column scales
        rs = 2.0 ** g.integers(-80, 80, m)
        A[0] = (A[0].reshape(k, m) * rs[None, :]).reshape(-1)
        A[1] = (A[1].reshape(k, m) * rs[None, :]).reshape(-1)
        cs = 2.0 ** g.integers(-80, 80, n)
        B[0] = (B[0].reshape(n, k) * cs[:, None]).reshape(-1)
        B[1] = (B[1].reshape(n, k) * cs[:, None]).reshape(-1)
    elif kind == "cancel":      # B column j = -(B column j-1): heavy cancellation
        B[0] = B[0].reshape(n, k)
        B[1] = B[1].reshape(n, k)
        B[0][1::2] = -B[0][0::2][: n // 2]
        B[1][1::2] = -B[1][0::2][: n // 2]
        A[0][::3] = A[0][::3] * 2.0 ** 30
        A[1][::3] = A[1][::3] * 2.0 ** 30
        B[0] = B[0].reshape(-1)
        B[1] = B[1].reshape(-1)
    return A, B


@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("kind", ["uniform", "disjoint", "graded", "rows", "cancel"])
@pytest.mark.parametrize("k", [1, 2, 3, 17, 300])
def test_fast_modes_bound_on_adversarial_patterns(mode, kind, k):
    m, n = 70, 66
    A, B = _pattern(kind, m, n, k, 5 + k)
    C = random_dd(m, n, m, 5, 3)
    alpha, beta = (1.5, 0.0), (0.5, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, _Scalar(alpha), a, m, b, k, _Scalar(beta), c, m, mode=mode)
    # fast: elements whose row / column exponent spreads are too wide for the
    # certified bound take the TwoSum fallback (route 5)
    assert _lib.last_route() in ((1, 5) if mode == "fast" else (3,))
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    I, J = list(range(0, m, 7)), list(range(0, n, 5))
    vals, scales = exact.exact_entries("N", "N", k, alpha, A[0], A[1], m, B[0], B[1], k,
                                       beta, C[0], C[1], m, I, J)
    worst = exact.error_ratios(gh, gl, m, I, J, vals, scales, k)
    assert worst <= 1.0, worst


# ---- split-K (fast modes fill the GPU when the tile grid is small) ----------

@pytest.mark.parametrize("mode", ["fast", "twosum"])
@pytest.mark.parametrize("shape", [(200, 130, 4096), (64, 64, 20000), (300, 70, 1500)])
def test_fast_split_k_within_bound(mode, shape):
    m, n, k = shape
    A = random_dd(m, k, m, 21, 1)
    B = random_dd(k, n, k, 21, 2)
    C = random_dd(m, n, m, 21, 3)
    alpha, beta = (1.5, 2 ** -60), (0.5, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, _Scalar(alpha), a, m, b, k, _Scalar(beta), c, m, mode=mode)
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    I, J = list(range(0, m, max(1, m // 6))), list(range(0, n, max(1, n // 6)))
    vals, scales = exact.exact_entries("N", "N", k, alpha, A[0], A[1], m, B[0], B[1], k,
                                       beta, C[0], C[1], m, I, J)
    assert exact.error_ratios(gh, gl, m, I, J, vals, scales, k) < 0.25


@pytest.mark.parametrize("uplo", ["U", "L"])
def test_fast_split_k_rsyrk_triangle_only(uplo):
    n, k = 150, 6000
    A = random_dd(n, k, n, 22, 1)
    C = random_dd(n, n, n, 22, 3)
    a, c = dev(n, k, n, A), dev(n, n, n, C)
    Rsyrk(uplo, "N", n, k, 1.5, a, n, 0.5, c, n, mode="fast")
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    iu = np.array([[(i <= j) if uplo == "U" else (i >= j) for j in range(n)] for i in range(n)])
    mask = iu.T.reshape(-1)          # column-major flat index i + j*n
    assert bits_equal(gh[~mask], C[0][~mask]) and bits_equal(gl[~mask], C[1][~mask])
    I = [0, 37, 74, 149]
    vals, scales = exact.exact_entries("N", "T", k, (1.5, 0.0), A[0], A[1], n, A[0], A[1], n,
                                       (0.5, 0.0), C[0], C[1], n, I, I)
    for x, i in enumerate(I):
        for y, j in enumerate(I):
            if (i <= j) if uplo == "U" else (i >= j):
                assert exact.error_ratios(gh, gl, n, [i], [j], [[vals[x][y]]], [[scales[x][y]]], k) < 0.25


def test_nccl_path_single_rank_selftest():
    """The NCCL code path of parallel.py (broadcast, P2P slabs, gather) on one
    rank, bit-exact against the single-GPU routines (scripts/dist_selftest.py)."""
    import subprocess
    import sys
    repo = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(repo, "scripts", "dist_selftest.py")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout + out.stderr[-2000:]
    assert "MISMATCH" not in out.stdout and out.stdout.count("OK") == 5


# ---- Cgemm ('cdd', 'c64') against the reference's outputs -------------------

def _cmat(prec, rows, cols, ld, arr, name, on_device=True):
    import torch
    from paper_2109_13406_b200.matrix import HostMatrix as HM
    if prec == "cdd":
        planes = [np.ascontiguousarray(arr[f"{name}_{p}"]) for p in ("rh", "rl", "ih", "il")]
    else:
        planes = [np.ascontiguousarray(arr[f"{name}_z"])]
    if on_device:
        return DeviceMatrix(rows, cols, prec, ld, store=tuple(torch.from_numpy(p.copy()).cuda()
                                                            for p in planes))
    h = HM(0, 0, prec)
    h.m, h.n, h.ld = rows, cols, ld
    h.store = tuple(p.copy() for p in planes)
    return h


def _run_cgemm(case, arr, mode, on_device=True):
    from paper_2109_13406_b200 import Cgemm
    prec = case["precision"]
    ta, tb = case["transa"].upper(), case["transb"].upper()
    m, n, k = case["m"], case["n"], case["k"]
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    a = _cmat(prec, nra, nca, case["lda"], arr, "A", on_device)
    b = _cmat(prec, nrb, ncb, case["ldb"], arr, "B", on_device)
    c = _cmat(prec, m, n, case["ldc"], arr, "C", on_device)
    al = complex(*case["alpha_v"]) if case["alpha"] != "zr" else case["alpha_v"][0]
    be = complex(*case["beta_v"])
    with np.errstate(all="ignore"):
        Cgemm(case["transa"], case["transb"], m, n, k, al, a, case["lda"], b, case["ldb"], be,
              c, case["ldc"], mode=mode)
    if on_device:
        return tuple(p.cpu().numpy() for p in c.store)
    return c.store


def _bits_equal_c(a, b):
    a, b = np.asarray(a), np.asarray(b)
    if a.dtype.kind == "c":
        return bits_equal(a.real.copy(), b.real.copy()) and bits_equal(a.imag.copy(), b.imag.copy())
    return bits_equal(a, b)


@pytest.mark.parametrize("idx", range(len(CCASES)))
def test_cgemm_golden_bitwise_exact(idx):
    case, arr, outs, _ = CCASES[idx]
    got = _run_cgemm(case, arr, "exact")
    for g_, o_ in zip(got, outs):
        assert _bits_equal_c(g_, o_), case


@pytest.mark.parametrize("idx", [i for i, c in enumerate(CCASES) if c[0]["precision"] == "cdd"])
def test_cgemm_cdd_fast_close_to_reference(idx):
    case, arr, outs, _ = CCASES[idx]
    got = _run_cgemm(case, arr, "fast")
    k = max(case["k"], 1)
    ref_re = outs[0] + outs[1]
    ref_im = outs[2] + outs[3]
    got_re, got_im = got[0] + got[1], got[2] + got[3]
    with np.errstate(all="ignore"):
        scale = np.maximum(1.0, np.abs(ref_re) + np.abs(ref_im))
        ok = (np.abs(got_re - ref_re) <= 1e-28 * k * scale) | (np.isnan(ref_re) & np.isnan(got_re))
        ok &= (np.abs(got_im - ref_im) <= 1e-28 * k * scale) | (np.isnan(ref_im) & np.isnan(got_im))
    assert ok.all(), case


@pytest.mark.parametrize("idx", [0, 9, 20])
def test_cgemm_host_path_bitwise(idx):
    case, arr, outs, _ = CCASES[idx]
    got = _run_cgemm(case, arr, "exact", on_device=False)
    for g_, o_ in zip(got, outs):
        assert _bits_equal_c(g_, o_), case


# ---- out-of-bounds guard: NaN sentinels around and inside the operands ------

def _guarded(planes, rows, cols, ld, guard=4096):
    """Device planes embedded in NaN-filled buffers (NaN also in the ld padding)."""
    import torch
    out, views = [], []
    for p in planes:
        buf = np.full(len(p) + 2 * guard, np.nan)
        body = p.copy()
        for j in range(cols):
            body[j * ld + rows:(j + 1) * ld] = np.nan        # padding rows of each column
        buf[guard:guard + len(p)] = body
        t = torch.from_numpy(buf).cuda()
        out.append(t)
        views.append(t[guard:guard + len(p)])
    return out, tuple(views)


@pytest.mark.parametrize("mode", ["exact", "fast", "twosum"])
@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T"), ("T", "T")])
def test_kernels_never_touch_outside_the_operands(mode, ta, tb):
    m, n, k, pad = 70, 45, 300, 2           # even ld: the TMA kernel takes NN
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra + pad, 31, 1)
    B = random_dd(nrb, ncb, nrb + pad, 31, 2)
    C = random_dd(m, n, m + pad, 31, 3)
    # reference run on clean operands
    a0, b0 = dev(nra, nca, nra + pad, A), dev(nrb, ncb, nrb + pad, B)
    c0 = dev(m, n, m + pad, C)
    Rgemm(ta, tb, m, n, k, 1.5, a0, nra + pad, b0, nrb + pad, 0.5, c0, m + pad, mode=mode)
    ref = [p.cpu().numpy() for p in c0.store]
    # guarded run: NaN everywhere the kernel must not read
    abufs, av = _guarded(A, nra, nca, nra + pad)
    bbufs, bv = _guarded(B, nrb, ncb, nrb + pad)
    cbufs, cv = _guarded(C, m, n, m + pad)
    a = DeviceMatrix(nra, nca, "dd", nra + pad, store=av)
    b = DeviceMatrix(nrb, ncb, "dd", nrb + pad, store=bv)
    c = DeviceMatrix(m, n, "dd", m + pad, store=cv)
    Rgemm(ta, tb, m, n, k, 1.5, a, nra + pad, b, nrb + pad, 0.5, c, m + pad, mode=mode)
    got = [p.cpu().numpy() for p in c.store]
    for g_, r_ in zip(got, ref):
        for j in range(n):
            col = slice(j * (m + pad), j * (m + pad) + m)
            assert bits_equal(g_[col], r_[col])
            assert np.all(np.isnan(g_[j * (m + pad) + m:(j + 1) * (m + pad)]))  # C padding untouched
    for buf in cbufs:
        h = buf.cpu().numpy()
        assert np.all(np.isnan(h[:4096])) and np.all(np.isnan(h[-4096:]))


def test_concurrent_calls_on_two_streams_from_two_threads():
    """The C ABI is reentrant: two host threads, two streams, fast mode (cuBLAS
    bound GEMM per thread) and exact mode at once, results as if sequential."""
    import threading
    import torch
    m, n, k = 200, 150, 700
    A, B, C = random_dd(m, k, m, 41, 1), random_dd(k, n, k, 41, 2), random_dd(m, n, m, 41, 3)
    refs = {}
    for mode in ("fast", "exact"):
        c = dev(m, n, m, C)
        Rgemm("N", "N", m, n, k, 1.5, dev(m, k, m, A), m, dev(k, n, k, B), k, 0.5, c, m, mode=mode)
        refs[mode] = [p.cpu().numpy() for p in c.store]
    out, errs = {}, []

    def worker(mode):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for _ in range(5):
                    c = dev(m, n, m, C)
                    Rgemm("N", "N", m, n, k, 1.5, dev(m, k, m, A), m, dev(k, n, k, B), k, 0.5,
                          c, m, mode=mode)
                s.synchronize()
                out[mode] = [p.cpu().numpy() for p in c.store]
        except Exception as e:   # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker, args=(md,)) for md in ("fast", "exact")]
    for t in ts:
        t.start()
    for t in ts:
        t.join()
    assert not errs, errs
    for mode in ("fast", "exact"):
        assert all(bits_equal(a, b) for a, b in zip(out[mode], refs[mode])), mode


@pytest.mark.parametrize("ta,tb,beta,k", [("N", "N", 0.5, 7680), ("T", "T", 0.0, 7680),
                                          ("N", "T", 1.0, 7680), ("N", "N", 0.5, 8704)])
def test_host_pipelined_path_matches_device_exact(ta, tb, beta, k):
    """ddb_rgemm_host with pinned buffers and a large problem runs column
    blocks with copies overlapped (capi.cu); exact mode must still be
    bit-identical to the device-resident call."""
    import torch
    m, n = 640, 2048                            # m n k >= 1e10: the pipelined branch
    # (k >= 8192: block 0 in 8 k panels)
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A, B, C = random_dd(nra, nca, nra, 4, 1), random_dd(nrb, ncb, nrb, 4, 2), random_dd(m, n, m, 4, 3)
    hm = []
    for (r, c, planes) in ((nra, nca, A), (nrb, ncb, B), (m, n, C)):
        h = HostMatrix(r, c, "dd", r, pinned=True)
        h.store[0][:] = planes[0]
        h.store[1][:] = planes[1]
        hm.append(h)
    Rgemm(ta, tb, m, n, k, 1.5, hm[0], nra, hm[1], nrb, beta, hm[2], m, mode="exact")
    c = dev(m, n, m, C)
    Rgemm(ta, tb, m, n, k, 1.5, dev(nra, nca, nra, A), nra, dev(nrb, ncb, nrb, B), nrb, beta, c,
          m, mode="exact")
    torch.cuda.synchronize()
    assert bits_equal(hm[2].store[0], c.store[0].cpu().numpy())
    assert bits_equal(hm[2].store[1], c.store[1].cpu().numpy())


def _mgpu_devices(count):
    import ctypes
    return (ctypes.c_int * count)(*([0] * count))


@pytest.mark.parametrize("ta,tb,beta,mode", [("N", "N", 0.5, "exact"), ("N", "T", 0.0, "exact"),
                                             ("T", "N", 1.5, "exact"), ("T", "T", 0.5, "exact"),
                                             ("N", "N", 0.5, "fast")])
@pytest.mark.parametrize("ndev", [1, 3])
def test_rgemm_mgpu_matches_single_call(ta, tb, beta, mode, ndev):
    """ddb_rgemm_mgpu with the device list [0]*ndev: the column slabs, peer
    copies and gathers of the multi-GPU entry point on one GPU; exact mode
    bitwise equal to ddb_rgemm, fast mode within its bound of it."""
    import torch
    L = _lib.load()
    m, n, k = 150, 333, 97
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A, B, C = random_dd(nra, nca, nra + 1, 6, 1), random_dd(nrb, ncb, nrb + 2, 6, 2), \
        random_dd(m, n, m + 3, 6, 3)
    d = [torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in (*A, *B, *C)]
    ref = [t.clone() for t in d[4:]]
    code = _lib.MODES[mode]
    rc = L.ddb_rgemm(ta.encode(), tb.encode(), m, n, k, 1.5, 0.0, d[0].data_ptr(), d[1].data_ptr(),
                     nra + 1, d[2].data_ptr(), d[3].data_ptr(), nrb + 2, beta, 0.0,
                     ref[0].data_ptr(), ref[1].data_ptr(), m + 3, code, None)
    assert rc == 0
    rc = L.ddb_rgemm_mgpu(ta.encode(), tb.encode(), m, n, k, 1.5, 0.0, d[0].data_ptr(),
                          d[1].data_ptr(), nra + 1, d[2].data_ptr(), d[3].data_ptr(), nrb + 2, beta,
                          0.0, d[4].data_ptr(), d[5].data_ptr(), m + 3, code, ndev,
                          _mgpu_devices(ndev))
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    if mode == "exact":
        assert bits_equal(d[4].cpu().numpy(), ref[0].cpu().numpy())
        assert bits_equal(d[5].cpu().numpy(), ref[1].cpu().numpy())
    else:
        diff = (d[4] - ref[0]) + (d[5] - ref[1])
        assert float(diff.abs().max()) <= 1e-28 * float(ref[0].abs().max())


@pytest.mark.parametrize("up,tr", [("U", "N"), ("L", "N"), ("U", "T"), ("L", "T")])
@pytest.mark.parametrize("ndev", [2, 4])
def test_rsyrk_mgpu_matches_single_call(up, tr, ndev):
    import torch
    L = _lib.load()
    n, k = 300, 41
    nra, nca = (n, k) if tr == "N" else (k, n)
    A, C = random_dd(nra, nca, nra, 7, 1), random_dd(n, n, n + 1, 7, 3)
    d = [torch.from_numpy(np.ascontiguousarray(p)).cuda() for p in (*A, *C)]
    ref = [t.clone() for t in d[2:]]
    rc = L.ddb_rsyrk(up.encode(), tr.encode(), n, k, 1.5, 0.0, d[0].data_ptr(), d[1].data_ptr(),
                     nra, 0.5, 0.0, ref[0].data_ptr(), ref[1].data_ptr(), n + 1, 0, None)
    assert rc == 0
    rc = L.ddb_rsyrk_mgpu(up.encode(), tr.encode(), n, k, 1.5, 0.0, d[0].data_ptr(),
                          d[1].data_ptr(), nra, 0.5, 0.0, d[2].data_ptr(), d[3].data_ptr(), n + 1,
                          0, ndev, _mgpu_devices(ndev))
    assert rc == 0, _lib.last_error()
    torch.cuda.synchronize()
    assert bits_equal(d[2].cpu().numpy(), ref[0].cpu().numpy())
    assert bits_equal(d[3].cpu().numpy(), ref[1].cpu().numpy())


@pytest.mark.parametrize("ta,tb", [("T", "N"), ("T", "T"), ("N", "N")])
def test_host_pipelined_fast_within_bound(ta, tb):
    """The pipelined host path streams the first column block's k in panels
    (fast modes, any transa): still inside the certified bound."""
    m, n, k = 512, 2048, 9728                   # m n k >= 1e10, k >= 4096: k-panels
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A, B, C = random_dd(nra, nca, nra, 8, 1), random_dd(nrb, ncb, nrb, 8, 2), random_dd(m, n, m, 8, 3)
    hm = []
    for (r, c, planes) in ((nra, nca, A), (nrb, ncb, B), (m, n, C)):
        h = HostMatrix(r, c, "dd", r, pinned=True)
        h.store[0][:] = planes[0]
        h.store[1][:] = planes[1]
        hm.append(h)
    alpha, beta = (1.5, 2 ** -60), (0.5, 0.0)
    Rgemm(ta, tb, m, n, k, _Scalar(alpha), hm[0], nra, hm[1], nrb, _Scalar(beta), hm[2], m,
          mode="fast")
    I, J = [0, 97, 255, 511], [0, 5, 300, 1023, 2047]      # J spans the first column block
    vals, scales = exact.exact_entries(ta, tb, k, alpha, A[0], A[1], nra, B[0], B[1], nrb, beta,
                                       C[0], C[1], m, I, J)
    assert exact.error_ratios(hm[2].store[0], hm[2].store[1], m, I, J, vals, scales, k) < 0.25
