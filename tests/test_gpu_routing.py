"""GPU: per-element routing (dd_prescan.cu, internal.h elem_class).

* Fast mode's certified anchor is only tight while an element's row / column
  exponent spreads stay moderate (dd_bound.cu); wider elements must take the
  TwoSum accumulation, so the north star's c*k*2^-104*sum|ab| bound (c = 4)
  holds for EVERY in-window input.  The adversarial inputs of the round-1
  review: A row i = [U(1,2), 2^-s U(1,2), ...], B column j = [2^-s U(1,2),
  U(1,2), 2^-s U(1,2), ...], normalised dd words with non-zero tails.
* Unsafe words (NaN, huge, tiny) reroute only their op(A) row / op(B) column
  to the reference-semantics kernel; everything else keeps its fast kernel.
"""

import os
import time

import numpy as np
import pytest

from oracle import exact
from paper_2109_13406_b200 import DeviceMatrix, Rgemm, Rsyrk, _lib
from paper_2109_13406_b200.synth import random_dd, two_sum

pytestmark = pytest.mark.gpu

C_BOUND = 4.0


@pytest.fixture(autouse=True)
def debug_sync(monkeypatch):
    monkeypatch.setenv("DDB_DEBUG_SYNC", "1")
    yield


def dev(m, n, ld, planes):
    import torch
    return DeviceMatrix(m, n, "dd", ld,
                        store=tuple(torch.from_numpy(np.ascontiguousarray(p)).cuda()
                                    for p in planes))


def bits_equal(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return bool(np.all((a.view(np.uint64) == b.view(np.uint64)) | (np.isnan(a) & np.isnan(b))))


def _dd_from(hi, g):
    lo = hi * g.uniform(-1.0, 1.0, hi.shape) * 2.0 ** -53
    return two_sum(hi, lo)


def spread_operands(m, n, k, s, seed, wide_rows=None):
    """A (m x k) rows [U(1,2), 2^-s U(1,2), ...]; B (k x n) columns
    [2^-s U, U(1,2), 2^-s U, ...].  wide_rows: only these rows of A / columns
    of B get the spread (the rest are plain U(1,2) entries)."""
    g = np.random.default_rng(seed)
    A = g.uniform(1.0, 2.0, (m, k))
    B = g.uniform(1.0, 2.0, (k, n))
    rows = range(m) if wide_rows is None else wide_rows
    cols = range(n) if wide_rows is None else [j for j in wide_rows if j < n]
    for i in rows:
        A[i, 1:] *= 2.0 ** -s
    for j in cols:
        B[:, j] *= 2.0 ** -s
        B[1 % k, j] *= 2.0 ** s
    A = A * np.where(g.random((m, k)) < 0.5, -1.0, 1.0)
    ah, al = _dd_from(A.reshape(-1, order="F"), g)
    bh, bl = _dd_from(B.reshape(-1, order="F"), g)
    return (ah, al), (bh, bl)


def _ratio(c, m, n, k, A, B, alpha, beta, C0, I, J, ta="N", tb="N", lda=None, ldb=None):
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    lda = lda or (m if ta == "N" else k)
    ldb = ldb or (k if tb == "N" else n)
    vals, scales = exact.exact_entries(ta, tb, k, alpha, A[0], A[1], lda, B[0], B[1], ldb,
                                       beta, C0[0], C0[1], m, I, J)
    return exact.error_ratios(gh, gl, m, I, J, vals, scales, k, c=C_BOUND)


@pytest.mark.parametrize("mode,split", [("fast", None), ("fast", "2"), ("fast", "0"),
                                        ("twosum", None)])
@pytest.mark.parametrize("k", [2, 6, 300])
@pytest.mark.parametrize("s", [20, 50, 100, 130, 180, 250])
def test_wide_spread_inputs_within_bound(monkeypatch, mode, split, k, s):
    if split is not None:
        monkeypatch.setenv("DDB_SPLIT", split)
    m, n = 96, 72
    A, B = spread_operands(m, n, k, s, 1000 + s + k)
    C = random_dd(m, n, m, 5, 3)
    alpha, beta = (1.5, 0.0), (0.0, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, alpha[0], a, m, b, k, beta[0], c, m, mode=mode)
    route = _lib.last_route()
    lg = max(0, int(np.ceil(np.log2(k))))
    if mode == "fast":
        # spread sum 2s against the limit 112 - ceil(log2 k)
        assert route == (5 if 2 * s > 112 - lg else 1), route
    else:
        assert route == 3
    I, J = list(range(0, m, 5)), list(range(0, n, 3))
    worst = _ratio(c, m, n, k, A, B, alpha, beta, C, I, J)
    assert worst <= 1.0, worst


@pytest.mark.parametrize("k", [300, 20000])
def test_mixed_wide_and_fast_elements(monkeypatch, k):
    """Some rows / columns wide, the rest not: the certified kernel and the
    TwoSum fallback write disjoint element sets (with split-K at k = 20000);
    every sampled element is inside the bound and nothing is left unwritten."""
    m, n = 130, 100
    wide = [0, 3, 64, 65, 127, 129]
    A, B = spread_operands(m, n, k, 200, 7 + k, wide_rows=wide)
    C = random_dd(m, n, m, 9, 3)
    sentinel = (np.full(m * n, np.nan), np.full(m * n, np.nan))
    alpha, beta = (1.5, 0.0), (0.0, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, sentinel)
    Rgemm("N", "N", m, n, k, alpha[0], a, m, b, k, beta[0], c, m, mode="fast")
    assert _lib.last_route() == 5
    gh = c.store[0].cpu().numpy()
    assert np.all(np.isfinite(gh)), "an element was skipped by both kernels"
    I = sorted(set(wide + list(range(1, m, 11))))
    J = sorted(set([j for j in wide if j < n] + list(range(2, n, 13))))
    worst = _ratio(c, m, n, k, A, B, alpha, beta, sentinel, I, J)
    assert worst <= 1.0, worst


@pytest.mark.parametrize("uplo", ["U", "L"])
@pytest.mark.parametrize("trans", ["N", "T"])
def test_rsyrk_wide_rows_within_bound(uplo, trans):
    n, k = 120, 40
    g = np.random.default_rng(3)
    X = g.uniform(1.0, 2.0, (n, k))
    X[::7, 1:] *= 2.0 ** -150          # op(A) rows with a 2^150 spread
    if trans == "T":
        X = X.T.copy()
    rows, cols = X.shape
    ah, al = _dd_from(X.reshape(-1, order="F"), g)
    C = random_dd(n, n, n, 4, 3)
    a, c = dev(rows, cols, rows, (ah, al)), dev(n, n, n, C)
    Rsyrk(uplo, trans, n, k, 1.5, a, rows, 0.5, c, n, mode="fast")
    assert _lib.last_route() == 5
    # Rsyrk N == Rgemm NT with B = A; T == TN with B = A (same entries)
    tb = "T" if trans == "N" else "N"
    ta = trans
    I = list(range(0, n, 7))
    J = list(range(0, n, 5))
    gh, gl = c.store[0].cpu().numpy(), c.store[1].cpu().numpy()
    vals, scales = exact.exact_entries(ta, tb, k, (1.5, 0.0), ah, al, rows, ah, al, rows,
                                       (0.5, 0.0), C[0], C[1], n, I, J)
    for x, i in enumerate(I):
        for y, j in enumerate(J):
            inside = i <= j if uplo == "U" else i >= j
            if inside:
                r = exact.error_ratios(gh, gl, n, [i], [j], [[vals[x][y]]], [[scales[x][y]]], k)
                assert r <= 1.0, (i, j, r)
            else:   # the other triangle is untouched
                assert gh[i + j * n] == C[0][i + j * n] and gl[i + j * n] == C[1][i + j * n]


def test_cert_depth_cap_routes_deep_calls_to_twosum():
    """k above 2^16: the certified bound's accumulation factor is no longer
    tight enough, the call takes the TwoSum MAC (route 3) and stays inside
    the bound."""
    m, n, k = 4, 4, (1 << 16) + 40
    A = random_dd(m, k, m, 11, 1)
    B = random_dd(k, n, k, 11, 2)
    C = random_dd(m, n, m, 11, 3)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, 1.5, a, m, b, k, 0.5, c, m, mode="fast")
    assert _lib.last_route() == 3
    worst = _ratio(c, m, n, k, A, B, (1.5, 0.0), (0.5, 0.0), C, [0, 3], [0, 2, 3])
    assert worst <= 1.0, worst


# ---- unsafe words: per-element reference routing ---------------------------

def _poison(planes, idx, value):
    h, l = planes[0].copy(), planes[1].copy()
    h[idx] = value
    l[idx] = 0.0
    return h, l


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "N"), ("N", "T")])
@pytest.mark.parametrize("value", [np.nan, np.inf, 2.0 ** 400, 2.0 ** -400])
def test_unsafe_words_exact_mode_bitwise_equals_reference(ta, tb, value):
    """Exact mode with one unsafe word in op(A) and one in op(B): the routed
    rows / columns come from the reference kernel, the rest from the exact
    tiled kernel, and the whole result is bit-identical to mode='reference'."""
    m, n, k = 200, 150, 90
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra, 21, 1)
    B = random_dd(nrb, ncb, nrb, 21, 2)
    C = random_dd(m, n, m, 21, 3)
    i0, l0, l1, j1 = 17, 40, 3, 77
    A = _poison(A, (i0 + l0 * nra) if ta == "N" else (l0 + i0 * nra), value)
    B = _poison(B, (l1 + j1 * nrb) if tb == "N" else (j1 + l1 * nrb), value)
    outs = []
    for md in ("exact", "reference"):
        a, b, c = dev(nra, nca, nra, A), dev(nrb, ncb, nrb, B), dev(m, n, m, C)
        Rgemm(ta, tb, m, n, k, 1.5, a, nra, b, nrb, 0.5, c, m, mode=md)
        if md == "exact":
            assert _lib.last_route() == 2
        outs.append((c.store[0].cpu().numpy(), c.store[1].cpu().numpy()))
    assert bits_equal(outs[0][0], outs[1][0]) and bits_equal(outs[0][1], outs[1][1])


@pytest.mark.parametrize("mode", ["fast", "twosum"])
def test_unsafe_words_fast_modes_route_only_their_rows_and_columns(mode):
    m, n, k = 256, 192, 1500
    A = random_dd(m, k, m, 23, 1)
    B = random_dd(k, n, k, 23, 2)
    C = random_dd(m, n, m, 23, 3)
    i0, j1 = 101, 33
    A = _poison(A, i0 + 700 * m, np.nan)
    B = _poison(B, 5 + j1 * k, 2.0 ** 500)
    outs = []
    for md in (mode, "reference"):
        a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
        Rgemm("N", "N", m, n, k, 1.5, a, m, b, k, 0.5, c, m, mode=md)
        outs.append((c.store[0].cpu().numpy().reshape(n, m).T,
                     c.store[1].cpu().numpy().reshape(n, m).T))
    (fh, fl), (rh, rl) = outs
    routed = np.zeros((m, n), bool)
    routed[i0, :] = True
    routed[:, j1] = True
    assert bits_equal(fh[routed], rh[routed]) and bits_equal(fl[routed], rl[routed])
    assert np.all(np.isfinite(fh[~routed]))
    # the other elements are the fast kernel's, inside the bound
    I, J = [0, 50, 100, 102, 255], [0, 32, 34, 191]
    c_fast = dev(m, n, m, (fh.T.reshape(-1).copy(), fl.T.reshape(-1).copy()))
    worst = _ratio(c_fast, m, n, k, A, B, (1.5, 0.0), (0.5, 0.0), C, I, J)
    assert worst <= 1.0, worst


def test_one_nan_in_a_large_call_costs_little():
    """One NaN in an 8192^3 fast call: only its row of C goes to the
    reference kernel (bitwise equal to mode='reference' there); the call
    stays within 1.2x of the clean call's time."""
    import torch
    n = 8192
    g = torch.Generator(device="cuda").manual_seed(5)
    planes = []
    for _ in range(3):
        h = torch.rand(n * n, device="cuda", dtype=torch.float64, generator=g) * 2 - 1
        planes.append((h, h * 2.0 ** -60))
    a, b, c = (DeviceMatrix(n, n, "dd", n, store=p) for p in planes)
    c_clean = [x.clone() for x in planes[2]]

    def timed(mat_a):
        times = []
        for _ in range(3):
            cc = DeviceMatrix(n, n, "dd", n, store=tuple(x.clone() for x in c_clean))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Rgemm("N", "N", n, n, n, 1.5, mat_a, n, b, n, 0.5, cc, n, mode="fast")
            torch.cuda.synchronize()
            times.append(time.perf_counter() - t0)
        return min(times), cc

    t_clean, _ = timed(a)
    ah = planes[0][0].clone()
    ah[4321 + 17 * n] = float("nan")
    a_bad = DeviceMatrix(n, n, "dd", n, store=(ah, planes[0][1]))
    t_bad, cc = timed(a_bad)
    assert t_bad <= 1.2 * t_clean, (t_bad, t_clean)
    # the routed row equals the reference semantics on that row alone
    row_a = DeviceMatrix(1, n, "dd", 1, store=(ah[4321::n].clone(), planes[0][1][4321::n].clone()))
    ref_c = DeviceMatrix(1, n, "dd", 1, store=(c_clean[0][4321::n].clone(),
                                                c_clean[1][4321::n].clone()))
    Rgemm("N", "N", 1, n, n, 1.5, row_a, 1, b, n, 0.5, ref_c, 1, mode="reference")
    assert bits_equal(cc.store[0][4321::n].cpu().numpy(), ref_c.store[0].cpu().numpy())
    assert bits_equal(cc.store[1][4321::n].cpu().numpy(), ref_c.store[1].cpu().numpy())
    assert torch.isfinite(cc.store[0][4322::n]).all()


@pytest.mark.parametrize("k,s", [(32768, 48), (32768, 49), (65536, 48), (65536, 49)])
def test_spread_at_the_limit_deep_k(monkeypatch, k, s):
    """Right at the wide limit (2s = 112 - ceil(log2 k) stays on the certified
    path, 2s + 2 takes the fallback) and at the deepest certified k, where the
    accumulation factor (1 + k 2^-21) and the floor k 2^-120 are largest: the
    split kernel must still be inside the c = 4 bound."""
    monkeypatch.setenv("DDB_SPLIT", "2")
    m, n = 24, 20
    A, B = spread_operands(m, n, k, s, 77 + s)
    C = random_dd(m, n, m, 5, 3)
    alpha, beta = (1.5, 0.0), (0.5, 0.0)
    a, b, c = dev(m, k, m, A), dev(k, n, k, B), dev(m, n, m, C)
    Rgemm("N", "N", m, n, k, alpha[0], a, m, b, k, beta[0], c, m, mode="fast")
    lim = 112 - int(np.ceil(np.log2(k)))
    assert _lib.last_route() == (5 if 2 * s > lim else 1)
    worst = _ratio(c, m, n, k, A, B, alpha, beta, C, [0, 7, 23], [0, 5, 19])
    assert worst <= 1.0, worst
