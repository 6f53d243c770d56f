"""Multi-rank host logic on CPU: world_size 2 over gloo.  The per-slab compute
is the bit-exact oracle (test infrastructure), so the test checks that the
column / triangle decomposition, broadcasts, scatters and gathers reproduce
the single-process result bit for bit -- the GPU analogue of the reference's
thread-count invariance (test_acceptance.py:431-468)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import oracle
from paper_2109_13406_b200 import parallel
from paper_2109_13406_b200.matrix import DeviceMatrix, to_dd
from paper_2109_13406_b200.synth import random_dd


def _np(t):
    return t.numpy()


def oracle_gemm(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, mode=None):
    """compute callable: the oracle on CPU-tensor views (shares memory)."""
    ch, cl = _np(c.store[0]), _np(c.store[1])
    ah, al = np.ascontiguousarray(_np(a.store[0])), np.ascontiguousarray(_np(a.store[1]))
    bh, bl = np.ascontiguousarray(_np(b.store[0])), np.ascontiguousarray(_np(b.store[1]))
    rc = oracle.rgemm(ta, tb, m, n, k, to_dd(alpha), ah, al, lda, bh, bl, ldb, to_dd(beta),
                      ch, cl, ldc, threads=1)
    assert rc == 0


def oracle_syrk(up, tr, n, k, alpha, a, lda, beta, c, ldc, mode=None):
    ch, cl = _np(c.store[0]), _np(c.store[1])
    ah, al = np.ascontiguousarray(_np(a.store[0])), np.ascontiguousarray(_np(a.store[1]))
    rc = oracle.rsyrk(up, tr, n, k, to_dd(alpha), ah, al, lda, to_dd(beta), ch, cl, ldc, threads=1)
    assert rc == 0


def oracle_gemm_np(ta, tb, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc, mode=None):
    """compute callable on host (numpy) matrices, writing C in place."""
    rc = oracle.rgemm(ta, tb, m, n, k, to_dd(alpha), np.ascontiguousarray(a.store[0]),
                      np.ascontiguousarray(a.store[1]), lda, np.ascontiguousarray(b.store[0]),
                      np.ascontiguousarray(b.store[1]), ldb, to_dd(beta), c.store[0], c.store[1],
                      ldc, threads=1)
    assert rc == 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _cpu_mat(rows, cols, seed, tag, pad=0):
    ld = max(1, rows) + pad
    hi, lo = random_dd(rows, cols, ld, seed, tag)
    return DeviceMatrix(rows, cols, "dd", ld,
                        store=(torch.from_numpy(hi.copy()), torch.from_numpy(lo.copy())))


def _worker(rank, world, port, case, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        if case[0] in ("gemm", "gemm_pad"):
            pad = 3 if case[0] == "gemm_pad" else 0
            _, ta, tb, m, n, k, beta, kchunks, mode = (case + (None, None))[:9]
            nra, nca = (m, k) if ta == "N" else (k, m)
            nrb, ncb = (k, n) if tb == "N" else (n, k)
            if rank == 0:
                A, B, C = (_cpu_mat(nra, nca, 3, 1, pad), _cpu_mat(nrb, ncb, 3, 2, pad),
                           _cpu_mat(m, n, 3, 3, pad))
            else:
                A = B = C = None
            plan = parallel.RgemmPlan(m, n, k, world, rank, torch.device("cpu"))
            parallel.rgemm_columns(plan, ta, tb, 1.5, A, B, beta, C, compute=oracle_gemm,
                                   kchunks=kchunks, mode=mode)
            if rank == 0:
                q.put((C.store[0].numpy().copy(), C.store[1].numpy().copy()))
        elif case[0] == "shared":
            from paper_2109_13406_b200.matrix import SharedHostMatrix
            _, ta, tb, m, n, k, pad = case
            nra, nca = (m, k) if ta == "N" else (k, m)
            nrb, ncb = (k, n) if tb == "N" else (n, k)
            dims = ((nra, nca, 1), (nrb, ncb, 2), (m, n, 3))
            names = [None, None, None]
            mats = []
            if rank == 0:
                for rows, cols, tag in dims:
                    sm = SharedHostMatrix(rows, cols, "dd", rows + pad, create=True)
                    hi, lo = random_dd(rows, cols, rows + pad, 6, tag)
                    sm.store[0][:] = hi
                    sm.store[1][:] = lo
                    mats.append(sm)
                names = [x.name for x in mats]
            dist.broadcast_object_list(names, src=0)
            if rank != 0:
                mats = [SharedHostMatrix(rows, cols, "dd", rows + pad, name=nm)
                        for (rows, cols, _), nm in zip(dims, names)]
            a, b, c = mats
            parallel.rgemm_host_shared(ta, tb, m, n, k, 1.5, a, b, 0.5, c, world, rank,
                                       compute=oracle_gemm_np)
            if rank == 0:
                q.put((np.array(c.store[0]), np.array(c.store[1])))
            dist.barrier()
            for x in mats:
                x.close()
        elif case[0] == "host":
            from paper_2109_13406_b200 import HostMatrix
            _, m, n, k = case
            hm = None
            if rank == 0:
                hm = []
                for rows, cols, tag in ((m, k, 1), (k, n, 2), (m, n, 3)):
                    h = HostMatrix(rows, cols, "dd", rows)
                    hi, lo = random_dd(rows, cols, rows, 5, tag)
                    h.store[0][:] = hi
                    h.store[1][:] = lo
                    hm.append(h)
            a, b, c = hm if hm else (None,) * 3
            # the bench's e2e call (bench.py _e2e), argument order as Rgemm's
            parallel.rgemm_host_columns("N", "N", m, n, k, 1.5, a, b, 0.5, c, world, rank,
                                        torch.device("cpu"), compute=oracle_gemm)
            if rank == 0:
                q.put((np.array(c.store[0]), np.array(c.store[1])))
        else:
            _, up, tr, n, k = case[:5]
            pad = case[5] if len(case) > 5 else 0
            nra, nca = (n, k) if tr == "N" else (k, n)
            if rank == 0:
                A, C = _cpu_mat(nra, nca, 4, 1, pad), _cpu_mat(n, n, 4, 3, pad)
            else:
                A = C = None
            parallel.rsyrk_columns(n, k, world, rank, torch.device("cpu"), up, tr, 1.5, A, 0.5, C,
                                   compute_gemm=oracle_gemm, compute_syrk=oracle_syrk)
            if rank == 0:
                q.put((C.store[0].numpy().copy(), C.store[1].numpy().copy()))
    finally:
        dist.destroy_process_group()


def _run(case, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


@pytest.mark.parametrize("ta,tb,beta", [("N", "N", 0.5), ("N", "T", 0.0), ("T", "N", 1.0),
                                        ("T", "T", 0.5)])
def test_rgemm_columns_bitwise_equal_single_process(ta, tb, beta):
    m, n, k = 70, 150, 33
    got = _run(("gemm", ta, tb, m, n, k, beta))
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra, 3, 1)
    B = random_dd(nrb, ncb, nrb, 3, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m, 3, 3))
    oracle.rgemm(ta, tb, m, n, k, (1.5, 0.0), A[0], A[1], nra, B[0], B[1], nrb, to_dd(beta),
                 ch, cl, m)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


def test_rgemm_host_columns_bitwise_equal_single_process():
    """The end-to-end multi-rank entry (host buffers on rank 0) the bench's
    N > 1 e2e leg calls: the single-process result bit for bit."""
    m, n, k = 64, 90, 40
    got = _run(("host", m, n, k))
    A = random_dd(m, k, m, 5, 1)
    B = random_dd(k, n, k, 5, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m, 5, 3))
    oracle.rgemm("N", "N", m, n, k, (1.5, 0.0), A[0], A[1], m, B[0], B[1], k, (0.5, 0.0),
                 ch, cl, m)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


@pytest.mark.parametrize("ta,tb,pad", [("N", "N", 0), ("T", "T", 3), ("N", "T", 1)])
def test_rgemm_host_shared_bitwise_equal_single_process(ta, tb, pad):
    """The per-rank host entry (every rank stages its own slab from shared
    host memory through its own link, no collective on the data path):
    the single-process result bit for bit, padding untouched."""
    m, n, k = 70, 150, 33
    got = _run(("shared", ta, tb, m, n, k, pad))
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra + pad, 6, 1)
    B = random_dd(nrb, ncb, nrb + pad, 6, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m + pad, 6, 3))
    oracle.rgemm(ta, tb, m, n, k, (1.5, 0.0), A[0], A[1], nra + pad, B[0], B[1], nrb + pad,
                 (0.5, 0.0), ch, cl, m + pad)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


@pytest.mark.parametrize("world", [3, 4])
def test_rgemm_and_rsyrk_columns_wider_worlds(world):
    """World sizes 3 and 4 (uneven column / triangle slabs, k-panels): still
    the single-process result bit for bit."""
    m, n, k = 70, 200, 130
    got = _run(("gemm", "N", "T", m, n, k, 0.5, 3, None), world=world)
    A = random_dd(m, k, m, 3, 1)
    B = random_dd(n, k, n, 3, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m, 3, 3))
    oracle.rgemm("N", "T", m, n, k, (1.5, 0.0), A[0], A[1], m, B[0], B[1], n, (0.5, 0.0),
                 ch, cl, m)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)
    nn, kk = 230, 19
    got = _run(("syrk", "L", "N", nn, kk), world=world)
    A = random_dd(nn, kk, nn, 4, 1)
    ch, cl = (x.copy() for x in random_dd(nn, nn, nn, 4, 3))
    oracle.rsyrk("L", "N", nn, kk, (1.5, 0.0), A[0], A[1], nn, (0.5, 0.0), ch, cl, nn)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


@pytest.mark.parametrize("ta,tb,beta,mode", [("N", "N", 0.5, None), ("N", "T", 0.0, None),
                                             ("T", "N", 0.5, "exact"), ("T", "T", 1.0, "exact")])
def test_rgemm_columns_k_panels_bitwise(ta, tb, beta, mode):
    """k streamed in 3 panels (transfers overlapped with compute): still the
    single-process result bit for bit -- transa 'N' by the axpy order,
    transa 'T' in exact mode because the panels are then suppressed."""
    m, n, k = 66, 150, 200
    got = _run(("gemm", ta, tb, m, n, k, beta, 3, mode))
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra, 3, 1)
    B = random_dd(nrb, ncb, nrb, 3, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m, 3, 3))
    oracle.rgemm(ta, tb, m, n, k, (1.5, 0.0), A[0], A[1], nra, B[0], B[1], nrb, to_dd(beta),
                 ch, cl, m)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


@pytest.mark.parametrize("ta,tb", [("N", "N"), ("T", "T")])
def test_rgemm_columns_padded_leading_dimensions(ta, tb):
    """lda / ldb / ldc = rows + 3 on the root: the operands are packed for the
    slabs and C comes back into its padded storage, padding untouched --
    bitwise the single-process result on the same padded layout."""
    m, n, k = 70, 150, 33
    got = _run(("gemm_pad", ta, tb, m, n, k, 0.5))
    nra, nca = (m, k) if ta == "N" else (k, m)
    nrb, ncb = (k, n) if tb == "N" else (n, k)
    A = random_dd(nra, nca, nra + 3, 3, 1)
    B = random_dd(nrb, ncb, nrb + 3, 3, 2)
    ch, cl = (x.copy() for x in random_dd(m, n, m + 3, 3, 3))
    oracle.rgemm(ta, tb, m, n, k, (1.5, 0.0), A[0], A[1], nra + 3, B[0], B[1], nrb + 3,
                 (0.5, 0.0), ch, cl, m + 3)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


@pytest.mark.parametrize("up,tr", [("U", "N"), ("L", "T")])
def test_rsyrk_columns_padded_leading_dimensions(up, tr):
    n, k = 120, 17
    got = _run(("syrk", up, tr, n, k, 2))
    nra, nca = (n, k) if tr == "N" else (k, n)
    A = random_dd(nra, nca, nra + 2, 4, 1)
    ch, cl = (x.copy() for x in random_dd(n, n, n + 2, 4, 3))
    oracle.rsyrk(up, tr, n, k, (1.5, 0.0), A[0], A[1], nra + 2, (0.5, 0.0), ch, cl, n + 2)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


def test_k_chunks_cover():
    for k in (1, 63, 64, 200, 4096, 8193):
        for c in (1, 2, 3, 4, 8):
            ch = parallel._k_chunks(k, c)
            assert ch[0][0] == 0 and ch[-1][1] == k
            assert all(a1 == b0 for (_, a1), (b0, _) in zip(ch, ch[1:]))
            assert all(l1 > l0 for l0, l1 in ch)


@pytest.mark.parametrize("up,tr", [("U", "N"), ("L", "N"), ("U", "T"), ("L", "T")])
def test_rsyrk_triangle_split_bitwise_equal_single_process(up, tr):
    n, k = 200, 17
    got = _run(("syrk", up, tr, n, k))
    nra, nca = (n, k) if tr == "N" else (k, n)
    A = random_dd(nra, nca, nra, 4, 1)
    ch, cl = (x.copy() for x in random_dd(n, n, n, 4, 3))
    oracle.rsyrk(up, tr, n, k, (1.5, 0.0), A[0], A[1], nra, (0.5, 0.0), ch, cl, n)
    assert np.array_equal(got[0], ch) and np.array_equal(got[1], cl)


def test_splits_cover_and_balance():
    for n in (1, 63, 64, 1000, 8192):
        for world in (1, 2, 3, 4, 8):
            b = parallel.column_split(n, world)
            assert b[0][0] == 0 and b[-1][1] == n
            assert all(b[i][1] == b[i + 1][0] for i in range(world - 1))
            t = parallel.triangle_split(n, world, "U")
            assert t[0][0] == 0 and t[-1][1] == n
            assert all(t[i][1] == t[i + 1][0] for i in range(world - 1))
    # triangle areas within a tile-row of each other at n = 8192, P = 8
    t = parallel.triangle_split(8192, 8, "U")
    areas = [(j1 * j1 - j0 * j0) / 2 for j0, j1 in t]
    assert max(areas) / min(areas) < 1.05
    t = parallel.triangle_split(8192, 8, "L")
    areas = [((8192 - j0) ** 2 - (8192 - j1) ** 2) / 2 for j0, j1 in t]
    assert max(areas) / min(areas) < 1.05
