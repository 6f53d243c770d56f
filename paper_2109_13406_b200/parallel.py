"""Multi-GPU dd Rgemm / Rsyrk: one process per GPU, torch.distributed (NCCL).

The partition is the reference's own thread decomposition lifted to GPUs:
``Rgemm_par`` splits C into contiguous column panels and runs the sequential
kernel on each (``/root/reference/pkg/src/mpkit/mpblas/parallel.py:102-157``,
``_chunks`` :37-47).  In exact mode every C(i, j) still sees exactly the same
sequence of dd operations, so the P-GPU result is bitwise equal to the 1-GPU
result (the reference pins this for threads: test_acceptance.py:431-468); the
fast modes keep their error bound under any split but may differ in the last
bits (the bound GEMM and the split-K choice depend on the slab shape).

Data movement (operands start on rank 0, the root, and C ends there):

  Rgemm  broadcast op(A)'s storage (every rank needs all rows of op(A));
         send rank r the columns J_r of op(B) (packed on the root when
         transb = 'T') and, unless beta == 0, the column slab C[:, J_r];
         each rank runs the single-GPU kernel on its slab; the slabs come back.
  Rsyrk  broadcast A; column slabs with triangle-balanced boundaries
         (j_r ~ n*sqrt(r/P) for 'U'), each rank computes its slab of the
         triangle as one Rgemm rectangle + one Rsyrk diagonal block -- the
         same per-element operation sequence as a full Rsyrk (Rsyrk 'N' is NT
         Rgemm with B = A, level23.py:250-258).

The compute callable is injectable so the host logic is testable on CPU with
the gloo backend (tests/test_parallel_gloo.py); the default is the CUDA path.

Set ``DDB_TMA_PERSISTENT=0`` before the first GEMM of a process that overlaps
these broadcasts with compute (bench.py does): the library's default
persistent tile walk holds every SM until a GEMM ends, and NCCL's kernels
need SMs to run beside it.
"""

from __future__ import annotations

import functools
import math

import torch
import torch.distributed as dist

from .matrix import DeviceMatrix, HostMatrix, SharedHostMatrix, to_dd
from .mpblas import Rgemm, Rsyrk

TILE = 64   # column boundaries are multiples of the kernel's BN


def column_split(n, world, tile=TILE):
    """Contiguous column blocks, sizes within one tile of each other."""
    ntiles = -(-n // tile) if n else 0
    out = []
    for r in range(world):
        t0 = ntiles * r // world
        t1 = ntiles * (r + 1) // world
        out.append((min(n, t0 * tile), min(n, t1 * tile)))
    return out


def triangle_split(n, world, uplo="U", tile=16):
    """Column blocks with equal triangle area (U: area of [0, j) ~ j^2)."""
    ntiles = -(-n // tile) if n else 0
    bounds = [0]
    for r in range(1, world):
        frac = math.sqrt(r / world) if uplo == "U" else 1.0 - math.sqrt((world - r) / world)
        t = int(round(frac * ntiles))
        bounds.append(max(bounds[-1], min(ntiles, t)))
    bounds.append(ntiles)
    return [(min(n, bounds[r] * tile), min(n, bounds[r + 1] * tile)) for r in range(world)]


class _Ops:
    """Collective helpers over torch.distributed (NCCL or gloo)."""

    def __init__(self, group=None):
        self.group = group

    def bcast(self, t, src=0):
        dist.broadcast(t, src=src, group=self.group)

    def exchange(self, ops):
        ops = [op for op in ops if op is not None]
        if ops:
            for req in dist.batch_isend_irecv(ops):
                req.wait()

    @staticmethod
    def send(t, peer, group=None):
        return dist.P2POp(dist.isend, t, peer, group=group)

    @staticmethod
    def recv(t, peer, group=None):
        return dist.P2POp(dist.irecv, t, peer, group=group)


class RgemmPlan:
    """Column split and cached receive buffers for one (m, n, k, world) shape."""

    def __init__(self, m, n, k, world, rank, device, tile=TILE):
        self.m, self.n, self.k = m, n, k
        self.world, self.rank, self.device = world, rank, device
        self.blocks = column_split(n, world, tile)
        self._bufs = {}

    def buf(self, name, numel, dtype=torch.float64):
        b = self._bufs.get(name)
        if b is None or b[0].numel() < numel:
            b = (torch.empty(numel, dtype=dtype, device=self.device),
                 torch.empty(numel, dtype=dtype, device=self.device))
            self._bufs[name] = b
        return b[0][:numel], b[1][:numel]


def _slab(store, start, length):
    return store[0][start:start + length], store[1][start:start + length]


def _k_chunks(k, kchunks, tile=TILE):
    """[l0, l1) boundaries of kchunks nearly equal k-panels (tile multiples)."""
    kchunks = max(1, min(kchunks, -(-k // tile) if k else 1))
    out = []
    for c in range(kchunks):
        l0 = (k * c // kchunks) // tile * tile if c else 0
        l1 = (k * (c + 1) // kchunks) // tile * tile if c + 1 < kchunks else k
        if l1 > l0:
            out.append((l0, l1))
    return out or [(0, k)]


def rgemm_columns(plan, transa, transb, alpha, a, b, beta, c, mode=None, group=None,
                  compute=None, kchunks=None):
    """C <- alpha op(A) op(B) + beta C with C split by column blocks over ranks.

    On the root, ``a``/``b``/``c`` are the full operands; padded leading
    dimensions are packed first (C's result is copied back into the padded
    storage, its padding untouched); on the other ranks they are ignored
    (None).  Returns nothing; on the root C holds the result (bitwise equal
    to ``Rgemm`` in exact mode).

    The k dimension is streamed in ``kchunks`` panels: panel c+1 of op(A)
    (broadcast) and of each rank's op(B) columns (point-to-point) is in
    flight on NCCL's stream while panel c computes, each panel an Rgemm with
    beta = 1 after the first.  For transa = 'N' that is the reference's own
    per-element sequence (beta-scale C, then c += a_il * (alpha b_lj) for l
    ascending, level23.py:120-125), so exact mode stays bitwise; for
    transa = 'T' the reference sums from zero and combines once, so exact
    mode keeps a single panel there (fast modes chunk either way)."""
    from .mpblas import default_mode
    ops = _Ops(group)
    compute = functools.partial(Rgemm, _check_storage=False) if compute is None else compute
    m, n, k = plan.m, plan.n, plan.k
    rank, world = plan.rank, plan.world
    ta, tb = transa.upper(), transb.upper()
    nra, nca = (m, k) if ta == "N" else (k, m)
    lda = max(1, nra)
    be = to_dd(beta)
    beta_zero = be[0] == 0.0 and be[1] == 0.0
    exact_like = (default_mode() if mode is None else mode) in ("exact", "reference")
    if kchunks is None:
        # panels exist to overlap the broadcast of op(A) with compute; one
        # rank has nothing to overlap (each panel is a separate kernel call)
        kchunks = 4 if world > 1 and k >= 4096 and (ta == "N" or not exact_like) else 1
    if ta != "N" and exact_like:
        kchunks = 1
    panels = _k_chunks(k, kchunks)
    j0, j1 = plan.blocks[rank]
    nb = j1 - j0
    c_user = None
    if rank == 0:
        # the slabs below assume tight leading dimensions: pack padded operands
        a, b = a.packed(), b.packed()
        if c.ld != max(1, m):
            c_user, c = c, c.packed()

    # 1. C column slabs to their owners (only read when beta != 0)
    sends, recvs = [], []
    if rank == 0:
        c_loc = _slab(c.store, j0 * m, nb * m)
        if not beta_zero:
            for r in range(1, world):
                r0, r1 = plan.blocks[r]
                if r1 > r0:
                    cs = _slab(c.store, r0 * m, (r1 - r0) * m)
                    sends += [ops.send(cs[0], r, group), ops.send(cs[1], r, group)]
    elif nb:
        c_loc = plan.buf("C", nb * m)
        if not beta_zero:
            recvs += [ops.recv(c_loc[0], 0, group), ops.recv(c_loc[1], 0, group)]
        else:
            c_loc[0].zero_()
            c_loc[1].zero_()
    ops.exchange(sends + recvs)

    # 2. k-panels: communication of panel c+1 overlaps the compute of panel c
    def a_panel(idx, l0, l1):
        """(store, ld) of op(A)(:, l0:l1): a slice of A ('N') or packed rows ('T')."""
        if ta == "N":
            if rank == 0:
                st = _slab(a.store, l0 * lda, (l1 - l0) * lda)
            else:
                full = plan.buf("A", lda * nca)
                st = _slab(full, l0 * lda, (l1 - l0) * lda)
            return st, lda
        kc = l1 - l0
        if rank == 0:
            st = tuple(p[:lda * nca].view(nca, lda)[:, l0:l1].contiguous().view(-1)
                       for p in a.store)
        else:
            st = plan.buf(f"A{idx}", kc * nca)
        return st, max(1, kc)

    def b_panel(idx, l0, l1, r0, r1, store=None):
        """op(B)(l0:l1, r0:r1) packed column-major; (store, ld)."""
        kc, w = l1 - l0, r1 - r0
        if store is not None:            # the root packs from the full B
            if tb == "N":
                st = tuple(p[:k * n].view(n, k)[r0:r1, l0:l1].contiguous().view(-1)
                           for p in store)
            else:
                st = tuple(p[:n * k].view(k, n)[l0:l1, r0:r1].contiguous().view(-1)
                           for p in store)
        else:
            st = plan.buf(f"B{idx}", kc * w)
        return st, (max(1, kc) if tb == "N" else max(1, w))

    def issue(idx):
        """Start panel idx's transfers; returns (waitables, local A, local B)."""
        l0, l1 = panels[idx]
        a_st, a_ld = a_panel(idx, l0, l1)
        works = [dist.broadcast(a_st[0], src=0, group=group, async_op=True),
                 dist.broadcast(a_st[1], src=0, group=group, async_op=True)]
        p2p = []
        b_loc = None
        if rank == 0:
            for r in range(world):
                r0, r1 = plan.blocks[r]
                if r1 == r0:
                    continue
                st, ld = b_panel(idx, l0, l1, r0, r1, store=b.store)
                if r == 0:
                    b_loc = (st, ld)
                else:
                    p2p += [ops.send(st[0], r, group), ops.send(st[1], r, group)]
        elif nb:
            st, ld = b_panel(idx, l0, l1, j0, j1)
            b_loc = (st, ld)
            p2p += [ops.recv(st[0], 0, group), ops.recv(st[1], 0, group)]
        if p2p:
            works += dist.batch_isend_irecv(p2p)
        return works, (a_st, a_ld), b_loc

    pending = issue(0)
    for idx, (l0, l1) in enumerate(panels):
        works, (a_st, a_ld), b_loc = pending
        if idx + 1 < len(panels):
            pending = issue(idx + 1)
        for w_ in works:
            w_.wait()
        if nb:
            kc = l1 - l0
            A = DeviceMatrix(*((m, kc) if ta == "N" else (kc, m)), "dd", a_ld, store=a_st)
            (b_st, b_ld) = b_loc
            B = DeviceMatrix(*((kc, nb) if tb == "N" else (nb, kc)), "dd", b_ld, store=b_st)
            C = DeviceMatrix(m, nb, "dd", max(1, m), store=c_loc)
            compute(ta, tb, m, nb, kc, alpha, A, a_ld, B, b_ld, beta if idx == 0 else 1.0, C,
                    max(1, m), mode=mode)

    # 3. slabs back to the root
    sends, recvs = [], []
    if rank == 0:
        for r in range(1, world):
            r0, r1 = plan.blocks[r]
            if r1 == r0:
                continue
            cs = _slab(c.store, r0 * m, (r1 - r0) * m)
            recvs += [ops.recv(cs[0], r, group), ops.recv(cs[1], r, group)]
    elif nb:
        sends += [ops.send(c_loc[0], 0, group), ops.send(c_loc[1], 0, group)]
    ops.exchange(sends + recvs)
    if c_user is not None:   # back into the caller's padded storage
        for dst, src in zip(c_user.store, c.store):
            dst[:c_user.ld * n].view(n, c_user.ld)[:, :m].copy_(src[:m * n].view(n, m))


def rsyrk_columns(n, k, world, rank, device, uplo, trans, alpha, a, beta, c, mode=None,
                  group=None, compute_gemm=None, compute_syrk=None):
    """Rsyrk with the uplo triangle split into triangle-balanced column slabs.

    Root holds A (lda = rows) and C (ldc = n); the result lands in the root's
    C (bitwise equal to ``Rsyrk`` in exact mode); the opposite triangle is
    never changed."""
    ops = _Ops(group)
    gemm = functools.partial(Rgemm, _check_storage=False) if compute_gemm is None else compute_gemm
    syrk = functools.partial(Rsyrk, _check_storage=False) if compute_syrk is None else compute_syrk
    up, tr = uplo.upper(), trans.upper()
    nra, nca = (n, k) if tr == "N" else (k, n)
    lda = max(1, nra)
    blocks = triangle_split(n, world, up)
    bufs = {}

    def buf(name, numel):
        if name not in bufs:
            bufs[name] = (torch.empty(numel, dtype=torch.float64, device=device),
                          torch.empty(numel, dtype=torch.float64, device=device))
        return bufs[name]

    c_user = None
    if rank == 0:   # the slabs below assume tight leading dimensions
        a = a.packed()
        if c.ld != max(1, n):
            c_user, c = c, c.packed()
    a_store = (a.store[0][:lda * nca], a.store[1][:lda * nca]) if rank == 0 else buf("A", lda * nca)
    ops.bcast(a_store[0])
    ops.bcast(a_store[1])

    j0, j1 = blocks[rank]
    nb = j1 - j0
    sends, recvs = [], []
    if rank == 0:
        for r in range(1, world):
            r0, r1 = blocks[r]
            if r1 > r0:
                cs = _slab(c.store, r0 * n, (r1 - r0) * n)
                sends += [ops.send(cs[0], r, group), ops.send(cs[1], r, group)]
        c_loc = _slab(c.store, j0 * n, nb * n)
    elif nb:
        c_loc = buf("C", nb * n)
        recvs += [ops.recv(c_loc[0], 0, group), ops.recv(c_loc[1], 0, group)]
    ops.exchange(sends + recvs)

    if nb:
        def sub(store, off):
            return store[0][off:], store[1][off:]

        # rows of op(A) [r0, r1) as a stored matrix view
        def a_rows(r0, r1):
            if tr == "N":   # rows r0.. of the n x k matrix: offset r0, same lda
                return DeviceMatrix(r1 - r0, k, "dd", lda, store=sub(a_store, r0))
            return DeviceMatrix(k, r1 - r0, "dd", lda, store=sub(a_store, r0 * lda))

        diag = DeviceMatrix(nb, nb, "dd", n, store=sub(c_loc, j0))
        syrk(up, tr, nb, k, alpha, a_rows(j0, j1), lda, beta, diag, n, mode=mode)
        ta, tb = ("N", "T") if tr == "N" else ("T", "N")
        if up == "U" and j0 > 0:        # rectangle rows [0, j0) x cols J
            rect = DeviceMatrix(j0, nb, "dd", n, store=c_loc)
            gemm(ta, tb, j0, nb, k, alpha, a_rows(0, j0), lda, a_rows(j0, j1), lda, beta,
                 rect, n, mode=mode)
        if up == "L" and j1 < n:        # rectangle rows [j1, n) x cols J
            rect = DeviceMatrix(n - j1, nb, "dd", n, store=sub(c_loc, j1))
            gemm(ta, tb, n - j1, nb, k, alpha, a_rows(j1, n), lda, a_rows(j0, j1), lda, beta,
                 rect, n, mode=mode)

    sends, recvs = [], []
    if rank == 0:
        for r in range(1, world):
            r0, r1 = blocks[r]
            if r1 > r0:
                cs = _slab(c.store, r0 * n, (r1 - r0) * n)
                recvs += [ops.recv(cs[0], r, group), ops.recv(cs[1], r, group)]
    elif nb:
        sends += [ops.send(c_loc[0], 0, group), ops.send(c_loc[1], 0, group)]
    ops.exchange(sends + recvs)
    if c_user is not None:   # back into the caller's padded storage
        for dst, src in zip(c_user.store, c.store):
            dst[:c_user.ld * n].view(n, c_user.ld)[:, :n].copy_(src[:n * n].view(n, n))


def rgemm_host_columns(transa, transb, m, n, k, alpha, a, b, beta, c, world, rank, device,
                       mode=None, group=None, compute=None):
    """End-to-end variant: host (numpy) operands on the root are staged to its
    GPU, the column-split Rgemm runs, and C is copied back to the host.
    Argument order as Rgemm's (alpha, a, b, beta, c); a, b, c are HostMatrix
    on rank 0 and None elsewhere."""
    plan = RgemmPlan(m, n, k, world, rank, device)
    if rank == 0:
        A, B, C = (DeviceMatrix.from_host(x, device) for x in (a, b, c))
    else:
        A = B = C = None
    rgemm_columns(plan, transa, transb, alpha, A, B, beta, C, mode=mode, group=group,
                  compute=compute)
    if rank == 0:
        # straight into the caller's (pinned) planes: one DMA per plane, no
        # pageable temporary
        for dst, src in zip(c.store, C.store):
            torch.from_numpy(dst).copy_(src)


def rgemm_host_shared(transa, transb, m, n, k, alpha, a, b, beta, c, world, rank, mode=None,
                      group=None, compute=None):
    """End-to-end multi-rank Rgemm from / to SHARED host buffers: every rank
    runs the host entry point (``ddb_rgemm_host``: copies pipelined with the
    kernels) on its column slab J_r of C, reading op(A) and its op(B) columns
    and writing its C columns through its OWN GPU and PCIe link -- no
    collective on the data path, and no rank's link carries another's slab.

    ``a``, ``b``, ``c`` are ``SharedHostMatrix`` objects mapped (and pinned)
    in every rank.  The per-element operation sequence is the single call's,
    so exact mode is bitwise equal to ``Rgemm``.  Returns after every rank's
    slab is back in ``c`` (a barrier)."""
    compute = functools.partial(Rgemm, _check_storage=False) if compute is None else compute
    ta, tb = transa.upper(), transb.upper()
    j0, j1 = column_split(n, world)[rank]
    w = j1 - j0
    if w > 0:
        nra, nca = (m, k) if ta == "N" else (k, m)
        # op(B)(:, J): columns J of B ('N', offset j0 * ldb) or rows J ('T', offset j0)
        boff = j0 * b.ld if tb == "N" else j0
        bv = HostMatrix.from_planes(k if tb == "N" else w, w if tb == "N" else k,
                                    *(p[boff:] for p in b.store), ld=b.ld)
        cv = HostMatrix.from_planes(m, w, *(p[j0 * c.ld:] for p in c.store), ld=c.ld)
        compute(ta, tb, m, w, k, alpha, a, a.ld, bv, b.ld, beta, cv, c.ld, mode=mode)
    if dist.is_initialized():
        dist.barrier(group=group)

