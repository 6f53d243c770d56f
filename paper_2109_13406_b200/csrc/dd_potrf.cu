// dd_potrf.cu -- blocked dd Cholesky (Rpotrf) whose trailing updates are
// Rsyrk calls, bit-identical to the reference's unblocked order in exact mode.
//
// The reference's Rpotrf (mplapack/chol.py:21-65) is unblocked and
// left-looking.  For column j (lower; upper is the transpose):
//   dot   = sum_ltr_{l<j} L(j,l) * L(j,l)              (chol.py:38-40)
//   ajj   = A(j,j) - dot ; fail (info = j+1, A(j,j) = ajj) if NaN or <= 0
//   L(j,j) = sqrt(ajj) ; rec = 1 / L(j,j)               (chol.py:41-49, :63)
//   lower: tail_i = A(i,j) + sum_{l<j} (-L(j,l)) * L(i,l), accumulated in
//          place left to right, then L(i,j) = rec * tail_i  (chol.py:57-64)
//   upper: temp_jj = sum_ltr_{l<j} U(l,jj) * U(l,j) (from zero), then
//          U(j,jj) = rec * (A(j,jj) - temp_jj)           (chol.py:50-56)
//
// Blocked right-looking form with the same per-element operation sequence:
//   * the pivots' dot products are kept in a vector D, each entry extended
//     by one product as soon as its row (column) gets a new factor entry, in
//     the reference's l order -- so a pivot costs O(1), and ajj = d0(j) - D(j)
//     with d0 the original diagonal;
//   * lower: after a block column [j0, j1) is factored, the trailing lower
//     triangle is updated IN PLACE by Rsyrk('L', 'N', alpha = -1, beta = 1):
//     per element c = c + L(i,l) * (-1 * L(j,l)), l = j0..j1-1 in order --
//     the reference's accumulation, continued (mul2 is symmetric and
//     mul2(-1, x) == -x inside the safe window; the diagonal entries of the
//     update are discarded, pivots come from D);
//   * upper: temp accumulates from ZERO, so the trailing updates go to a
//     separate accumulator S (lower-stored, S(jj, j) for U(j, jj)) by
//     Rsyrk('L', 'N', alpha = 1, beta = 1) on T = U12^T;
//   * per middle panel (<= 256 columns): its diagonal block by 64-column
//     inner blocks -- potrf_diag_kernel factors the inner diagonal block in
//     one CTA (right-looking, a barrier per column; the pivots are the only
//     serial chain), potrf_rows_kernel the diagonal block's rows below it,
//     potrf_blockupd_kernel the rest of the diagonal block -- then every row
//     below the panel ('U': column right of it) in one potrf_rows_kernel
//     launch against all of the panel's columns, each row an independent
//     sequence run by a warp.
// So in exact mode (Rsyrk exact) the factor is bit-identical to the
// reference for operands inside the safe window; fast / twosum modes differ
// only by their Rsyrk accumulation.  On failure the device info is set,
// later column kernels exit, and restore_kernel puts back the original
// entries the reference would not have touched yet (trailing updates of the
// lower form write in place; a backup copy is kept for that).
// dd sqrt / div / sub are the reference's scalar forms (ddarith.py:79-163);
// element-wise add / mul the vectorised ones (elem.py:54-78).
#include "lapack_num.cuh"

namespace ddb {

// Diagonal block [j0, j1) in one CTA, staged in shared memory, right-looking:
// per column j the pivot (thread 0), the column inside the block, then the
// block's trailing strictly-lower entries, each update in the reference's
// l order.  X(q, c) (q > c) is the block entry the factor overwrites: A(q, c)
// for 'L', A(c, q) for 'U'; for 'U' the running dot products S(q, c) are
// staged too.  The reciprocals go to p.rec for the panel kernel.
// The pivot chain (thread 0: sqrt and reciprocal, the reference's scalar
// forms) is the kernel's critical path, so the trailing updates run on the
// warps of the other three SM sub-partitions (warp w on w % 4) and leave
// warp 0's FP64 pipe to it; while the block stays inside the safe window
// (checked at load, then every new column value) they use the check-free
// forms, bit-identical there.
#ifdef DDB_DIAG_TIMING
// diagnostics build only: per-step clock64 stamps of the last diagonal block
__device__ long long g_diag_t[64][8];
#define DIAG_T(j, k) (g_diag_t[j][k] = clock64())
#else
#define DIAG_T(j, k) ((void)0)
#endif

// RK_TWOSUM (fast / twosum modes): the accumulators are unnormalised (H, L)
// pairs -- per product p = xh yh, its FMA residual and the cross terms go to
// L together with TwoSum(H, p)'s error: 13 FP64 operations instead of the
// exact-order add2(mul2()) 29, the TwoSum mode's error bound (every rounding
// lands in L, |L| ~ u |H|).  Normalised when an entry is finalised.
__device__ __forceinline__ dd ts_mac(dd acc, dd x, dd y) {
  const double p = dmul(x.h, y.h);
  const double e = dfma(x.h, y.h, -p);
  const double c = dfma(x.h, y.l, dmul(x.l, y.h));
  double s, err;
  two_sum(acc.h, p, s, err);
  return dd{s, dadd(acc.l, dadd(err, dadd(e, c)))};
}
__device__ __forceinline__ dd ts_norm(dd a) {
  double s, e;
  quick_two_sum(a.h, a.l, s, e);
  return dd{s, e};
}
// binary64 instantiations never select RK_TWOSUM (fastacc is dd only)
__device__ __forceinline__ double ts_mac(double acc, double x, double y) { return dadd(acc, dmul(x, y)); }
__device__ __forceinline__ double ts_norm(double a) { return a; }

// Fast / twosum modes (FA): the pivot's square root and reciprocal by one
// Newton correction each on the IEEE sqrt / reciprocal of the high word
// (dd-accurate; ~500 instead of ~2100 cycles of the reference's scalar
// forms), the trailing update with the TwoSum accumulation (entries stay
// unnormalised until their column is finalised); both inside the safe
// window only, the exact forms otherwise.
__device__ __forceinline__ dd fast_sqrt_dd(dd a) {
  const double y = __dsqrt_rn(a.h);
  const double r = dadd(dfma(-y, y, a.h), a.l);
  double s, e;
  quick_two_sum(y, __ddiv_rn(r, dmul(2.0, y)), s, e);
  return dd{s, e};
}
__device__ __forceinline__ dd fast_rec_dd(dd s) {
  const double r0 = __drcp_rn(s.h);
  const double e = dsub(dfma(-s.h, r0, 1.0), dmul(s.l, r0));
  double h, l;
  quick_two_sum(r0, dmul(r0, e), h, l);
  return dd{h, l};
}
__device__ __forceinline__ double fast_sqrt_dd(double a) { return __dsqrt_rn(a); }
__device__ __forceinline__ double fast_rec_dd(double s) { return __ddiv_rn(1.0, s); }

template <class N, bool FA>
__global__ void __launch_bounds__(512)
potrf_diag_kernel(PotrfArgs p, int64_t j0, int nb) {
  using T = typename N::T;
  extern __shared__ double sm[];
  __shared__ T rec_s;
  __shared__ int ok_s, nc_s;
  if (*p.info != 0) return;
  const int64_t lda = p.lda, lds = p.lds;
  const int sq = nb * nb;
  double* xh = sm;
  double* xl = sm + sq;
  double* sh = sm + 2 * sq;                      // 'U' only
  double* sl = sm + 3 * sq;
  double* dh = sm + (p.upper ? 4 : 2) * sq;
  double* dl = dh + nb;
  double* d0h = dl + nb;
  double* d0l = d0h + nb;
  bool win = true;
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    const T xv = N::ld(p.a_hi, p.a_lo, x);
    N::st(xh, xl, t, xv);
    win &= N::win(xv);
    if (p.upper) {
      const T sv = N::ld(p.s_hi, p.s_lo, (j0 + q) + (j0 + c) * lds);
      N::st(sh, sl, t, sv);
      win &= N::win(sv);
    }
  }
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    const T dv = N::ld(p.dh, p.dl, j0 + t);
    N::st(dh, dl, t, dv);
    N::st(d0h, d0l, t, N::ld(p.d0_hi, p.d0_lo, j0 + t));
    win &= N::win(dv);
  }
  if (threadIdx.x == 0) nc_s = 1;
  win = __syncthreads_and(win) && !N::kF64;
  if (threadIdx.x == 0) nc_s = win;
  __syncthreads();
  // thread 0 computes pivot j+1 while warps 1.. run step j's trailing
  // update (pivot j+1 needs only D(j+1), final after step j's column phase)
  auto pivot = [&](int j) {
    const T d0 = N::ld(d0h, d0l, j), dj = N::ld(dh, dl, j);
    const bool fa = FA && nc_s && N::win(d0) && N::win(dj);
    const T ajj = fa ? N::fadd2(d0, N::neg(dj)) : N::ssub(d0, dj);   // chol.py:41
    const int64_t djj = (j0 + j) * (lda + 1);
    ok_s = !N::bad_pivot(ajj);
    DIAG_T(j, 5);
    if (!ok_s) {
      N::st(p.a_hi, p.a_lo, djj, ajj);
      *p.info = (int)(j0 + j + 1);
    } else {
      const bool fs = fa && N::win(ajj);
      const T s = fs ? fast_sqrt_dd(ajj) : N::ssqrt(ajj);
      N::st(p.a_hi, p.a_lo, djj, s);
      DIAG_T(j, 6);
      const T rec = fs ? fast_rec_dd(s) : N::sdiv(N::one(), s);
      rec_s = rec;
      N::st(p.rec_hi, p.rec_lo, j, rec);
      DIAG_T(j, 7);
    }
  };
  // trailing-update ownership: every strictly-lower entry (q, c) of the
  // block belongs to one thread of the warps off sub-partition 0 for the
  // whole kernel and lives in its registers -- per step j the owner adds the
  // product of column j's entries (c > j) and stores the entry once, when
  // its column is next (c = j + 1).  No per-step index arithmetic and no
  // shared-memory read-modify-write of the accumulators.
  constexpr int kE = 6;                    // 6 x 384 >= 2016 entries (nb <= 64)
  const int warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const bool owner = (warp & 3) != 0;
  const int nthr = (nw - (nw + 3) / 4) * 32;                  // warps not on sub-partition 0
  const int me = (warp - warp / 4 - 1) * 32 + (threadIdx.x & 31);
  int eq[kE], ec[kE];
  T eacc[kE];
  {
    const int npairs = nb * (nb - 1) / 2;
#pragma unroll
    for (int k = 0; k < kE; ++k) {
      const int t = me + k * nthr;
      eq[k] = -1;
      ec[k] = nb;
      eacc[k] = N::zero();
      if (owner && t < npairs) {
        // column c of pair t, column-major over the strictly-lower triangle
        int ci = (int)((2.0f * nb - 1.0f - sqrtf((2.0f * nb - 1.0f) * (2.0f * nb - 1.0f) - 8.0f * t)) * 0.5f);
        while (ci > 0 && ci * (2 * nb - ci - 1) / 2 > t) --ci;
        while ((ci + 1) * (2 * nb - ci - 2) / 2 <= t) ++ci;
        eq[k] = ci + 1 + (t - ci * (2 * nb - ci - 1) / 2);
        ec[k] = ci;
        eacc[k] = p.upper ? N::ld(sh, sl, eq[k] + ec[k] * nb) : N::ld(xh, xl, eq[k] + ec[k] * nb);
      }
    }
  }
  if (threadIdx.x == 0) pivot(0);
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (!ok_s) break;
    if (threadIdx.x == 0) DIAG_T(j, 0);
    const T rec = rec_s;
    for (int q = j + 1 + threadIdx.x; q < nb; q += blockDim.x) {
      const int t = q + j * nb;
      T a = N::ld(xh, xl, t);
      if (FA && !p.upper) a = ts_norm(a);            // TwoSum-accumulated entry
      if (p.upper) a = N::add(a, N::neg(FA ? ts_norm(N::ld(sh, sl, t)) : N::ld(sh, sl, t)));
      const T v = N::mul(rec, a);
      N::st(xh, xl, t, v);
      const bool f = nc_s && N::win(v);
      if (!f) nc_s = 0;
      const T d = N::ld(dh, dl, q);
      N::st(dh, dl, q, f ? N::fadd2(d, N::fmul(v, v)) : N::add(d, N::mul(v, v)));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      DIAG_T(j, 1);
      if (j + 1 < nb) pivot(j + 1);
      DIAG_T(j, 2);
    } else if (owner) {
      const bool fast = nc_s;
#pragma unroll
      for (int k = 0; k < kE; ++k) {
        if (ec[k] <= j) continue;              // entry final (or none)
        const int q = eq[k], c = ec[k];
        const T vq = N::ld(xh, xl, q + j * nb), vc = N::ld(xh, xl, c + j * nb);
        T f1, f2;
        if (!p.upper) { f1 = N::neg(vc); f2 = vq; }
        else { f1 = vq; f2 = vc; }
        T r;
        if (FA && fast) r = ts_mac(eacc[k], f1, f2);
        else if (fast) r = N::fadd2(eacc[k], N::fmul(f1, f2));
        else r = N::add(FA ? ts_norm(eacc[k]) : eacc[k], N::mul(f1, f2));
        eacc[k] = r;
        if (c == j + 1) {                       // its column is next: hand it over
          if (!p.upper) N::st(xh, xl, q + c * nb, r);
          else N::st(sh, sl, q + c * nb, r);
        }
      }
      if (threadIdx.x == 32) DIAG_T(j, 3);
    }
    __syncthreads();
    if (threadIdx.x == 0) DIAG_T(j, 4);
  }
  // write the block back ('U': the untouched part is written back unchanged;
  // 'L': entries the reference would not have touched yet are restored from
  // the backup by potrf_restore_kernel)
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    N::st(p.a_hi, p.a_lo, x, N::ld(xh, xl, t));
  }
}

// Factor rows below a factored diagonal block.  Rows q in [q0, q1) ('U':
// columns of U) against the w <= 32 * NPER columns [j0, j0 + w): each q is an
// independent recurrence, one warp per q, lane t holding the accumulators of
// columns c = t + 32 i ("chain" i).  Step c: entry c is finalised (rec_c *
// acc, or rec_c * (A - acc) for 'U'), broadcast, and every lane extends its
// later columns by one product -- the reference's per-element order
// (chol.py:50-64) and the same operation sequence the blocked path's Rsyrk /
// Rgemm updates apply, so one launch covers a whole (up to 256-wide) panel.
// The diagonal block's factor P(c2, c) = L(j0 + c2, j0 + c) ('U': U(j0 + c,
// j0 + c2)) is read at ph[c2 * sr + c * sc] through L1 (the w x w block is
// L2-resident) one step ahead of its use; the reciprocals sit in shared
// memory.  The steps run in 32-step segments, one per chain, unrolled over
// the chains: in segment s chains < s are finished and compiled out, chains >
// s are fully live, so a 256-wide panel keeps ~89 % of the lanes busy with no
// per-chain predicates.  Every lane forms rec_c * acc on its own chain-s
// accumulator and the owner's is broadcast (no divergent owner branch).
// Arithmetic (MODE): the check-free forms are bit-identical to the checked
// ones inside the safe window (lapack_num.cuh: NumDD::win); RK_FAST when every
// P row this warp reads is inside it (pmask, potrf_psafe_kernel) and so are
// the starting accumulators and D -- then only the broadcast value is checked
// per step; RK_CHECK checks every P entry at use (no mask: the narrow inner
// panels); RK_SLOW the checked forms throughout.
constexpr int kRowsThreads = 256;    // 8 rows per CTA
#ifndef DDB_ROWS_MINB
#define DDB_ROWS_MINB 2      // CTAs per SM the register allocation targets (2: 128 registers; 86.8 vs 89.4 ms)
#endif
#ifndef DDB_ROWS_SEL
#define DDB_ROWS_SEL 0       // 1: the ordered-Fast2Sum add (fewer FP64 ops, more selects; 86.8 vs 86.0 ms)
#endif
enum RowsMode { RK_SLOW = 0, RK_CHECK = 1, RK_FAST = 2, RK_TWOSUM = 3 };


template <class N>
__device__ __forceinline__ typename N::T rfadd(typename N::T x, typename N::T y) {
  return DDB_ROWS_SEL ? N::fadd(x, y) : N::fadd2(x, y);
}

template <class N, int NPER, bool UP, int MODE, bool TCHK = false>
__device__ __forceinline__ void rows_steps(const PotrfArgs& p, int64_t j0, int w, int ncols, int64_t q,
                                           const double* __restrict__ ph, const double* __restrict__ pl,
                                           int sr, int sc, const typename N::T* rec_s,
                                           typename N::T (&acc)[NPER], const typename N::T (&au)[NPER],
                                           typename N::T& dq) {
  using T = typename N::T;
  const int lane = threadIdx.x & 31;
  const int64_t lda = p.lda;
  T tn[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) tn[i] = N::zero();
  int off = lane * sr;                       // P(lane + 32 i, c) at off + 32 i sr
  auto fetch = [&](int s) {                  // chains >= s of the step at column offset off
#pragma unroll
    for (int i = 0; i < NPER; ++i)
      if (i >= s && lane + 32 * i < w) tn[i] = N::ldg(ph, pl, off + 32 * i * sr);
  };
  if (ncols > 0) fetch(0);
#pragma unroll
  for (int s = 0; s < NPER; ++s) {
    if (32 * s >= ncols) break;
    const int cend = min(32, ncols - 32 * s);
    for (int cc = 0; cc < cend; ++cc) {
      const int c = 32 * s + cc;
      T t[NPER];
#pragma unroll
      for (int i = s; i < NPER; ++i) t[i] = tn[i];
      off += sc;
      if (c + 1 < ncols) fetch(cc + 1 < 32 ? s : s + 1);
      // finalise entry c: every lane forms it from its own chain-s
      // accumulator, the owner's (lane cc) is broadcast and stored
      T as = acc[s];
      if constexpr (MODE == RK_TWOSUM) as = ts_norm(as);
      const T a = UP ? N::add(au[s], N::neg(as)) : as;
      const T v = N::shfl(N::mul(rec_s[c], a), cc);
      if (lane == cc) N::st(p.a_hi, p.a_lo, UP ? (j0 + c) + q * lda : q + (j0 + c) * lda, v);
      // extend the later columns.  Lanes whose chain-s column is already
      // final (c2 <= c) and lanes past w update too: those accumulators are
      // never read again, so no per-lane predicate is needed
      if constexpr (MODE == RK_TWOSUM) {
        if (N::win(v)) {                              // warp-uniform
          dq = ts_mac(dq, v, v);
#pragma unroll
          for (int i = s; i < NPER; ++i) {
            if (TCHK && !N::win(t[i]))          // an unchecked P entry outside the window
              acc[i] = UP ? N::add(ts_norm(acc[i]), N::mul(v, t[i]))
                          : N::add(ts_norm(acc[i]), N::mul(N::neg(t[i]), v));
            else
              acc[i] = UP ? ts_mac(acc[i], v, t[i]) : ts_mac(acc[i], N::neg(t[i]), v);
          }
        } else {                                      // checked forms on normalised values
          dq = N::add(ts_norm(dq), N::mul(v, v));
#pragma unroll
          for (int i = s; i < NPER; ++i)
            acc[i] = UP ? N::add(ts_norm(acc[i]), N::mul(v, t[i]))
                        : N::add(ts_norm(acc[i]), N::mul(N::neg(t[i]), v));
        }
        continue;
      }
      if (MODE != RK_SLOW && N::win(v)) {           // warp-uniform
        dq = rfadd<N>(dq, N::fmul(v, v));
#pragma unroll
        for (int i = s; i < NPER; ++i) {
          if (MODE == RK_CHECK && !N::win(t[i]))
            acc[i] = UP ? N::add(acc[i], N::mul(v, t[i])) : N::add(acc[i], N::mul(N::neg(t[i]), v));
          else
            acc[i] = UP ? rfadd<N>(acc[i], N::fmul(v, t[i])) : rfadd<N>(acc[i], N::fmul(N::neg(t[i]), v));
        }
      } else {
        dq = N::add(dq, N::mul(v, v));
#pragma unroll
        for (int i = s; i < NPER; ++i)
          acc[i] = UP ? N::add(acc[i], N::mul(v, t[i])) : N::add(acc[i], N::mul(N::neg(t[i]), v));
      }
    }
  }
}

// FA: the fast / twosum modes' instantiation (RK_TWOSUM on the masked
// panel), else the exact modes' (RK_FAST): one accumulation form per
// kernel keeps its code and register use down
template <class N, int NPER, bool UP, bool FA>
__global__ void __launch_bounds__(kRowsThreads, DDB_ROWS_MINB)
potrf_rows_kernel(PotrfArgs p, int64_t j0, int w, int64_t q0, int64_t q1,
                  const double* __restrict__ ph, const double* __restrict__ pl, int sr, int sc,
                  const double* __restrict__ rh, const double* __restrict__ rl,
                  const unsigned* __restrict__ pmask) {
  using T = typename N::T;
  __shared__ T rec_s[32 * NPER];
  // a failure inside the diagonal block still leaves the columns before it
  // complete, as the reference does (chol.py:44-46)
  int ncols = w;
  const int inf = *p.info;
  if (inf != 0) {
    if (inf - 1 < j0) return;
    ncols = (int)min((int64_t)w, inf - 1 - j0);
  }
  for (int c = threadIdx.x; c < w; c += blockDim.x) rec_s[c] = N::ld(rh, rl, c);
  __syncthreads();
  const int64_t lda = p.lda, lds = p.lds;
  const int lane = threadIdx.x & 31;
  const int64_t q = q0 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (q >= q1) return;                  // whole warps exit together
  T acc[NPER], au[NPER];
  bool ok = true;
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + 32 * i;
    acc[i] = N::zero();
    au[i] = N::zero();
    if (c < w) {
      acc[i] = UP ? N::ld(p.s_hi, p.s_lo, q + (j0 + c) * lds) : N::ld(p.a_hi, p.a_lo, q + (j0 + c) * lda);
      if (UP) au[i] = N::ld(p.a_hi, p.a_lo, (j0 + c) + q * lda);    // 'U': A(j0 + c, q)
      ok &= N::win(acc[i]);
      if (pmask != nullptr) ok &= (pmask[i] >> lane & 1u) != 0;
    }
  }
  // D(q), the running pivot dot product, kept by every lane (same value)
  T dq = N::ld(p.dh, p.dl, q);
  ok &= N::win(dq);
  const bool all_ok = __all_sync(0xffffffffu, ok);
  if (N::kF64 || !all_ok)
    rows_steps<N, NPER, UP, RK_SLOW>(p, j0, w, ncols, q, ph, pl, sr, sc, rec_s, acc, au, dq);
  else if (pmask == nullptr && p.fastacc) {   // narrow launch, fast modes: TwoSum, P checked per entry
    rows_steps<N, NPER, UP, RK_TWOSUM, true>(p, j0, w, ncols, q, ph, pl, sr, sc, rec_s, acc, au, dq);
    dq = ts_norm(dq);
  } else if (pmask == nullptr)
    rows_steps<N, NPER, UP, RK_CHECK>(p, j0, w, ncols, q, ph, pl, sr, sc, rec_s, acc, au, dq);
  else if constexpr (FA) {
    rows_steps<N, NPER, UP, RK_TWOSUM>(p, j0, w, ncols, q, ph, pl, sr, sc, rec_s, acc, au, dq);
    dq = ts_norm(dq);
  } else
    rows_steps<N, NPER, UP, RK_FAST>(p, j0, w, ncols, q, ph, pl, sr, sc, rec_s, acc, au, dq);
  if (lane == 0) N::st(p.dh, p.dl, q, dq);
}

// Window mask of the w x w factor block P (potrf_rows_kernel): bit r % 32 of
// mask[r / 32] set when every P(r, c), c < r, is inside the safe window.  One
// warp per row, 32 rows per CTA.
__global__ void __launch_bounds__(1024)
potrf_psafe_kernel(const double* __restrict__ ph, const double* __restrict__ pl, int w, int sr,
                   int sc, unsigned* __restrict__ mask) {
  const int lane = threadIdx.x & 31, r = blockIdx.x * 32 + threadIdx.x / 32;
  bool ok = true;
  if (r < w)
    for (int c = lane; c < r; c += 32) ok &= NumDD::win(NumDD::ldg(ph, pl, (int64_t)r * sr + (int64_t)c * sc));
  ok = __all_sync(0xffffffffu, ok);
  __shared__ unsigned word;
  if (threadIdx.x == 0) word = 0;
  __syncthreads();
  if (lane == 0 && ok) atomicOr(&word, 1u << (threadIdx.x / 32));
  __syncthreads();
  if (threadIdx.x == 0) mask[blockIdx.x] = word;
}

// Trailing update of the diagonal block [i1, j1)^2 by the factored inner
// block [i0, i1) (<= 64 columns): entries i1 <= c < q < j1, one thread each,
// products in l order -- what Rsyrk('L', 'N') applies there in the blocked
// path ('L': A(q, c) += (-L(c, l)) L(q, l) in place; 'U': S(q, c) += U(l, q)
// U(l, c)).  The CTA's 32 rows and 8 columns of the inner block's factor are
// staged in shared memory first.  Diagonal entries are not updated: pivots
// come from D.
template <class N>
__global__ void __launch_bounds__(256)
potrf_blockupd_kernel(PotrfArgs p, int64_t i0, int64_t i1, int64_t j1) {
  using T = typename N::T;
  __shared__ T fq[kPotrfMaxNb][33], fc[kPotrfMaxNb][8];
  __shared__ int fok;
  if (*p.info != 0) return;
  const int64_t qb = i1 + (int64_t)blockIdx.x * 32, cb = i1 + (int64_t)blockIdx.y * 8;
  if (cb >= qb + 31) return;                       // tile strictly above the diagonal
  if (threadIdx.x == 0 && threadIdx.y == 0) fok = !N::kF64;
  __syncthreads();
  const int kb = (int)(i1 - i0);
  const int64_t lda = p.lda;
  const int tx = threadIdx.x, ty = threadIdx.y;
  // F(x, l) = L(x, i0 + l) ('L') / U(i0 + l, x) ('U')
  auto f = [&](int64_t x, int l) {
    return p.upper ? N::ld(p.a_hi, p.a_lo, (i0 + l) + x * lda) : N::ld(p.a_hi, p.a_lo, x + (i0 + l) * lda);
  };
  bool ok = true;
  for (int l = ty; l < kb; l += 8) {
    if (qb + tx < j1) { fq[l][tx] = f(qb + tx, l); ok &= N::win(fq[l][tx]); }
    if (tx < 8 && cb + tx < j1) { fc[l][tx] = f(cb + tx, l); ok &= N::win(fc[l][tx]); }
  }
  if (!ok) fok = 0;
  __syncthreads();
  const int64_t q = qb + tx, c = cb + ty;
  if (q >= j1 || c >= q) return;
  // inside the safe window: the check-free forms (exact: bit-identical) or,
  // in the fast / twosum modes, the TwoSum accumulation
  T acc = !p.upper ? N::ld(p.a_hi, p.a_lo, q + c * lda) : N::ld(p.s_hi, p.s_lo, q + c * p.lds);
  const bool fast = fok && N::win(acc);
  for (int l = 0; l < kb; ++l) {
    const T f1 = !p.upper ? N::neg(fc[l][ty]) : fq[l][tx];
    const T f2 = !p.upper ? fq[l][tx] : fc[l][ty];
    if (fast && p.fastacc) acc = ts_mac(acc, f1, f2);
    else if (fast) acc = N::fadd2(acc, N::fmul(f1, f2));
    else acc = N::add(acc, N::mul(f1, f2));
  }
  if (fast && p.fastacc) acc = ts_norm(acc);
  if (!p.upper) N::st(p.a_hi, p.a_lo, q + c * lda, acc);
  else N::st(p.s_hi, p.s_lo, q + c * p.lds, acc);
}

// Fast / twosum modes, late in the factorization: the lookahead update of
// the next (<= 256-column) block column as one lean launch instead of an
// Rsyrk and an Rgemm call (each ~10 launches of routing / bound / split
// machinery: ~0.12 ms apiece for a few microseconds of work).  C(r, c) +=
// sgn F(c, l) F(r, l), l < kb, for rows [r0, r1) and columns [c0, c0 + wd),
// c <= r; F(x, l) at fh[x + l ldf].  CTA: 128 rows (one per thread) x 8
// columns with the columns' F(c, :) slice in shared memory; the TwoSum
// accumulation while the operands are inside the safe window, the checked
// dd forms otherwise.
__global__ void __launch_bounds__(128)
potrf_lean_upd_kernel(const double* __restrict__ fh, const double* __restrict__ fl, int64_t ldf,
                      int kb, double sgn, double* __restrict__ ch, double* __restrict__ cl,
                      int64_t ldc, int64_t r0, int64_t r1, int64_t c0, int wd,
                      const int* __restrict__ info) {
  constexpr int CW = 8, KMAX = 256;
  __shared__ dd fs[KMAX][CW];
  __shared__ int fok;
  if (*info != 0) return;                    // a failed factorization: the restore pass owns the rest
  const int64_t cb = c0 + (int64_t)blockIdx.y * CW;
  const int64_t rbase = r0 + (int64_t)blockIdx.x * blockDim.x;
  if (rbase + blockDim.x - 1 < cb) return;   // the whole tile lies above the diagonal
  if (threadIdx.x == 0) fok = 1;
  __syncthreads();
  for (int e = threadIdx.x; e < kb * CW; e += blockDim.x) {
    const int l = e / CW, cc = e % CW;
    dd f{0.0, 0.0};
    if (cb + cc < c0 + wd) f = NumDD::ld(fh, fl, cb + cc + (int64_t)l * ldf);
    fs[l][cc] = dd{sgn * f.h, sgn * f.l};
    if (!NumDD::win(f)) fok = 0;
  }
  __syncthreads();
  const int64_t r = rbase + threadIdx.x;
  if (r >= r1) return;
  dd acc[CW];
  bool ok = fok != 0;
#pragma unroll
  for (int cc = 0; cc < CW; ++cc) {
    acc[cc] = dd{0.0, 0.0};
    if (cb + cc < c0 + wd && cb + cc <= r) {
      acc[cc] = NumDD::ld(ch, cl, r + (cb + cc) * ldc);
      ok &= NumDD::win(acc[cc]);
    }
  }
  dd fn = NumDD::ld(fh, fl, r);
  for (int l = 0; l < kb; ++l) {
    const dd fr = fn;
    if (l + 1 < kb) fn = NumDD::ld(fh, fl, r + (int64_t)(l + 1) * ldf);
    if (ok && NumDD::win(fr)) {
#pragma unroll
      for (int cc = 0; cc < CW; ++cc) acc[cc] = ts_mac(acc[cc], fs[l][cc], fr);
    } else {
#pragma unroll
      for (int cc = 0; cc < CW; ++cc) acc[cc] = NumDD::add(ts_norm(acc[cc]), NumDD::mul(fs[l][cc], fr));
    }
  }
#pragma unroll
  for (int cc = 0; cc < CW; ++cc)
    if (cb + cc < c0 + wd && cb + cc <= r) NumDD::st(ch, cl, r + (cb + cc) * ldc, ts_norm(acc[cc]));
}

cudaError_t launch_potrf_lean_upd(const double* fh, const double* fl, int64_t ldf, int kb, double sgn,
                                  double* ch, double* cl, int64_t ldc, int64_t r0, int64_t r1,
                                  int64_t c0, int wd, const int* info, cudaStream_t s) {
  if (r1 <= r0 || wd <= 0 || kb <= 0) return cudaSuccess;
  if (kb > 256) return cudaErrorInvalidValue;
  dim3 grid((unsigned)((r1 - r0 + 127) / 128), (unsigned)((wd + 7) / 8));
  potrf_lean_upd_kernel<<<grid, 128, 0, s>>>(fh, fl, ldf, kb, sgn, ch, cl, ldc, r0, r1, c0, wd, info);
  return cudaGetLastError();
}

// T(r, l) = U(j0 + l, j1 + r), r < rows, l < nb  (ld = rows)
__global__ void __launch_bounds__(256)
potrf_transpose_kernel(PotrfArgs p, int64_t j0, int64_t j1, int nb, int64_t rows) {
  __shared__ double th[32][33], tl[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, l0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {          // read: l fastest in memory
    const int64_t r = r0 + y, l = l0 + threadIdx.x;
    if (r < rows && l < nb) {
      const int64_t x = (j0 + l) + (j1 + r) * p.lda;
      th[y][threadIdx.x] = p.a_hi[x];
      if (!p.f64) tl[y][threadIdx.x] = p.a_lo[x];
    }
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {          // write: r fastest
    const int64_t l = l0 + y, r = r0 + threadIdx.x;
    if (r < rows && l < nb) {
      p.t_hi[r + l * rows] = th[threadIdx.x][y];
      if (!p.f64) p.t_lo[r + l * rows] = tl[threadIdx.x][y];
    }
  }
}

// After a failure at column f = info - 1 (lower form): the reference leaves
// column f below the diagonal and every later column untouched; put back the
// original lower-triangle entries there from the backup (ld = n).
__global__ void __launch_bounds__(256)
potrf_restore_kernel(PotrfArgs p) {
  const int info = *p.info;
  if (info == 0) return;
  const int64_t f = info - 1;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= p.n) return;
  for (int64_t c = f + blockIdx.y; c <= i && c < p.n; c += gridDim.y) {
    if (i == c && c == f) continue;
    p.a_hi[i + c * p.lda] = p.b_hi[i + c * p.n];
    if (!p.f64) p.a_lo[i + c * p.lda] = p.b_lo[i + c * p.n];
  }
}

#ifdef DDB_DIAG_TIMING
extern "C" int ddb_debug_diag_timing(long long* out) {
  return (int)cudaMemcpyFromSymbol(out, g_diag_t, sizeof(g_diag_t));
}
#endif

cudaError_t launch_potrf_diag(const PotrfArgs& p, int64_t j0, int64_t j1, cudaStream_t s) {
  const int nb = (int)(j1 - j0);
  const size_t smem = sizeof(double) * ((size_t)(p.upper ? 4 : 2) * nb * nb + 4 * (size_t)nb);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(potrf_diag_kernel<NumDD, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(potrf_diag_kernel<NumDD, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(potrf_diag_kernel<NumF64, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  if (p.f64) potrf_diag_kernel<NumF64, false><<<1, 512, smem, s>>>(p, j0, nb);
  else if (p.fastacc) potrf_diag_kernel<NumDD, true><<<1, 512, smem, s>>>(p, j0, nb);
  else potrf_diag_kernel<NumDD, false><<<1, 512, smem, s>>>(p, j0, nb);
  return cudaGetLastError();
}

template <class N, int NPER>
static cudaError_t rows_launch(const PotrfArgs& p, int64_t j0, int w, int64_t q0, int64_t q1,
                               const double* ph, const double* pl, int sr, int sc,
                               const double* rh, const double* rl, const unsigned* pmask,
                               cudaStream_t s) {
  const int64_t threads = (q1 - q0) * 32;
  const unsigned grid = (unsigned)((threads + kRowsThreads - 1) / kRowsThreads);
  const bool fa = p.fastacc && pmask != nullptr;
  if (p.upper) {
    if (fa) potrf_rows_kernel<N, NPER, true, true><<<grid, kRowsThreads, 0, s>>>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask);
    else potrf_rows_kernel<N, NPER, true, false><<<grid, kRowsThreads, 0, s>>>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask);
  } else {
    if (fa) potrf_rows_kernel<N, NPER, false, true><<<grid, kRowsThreads, 0, s>>>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask);
    else potrf_rows_kernel<N, NPER, false, false><<<grid, kRowsThreads, 0, s>>>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask);
  }
  return cudaGetLastError();
}

template <class N>
static cudaError_t rows_dispatch(const PotrfArgs& p, int64_t j0, int w, int64_t q0, int64_t q1,
                                 const double* ph, const double* pl, int sr, int sc,
                                 const double* rh, const double* rl, const unsigned* pmask,
                                 cudaStream_t s) {
  if (w <= 64) return rows_launch<N, 2>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask, s);
  if (w <= 128) return rows_launch<N, 4>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask, s);
  return rows_launch<N, 8>(p, j0, w, q0, q1, ph, pl, sr, sc, rh, rl, pmask, s);
}

cudaError_t launch_potrf_rows(const PotrfArgs& p, int64_t j0, int w, int64_t q0, int64_t q1,
                              const double* ph, const double* pl, int64_t sr, int64_t sc,
                              const double* rh, const double* rl, unsigned* pmask, cudaStream_t s) {
  if (q1 <= q0 || w <= 0) return cudaSuccess;
  // P offsets are 32-bit: the w x w block spans < 2^31 elements
  if (w > kPotrfMaxPanel || (w - 1) * (sr + sc) >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  if (pmask != nullptr && !p.f64) {
    const cudaError_t e = launch_window_mask(ph, pl, w, sr, sc, pmask, s);
    if (e != cudaSuccess) return e;
  }
  return p.f64 ? rows_dispatch<NumF64>(p, j0, w, q0, q1, ph, pl, (int)sr, (int)sc, rh, rl, nullptr, s)
               : rows_dispatch<NumDD>(p, j0, w, q0, q1, ph, pl, (int)sr, (int)sc, rh, rl, pmask, s);
}

cudaError_t launch_window_mask(const double* ph, const double* pl, int w, int64_t sr, int64_t sc,
                               unsigned* mask, cudaStream_t s) {
  if (w <= 0) return cudaSuccess;
  if ((w - 1) * (sr + sc) >= (int64_t(1) << 31)) return cudaErrorInvalidValue;
  potrf_psafe_kernel<<<(w + 31) / 32, 1024, 0, s>>>(ph, pl, w, (int)sr, (int)sc, mask);
  return cudaGetLastError();
}

cudaError_t launch_potrf_blockupd(const PotrfArgs& p, int64_t i0, int64_t i1, int64_t j1,
                                  cudaStream_t s) {
  const int64_t m = j1 - i1;
  if (m <= 1) return cudaSuccess;
  dim3 grid((unsigned)((m + 31) / 32), (unsigned)((m + 7) / 8));
  if (p.f64) potrf_blockupd_kernel<NumF64><<<grid, dim3(32, 8), 0, s>>>(p, i0, i1, j1);
  else potrf_blockupd_kernel<NumDD><<<grid, dim3(32, 8), 0, s>>>(p, i0, i1, j1);
  return cudaGetLastError();
}

cudaError_t launch_potrf_transpose(const PotrfArgs& p, int64_t j0, int64_t j1, int nb,
                                   int64_t rows, cudaStream_t s) {
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((nb + 31) / 32));
  potrf_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(p, j0, j1, nb, rows);
  return cudaGetLastError();
}

cudaError_t launch_potrf_restore(const PotrfArgs& p, cudaStream_t s) {
  dim3 grid((unsigned)((p.n + 255) / 256), 64);
  potrf_restore_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ddb
