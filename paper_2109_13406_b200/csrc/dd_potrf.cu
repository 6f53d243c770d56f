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
//   * per block: potrf_diag_kernel factors the diagonal block in one CTA
//     (right-looking, a barrier per column; the pivots are the only serial
//     chain), potrf_panel_kernel the rows below it ('U': the columns right of
//     it), each row an independent sequence over the block's columns run by
//     a group of lanes; block width <= 64 (the diagonal block lives in
//     shared memory).
// So in exact mode (Rsyrk exact) the factor is bit-identical to the
// reference for operands inside the safe window; fast / twosum modes differ
// only by their Rsyrk accumulation.  On failure the device info is set,
// later column kernels exit, and restore_kernel puts back the original
// entries the reference would not have touched yet (trailing updates of the
// lower form write in place; a backup copy is kept for that).
// dd sqrt / div / sub are the reference's scalar forms (ddarith.py:79-163);
// element-wise add / mul the vectorised ones (elem.py:54-78).
#include "internal.h"

namespace ddb {

namespace {

__device__ __forceinline__ dd neg2(dd x) { return dd{-x.h, -x.l}; }

__device__ __forceinline__ bool isfin(double x) { return finite_(x); }

// _canon (ddarith.py:68-71)
__device__ __forceinline__ dd canon(double h, double l) { return dd{h, isfin(h) ? l : 0.0}; }

// scalar _add2 (ddarith.py:79-90): the element form plus the final _canon
__device__ dd add2_s(dd x, dd y) {
  const double s0 = dadd(x.h, y.h);
  if (!isfin(s0)) return dd{s0, 0.0};
  const dd r = add2_chk(x, y);
  return canon(r.h, r.l);
}

// _mul21 (ddarith.py:103-110): dd * double
__device__ dd mul21_s(dd x, double y) {
  double p, e;
  two_prod_dekker(x.h, y, p, e);
  if (!(isfin(p) && isfin(e))) return canon(p, 0.0);
  e = dadd(e, dmul(x.l, y));
  double s, t;
  quick_two_sum(p, e, s, t);
  return canon(s, t);
}

// _div2 (ddarith.py:113-131)
__device__ dd div2_s(dd x, dd y) {
  if (y.h == 0.0) {
    if (x.h == 0.0) return dd{__longlong_as_double(0x7ff8000000000000LL), 0.0};
    return dd{copysign(__longlong_as_double(0x7ff0000000000000LL), x.h) * copysign(1.0, y.h), 0.0};
  }
  if (!(isfin(x.h) && isfin(y.h))) {
    if (!isfin(y.h) && !isnan(y.h)) {
      if (!isfin(x.h) && !isnan(x.h)) return dd{__longlong_as_double(0x7ff8000000000000LL), 0.0};
      return dd{dmul(copysign(0.0, x.h), copysign(1.0, y.h)), 0.0};
    }
    return canon(dmul(x.h, copysign(1.0, y.h)), 0.0);
  }
  const double q1 = x.h / y.h;
  dd r = add2_s(x, neg2(mul21_s(y, q1)));
  const double q2 = r.h / y.h;
  r = add2_s(r, neg2(mul21_s(y, q2)));
  const double q3 = r.h / y.h;
  double a, b;
  quick_two_sum(q1, q2, a, b);
  return add2_s(dd{a, b}, dd{q3, 0.0});
}

// _sqrt2 (ddarith.py:142-163): Newton correction on 1/sqrt(hi), with the
// exact even-power pre-scaling for very large / small arguments
__device__ dd sqrt2_s(dd v) {
  if (v.h == 0.0 && v.l == 0.0) return dd{0.0, 0.0};
  if (!isfin(v.h)) return dd{v.h, 0.0};
  double h = v.h, l = v.l;
  int shift = 0;
  if (h >= 0x1p996) { h = dmul(h, 0x1p-106); l = dmul(l, 0x1p-106); shift = 53; }
  else if (h <= 0x1p-996) { h = dmul(h, 0x1p106); l = dmul(l, 0x1p106); shift = -53; }
  const double x = 1.0 / sqrt(h);
  const double ax = dmul(h, x);
  double p, e;
  two_prod_dekker(ax, ax, p, e);
  const dd r = add2_s(dd{h, l}, dd{-p, -e});
  double s, e2;
  quick_two_sum(ax, dmul(r.h, dmul(x, 0.5)), s, e2);
  if (shift == 53) { s = dmul(s, 0x1p53); e2 = dmul(e2, 0x1p53); }
  else if (shift == -53) { s = dmul(s, 0x1p-53); e2 = dmul(e2, 0x1p-53); }
  return canon(s, e2);
}

// chol.py:42: _isnan(ajj) (float(ajj) = hi + lo) or ajj <= 0 (_cmp2 order)
__device__ __forceinline__ bool bad_pivot(dd a) {
  if (isnan(dadd(a.h, a.l))) return true;
  if (a.h < 0.0) return true;
  if (a.h > 0.0) return false;
  return !(a.l > 0.0);
}

}  // namespace

// Diagonal block [j0, j1) in one CTA, staged in shared memory, right-looking:
// per column j the pivot (thread 0), the column inside the block, then the
// block's trailing strictly-lower entries, each update in the reference's
// l order.  X(q, c) (q > c) is the block entry the factor overwrites: A(q, c)
// for 'L', A(c, q) for 'U'; for 'U' the running dot products S(q, c) are
// staged too.  The reciprocals go to p.rec for the panel kernel.
__global__ void __launch_bounds__(512)
potrf_diag_kernel(PotrfArgs p, int64_t j0, int nb) {
  extern __shared__ double sm[];
  __shared__ dd rec_s;
  __shared__ int ok_s;
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
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    xh[t] = p.a_hi[x];
    xl[t] = p.a_lo[x];
    if (p.upper) {
      const int64_t y = (j0 + q) + (j0 + c) * lds;
      sh[t] = p.s_hi[y];
      sl[t] = p.s_lo[y];
    }
  }
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    dh[t] = p.dh[j0 + t];
    dl[t] = p.dl[j0 + t];
    d0h[t] = p.d0_hi[j0 + t];
    d0l[t] = p.d0_lo[j0 + t];
  }
  __syncthreads();
  // thread 0 computes pivot j+1 while warps 1.. run step j's trailing
  // update (pivot j+1 needs only D(j+1), final after step j's column phase)
  auto pivot = [&](int j) {
    const dd ajj = add2_s(dd{d0h[j], d0l[j]}, neg2(dd{dh[j], dl[j]}));   // chol.py:41
    const int64_t djj = (j0 + j) * (lda + 1);
    ok_s = !bad_pivot(ajj);
    if (!ok_s) {
      p.a_hi[djj] = ajj.h;
      p.a_lo[djj] = ajj.l;
      *p.info = (int)(j0 + j + 1);
    } else {
      const dd s = sqrt2_s(ajj);
      p.a_hi[djj] = s.h;
      p.a_lo[djj] = s.l;
      const dd rec = div2_s(dd{1.0, 0.0}, s);
      rec_s = rec;
      p.rec_hi[j] = rec.h;
      p.rec_lo[j] = rec.l;
    }
  };
  if (threadIdx.x == 0) pivot(0);
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (!ok_s) break;
    const dd rec = rec_s;
    for (int q = j + 1 + threadIdx.x; q < nb; q += blockDim.x) {
      const int t = q + j * nb;
      dd a{xh[t], xl[t]};
      if (p.upper) a = add2_chk(a, neg2(dd{sh[t], sl[t]}));
      const dd v = mul2_chk(rec, a);
      xh[t] = v.h;
      xl[t] = v.l;
      const dd d = add2_chk(dd{dh[q], dl[q]}, mul2_chk(v, v));
      dh[q] = d.h;
      dl[q] = d.l;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (j + 1 < nb) pivot(j + 1);
    } else if (threadIdx.x >= 32) {
      // pairs (q, c), j < c < q < nb, enumerated column by column; batches
      // of kB independent updates (operands gathered before any store)
      const int rem = nb - j - 1;
      const int npairs = rem * (rem - 1) / 2;
      constexpr int kB = 4;
      const int nthr = blockDim.x - 32;
      for (int base = threadIdx.x - 32; base < npairs; base += nthr * kB) {
        int xs[kB];
        dd acc[kB], f1[kB], f2[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int t = base + b * nthr;
          xs[b] = -1;
          if (t < npairs) {
            // column ci (0-based within the rem trailing columns) of pair t
            int ci = (int)((2.0f * rem - 1.0f - sqrtf((2.0f * rem - 1.0f) * (2.0f * rem - 1.0f) - 8.0f * t)) * 0.5f);
            while (ci > 0 && ci * (2 * rem - ci - 1) / 2 > t) --ci;
            while ((ci + 1) * (2 * rem - ci - 2) / 2 <= t) ++ci;
            const int qi = ci + 1 + (t - ci * (2 * rem - ci - 1) / 2);
            const int c = j + 1 + ci, q = j + 1 + qi;
            xs[b] = q + c * nb;
            const dd vq{xh[q + j * nb], xl[q + j * nb]}, vc{xh[c + j * nb], xl[c + j * nb]};
            if (!p.upper) { acc[b] = dd{xh[xs[b]], xl[xs[b]]}; f1[b] = neg2(vc); f2[b] = vq; }
            else { acc[b] = dd{sh[xs[b]], sl[xs[b]]}; f1[b] = vq; f2[b] = vc; }
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          if (xs[b] < 0) continue;
          const dd r = add2_chk(acc[b], mul2_chk(f1[b], f2[b]));
          if (!p.upper) { xh[xs[b]] = r.h; xl[xs[b]] = r.l; }
          else { sh[xs[b]] = r.h; sl[xs[b]] = r.l; }
        }
      }
    }
    __syncthreads();
  }
  // write the block back ('U': the untouched part is written back unchanged;
  // 'L': entries the reference would not have touched yet are restored from
  // the backup by potrf_restore_kernel)
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    p.a_hi[x] = xh[t];
    p.a_lo[x] = xl[t];
  }
}

// Panel below ('L': rows q >= j1) / right of ('U': columns q >= j1) the
// diagonal block.  Each q is independent: a group of G lanes owns it, lane t
// holding the accumulators of block columns c = j0 + t + G*i.  Step c: the
// owner finalises entry c (rec_c * acc, or rec_c * (A - acc) for 'U'),
// broadcasts it, and every lane extends its later columns by one product --
// the reference's per-element order (chol.py:50-64), with NPER independent
// chains per lane.  The block's factor (strictly-lower part, transposed for
// 'U') and the reciprocals sit in shared memory.
constexpr int kPanelG = 32;          // lanes per row: one warp
constexpr int kPanelThreads = 256;    // 8 rows per CTA

template <int NPER>
__global__ void __launch_bounds__(kPanelThreads)
potrf_panel_kernel(PotrfArgs p, int64_t j0, int nb) {
  extern __shared__ double sm[];
  // a failure inside this block's diagonal part still leaves the columns
  // before it complete, as the reference does (chol.py:44-46)
  int ncols = nb;
  const int inf = *p.info;
  if (inf != 0) {
    if (inf - 1 < j0) return;
    ncols = (int)(inf - 1 - j0);
  }
  const int64_t lda = p.lda, lds = p.lds;
  const int64_t j1 = j0 + nb;
  // packed strictly-lower triangle: T(c2, c) (c < c2) at off(c) + c2 - c - 1
  const int ntri = nb * (nb - 1) / 2;
  double* th = sm;
  double* tl = sm + ntri;
  double* rh = sm + 2 * ntri;
  double* rl = rh + nb;
  auto off = [nb](int c) { return c * (2 * nb - c - 1) / 2; };
  for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
    const int c2 = t % nb, c = t / nb;
    if (c2 <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + c2) * lda : (j0 + c2) + (j0 + c) * lda;
    th[off(c) + c2 - c - 1] = p.a_hi[x];
    tl[off(c) + c2 - c - 1] = p.a_lo[x];
  }
  for (int c = threadIdx.x; c < nb; c += blockDim.x) {
    rh[c] = p.rec_hi[c];
    rl[c] = p.rec_lo[c];
  }
  __syncthreads();
  const int lane = threadIdx.x % kPanelG;
  const int64_t q = j1 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kPanelG;
  if (q >= p.n) return;                 // whole warps exit together
  dd acc[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + kPanelG * i;
    acc[i] = dd{0.0, 0.0};
    if (c < nb) {
      const int64_t x = p.upper ? q + (j0 + c) * lds : q + (j0 + c) * lda;
      acc[i] = p.upper ? dd{p.s_hi[x], p.s_lo[x]} : dd{p.a_hi[x], p.a_lo[x]};
    }
  }
  dd dq{0.0, 0.0};
  if (lane == 0) dq = dd{p.dh[q], p.dl[q]};
  for (int c = 0; c < ncols; ++c) {
    const int owner = c % kPanelG, ic = c / kPanelG;
    dd v{0.0, 0.0};
    if (lane == owner) {
      dd a{0.0, 0.0};
#pragma unroll
      for (int i = 0; i < NPER; ++i)
        if (i == ic) a = acc[i];
      const dd rec{rh[c], rl[c]};
      const int64_t x = p.upper ? (j0 + c) + q * lda : q + (j0 + c) * lda;
      if (p.upper) a = add2_chk(dd{p.a_hi[x], p.a_lo[x]}, neg2(a));
      v = mul2_chk(rec, a);
      p.a_hi[x] = v.h;
      p.a_lo[x] = v.l;
    }
    v.h = __shfl_sync(0xffffffffu, v.h, owner);
    v.l = __shfl_sync(0xffffffffu, v.l, owner);
    if (lane == 0) dq = add2_chk(dq, mul2_chk(v, v));
#pragma unroll
    for (int i = 0; i < NPER; ++i) {
      const int c2 = lane + kPanelG * i;
      if (c2 > c && c2 < nb) {
        const int o = off(c) + c2 - c - 1;
        const dd t{th[o], tl[o]};
        acc[i] = p.upper ? add2_chk(acc[i], mul2_chk(v, t))
                         : add2_chk(acc[i], mul2_chk(neg2(t), v));
      }
    }
  }
  if (lane == 0) {
    p.dh[q] = dq.h;
    p.dl[q] = dq.l;
  }
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
      tl[y][threadIdx.x] = p.a_lo[x];
    }
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {          // write: r fastest
    const int64_t l = l0 + y, r = r0 + threadIdx.x;
    if (r < rows && l < nb) {
      p.t_hi[r + l * rows] = th[threadIdx.x][y];
      p.t_lo[r + l * rows] = tl[threadIdx.x][y];
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
    p.a_lo[i + c * p.lda] = p.b_lo[i + c * p.n];
  }
}

cudaError_t launch_potrf_diag(const PotrfArgs& p, int64_t j0, int64_t j1, cudaStream_t s) {
  const int nb = (int)(j1 - j0);
  const size_t smem = sizeof(double) * ((size_t)(p.upper ? 4 : 2) * nb * nb + 4 * (size_t)nb);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(potrf_diag_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_dev = dev;
  }
  potrf_diag_kernel<<<1, 512, smem, s>>>(p, j0, nb);
  return cudaGetLastError();
}

template <int NPER>
static cudaError_t panel_launch(const PotrfArgs& p, int64_t j0, int nb, int64_t rows,
                                cudaStream_t s) {
  const size_t smem = sizeof(double) * ((size_t)nb * (nb - 1) + 2 * (size_t)nb);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(potrf_panel_kernel<NPER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  const int64_t threads = rows * kPanelG;
  potrf_panel_kernel<NPER><<<(unsigned)((threads + kPanelThreads - 1) / kPanelThreads),
                             kPanelThreads, smem, s>>>(p, j0, nb);
  return cudaGetLastError();
}

cudaError_t launch_potrf_panel(const PotrfArgs& p, int64_t j0, int nb, int64_t rows,
                               cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int nper = (nb + kPanelG - 1) / kPanelG;
  (void)nper;   // nb <= 64 = 2 * kPanelG
  return panel_launch<2>(p, j0, nb, rows, s);
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
