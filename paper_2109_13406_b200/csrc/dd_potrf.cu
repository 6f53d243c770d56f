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
//   * potrf_col_kernel finishes column j of the current block: the pivot
//     (every CTA recomputes it, CTA 0 stores it), then one thread per
//     trailing row (column) continues the sequence over l in [j0, j).
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

// Column j of the block starting at j0.  d0 = original diagonal, D = pivot
// dot products so far, S (upper only) = the lower-stored accumulator.
__global__ void __launch_bounds__(128)
potrf_col_kernel(PotrfArgs p, int64_t j0, int64_t j) {
  if (*p.info != 0) return;
  const dd ajj = add2_s(dd{p.d0_hi[j], p.d0_lo[j]}, neg2(dd{p.dh[j], p.dl[j]}));
  const int64_t djj = j + j * p.lda;
  if (bad_pivot(ajj)) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.a_hi[djj] = ajj.h;
      p.a_lo[djj] = ajj.l;
      *p.info = (int)(j + 1);
    }
    return;
  }
  const dd s = sqrt2_s(ajj);
  const dd rec = div2_s(dd{1.0, 0.0}, s);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.a_hi[djj] = s.h;
    p.a_lo[djj] = s.l;
  }
  const int64_t q = j + 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= p.n) return;
  const int64_t lda = p.lda;
  dd v;
  if (!p.upper) {
    dd acc{p.a_hi[q + j * lda], p.a_lo[q + j * lda]};
    for (int64_t l = j0; l < j; ++l) {
      const dd t = neg2(dd{p.a_hi[j + l * lda], p.a_lo[j + l * lda]});
      acc = add2_chk(acc, mul2_chk(t, dd{p.a_hi[q + l * lda], p.a_lo[q + l * lda]}));
    }
    v = mul2_chk(rec, acc);
    p.a_hi[q + j * lda] = v.h;
    p.a_lo[q + j * lda] = v.l;
  } else {
    dd acc{0.0, 0.0};                     // S is absent for a single block
    if (p.s_hi != nullptr) acc = dd{p.s_hi[q + j * p.lds], p.s_lo[q + j * p.lds]};
    for (int64_t l = j0; l < j; ++l)
      acc = add2_chk(acc, mul2_chk(dd{p.a_hi[l + q * lda], p.a_lo[l + q * lda]},
                                   dd{p.a_hi[l + j * lda], p.a_lo[l + j * lda]}));
    const dd elt = add2_chk(dd{p.a_hi[j + q * lda], p.a_lo[j + q * lda]}, neg2(acc));
    v = mul2_chk(rec, elt);
    p.a_hi[j + q * lda] = v.h;
    p.a_lo[j + q * lda] = v.l;
  }
  const dd d = add2_chk(dd{p.dh[q], p.dl[q]}, mul2_chk(v, v));
  p.dh[q] = d.h;
  p.dl[q] = d.l;
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

cudaError_t launch_potrf_col(const PotrfArgs& p, int64_t j0, int64_t j, cudaStream_t s) {
  const int64_t rows = p.n - j - 1;
  const unsigned grid = rows > 0 ? (unsigned)((rows + 127) / 128) : 1u;
  potrf_col_kernel<<<grid, 128, 0, s>>>(p, j0, j);
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
