// dd_prescan.cu -- one HBM-bound pass over the operands before the tiled
// kernels run.
//
// It produces, in a per-call workspace:
//   * row_exp[i]  max biased exponent of the hi words of row i of op(A)
//   * col_exp[j]  max biased exponent of the hi words of column j of op(B)
//     (fast mode only: the scales of the certified bound GEMM, dd_bound.cu)
//   * flag        nonzero if any word lies outside the safe window:
//       hi: zero, or 2**-300 <= |hi| < 2**301;   lo: finite and |lo| < 2**301.
//     Inside the window the tiled kernels' check-free dd arithmetic is
//     bit-identical to the reference's checked arithmetic (dd_arith.cuh) and
//     the fast accumulator's residual captures stay exact.  Outside it the
//     tiled kernels exit at once and the reference-semantics kernel
//     (dd_reference.cu) computes the call, so every input is handled with
//     the reference's own inf / nan / overflow behaviour.
//     In the fast modes (canon != 0) a word is also unsafe when it is not a
//     normalised dd, |lo| > 2^-53 |hi| (e.g. hi = 0, lo != 0): their error
//     analyses bound the lo * hi terms by the hi * hi ones (dd_tiled.cuh),
//     and the certified bound is built from |hi| alone (dd_bound.cu).  The
//     reference's own operations only ever produce normalised values; such
//     hand-made inputs get the reference semantics instead.
//
// Traffic: 16 B per scanned element (hi + lo), coalesced along the
// contiguous (column-major) dimension; one block = 32 rows x 64 columns.
#include "internal.h"

namespace ddb {

__device__ __forceinline__ int bexp(double x) {
  return (int)((__double_as_longlong(x) >> 52) & 0x7ff);
}

__global__ void __launch_bounds__(256)
prescan_kernel(const double* __restrict__ hi, const double* __restrict__ lo, int64_t ld,
               int64_t rows, int64_t cols, int* __restrict__ out_row,
               int* __restrict__ out_col, int* __restrict__ flag, int tri,
               int64_t col_off, int canon) {
  __shared__ int srow[8][33];
  const int x = threadIdx.x, y = threadIdx.y;
  const int64_t r = (int64_t)blockIdx.x * 32 + x;
  const int64_t c0 = (int64_t)blockIdx.y * 64;
  int rmax = 0;
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t c = c0 + y + 8 * q;
    int e = 0;
    // tri: 1 = only the upper triangle (r <= c) is live, 2 = only the lower
    const int64_t cg = c + col_off;
    const bool live = tri == 0 || (tri == 1 ? r <= cg : r >= cg);
    if (r < rows && c < cols && live) {
      const double h = hi[r + c * ld];
      const double l = lo[r + c * ld];
      const int eh = bexp(h), el = bexp(l);
      bad |= (h != 0.0 && eh < WIN_LO) || eh > WIN_HI || el > WIN_HI;
      // h * 2^-53 is exact inside the window (|h| >= 2^-300)
      bad |= canon && fabs(l) > fabs(h) * 0x1p-53;
      e = eh;
    }
    rmax = max(rmax, e);
    if (out_col != nullptr) {
      int cm = e;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, off));
      if (x == 0 && c < cols && cm > 0) atomicMax(&out_col[c], cm);
    }
  }
  if (out_row != nullptr) {
    srow[y][x] = rmax;
    __syncthreads();
    if (y == 0) {
      int m = srow[0][x];
#pragma unroll
      for (int t = 1; t < 8; ++t) m = max(m, srow[t][x]);
      if (r < rows && m > 0) atomicMax(&out_row[r], m);
    }
  }
  if (__syncthreads_or(bad) && x == 0 && y == 0) atomicOr(flag, ROUTE_UNSAFE);
}

static cudaError_t scan(const double* hi, const double* lo, int64_t ld, int64_t rows,
                        int64_t cols, int* out_row, int* out_col, int* flag,
                        cudaStream_t s, int* nlaunch, int canon, int tri = 0) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t gx = (rows + 31) / 32, gy_total = (cols + 63) / 64;
  // gridDim.y is limited to 65535: split very wide matrices into column slabs
  for (int64_t y0 = 0; y0 < gy_total; y0 += 65535) {
    const int64_t gy = gy_total - y0 < 65535 ? gy_total - y0 : 65535;
    const int64_t cbase = y0 * 64;
    dim3 grid((unsigned)gx, (unsigned)gy), block(32, 8);
    prescan_kernel<<<grid, block, 0, s>>>(hi + cbase * ld, lo + cbase * ld, ld, rows,
                                          cols - cbase, out_row,
                                          out_col ? out_col + cbase : nullptr, flag, tri,
                                          cbase, canon);
    ++*nlaunch;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// Scans op(A) rows and op(B) columns (and C when the exact kernel will use
// it as its starting accumulator).
cudaError_t launch_prescan(const GemmArgs& g, int alg, int* row_exp, int* col_exp,
                           int* flag, cudaStream_t s, int* nlaunch) {
  // only the certified-anchor algorithm consumes the exponent maxima
  const bool fast = alg == ALG_CERT;
  // the fast algorithms' error analyses assume normalised dd operands
  const int canon = alg == ALG_CERT || alg == ALG_TWOSUM;
  cudaError_t e;
  // op(A) is m x k: stored m x k (N) or k x m (T)
  if (g.ta == 0)
    e = scan(g.a_hi, g.a_lo, g.lda, g.m, g.k, fast ? row_exp : nullptr, nullptr, flag, s, nlaunch, canon);
  else
    e = scan(g.a_hi, g.a_lo, g.lda, g.k, g.m, nullptr, fast ? row_exp : nullptr, flag, s, nlaunch, canon);
  if (e != cudaSuccess) return e;
  if (g.syrk == 0) {
    // op(B) is k x n: stored k x n (N) or n x k (T)
    if (g.tb == 0)
      e = scan(g.b_hi, g.b_lo, g.ldb, g.k, g.n, nullptr, fast ? col_exp : nullptr, flag, s, nlaunch, canon);
    else
      e = scan(g.b_hi, g.b_lo, g.ldb, g.n, g.k, fast ? col_exp : nullptr, nullptr, flag, s, nlaunch, canon);
    if (e != cudaSuccess) return e;
  }
  // The exact kernel's axpy form (transa = 'N') starts its unchecked
  // accumulation from beta*C, so C must be in the window too.
  if (alg == ALG_EXACT && g.ta == 0 && !(g.beta.h == 0.0 && g.beta.l == 0.0)) {
    // Rsyrk: only the uplo triangle is ever read (level23.py:245-246)
    e = scan(g.c_hi, g.c_lo, g.ldc, g.m, g.n, nullptr, nullptr, flag, s, nlaunch, 0, g.syrk);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace ddb
