// dd_prescan.cu -- one HBM-bound pass over the operands before the tiled
// kernels run, and the per-element routing it feeds.
//
// Per op(A) row i and op(B) column j it produces, in a per-call workspace
// (RouteWs, zeroed before the call):
//   * rmax / cmax  max biased exponent of the nonzero hi words (the scales of
//     the certified bound GEMM, dd_bound.cu);
//   * rneg / cneg  2047 - min biased exponent of the nonzero hi words, with
//     bit 16 set when the row / column holds a word outside the safe window:
//       hi: zero, or 2**-300 <= |hi| < 2**301;   lo: finite and |lo| < 2**301.
//     Inside the window the tiled kernels' check-free dd arithmetic is
//     bit-identical to the reference's checked arithmetic (dd_arith.cuh) and
//     the fast accumulators' residual captures stay exact.  Each element of
//     C depends on row i of op(A), column j of op(B) and C(i, j) only, so an
//     unsafe word reroutes just the elements of its row (A) or column (B)
//     to the reference-semantics kernel (dd_reference.cu), which reproduces
//     the reference's own inf / nan / overflow behaviour bit for bit; the
//     tiled kernels skip those elements.  In exact mode with transa = 'N'
//     the accumulator starts from beta * C, so an unsafe C(i, j) marks row i.
//     In the fast modes (canon != 0) a word is also unsafe when it is not a
//     normalised dd, |lo| > 2^-53 |hi| (e.g. hi = 0, lo != 0): their error
//     analyses bound the lo * hi terms by the hi * hi ones (dd_tiled.cuh),
//     and the certified bound is built from |hi| alone (dd_bound.cu).  The
//     reference's own operations only ever produce normalised values.
//   * flag[0]      nonzero if any word is unsafe (gates dd_reference.cu).
//
// route_summary_kernel then turns them into the exponent spread of each row /
// column (rsp / csp: max - min exponent of its nonzero hi words, SPREAD_BAD
// if unsafe), the spread maxima over blocks of ROUTE_BLK rows / columns (rsb
// / csb) and over the call (flag[1] rows, flag[2] columns).  The fast mode's
// certified bound is tight only while rsp[i] + csp[j] stays below a limit
// (dd_bound.cu derives it); wider elements are EC_WIDE and computed by the
// TwoSum accumulation instead (elem_class, internal.h).
//
// Traffic: 16 B per scanned element (hi + lo), coalesced along the
// contiguous (column-major) dimension; one block = 32 rows x 64 columns.
#include "internal.h"

namespace ddb {

__device__ __forceinline__ int bexp(double x) {
  return (int)((__double_as_longlong(x) >> 52) & 0x7ff);
}

// Row / column outputs: (max, neg) pairs; a null max with a non-null neg
// records only the unsafe bit (badonly: the C scan).
__global__ void __launch_bounds__(256)
prescan_kernel(const double* __restrict__ hi, const double* __restrict__ lo, int64_t ld,
               int64_t rows, int64_t cols, int* __restrict__ rmax_out,
               int* __restrict__ rneg_out, int* __restrict__ cmax_out, int* __restrict__ cneg_out,
               int* __restrict__ flag, int tri, int64_t col_off, int canon, int badonly) {
  __shared__ int smax[8][33], sneg[8][33];
  const int x = threadIdx.x, y = threadIdx.y;
  const int64_t r = (int64_t)blockIdx.x * 32 + x;
  const int64_t c0 = (int64_t)blockIdx.y * 64;
  int rmax = 0, rneg = 0;
  bool bad = false;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const int64_t c = c0 + y + 8 * q;
    int e = 0, ng = 0;
    // tri: 1 = only the upper triangle (r <= c) is live, 2 = only the lower
    const int64_t cg = c + col_off;
    const bool live = tri == 0 || (tri == 1 ? r <= cg : r >= cg);
    if (r < rows && c < cols && live) {
      const double h = hi[r + c * ld];
      const double l = lo[r + c * ld];
      const int eh = bexp(h), el = bexp(l);
      bool b = (h != 0.0 && eh < WIN_LO) || eh > WIN_HI || el > WIN_HI;
      // h * 2^-53 is exact inside the window (|h| >= 2^-300)
      b |= canon && fabs(l) > fabs(h) * 0x1p-53;
      bad |= b;
      if (!badonly && h != 0.0) { e = eh; ng = 2047 - eh; }
      ng |= b ? (1 << 16) : 0;
    }
    rmax = max(rmax, e);
    rneg = max(rneg, ng);
    if (cneg_out != nullptr) {
      int cm = e, cn = ng;
#pragma unroll
      for (int off = 16; off > 0; off >>= 1) {
        cm = max(cm, __shfl_xor_sync(0xffffffffu, cm, off));
        cn = max(cn, __shfl_xor_sync(0xffffffffu, cn, off));
      }
      if (x == 0 && c < cols) {
        if (cm > 0 && cmax_out != nullptr) atomicMax(&cmax_out[c], cm);
        if (cn > 0) atomicMax(&cneg_out[c], cn);
      }
    }
  }
  if (rneg_out != nullptr) {
    smax[y][x] = rmax;
    sneg[y][x] = rneg;
    __syncthreads();
    if (y == 0) {
      int m = smax[0][x], n = sneg[0][x];
#pragma unroll
      for (int t = 1; t < 8; ++t) { m = max(m, smax[t][x]); n = max(n, sneg[t][x]); }
      if (r < rows) {
        if (m > 0 && rmax_out != nullptr) atomicMax(&rmax_out[r], m);
        if (n > 0) atomicMax(&rneg_out[r], n);
      }
    }
  }
  if (__syncthreads_or(bad) && x == 0 && y == 0) atomicOr(flag, ROUTE_UNSAFE);
}

static cudaError_t scan(const double* hi, const double* lo, int64_t ld, int64_t rows,
                        int64_t cols, int* rmax, int* rneg, int* cmax, int* cneg, int* flag,
                        cudaStream_t s, int* nlaunch, int canon, int tri = 0, int badonly = 0) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  const int64_t gx = (rows + 31) / 32, gy_total = (cols + 63) / 64;
  // gridDim.y is limited to 65535: split very wide matrices into column slabs
  for (int64_t y0 = 0; y0 < gy_total; y0 += 65535) {
    const int64_t gy = gy_total - y0 < 65535 ? gy_total - y0 : 65535;
    const int64_t cbase = y0 * 64;
    dim3 grid((unsigned)gx, (unsigned)gy), block(32, 8);
    prescan_kernel<<<grid, block, 0, s>>>(hi + cbase * ld, lo + cbase * ld, ld, rows,
                                          cols - cbase, rmax, rneg,
                                          cmax ? cmax + cbase : nullptr,
                                          cneg ? cneg + cbase : nullptr, flag, tri, cbase,
                                          canon, badonly);
    ++*nlaunch;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// rsp / rsb / flag[1] from (rmax, rneg) for the first nr entries, then csp /
// csb / flag[2] for nc more (Rsyrk: nc = 0, the row results serve both).
__global__ void __launch_bounds__(256)
route_summary_kernel(const int* __restrict__ rmax, const int* __restrict__ rneg, int* rsp,
                     int* rsb, int64_t nr, int64_t nr_pad, const int* __restrict__ cmax,
                     const int* __restrict__ cneg, int* csp, int* csb, int64_t nc, int* flag,
                     int syrk, int* bad_rows, int* bad_cols) {
  const int64_t t = (int64_t)blockIdx.x * 256 + threadIdx.x;
  const bool is_row = t < nr_pad;
  const int64_t i = is_row ? t : t - nr_pad;
  const int64_t n = is_row ? nr : nc;
  int sp = 0, live = 0;
  if (i < n) {
    const int mx = is_row ? rmax[i] : cmax[i];
    const int ng = is_row ? rneg[i] : cneg[i];
    if (ng >> 16) {
      sp = SPREAD_BAD;
      const int pos = atomicAdd(&flag[is_row ? 3 : 4], 1);   // listed for dd_reference.cu
      (is_row ? bad_rows : bad_cols)[pos] = (int)i;
    } else if ((ng & 0xffff) != 0) {
      const int d = mx - (2047 - (ng & 0xffff));
      live = sp = d > 0 ? d : 0;
    }
    (is_row ? rsp : csp)[i] = sp;
  }
  // warps cover ROUTE_BLK = 32 aligned entries (nr_pad is a multiple of 32)
  int m = live;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, off));
  if ((threadIdx.x & 31) == 0 && i < n) {
    (is_row ? rsb : csb)[i / ROUTE_BLK] = m;
    if (m > 0) {
      atomicMax(&flag[is_row ? 1 : 2], m);
      if (syrk) atomicMax(&flag[2], m);
    }
  }
}

static size_t al256(size_t b) { return (b + 255) / 256 * 256; }

size_t route_ws_bytes(int64_t m, int64_t n, int syrk) {
  const size_t per = 4 * (size_t)m + (m / ROUTE_BLK + 1);
  const size_t perc = syrk ? 0 : 4 * (size_t)n + (n / ROUTE_BLK + 1);
  return al256(sizeof(int) * (16 + per + perc));
}

RouteWs route_ws_carve(void* base, int64_t m, int64_t n, int syrk) {
  RouteWs r;
  int* p = static_cast<int*>(base);
  r.flag = p; p += 16;
  r.rmax = p; p += m;
  r.rneg = p; p += m;
  r.rsp = p; p += m;
  r.rsb = p; p += m / ROUTE_BLK + 1;
  r.bad_rows = p; p += m;
  if (syrk) {
    r.cmax = r.rmax; r.cneg = r.rneg; r.csp = r.rsp; r.csb = r.rsb; r.bad_cols = r.bad_rows;
  } else {
    r.cmax = p; p += n;
    r.cneg = p; p += n;
    r.csp = p; p += n;
    r.csb = p; p += n / ROUTE_BLK + 1;
    r.bad_cols = p;
  }
  return r;
}

// Scans op(A) rows and op(B) columns (and C when the exact kernel will use
// it as its starting accumulator), then summarises the spreads.
cudaError_t launch_prescan(const GemmArgs& g, int alg, const RouteWs& r, cudaStream_t s,
                           int* nlaunch) {
  // the fast algorithms' error analyses assume normalised dd operands
  const int canon = alg == ALG_CERT || alg == ALG_TWOSUM;
  cudaError_t e;
  // op(A) is m x k: stored m x k (N) or k x m (T); its rows are op(A)'s rows
  if (g.ta == 0)
    e = scan(g.a_hi, g.a_lo, g.lda, g.m, g.k, r.rmax, r.rneg, nullptr, nullptr, r.flag, s,
             nlaunch, canon);
  else
    e = scan(g.a_hi, g.a_lo, g.lda, g.k, g.m, nullptr, nullptr, r.rmax, r.rneg, r.flag, s,
             nlaunch, canon);
  if (e != cudaSuccess) return e;
  if (g.syrk == 0) {
    // op(B) is k x n: stored k x n (N) or n x k (T)
    if (g.tb == 0)
      e = scan(g.b_hi, g.b_lo, g.ldb, g.k, g.n, nullptr, nullptr, r.cmax, r.cneg, r.flag, s,
               nlaunch, canon);
    else
      e = scan(g.b_hi, g.b_lo, g.ldb, g.n, g.k, r.cmax, r.cneg, nullptr, nullptr, r.flag, s,
               nlaunch, canon);
    if (e != cudaSuccess) return e;
  }
  // The exact kernel's axpy form (transa = 'N') starts its unchecked
  // accumulation from beta*C, so C must be in the window too.
  if (alg == ALG_EXACT && g.ta == 0 && !(g.beta.h == 0.0 && g.beta.l == 0.0)) {
    // Rsyrk: only the uplo triangle is ever read (level23.py:245-246)
    e = scan(g.c_hi, g.c_lo, g.ldc, g.m, g.n, nullptr, r.rneg, nullptr, nullptr, r.flag, s,
             nlaunch, 0, g.syrk, 1);
    if (e != cudaSuccess) return e;
  }
  const int64_t nr_pad = (g.m + 31) / 32 * 32;
  const int64_t nc = g.syrk ? 0 : g.n;
  const int64_t total = nr_pad + nc;
  route_summary_kernel<<<(unsigned)((total + 255) / 256), 256, 0, s>>>(
      r.rmax, r.rneg, r.rsp, r.rsb, g.m, nr_pad, r.cmax, r.cneg, r.csp, r.csb, nc, r.flag,
      g.syrk != 0, r.bad_rows, r.bad_cols);
  ++*nlaunch;
  return cudaGetLastError();
}

}  // namespace ddb
