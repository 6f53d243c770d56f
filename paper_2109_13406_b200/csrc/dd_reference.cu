// dd_reference.cu -- reference-semantics kernel: one thread per C element,
// operands read straight from HBM, every dd operation in its checked form
// (Dekker TwoProd + the reference's finiteness fix-ups).
//
// It is the complete per-element restatement of the reference:
//   alpha == 0        level23.py:110-115  (_gemm_core) / :247-249 (Rsyrk)
//   transa = 'N'      level23.py:120-125, :134-140  (beta rule, then
//                     c = add2(c, mul2(A(i,l), mul2(alpha, op(B)(l,j)))))
//   transa = 'T'/'C'  level23.py:126-133, :141-149  (acc from 0, _combine)
//   Rsyrk             level23.py:226-285 == NT / TN Rgemm with B = A, only
//                     the uplo triangle written
// and runs for the elements whose op(A) row or op(B) column holds a value
// outside the safe window (inf, nan, |x| >= 2**301, 0 < |hi| < 2**-300;
// dd_prescan.cu routes per element), for alpha == 0, for k == 0, and for
// mode DDB_MODE_REFERENCE.  It is not the fast path: throughput is a
// few percent of the tiled kernels (dd_gemm.cu).
#include "internal.h"

namespace ddb {

// One element of C with the reference's own semantics.
__device__ __forceinline__ void reference_elem(const GemmArgs& g, int64_t i, int64_t j,
                                               bool alpha_zero) {
  const int64_t ci = i + j * g.ldc;
  const dd c0{g.c_hi[ci], g.c_lo[ci]};
  dd out;
  if (alpha_zero) {
    if (dd_is_one(g.beta)) return;
    out = scale_beta(g.beta, c0);
  } else if (g.ta == 0) {
    dd c = g.sub ? c0 : scale_beta(g.beta, c0);
    for (int64_t l = 0; l < g.k; ++l) {
      const int64_t bi = g.tb == 0 ? l + j * g.ldb : j + l * g.ldb;
      const dd b{g.b_hi[bi], g.b_lo[bi]};
      const int64_t ai = i + l * g.lda;
      if (g.sub) {   // be.sub(c, be.mul(a, b)) (level23.py:334-336)
        const dd p = mul2_chk(dd{g.a_hi[ai], g.a_lo[ai]}, b);
        c = add2_chk(c, dd{-p.h, -p.l});
      } else {
        c = add2_chk(c, mul2_chk(dd{g.a_hi[ai], g.a_lo[ai]}, mul2_chk(g.alpha, b)));
      }
    }
    out = c;
  } else {
    dd acc{0.0, 0.0};
    for (int64_t l = 0; l < g.k; ++l) {
      const int64_t bi = g.tb == 0 ? l + j * g.ldb : j + l * g.ldb;
      const int64_t ai = l + i * g.lda;
      acc = add2_chk(acc, mul2_chk(dd{g.a_hi[ai], g.a_lo[ai]}, dd{g.b_hi[bi], g.b_lo[bi]}));
    }
    out = combine(g.alpha, acc, g.beta, c0);
  }
  g.c_hi[ci] = out.h;
  g.c_lo[ci] = out.l;
}

// GATE_ALWAYS: every element (2-D grid).  GATE_IF_UNSAFE: only the EC_REF
// elements: the rows of C whose op(A) row holds an unsafe word and the
// columns whose op(B) column does (the prescan's lists, dd_prescan.cu),
// walked as R*n + C*m virtual elements so that the elements of one routed
// row or column land on consecutive threads; exits at once when the call has
// none.
__global__ void __launch_bounds__(256)
reference_kernel(GemmArgs g, const int* __restrict__ flag, int gate) {
  const bool alpha_zero = dd_is_zero(g.alpha);
  if (gate == GATE_IF_UNSAFE) {
    if (flag[0] == ROUTE_SAFE) return;
    const int64_t R = flag[3], Cn = g.syrk ? flag[3] : flag[4];
    const int* cols = g.syrk ? g.bad_rows : g.bad_cols;
    const int64_t total = R * g.n + Cn * g.m, stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
      int64_t i, j;
      if (t < R * g.n) {
        i = g.bad_rows[t / g.n];
        j = t % g.n;
      } else {
        const int64_t u = t - R * g.n;
        j = cols[u / g.m];
        i = u % g.m;
        if (g.rsp[i] >= SPREAD_BAD) continue;   // its row is walked above
      }
      if (g.syrk == 1 && i > j) continue;
      if (g.syrk == 2 && i < j) continue;
      reference_elem(g, i, j, alpha_zero);
    }
    return;
  }
  for (int64_t i = (int64_t)blockIdx.x * 32 + threadIdx.x; i < g.m; i += (int64_t)gridDim.x * 32)
  for (int64_t j = (int64_t)blockIdx.y * 8 + threadIdx.y; j < g.n; j += (int64_t)gridDim.y * 8) {
    if (g.syrk == 1 && i > j) continue;
    if (g.syrk == 2 && i < j) continue;
    reference_elem(g, i, j, alpha_zero);
  }
}

// Binary64 precision (the F64 backend, elem.py:149-197): the same loop orders
// with plain IEEE operations; used for alpha == 0 and k == 0.
__global__ void __launch_bounds__(256) reference_f64_kernel(GemmArgs g) {
  const int64_t i = (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (i >= g.m) return;
  const double alpha = g.alpha.h, beta = g.beta.h;
  for (int64_t j = (int64_t)blockIdx.y * 8 + threadIdx.y; j < g.n; j += (int64_t)gridDim.y * 8) {
    if (g.syrk == 1 && i > j) continue;
    if (g.syrk == 2 && i < j) continue;
    const int64_t ci = i + j * g.ldc;
    const double c0 = g.c_hi[ci];
    double out;
    if (alpha == 0.0) {
      if (beta == 1.0) continue;
      out = beta == 0.0 ? 0.0 : dmul(beta, c0);
    } else if (g.ta == 0) {
      double c = beta == 0.0 ? 0.0 : (beta == 1.0 ? c0 : dmul(beta, c0));
      for (int64_t l = 0; l < g.k; ++l) {
        const int64_t bi = g.tb == 0 ? l + j * g.ldb : j + l * g.ldb;
        c = dadd(c, dmul(g.a_hi[i + l * g.lda], dmul(alpha, g.b_hi[bi])));
      }
      out = c;
    } else {
      double acc = 0.0;
      for (int64_t l = 0; l < g.k; ++l) {
        const int64_t bi = g.tb == 0 ? l + j * g.ldb : j + l * g.ldb;
        acc = dadd(acc, dmul(g.a_hi[l + i * g.lda], g.b_hi[bi]));
      }
      const double at = dmul(alpha, acc);
      out = beta == 0.0 ? at : dadd(at, dmul(beta, c0));
    }
    g.c_hi[ci] = out;
  }
}

cudaError_t launch_reference(const GemmArgs& g, const int* flag, int gate, cudaStream_t s,
                             int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  if (g.f64) {
    const int64_t gx = (g.m + 31) / 32;
    int64_t gy = (g.n + 7) / 8;
    if (gy > 65535) gy = 65535;
    reference_f64_kernel<<<dim3((unsigned)gx, (unsigned)gy), dim3(32, 8), 0, s>>>(g);
    ++*nlaunch;
    return cudaGetLastError();
  }
  if (gate == GATE_IF_UNSAFE) {
    // flat walk: 8 CTAs of 256 threads per SM, at most one thread per element
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    int64_t blocks = (g.m * g.n + 255) / 256;
    if (blocks > 8 * (int64_t)sms) blocks = 8 * (int64_t)sms;
    reference_kernel<<<(unsigned)blocks, 256, 0, s>>>(g, flag, gate);
    ++*nlaunch;
    return cudaGetLastError();
  }
  const int64_t cap_x = INT32_MAX, cap_y = 65535;
  int64_t gx = (g.m + 31) / 32;
  int64_t gy = (g.n + 7) / 8;
  if (gx > cap_x) gx = cap_x;
  if (gy > cap_y) gy = cap_y;
  dim3 grid((unsigned)gx, (unsigned)gy), block(32, 8);
  reference_kernel<<<grid, block, 0, s>>>(g, flag, gate);
  ++*nlaunch;
  return cudaGetLastError();
}

}  // namespace ddb
