// dd_gemm.cu -- tiled sm_100a dd GEMM / SYRK kernels on the FP64 pipe.
//
// One CTA computes a BM x BN = 128 x 64 tile of C; 256 threads, each owning
// an 8 x 4 register micro-tile.  op(A) / op(B) k-slices of BK = 16 are staged
// hi + lo planes through shared memory by a 3-stage cp.async pipeline
// (8-byte copies: any lda / ldb / alignment, any transpose -- the copy
// scatters each double to its k-major smem slot, so every trans variant reads
// smem the same way).  Tensor cores are not used: tcgen05 has no fp64 kind
// and DMMA rounds away the per-product error terms dd needs.
//
// Two accumulation modes (template MODE):
//
//  * MODE_EXACT -- bit-identical to the reference.  Per element exactly the
//    reference's sequence (level23.py:120-149): transa='N' starts from the
//    beta-scaled C and adds mul2(A(i,l), t_l) with t = mul2(alpha, op(B)) (t is
//    formed once per smem tile with the checked Dekker product); transa='T'
//    accumulates add2(acc, mul2(A(l,i), op(B)(l,j))) from zero and applies
//    _combine.  Inner loop: add2_nc(mul2_nc) = 29 FP64 instructions per MAC,
//    valid bit-for-bit inside the prescan's safe window (dd_arith.cuh).
//
//  * MODE_FAST -- error-bounded "anchored" accumulation, 6 FP64 instructions
//    per MAC.  Each element keeps T (offset-anchored hi part) and L (tail):
//        Tn = fma(ah, bh, T)       // T + ah*bh rounded onto T's fixed grid
//        d  = T - Tn               // exact (Sterbenz: Tn in [T/2, 2T])
//        r  = fma(ah, bh, d)       // = ah*bh - (Tn - T): the exact rounding
//                                  //   residual of T + ah*bh, rounded once
//        L  = fma(ah, bl, L); L = fma(al, bh, L); L += r;  T = Tn
//    T is kept inside [1.25, 1.75] * 2**E with sigma = 1.5 * 2**E, where E is
//    chosen (every KB = 32 k-steps, "re-anchor") so that |running sum| + the
//    next block's bound KB * 2**(row_exp + col_exp - 2044) <= 2**(E-2).  Then
//    T - sigma is exact, every Fast2Sum above is exact, and the only
//    roundings are r's and L's: the per-element error is bounded like a dd
//    accumulation, far inside c*k*2**-104 * sum|a*b| ("fast mode
//    error").  At each re-anchor T - sigma and L are folded onto the new grid
//    with two Fast2Sums, so |L| stays below one grid step.  The epilogue is
//    C = add2(mul2(alpha, acc), beta-rule(C)) in checked dd arithmetic.
//
// Rsyrk (SYRK = 1 upper / 2 lower) is NT (trans='N') or TN (trans='T')
// Rgemm with B = A: tiles fully outside the triangle exit at once, diagonal
// tiles mask their stores, so the opposite triangle is never written
// (level23.py:245-285).
#include "internal.h"

namespace ddb {

constexpr int BM = 128, BN = 64, BK = 16, NT = 256, STAGES = 3;
constexpr int ASTR = BM + 2, BSTR = BN + 2;        // smem row strides (doubles)
constexpr int A_STAGE = 2 * BK * ASTR, B_STAGE = 2 * BK * BSTR;
constexpr size_t SMEM_BYTES = (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double);
constexpr int RB = 2;                              // k-tiles per anchor block
constexpr int LG_KB = 5;                           // log2(RB * BK)
constexpr int GROUP_M = 8;                         // raster group (L2 reuse)

__device__ __forceinline__ void cp_async8(double* dst, const double* src, bool valid) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(d), "l"(src),
               "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ long long dbits(double x) { return __double_as_longlong(x); }
__device__ __forceinline__ double bitsd(long long x) { return __longlong_as_double(x); }

// sigma = 1.5 * 2**E for the binade T lives in (T > 0 always)
__device__ __forceinline__ double anchor_of(double T) {
  return bitsd((dbits(T) & 0x7ff0000000000000LL) | 0x0008000000000000LL);
}
__device__ __forceinline__ double anchor_from_bexp(int eb) {
  eb = eb < 64 ? 64 : (eb > 2000 ? 2000 : eb);
  return bitsd(((long long)eb << 52) | 0x0008000000000000LL);
}

template <int TA, int TB>
__device__ __forceinline__ void load_stage(const GemmArgs& g, double* sA, double* sB,
                                           int64_t i0, int64_t j0, int64_t l0, int tid) {
  // op(A) tile: BM x BK -> sA[plane][kk][ii]
#pragma unroll
  for (int r = 0; r < BM * BK / NT; ++r) {
    const int idx = tid + r * NT;
    int ii, kk;
    if (TA == 0) { ii = idx % BM; kk = idx / BM; } else { kk = idx % BK; ii = idx / BK; }
    const int64_t gi = i0 + ii, gl = l0 + kk;
    const bool v = gi < g.m && gl < g.k;
    const int64_t off = v ? (TA == 0 ? gi + gl * g.lda : gl + gi * g.lda) : 0;
    cp_async8(sA + kk * ASTR + ii, g.a_hi + off, v);
    cp_async8(sA + BK * ASTR + kk * ASTR + ii, g.a_lo + off, v);
  }
  // op(B) tile: BK x BN -> sB[plane][kk][jj]
#pragma unroll
  for (int r = 0; r < BN * BK / NT; ++r) {
    const int idx = tid + r * NT;
    int jj, kk;
    if (TB == 0) { kk = idx % BK; jj = idx / BK; } else { jj = idx % BN; kk = idx / BN; }
    const int64_t gj = j0 + jj, gl = l0 + kk;
    const bool v = gj < g.n && gl < g.k;
    const int64_t off = v ? (TB == 0 ? gl + gj * g.ldb : gj + gl * g.ldb) : 0;
    cp_async8(sB + kk * BSTR + jj, g.b_hi + off, v);
    cp_async8(sB + BK * BSTR + kk * BSTR + jj, g.b_lo + off, v);
  }
}

template <int TA, int TB, int MODE, int SYRK>
__global__ void __launch_bounds__(NT, 1)
dd_tiled_kernel(GemmArgs g, const int* __restrict__ row_exp, const int* __restrict__ col_exp,
                const int* __restrict__ flag, int tiles_m, int tiles_n) {
  if (*flag != ROUTE_SAFE) return;  // dd_reference.cu handles this call

  // grouped raster over the tile grid
  const int bid = blockIdx.x;
  const int group_size = GROUP_M * tiles_n;
  const int first_m = (bid / group_size) * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int local = bid % group_size;
  const int bm = first_m + local % gm, bn = local / gm;
  const int64_t i0 = (int64_t)bm * BM, j0 = (int64_t)bn * BN;
  if (SYRK == 1 && i0 > j0 + BN - 1) return;   // tile entirely below the diagonal
  if (SYRK == 2 && i0 + BM - 1 < j0) return;   // tile entirely above the diagonal

  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * A_STAGE;

  const int tid = threadIdx.x;
  const int tx = tid & 15, ty = tid >> 4;
  // rows i = g*32 + tx*2 + q (g<4, q<2); cols j = g*32 + ty*2 + q (g<2, q<2)

  double acc_h[8][4], acc_l[8][4];   // exact: (c_h, c_l);  fast: (T, L)
  int eb_row[8], eb_col[4];

  if (MODE == MODE_FAST) {
#pragma unroll
    for (int a = 0; a < 8; ++a) {
      const int64_t gi = i0 + (a >> 1) * 32 + tx * 2 + (a & 1);
      eb_row[a] = gi < g.m ? row_exp[gi] : 0;
    }
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gj = j0 + (b >> 1) * 32 + ty * 2 + (b & 1);
      eb_col[b] = gj < g.n ? col_exp[gj] : 0;
    }
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        acc_h[a][b] = anchor_from_bexp(eb_row[a] + eb_col[b] - 1018 + LG_KB);
        acc_l[a][b] = 0.0;
      }
  } else {
#pragma unroll
    for (int a = 0; a < 8; ++a)
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        acc_h[a][b] = 0.0;
        acc_l[a][b] = 0.0;
        if (TA == 0) {  // axpy form: start from the beta-scaled C (_scale_full)
          const int64_t gi = i0 + (a >> 1) * 32 + tx * 2 + (a & 1);
          const int64_t gj = j0 + (b >> 1) * 32 + ty * 2 + (b & 1);
          if (gi < g.m && gj < g.n) {
            const dd c = scale_beta(g.beta, dd{g.c_hi[gi + gj * g.ldc], g.c_lo[gi + gj * g.ldc]});
            acc_h[a][b] = c.h;
            acc_l[a][b] = c.l;
          }
        }
      }
  }

  const int ktiles = (int)((g.k + BK - 1) / BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage<TA, TB>(g, sA + s * A_STAGE, sB + s * B_STAGE, i0, j0, (int64_t)s * BK, tid);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    {
      const int nk = kt + STAGES - 1;
      const int ns = nk % STAGES;
      if (nk < ktiles) load_stage<TA, TB>(g, sA + ns * A_STAGE, sB + ns * B_STAGE, i0, j0, (int64_t)nk * BK, tid);
      cp_async_commit();
    }
    const int st = kt % STAGES;
    const double* a_h = sA + st * A_STAGE;
    const double* a_l = a_h + BK * ASTR;
    double* b_h = sB + st * B_STAGE;
    double* b_l = b_h + BK * BSTR;

    if (MODE == MODE_EXACT && TA == 0) {
      // t = mul2(alpha, op(B)(l, j)), once per tile element (level23.py:122, :137)
#pragma unroll
      for (int r = 0; r < BN * BK / NT; ++r) {
        const int idx = tid + r * NT;
        const int kk = idx / BN, jj = idx % BN;
        const dd t = mul2_chk(g.alpha, dd{b_h[kk * BSTR + jj], b_l[kk * BSTR + jj]});
        b_h[kk * BSTR + jj] = t.h;
        b_l[kk * BSTR + jj] = t.l;
      }
      __syncthreads();
    }

    int kcount = BK;
    if (MODE == MODE_EXACT) {
      const int64_t rem = g.k - (int64_t)kt * BK;
      kcount = rem < BK ? (int)rem : BK;   // exact: never run a padded k-step
    }

#pragma unroll 2
    for (int kk = 0; kk < kcount; ++kk) {
      double ah[8], al[8], bh[4], bl[4];
#pragma unroll
      for (int gq = 0; gq < 4; ++gq) {
        const double2 vh = *reinterpret_cast<const double2*>(a_h + kk * ASTR + gq * 32 + tx * 2);
        const double2 vl = *reinterpret_cast<const double2*>(a_l + kk * ASTR + gq * 32 + tx * 2);
        ah[2 * gq] = vh.x; ah[2 * gq + 1] = vh.y;
        al[2 * gq] = vl.x; al[2 * gq + 1] = vl.y;
      }
#pragma unroll
      for (int gq = 0; gq < 2; ++gq) {
        const double2 vh = *reinterpret_cast<const double2*>(b_h + kk * BSTR + gq * 32 + ty * 2);
        const double2 vl = *reinterpret_cast<const double2*>(b_l + kk * BSTR + gq * 32 + ty * 2);
        bh[2 * gq] = vh.x; bh[2 * gq + 1] = vh.y;
        bl[2 * gq] = vl.x; bl[2 * gq + 1] = vl.y;
      }
      if (MODE == MODE_FAST) {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const double T = acc_h[a][b];
            const double Tn = dfma(ah[a], bh[b], T);
            const double d = dsub(T, Tn);
            const double r = dfma(ah[a], bh[b], d);
            double L = dfma(ah[a], bl[b], acc_l[a][b]);
            L = dfma(al[a], bh[b], L);
            acc_l[a][b] = dadd(L, r);
            acc_h[a][b] = Tn;
          }
      } else {
#pragma unroll
        for (int a = 0; a < 8; ++a)
#pragma unroll
          for (int b = 0; b < 4; ++b) {
            const dd p = mul2_nc(dd{ah[a], al[a]}, dd{bh[b], bl[b]});
            const dd c = add2_nc(dd{acc_h[a][b], acc_l[a][b]}, p);
            acc_h[a][b] = c.h;
            acc_l[a][b] = c.l;
          }
      }
    }

    if (MODE == MODE_FAST && ((kt + 1) % RB) == 0 && kt + 1 < ktiles) {
      // re-anchor: fold (T - sigma) and L onto a grid sized for the running
      // sum plus the next KB-step block
#pragma unroll
      for (int a = 0; a < 8; ++a)
#pragma unroll
        for (int b = 0; b < 4; ++b) {
          const double T = acc_h[a][b];
          const double h = dsub(T, anchor_of(T));          // exact
          const int eh = (int)((dbits(h) >> 52) & 0x7ff);
          const int e_blk = eb_row[a] + eb_col[b] - 1018 + LG_KB;
          const double sg = anchor_from_bexp(max(eh + 4, e_blk));
          const double T2 = dadd(sg, h);
          const double e1 = dsub(h, dsub(T2, sg));          // exact (Fast2Sum)
          const double L = acc_l[a][b];
          const double T3 = dadd(T2, L);
          const double e2 = dsub(L, dsub(T3, T2));          // exact (Fast2Sum)
          acc_h[a][b] = T3;
          acc_l[a][b] = dadd(e1, e2);
        }
    }
  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int a = 0; a < 8; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) {
      const int64_t gi = i0 + (a >> 1) * 32 + tx * 2 + (a & 1);
      const int64_t gj = j0 + (b >> 1) * 32 + ty * 2 + (b & 1);
      if (gi >= g.m || gj >= g.n) continue;
      if (SYRK == 1 && gi > gj) continue;
      if (SYRK == 2 && gi < gj) continue;
      const int64_t ci = gi + gj * g.ldc;
      dd out;
      if (MODE == MODE_FAST) {
        const double T = acc_h[a][b];
        const double h = dsub(T, anchor_of(T));
        double s, e;
        two_sum(h, acc_l[a][b], s, e);
        const dd at = mul2_chk(g.alpha, dd{s, e});
        out = add2_chk(at, scale_beta(g.beta, dd{g.c_hi[ci], g.c_lo[ci]}));
      } else if (TA == 0) {
        out = dd{acc_h[a][b], acc_l[a][b]};
      } else {
        out = combine(g.alpha, dd{acc_h[a][b], acc_l[a][b]}, g.beta, dd{g.c_hi[ci], g.c_lo[ci]});
      }
      g.c_hi[ci] = out.h;
      g.c_lo[ci] = out.l;
    }
}

template <int TA, int TB, int MODE, int SYRK>
static cudaError_t launch_one(const GemmArgs& g, const int* row_exp, const int* col_exp,
                              const int* flag, cudaStream_t s) {
  auto kern = dd_tiled_kernel<TA, TB, MODE, SYRK>;
  // per-device attribute: set on every call (cheap, idempotent, thread-safe)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (int)((g.m + BM - 1) / BM), tiles_n = (int)((g.n + BN - 1) / BN);
  kern<<<tiles_m * tiles_n, NT, SMEM_BYTES, s>>>(g, row_exp, col_exp, flag, tiles_m, tiles_n);
  return cudaGetLastError();
}

cudaError_t launch_tiled(const GemmArgs& g, int mode, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  ++*nlaunch;
  const bool fast = mode == MODE_FAST;
  if (g.syrk == 0) {
    const int v = g.ta * 2 + g.tb;
    if (fast) {
      switch (v) {
        case 0: return launch_one<0, 0, MODE_FAST, 0>(g, row_exp, col_exp, flag, s);
        case 1: return launch_one<0, 1, MODE_FAST, 0>(g, row_exp, col_exp, flag, s);
        case 2: return launch_one<1, 0, MODE_FAST, 0>(g, row_exp, col_exp, flag, s);
        default: return launch_one<1, 1, MODE_FAST, 0>(g, row_exp, col_exp, flag, s);
      }
    }
    switch (v) {
      case 0: return launch_one<0, 0, MODE_EXACT, 0>(g, row_exp, col_exp, flag, s);
      case 1: return launch_one<0, 1, MODE_EXACT, 0>(g, row_exp, col_exp, flag, s);
      case 2: return launch_one<1, 0, MODE_EXACT, 0>(g, row_exp, col_exp, flag, s);
      default: return launch_one<1, 1, MODE_EXACT, 0>(g, row_exp, col_exp, flag, s);
    }
  }
  // Rsyrk: trans 'N' == NT with B = A, trans 'T' == TN with B = A
  const bool up = g.syrk == 1;
  if (g.ta == 0) {
    if (fast) return up ? launch_one<0, 1, MODE_FAST, 1>(g, row_exp, col_exp, flag, s)
                        : launch_one<0, 1, MODE_FAST, 2>(g, row_exp, col_exp, flag, s);
    return up ? launch_one<0, 1, MODE_EXACT, 1>(g, row_exp, col_exp, flag, s)
              : launch_one<0, 1, MODE_EXACT, 2>(g, row_exp, col_exp, flag, s);
  }
  if (fast) return up ? launch_one<1, 0, MODE_FAST, 1>(g, row_exp, col_exp, flag, s)
                      : launch_one<1, 0, MODE_FAST, 2>(g, row_exp, col_exp, flag, s);
  return up ? launch_one<1, 0, MODE_EXACT, 1>(g, row_exp, col_exp, flag, s)
            : launch_one<1, 0, MODE_EXACT, 2>(g, row_exp, col_exp, flag, s);
}

}  // namespace ddb
