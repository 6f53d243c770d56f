// dd_tiled.cuh -- tiled sm_100a dd GEMM / SYRK kernel template (FP64 pipe).
//
// One CTA computes a BM x BN = 128 x 64 tile of C with 256 threads, each
// owning an 8 x 4 register micro-tile (rows g*32 + tx*2 + q, cols
// g*32 + ty*2 + q).  op(A) / op(B) k-slices of BK = 16 are staged (hi and lo
// planes) through shared memory by a 3-stage cp.async pipeline.  8-byte
// copies handle any lda / ldb / alignment / transpose: each double lands in
// its k-major smem slot, so every trans variant reads smem identically with
// 16-byte LDS.  The dd MAC stays on the FP64 pipe: tcgen05 has no fp64 kind
// and DMMA rounds away the per-product error terms dd needs (the fast mode's
// auxiliary cross-term and bound GEMMs do use DMMA / tcgen05: dd_cross.cu,
// dd_bound.cu).
//
// Accumulation algorithms (template ALG), per output element:
//
//  ALG_EXACT  -- the reference's own sequence, bit for bit (level23.py:120-149):
//      transa='N': c = beta-rule(C); c = add2(c, mul2(A(i,l), t_l)),
//                  t = mul2(alpha, op(B)(l,j)) formed once per smem tile;
//      transa='T': acc = add2(acc, mul2(A(l,i), op(B)(l,j))) from 0, _combine.
//      add2_nc(mul2_nc) = 29 FP64-pipe instructions per MAC.
//
//  ALG_TWOSUM -- error-bounded dd accumulation, (S, L) per element:
//      p = ah*bh; e = fma(ah,bh,-p) + ah*bl + al*bh (two more fma);
//      (S, t) = TwoSum(S, p) [Knuth, 6 ops]; L += t + e;
//      every RN = 8 steps (S, L) = QuickTwoSum(S, L).   ~12.4 FP64 / MAC.
//
//  ALG_SELECT -- as TWOSUM but the sum error comes from a Fast2Sum whose
//      operands are ordered by an integer compare of |S| and |p| (the ALU
//      pipe, which the FP64-bound loop leaves idle): s = S + p;
//      t = small - (s - big).  ~9.4 FP64 + 8 ALU / MAC.
//      Both fast variants: |L| <= (RN + 4) u sum|ab|, so the rounding error
//      per step is <= (RN + 4) u^2 sum|ab| < 16 u^2 sum|ab| = 2^-102 sum|ab|,
//      i.e. inside c*k*2^-104*sum|ab| with c = 4 for every in-window input.
//
//  ALG_CERT   -- certified-anchor accumulation (the fast mode), 7.5 FP64/MAC:
//      T = sigma + running sum, sigma = 1.5*2^E with 2^E >= 2*Sigma'_ij, where
//      Sigma'_ij >= sum_l |a_il b_lj| is the certified bound of dd_bound.cu.
//      Every partial sum then keeps T inside [2^E, 2^(E+1)), so
//        Tn = fma(ah, bh, T)        T + ah*bh rounded onto T's fixed grid
//        r  = fma(ah, bh, T - Tn)   its rounding residual (T - Tn is exact)
//        L  = fma(al, bh, fma(ah, bl, L)) + r
//      and every RF = 2 steps L is folded into T with a Fast2Sum (exact).
//      With 2^E < 4 Sigma' the per-step error is <= 14 u^2 Sigma' < 2^-102
//      Sigma' (u = 2^-53): inside c*k*2^-104*sum|ab| (c = 4) for every input
//      in the safe window, like TWOSUM, at 7.5 instead of 12.4 instructions.
//
// Rsyrk (SYRK = 1 upper / 2 lower) is NT (trans='N') or TN (trans='T') Rgemm
// with B = A: tiles fully outside the triangle exit at once, diagonal tiles
// mask their stores (level23.py:245-285).
#pragma once
#include "internal.h"

namespace ddb {

namespace tiled {

// Tile configuration: NT threads as NX (along m) x NT/NX (along n), each
// owning a TM x TN micro-tile (TM, TN even) at rows g*2NX + tx*2 + q and
// columns g*2NY + ty*2 + q; MINB CTAs per SM (registers 65536/(NT*MINB)).
// PF: double-buffer the next k-step's operands in registers.
template <int TM_, int TN_, int MINB_, int NT_ = 256, int NX_ = 16, int PF_ = 1>
struct Cfg {
  static constexpr int TM = TM_, TN = TN_, MINB = MINB_, NT = NT_, NX = NX_, NY = NT_ / NX_;
  static constexpr int PF = PF_;
  static constexpr int BM = NX * TM, BN = NY * TN, BK = 16, STAGES = 3;
  static constexpr int ASTR = BM + 2, BSTR = BN + 2;   // smem row strides (doubles)
  static constexpr int A_STAGE = 2 * BK * ASTR, B_STAGE = 2 * BK * BSTR;
  static constexpr size_t SMEM_BYTES =
      (size_t)STAGES * (A_STAGE + B_STAGE) * sizeof(double) + (BM + BN) * sizeof(int);
};
using CfgBig = Cfg<8, 4, 1>;                 // 128 x 64 tile, 8 warps / SM
using CfgSmall = Cfg<4, 4, 2, 256, 16, 0>;   // 64 x 64 tile, 2 CTAs: 16 warps / SM
using CfgWide = Cfg<4, 4, 1, 512, 32, 0>;    // 128 x 64 tile, 16 warps / SM

constexpr int BK = 16;
#ifndef DDB_PHASE
#define DDB_PHASE 0      // phase-ordered CERT MAC step (experiment switch)
#endif
#ifndef DDB_ABLATE
#define DDB_ABLATE 0     // measurement-only ablations (wrong results): 1 = operands of
                         // step 0 reused for the whole k-tile, 2 = skip the k-tile
                         // loads + barrier after the first tile
#endif
#ifndef DDB_EXACT_SEL
#define DDB_EXACT_SEL 0  // exact mode: ordered-Fast2Sum TwoSums (bit-identical, 23 vs 29 ops)
#endif
#ifndef DDB_UNR
#define DDB_UNR 16       // fast modes: k-steps per loop body (divides BK, multiple of RF)
#endif
#ifndef DDB_PREFETCH
#define DDB_PREFETCH 1   // fast modes: load step kk+1's operands before step kk's math
#endif
constexpr int RN = 8;                              // fast: renormalise every RN steps
constexpr int RF = 2;                              // cert: fold L into T every RF steps
constexpr int GROUP_M = 4;    // raster group height: 4 -> 34 GB of DRAM reads at 8192^3, 12 -> 81 GB (scripts/dram_sweep.sh)

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

// cert: sigma = 1.5 * 2**E for the binade T lives in (T > 0 always)
__device__ __forceinline__ double anchor_of(double T) {
  return bitsd((dbits(T) & 0x7ff0000000000000LL) | 0x0008000000000000LL);
}
__device__ __forceinline__ double anchor_from_bexp(int eb) {
  eb = eb < 64 ? 64 : (eb > 2000 ? 2000 : eb);
  return bitsd(((long long)eb << 52) | 0x0008000000000000LL);
}

// |x| >= |y| on the bit patterns (integer pipe): IEEE order of magnitudes.
// The sign bit is cleared with a 32-bit LOP3 in inline PTX: written in C the
// 64-bit mask is recognised as fabs and lowered to a DADD on the FP64 pipe.
__device__ __forceinline__ unsigned long long abs_bits(double x) {
  unsigned long long r;
  asm("{\n\t.reg .b32 lo, hi;\n\tmov.b64 {lo, hi}, %1;\n\t"
      "and.b32 hi, hi, 0x7fffffff;\n\tmov.b64 %0, {lo, hi};\n\t}"
      : "=l"(r) : "d"(x));
  return r;
}
__device__ __forceinline__ bool abs_ge(double x, double y) { return abs_bits(x) >= abs_bits(y); }

template <class C, int TA, int TB, bool LO = true>
__device__ __forceinline__ void load_stage(const GemmArgs& g, double* sA, double* sB,
                                           int64_t i0, int64_t j0, int64_t l0, int64_t kend,
                                           int tid) {
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT, ASTR = C::ASTR, BSTR = C::BSTR;
  // op(A) tile: BM x BK -> sA[plane][kk][ii]
#pragma unroll
  for (int r = 0; r < BM * BK / NT; ++r) {
    const int idx = tid + r * NT;
    int ii, kk;
    if (TA == 0) { ii = idx % BM; kk = idx / BM; } else { kk = idx % BK; ii = idx / BK; }
    const int64_t gi = i0 + ii, gl = l0 + kk;
    const bool v = gi < g.m && gl < kend;
    const int64_t off = v ? (TA == 0 ? gi + gl * g.lda : gl + gi * g.lda) : 0;
    cp_async8(sA + kk * ASTR + ii, g.a_hi + off, v);
    if (LO) cp_async8(sA + BK * ASTR + kk * ASTR + ii, g.a_lo + off, v);
  }
  // op(B) tile: BK x BN -> sB[plane][kk][jj]
#pragma unroll
  for (int r = 0; r < BN * BK / NT; ++r) {
    const int idx = tid + r * NT;
    int jj, kk;
    if (TB == 0) { kk = idx % BK; jj = idx / BK; } else { jj = idx % BN; kk = idx / BN; }
    const int64_t gj = j0 + jj, gl = l0 + kk;
    const bool v = gj < g.n && gl < kend;
    const int64_t off = v ? (TB == 0 ? gl + gj * g.ldb : gj + gl * g.ldb) : 0;
    cp_async8(sB + kk * BSTR + jj, g.b_hi + off, v);
    if (LO) cp_async8(sB + BK * BSTR + kk * BSTR + jj, g.b_lo + off, v);
  }
}

template <int ALG, int TM, int TN, bool SUB = false>
__device__ __forceinline__ void mac_step(double (&H)[TM][TN], double (&L)[TM][TN],
                                         const double (&ah)[TM], const double (&al)[TM],
                                         const double (&bh)[TN], const double (&bl)[TN]) {
  if (ALG == ALG_CERT && DDB_PHASE) {
    // phase-ordered so that consecutive FP64 instructions are independent
    // (each phase touches all TM*TN elements before the next phase starts)
    double D[TM][TN];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        const double Tn = dfma(ah[a], bh[b], H[a][b]);
        D[a][b] = dsub(H[a][b], Tn);
        H[a][b] = Tn;
      }
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) L[a][b] = dfma(ah[a], bl[b], L[a][b]);
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) D[a][b] = dfma(ah[a], bh[b], D[a][b]);
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) L[a][b] = dfma(al[a], bh[b], L[a][b]);
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) L[a][b] = dadd(L[a][b], D[a][b]);
    return;
  }
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      if (ALG == ALG_F64) {     // f64: c = c + a*t (NN) / acc = acc + a*b (TN), unfused
        H[a][b] = dadd(H[a][b], dmul(ah[a], bh[b]));
      } else if (ALG == ALG_CERT) {
        const double T = H[a][b];
        const double Tn = dfma(ah[a], bh[b], T);
        const double r = dfma(ah[a], bh[b], dsub(T, Tn));
        double l = dfma(ah[a], bl[b], L[a][b]);
        l = dfma(al[a], bh[b], l);
        L[a][b] = dadd(l, r);
        H[a][b] = Tn;
      } else if (ALG == ALG_EXACT) {
        dd p = mul2_nc(dd{ah[a], al[a]}, dd{bh[b], bl[b]});
        if (SUB) p = dd{-p.h, -p.l};
        const dd c = DDB_EXACT_SEL ? add2_nc_sel(dd{H[a][b], L[a][b]}, p)
                                   : add2_nc(dd{H[a][b], L[a][b]}, p);
        H[a][b] = c.h;
        L[a][b] = c.l;
      } else {
        const double p = dmul(ah[a], bh[b]);
        double e = dfma(ah[a], bh[b], -p);
        e = dfma(ah[a], bl[b], e);
        e = dfma(al[a], bh[b], e);
        const double S = H[a][b];
        const double s = dadd(S, p);
        double t;
        if (ALG == ALG_TWOSUM) {
          const double bb = dsub(s, S);
          t = dadd(dsub(S, dsub(s, bb)), dsub(p, bb));
        } else {
          const bool ge = abs_ge(S, p);
          const double big = ge ? S : p, small = ge ? p : S;
          t = dsub(small, dsub(s, big));
        }
        L[a][b] = dadd(L[a][b], dadd(t, e));
        H[a][b] = s;
      }
    }
}

template <class C, int TA, int TB, int ALG, int SYRK>
__global__ void __launch_bounds__(C::NT, C::MINB)
dd_tiled_kernel(GemmArgs g, const int* __restrict__ row_exp, const int* __restrict__ col_exp,
                const int* __restrict__ flag, int tiles_m, int tiles_n) {
  constexpr int TM = C::TM, TN = C::TN, BM = C::BM, BN = C::BN, NT = C::NT;
  constexpr int RX = 2 * C::NX, RY = 2 * C::NY;   // row / column group strides
  constexpr int STAGES = C::STAGES, ASTR = C::ASTR, BSTR = C::BSTR;
  constexpr int A_STAGE = C::A_STAGE, B_STAGE = C::B_STAGE;

  // grouped raster over the tile grid
  const int bid = blockIdx.x;
  const int GM_ = g.group_m > 0 ? g.group_m : GROUP_M;
  const int group_size = GM_ * tiles_n;
  const int first_m = (bid / group_size) * GM_;
  const int gm = min(tiles_m - first_m, GM_);
  const int local = bid % group_size;
  const int bm = first_m + local % gm, bn = local / gm;
  const int64_t i0 = (int64_t)bm * BM, j0 = (int64_t)bn * BN;
  if (SYRK == 1 && i0 > j0 + BN - 1) return;   // tile entirely below the diagonal
  if (SYRK == 2 && i0 + BM - 1 < j0) return;   // tile entirely above the diagonal
  // TwoSum fallback launch (fast mode): only tiles that may hold EC_WIDE elements
  if (g.only_wide && !tile_maybe_wide(g, i0, j0, BM, BN)) return;

  extern __shared__ __align__(16) double smem[];
  double* sA = smem;
  double* sB = smem + STAGES * A_STAGE;
  int* sRowExp = reinterpret_cast<int*>(sB + STAGES * B_STAGE);
  int* sColExp = sRowExp + BM;

  const int tid = threadIdx.x;
  const int tx = tid % C::NX, ty = tid / C::NX;

  double H[TM][TN], L[TM][TN];   // exact: (c_h, c_l); twosum/select: (S, L); anchor: (T, L)

  if (ALG == ALG_CERT) {
    for (int r = tid; r < BM + BN; r += NT) {
      if (r < BM) {
        const int64_t gi = i0 + r;
        sRowExp[r] = gi < g.m ? row_exp[gi] : 0;
      } else {
        const int64_t gj = j0 + (r - BM);
        sColExp[r - BM] = gj < g.n ? col_exp[gj] : 0;
      }
    }
    __syncthreads();
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        const int ri = (a >> 1) * RX + tx * 2 + (a & 1), cj = (b >> 1) * RY + ty * 2 + (b & 1);
        const int64_t gi = i0 + ri, gj = j0 + cj;
        const float sb = (gi < g.m && gj < g.n) ? g.bound[gi + gj * g.m] : 0.f;
        // Sigma' = sd * 2^(rowexp + colexp - 2044), sd < 2^(es - 1022);
        // 2^E >= 2 Sigma'  <=>  biased E = es + rowexp + colexp - 2042
        const double sd = dfma((double)sb, g.bnd_fac, g.bnd_floor);
        const int es = (int)((dbits(sd) >> 52) & 0x7ff);
        H[a][b] = anchor_from_bexp(es + sRowExp[ri] + sColExp[cj] - 2042);
        L[a][b] = 0.0;
      }
  } else {
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TN; ++b) {
        H[a][b] = 0.0;
        L[a][b] = 0.0;
        if (ALG == ALG_F64 && TA == 0) {    // _scale_full in binary64
          const int64_t gi = i0 + (a >> 1) * RX + tx * 2 + (a & 1);
          const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
          if (gi < g.m && gj < g.n) {
            const double c = g.c_hi[gi + gj * g.ldc];
            H[a][b] = g.beta.h == 0.0 ? 0.0 : (g.beta.h == 1.0 ? c : dmul(g.beta.h, c));
          }
        }
        if (ALG == ALG_EXACT && TA == 0) {  // axpy form: start from beta-scaled C
          const int64_t gi = i0 + (a >> 1) * RX + tx * 2 + (a & 1);
          const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
          if (gi < g.m && gj < g.n) {
            const dd c = scale_beta(g.beta, dd{g.c_hi[gi + gj * g.ldc], g.c_lo[gi + gj * g.ldc]});
            H[a][b] = c.h;
            L[a][b] = c.l;
          }
        }
      }
  }

  // split-K (fast modes): blockIdx.y owns k in [kbeg, kend), a multiple of BK
  const int64_t kbeg = (int64_t)blockIdx.y * g.kchunk;
  const int64_t kend = g.kchunk >= g.k ? g.k : min(g.k, kbeg + g.kchunk);
  const int ktiles = (int)((kend - kbeg + BK - 1) / BK);
#pragma unroll
  for (int s = 0; s < STAGES - 1; ++s) {
    if (s < ktiles) load_stage<C, TA, TB, ALG != ALG_F64>(g, sA + s * A_STAGE, sB + s * B_STAGE, i0, j0, kbeg + (int64_t)s * BK, kend, tid);
    cp_async_commit();
  }

  for (int kt = 0; kt < ktiles; ++kt) {
    if ((DDB_ABLATE & 2) == 0 || kt == 0) {
    cp_async_wait<STAGES - 2>();
    __syncthreads();
    }
    if ((DDB_ABLATE & 2) == 0 || kt == 0) {
      const int nk = kt + STAGES - 1;
      const int ns = nk % STAGES;
      if (nk < ktiles) load_stage<C, TA, TB, ALG != ALG_F64>(g, sA + ns * A_STAGE, sB + ns * B_STAGE, i0, j0, kbeg + (int64_t)nk * BK, kend, tid);
      cp_async_commit();
    }
    const int st = kt % STAGES;
    const double* a_h = sA + st * A_STAGE;
    const double* a_l = a_h + BK * ASTR;
    double* b_h = sB + st * B_STAGE;
    double* b_l = b_h + BK * BSTR;

    if (ALG == ALG_F64 && TA == 0) {
      // temp = alpha * op(B)(l, j) in binary64 (level23.py:122, :137)
#pragma unroll
      for (int r = 0; r < BN * BK / NT; ++r) {
        const int idx = tid + r * NT;
        const int kk = idx / BN, jj = idx % BN;
        b_h[kk * BSTR + jj] = dmul(g.alpha.h, b_h[kk * BSTR + jj]);
      }
      __syncthreads();
    }
    if (ALG == ALG_EXACT && TA == 0 && SYRK != 3) {
      // t = mul2(alpha, op(B)(l, j)) once per tile element (level23.py:122, :137)
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
    if (ALG == ALG_EXACT || ALG == ALG_F64) {
      const int64_t rem = kend - kbeg - (int64_t)kt * BK;
      kcount = rem < BK ? (int)rem : BK;   // exact: never run a padded k-step
    }

    auto load_ops = [&](int kk, double (&ah)[TM], double (&al)[TM], double (&bh)[TN],
                        double (&bl)[TN]) {
#pragma unroll
      for (int gq = 0; gq < TM / 2; ++gq) {
        const double2 vh = *reinterpret_cast<const double2*>(a_h + kk * ASTR + gq * RX + tx * 2);
        ah[2 * gq] = vh.x; ah[2 * gq + 1] = vh.y;
        if (ALG != ALG_F64) {
          const double2 vl = *reinterpret_cast<const double2*>(a_l + kk * ASTR + gq * RX + tx * 2);
          al[2 * gq] = vl.x; al[2 * gq + 1] = vl.y;
        }
      }
#pragma unroll
      for (int gq = 0; gq < TN / 2; ++gq) {
        const double2 vh = *reinterpret_cast<const double2*>(b_h + kk * BSTR + gq * RY + ty * 2);
        bh[2 * gq] = vh.x; bh[2 * gq + 1] = vh.y;
        if (ALG != ALG_F64) {
          const double2 vl = *reinterpret_cast<const double2*>(b_l + kk * BSTR + gq * RY + ty * 2);
          bl[2 * gq] = vl.x; bl[2 * gq + 1] = vl.y;
        }
      }
    };
    auto k_step = [&](int kk) {
      double ah[TM], al[TM], bh[TN], bl[TN];
      load_ops(kk, ah, al, bh, bl);
      mac_step<ALG, TM, TN, SYRK == 3>(H, L, ah, al, bh, bl);
    };
    auto renorm = [&]() {
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          double s, e;
          quick_two_sum(H[a][b], L[a][b], s, e);
          H[a][b] = s;
          L[a][b] = e;
        }
    };
    auto fold = [&]() {   // (T, L) -> (T + L, exact rounding error): Fast2Sum, |T| >> |L|
#pragma unroll
      for (int a = 0; a < TM; ++a)
#pragma unroll
        for (int b = 0; b < TN; ++b) {
          const double T2 = dadd(H[a][b], L[a][b]);
          L[a][b] = dsub(L[a][b], dsub(T2, H[a][b]));
          H[a][b] = T2;
        }
    };
    if (ALG == ALG_EXACT || ALG == ALG_F64) {
#pragma unroll 1
      for (int kk = 0; kk < kcount; ++kk) k_step(kk);
    } else {
      // fast modes: the k-tile runs as BK/2 iterations of a 2-step body.
      // Unrolling the whole 16-step tile (~66 KB of SASS for the 8 x 4 tile)
      // overflows the instruction cache: measured 63 % of the FP64 pipe vs
      // 99 % for a 2- or 4-step body (scripts/cert_mix.cu).  Operands are
      // double-buffered in registers across the two steps; CERT folds every 2
      // steps, TWOSUM renormalises every RN = 8.
      if (DDB_ABLATE & 1) {   // ablation: operands loaded once per k-tile (no LDS in the steps)
        double ah[TM], al[TM], bh[TN], bl[TN];
        load_ops(0, ah, al, bh, bl);
#pragma unroll 1
        for (int kk = 0; kk < BK; kk += 2) {
          mac_step<ALG, TM, TN, SYRK == 3>(H, L, ah, al, bh, bl);
          mac_step<ALG, TM, TN, SYRK == 3>(H, L, ah, al, bh, bl);
          if (ALG == ALG_CERT) fold();
        }
      } else
#pragma unroll 1
      for (int kk = 0; kk < BK; kk += DDB_UNR) {
        if (C::PF) {   // step j+1's operands load while step j computes; nothing
                       // stays live across the back-edge but H and L
          double ah[2][TM], al[2][TM], bh[2][TN], bl[2][TN];
          load_ops(kk, ah[0], al[0], bh[0], bl[0]);
#pragma unroll
          for (int j = 0; j < DDB_UNR; ++j) {
            if (j + 1 < DDB_UNR)
              load_ops(kk + j + 1, ah[(j + 1) & 1], al[(j + 1) & 1], bh[(j + 1) & 1], bl[(j + 1) & 1]);
            mac_step<ALG, TM, TN, SYRK == 3>(H, L, ah[j & 1], al[j & 1], bh[j & 1], bl[j & 1]);
            if (ALG == ALG_CERT && (j % RF) == RF - 1) fold();
            if ((ALG == ALG_TWOSUM || ALG == ALG_SELECT) && ((kk + j + 1) % RN) == 0) renorm();
          }
        } else {
#pragma unroll
          for (int j = 0; j < DDB_UNR; ++j) {
            k_step(kk + j);
            if (ALG == ALG_CERT && (j % RF) == RF - 1) fold();
            if ((ALG == ALG_TWOSUM || ALG == ALG_SELECT) && ((kk + j + 1) % RN) == 0) renorm();
          }
        }
      }
    }

  }
  cp_async_wait<0>();

  // epilogue
#pragma unroll
  for (int a = 0; a < TM; ++a)
#pragma unroll
    for (int b = 0; b < TN; ++b) {
      const int64_t gi = i0 + (a >> 1) * RX + tx * 2 + (a & 1);
      const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
      if (gi >= g.m || gj >= g.n) continue;
      if (SYRK == 1 && gi > gj) continue;
      if (SYRK == 2 && gi < gj) continue;
      if (!elem_mine(g, gi, gj)) continue;   // routed elsewhere (internal.h: elem_class)
      const int64_t ci = gi + gj * g.ldc;
      if (ALG == ALG_F64) {    // level23.py:120-149 with the F64 backend (elem.py:149-197)
        if (TA == 0) {
          g.c_hi[ci] = H[a][b];
        } else {                // _combine: at = alpha*acc; beta == 0 ? at : at + beta*C
          const double at = dmul(g.alpha.h, H[a][b]);
          g.c_hi[ci] = g.beta.h == 0.0 ? at : dadd(at, dmul(g.beta.h, g.c_hi[ci]));
        }
        continue;
      }
      dd out;
      if (ALG == ALG_EXACT) {
        if (TA == 0) out = dd{H[a][b], L[a][b]};
        else out = combine(g.alpha, dd{H[a][b], L[a][b]}, g.beta, dd{g.c_hi[ci], g.c_lo[ci]});
      } else {
        double s, e;
        const double hv = ALG == ALG_CERT ? dsub(H[a][b], anchor_of(H[a][b])) : H[a][b];
        two_sum(hv, L[a][b], s, e);
        if (g.part != nullptr) {   // split-K: this slice's sum, combined by splitk_reduce
          double* ph = g.part + (size_t)blockIdx.y * 2 * g.m * g.n;
          ph[gi + gj * g.m] = s;
          ph[(size_t)g.m * g.n + gi + gj * g.m] = e;
          continue;
        }
        const dd at = mul2_chk(g.alpha, dd{s, e});
        out = add2_chk(at, scale_beta(g.beta, dd{g.c_hi[ci], g.c_lo[ci]}));
      }
      g.c_hi[ci] = out.h;
      g.c_lo[ci] = out.l;
    }
}

template <class C, int TA, int TB, int ALG, int SYRK>
cudaError_t launch_one(const GemmArgs& g, const int* row_exp, const int* col_exp,
                       const int* flag, cudaStream_t s) {
  constexpr int BM = C::BM, BN = C::BN, NT = C::NT;
  constexpr size_t SMEM_BYTES = C::SMEM_BYTES;
  auto kern = dd_tiled_kernel<C, TA, TB, ALG, SYRK>;
  // per-device attribute: set on every call (cheap, idempotent, thread-safe)
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (int)((g.m + BM - 1) / BM), tiles_n = (int)((g.n + BN - 1) / BN);
  const int splits = g.kchunk >= g.k ? 1 : (int)((g.k + g.kchunk - 1) / g.kchunk);
  kern<<<dim3(tiles_m * tiles_n, splits), NT, SMEM_BYTES, s>>>(g, row_exp, col_exp, flag,
                                                                tiles_m, tiles_n);
  return cudaGetLastError();
}

// All trans / uplo variants of one algorithm (instantiated per .cu file).
template <class C, int ALG>
cudaError_t launch_alg(const GemmArgs& g, const int* row_exp, const int* col_exp,
                       const int* flag, cudaStream_t s) {
  if constexpr (ALG == ALG_EXACT) {
    if (g.sub && g.syrk == 0 && g.ta == 0)   // SYRK = 3: the subtract-product form
      return g.tb == 0 ? launch_one<C, 0, 0, ALG, 3>(g, row_exp, col_exp, flag, s)
                       : launch_one<C, 0, 1, ALG, 3>(g, row_exp, col_exp, flag, s);
  }
  if (g.syrk == 0) {
    switch (g.ta * 2 + g.tb) {
      case 0: return launch_one<C, 0, 0, ALG, 0>(g, row_exp, col_exp, flag, s);
      case 1: return launch_one<C, 0, 1, ALG, 0>(g, row_exp, col_exp, flag, s);
      case 2: return launch_one<C, 1, 0, ALG, 0>(g, row_exp, col_exp, flag, s);
      default: return launch_one<C, 1, 1, ALG, 0>(g, row_exp, col_exp, flag, s);
    }
  }
  // Rsyrk: trans 'N' == NT with B = A, trans 'T' == TN with B = A
  if (g.ta == 0)
    return g.syrk == 1 ? launch_one<C, 0, 1, ALG, 1>(g, row_exp, col_exp, flag, s)
                       : launch_one<C, 0, 1, ALG, 2>(g, row_exp, col_exp, flag, s);
  return g.syrk == 1 ? launch_one<C, 1, 0, ALG, 1>(g, row_exp, col_exp, flag, s)
                     : launch_one<C, 1, 0, ALG, 2>(g, row_exp, col_exp, flag, s);
}

}  // namespace tiled
}  // namespace ddb
