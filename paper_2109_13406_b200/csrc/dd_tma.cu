// dd_tma.cu -- TMA + mbarrier pipeline variant of the fast-mode tiled kernel
// for the NN layout (the benchmark case) with 16-byte aligned operands.
//
// Same arithmetic as dd_tiled.cuh (mac_step / fold / renorm / epilogue), a
// different feed: a dedicated producer warp issues cp.async.bulk.tensor (TMA)
// copies of the A hi/lo (128 x 16, m-major) and B hi/lo (16 x 64, k-major) tiles
// into a 4-stage ring; 8 consumer warps wait on per-stage "full" mbarriers
// (transaction-counted) and release stages through "empty" mbarriers, so there
// is no __syncthreads, no per-thread address arithmetic and no cp.async issue
// in the k-loop.  TMA zero-fills the ragged edges.  A is read m-major exactly
// as before; B is read k-major: one 16-byte LDS gives a column's operands for
// two consecutive k-steps, so the 2-step loop body needs the same number of
// LDS as the cp.async kernel.
//
// Used when transa = transb = 'N', both planes 16-byte aligned, lda and ldb
// even (TMA global strides are multiples of 16 bytes); anything else runs
// dd_tiled.cuh.
//
// ALG_SPLIT (fast mode's default here): the dd product a*b = ah bh + (al bh +
// ah bl) + al bl splits into the hi * hi part, accumulated by this kernel with
// the certified anchor (Tn = fma(ah, bh, T), r = fma(ah, bh, T - Tn), L += r,
// the two residuals of a step pair summed before they enter L, (T, L)
// folded every 4 steps: 4.75 FP64 instructions per MAC instead of 7.5, and
// only the hi planes staged, 32-deep k-tiles), and the cross terms
// X = A_lo B_hi + A_hi B_lo, computed first by the hand-written DMMA kernel
// (dd_cross.cu; for Rsyrk on the triangle tiles only) and added to L in the
// epilogue; al bl (< u^2 |ab|) is dropped, as in every dd product.  Error per
// element, with the unit v = 2^(E-106) < 2^-104 S' (2^E < 4 S', S' >= sum
// |ah bh| the certified bound): each residual r (|r| <= ulp(T)/2 =
// 2^(E-53)) rounds by <= v/2; a pair sum r0 + r1 (<= 2^(E-52)) by <= v;
// after a fold |L| <= 2^(E-53), so by monotone rounding the two additions
// into L stay <= 1.5 * 2^(E-52) and 2.5 * 2^(E-52) and round by <= 2v, 4v:
// 4 (v/2) + 2 v + 2v + 4v = 10 v per 4 steps, c = 2.5 rho with rho = S' /
// sum|ab| (per-step accumulation with the same period: 2.75 rho; a period
// of 3: 2.17 rho).  The cross sums' recursive-summation bound is 2k u *
// sum (|al bh| + |ah bl|) <= 4k u^2 sum|ab| (operands normalised, |lo| <=
// 2^-53 |hi|, which the prescan enforces): c = 1; the dropped al bl c =
// 0.25.  rho <= 1.064 for every element the routing leaves here
// (dd_bound.cu: k <= 2^16 and row + column exponent spreads within 112 -
// ceil(log2 k); wider elements take the TwoSum fallback), so c <= 2.5 *
// 1.064 + 1.25 = 3.91 (+ O(u^2) epilogue roundings, << 0.09 k at the
// k >= 256 this kernel runs) against the north star's c = 4.
// Measured at 8192^3: 167 ms for this kernel + 60.5 ms of cross terms.
#include <cuda.h>

#include <cstdlib>

#include "dd_tiled.cuh"
#include "tma_util.cuh"

namespace ddb {
namespace tma {

using tiled::anchor_from_bexp;
using tiled::anchor_of;
using tiled::dbits;

#ifndef DDB_TMA_UNROLL
#define DDB_TMA_UNROLL 2   // 2-step bodies unrolled per loop trip (8 = the whole k-tile; 2 measured best)
#endif

constexpr int kTmaUnroll = DDB_TMA_UNROLL;
#ifndef DDB_TMA_EPI_NC
#define DDB_TMA_EPI_NC 1      // 1: check-free epilogue arithmetic inside the safe window
#endif
// (EPI_NC: 8192 x 7936 x 256 in 8.51 vs 8.59 ms; L1 / L2 prefetches of the
// epilogue's C and cross-term lines did not help)
constexpr int BM = 128, BN = 64, BK = 16, STAGES = 4;
constexpr int NT = 256;       // 8 consumer warps
#ifndef DDB_TMA_WS
#define DDB_TMA_WS 1          // 1: a separate producer warpgroup issues the TMA loads
#endif
// DDB_TMA_WS = 1: warps 8..11 form a producer warpgroup (one lane issues every
// TMA load; setmaxnreg hands its registers to the consumers, 24 / 240 per
// thread); 0: thread 0 of consumer warp 0 doubles as the producer
constexpr int NTK = NT + (DDB_TMA_WS ? 128 : 0);
#ifndef DDB_TMA_REGC
#define DDB_TMA_REGC 240      // consumer registers per thread after setmaxnreg (final kernel: 240 225.8 ms at 8192^3, 224 226.6, 208 226.2, 184 237.4 with spills)
#endif
constexpr int REG_CONSUMER = DDB_TMA_REGC, REG_PRODUCER = 24;
constexpr int TM = 8, TN = 4, RX = 32, RY = 32;
constexpr int A_PLANE = BK * BM, B_PLANE = BN * BK;          // doubles
constexpr int STAGE_DOUBLES = 2 * A_PLANE + 2 * B_PLANE;     // 6144 doubles = 48 KB
constexpr uint32_t STAGE_BYTES = STAGE_DOUBLES * 8;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;

// ALG_SPLIT: k-tile depth and fold period (steps between (T, L) folds).  The
// stage holds only the hi planes, so a deeper tile fits the same ring.  A
// fold period of 4 with pair-summed residuals: error <= 10 units per 4 steps
// (see the header); 229.3 vs 235.4 ms per 8192^3 step against a period of 3
// (6.5 units per 3 steps).
#ifndef DDB_SPLIT_BK
#define DDB_SPLIT_BK 32      // 32 x (128 + 64) doubles = the ring's 48 KB stage (24: 229.3 vs 228.8 ms)
#endif
#ifndef DDB_SPLIT_FOLD
#define DDB_SPLIT_FOLD 4
#endif
#ifndef DDB_SPLIT_CHAIN
#define DDB_SPLIT_CHAIN 0     // 1: per-element step chains instead of per-step sweeps
#endif
#ifndef DDB_SPLIT_PAIR
#define DDB_SPLIT_PAIR 1      // 1: the two residuals of a step pair summed before entering L
#endif
#ifndef DDB_SPLIT_UNROLL
#define DDB_SPLIT_UNROLL 2    // k-loop bodies unrolled per trip (2: 240.4 vs 241.8 ms at 8192^3)
#endif
#ifndef DDB_SPLIT_TN
#define DDB_SPLIT_TN 4        // split kernel: columns per thread (tile width SPLIT_TN / 2 * 32)
#endif
constexpr int SPLIT_BK = DDB_SPLIT_BK, SPLIT_FOLD = DDB_SPLIT_FOLD;
constexpr int SPLIT_TN = DDB_SPLIT_TN, SPLIT_BN = SPLIT_TN / 2 * RY;
constexpr bool SPLIT_CHAIN = DDB_SPLIT_CHAIN, SPLIT_PAIR = DDB_SPLIT_PAIR;
static_assert(!SPLIT_PAIR || SPLIT_FOLD % 2 == 0, "pairs fold on pair boundaries");
constexpr int SPLIT_UNROLL = DDB_SPLIT_UNROLL;
constexpr int SPLIT_BODY = SPLIT_FOLD % 2 == 0 ? SPLIT_FOLD : 2 * SPLIT_FOLD;   // even
static_assert(SPLIT_BK % SPLIT_BODY == 0 && SPLIT_BK % 2 == 0, "split k-tile");
static_assert((SPLIT_BK * (BM + SPLIT_BN)) * 8 <= STAGE_BYTES, "split stage fits the ring");
// split-K chunks must be whole k-tiles of every kernel (dd_gemm.cu)
static_assert(96 % SPLIT_BK == 0 || SPLIT_BK == 32, "chunk rounding");

// Work unit = one (tile, k-slice).  PERSISTENT: gridDim.x CTAs (one per SM)
// walk the units u = blockIdx.x + i * gridDim.x in raster order, so all SMs
// work on the same wave of tiles at nearly the same k (the wave's A / B panel
// k-slices are read from DRAM once and shared through L2); the producer runs
// ahead across unit boundaries, overlapping the epilogue with the next loads.
// the prescan's safe window on one dd value (hi zero or 2^-300 <= |hi| <
// 2^301, lo below 2^301): the epilogue's check-free forms are bit-identical
// to the checked ones when the products' factors and the sums' operands lie
// in it (mul2: two_prod_g takes the FMA residual and nothing overflows; add2:
// s0 = xh + yh is finite, and add2_nc_sel == add2_nc for finite operands)
__device__ __forceinline__ bool epi_win(double h, double l) {
  const int eh = (int)((__double_as_longlong(h) >> 52) & 0x7ff);
  const int el = (int)((__double_as_longlong(l) >> 52) & 0x7ff);
  return (eh >= WIN_LO || (__double_as_longlong(h) << 1) == 0) && eh <= WIN_HI && el <= WIN_HI;
}

template <int ALG, int SYRK>
__global__ void __launch_bounds__(NTK, 1)
dd_tma_nn_kernel(GemmArgs g, const __grid_constant__ CUtensorMap mAh,
                 const __grid_constant__ CUtensorMap mAl, const __grid_constant__ CUtensorMap mBh,
                 const __grid_constant__ CUtensorMap mBl, const int* __restrict__ row_exp,
                 const int* __restrict__ col_exp, const int* __restrict__ flag, int tiles_m,
                 int tiles_n, int splits) {
  constexpr bool CERTLIKE = ALG == ALG_CERT || ALG == ALG_SPLIT;
  constexpr int KB = ALG == ALG_SPLIT ? SPLIT_BK : BK;            // k-tile depth
  constexpr int AP = KB * BM;                                     // A hi plane, doubles
  // stage layout: A hi | A lo | B hi | B lo (split: A hi | B hi)
  constexpr int B_OFF = ALG == ALG_SPLIT ? AP : 2 * A_PLANE;
  // per-thread columns / tile width (split: SPLIT_TN, the hi planes leave room)
  constexpr int TNK = ALG == ALG_SPLIT ? SPLIT_TN : TN, BNK = TNK / 2 * RY;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align by an offset from the __shared__ array (an integer round trip of
  // the pointer would lose its address space: generic LD instead of LDS)
  double* ring = reinterpret_cast<double*>(smem_raw + ((1024u - (saddr(smem_raw) & 1023u)) & 1023u));
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE_DOUBLES);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  const int tiles = tiles_m * tiles_n;
  const int units = tiles * splits;
  // every unit has the same number of k-tiles except possibly the last slice
  const int64_t kchunk = g.kchunk >= g.k ? g.k : g.kchunk;
  auto unit_origin = [&](int u, int64_t& i0, int64_t& j0, int64_t& kbeg, int& ktiles) {
    const int tile = u % tiles, split = u / tiles;
    const int GM_ = g.group_m > 0 ? g.group_m : tiled::GROUP_M;
    const int group_size = GM_ * tiles_n;
    const int first_m = (tile / group_size) * GM_;
    const int gm = min(tiles_m - first_m, GM_);
    const int local = tile % group_size;
    i0 = (int64_t)(first_m + local % gm) * BM;
    j0 = (int64_t)(local / gm) * BNK;
    kbeg = (int64_t)split * kchunk;
    const int64_t kend = min(g.k, kbeg + kchunk);
    ktiles = (int)((kend - kbeg + KB - 1) / KB);
  };

  // Rsyrk (SYRK = 1 upper / 2 lower): units whose tile lies entirely in the
  // other triangle are skipped by producer and consumers alike
  auto skipped = [&](int u) {
    if (SYRK == 0) return false;
    int64_t i0, j0, kb;
    int kt;
    unit_origin(u, i0, j0, kb, kt);
    return SYRK == 1 ? i0 > j0 + BNK - 1 : i0 + BM - 1 < j0;
  };
  auto next_unit = [&](int u) {   // first unit >= u in this CTA's stride that is not skipped
    while (u < units && skipped(u)) u += gridDim.x;
    return u;
  };

  // ---- producer state (thread 0): walks (unit, k-tile) items ahead ----
  int p_unit = next_unit(blockIdx.x), p_kt = 0, p_ktiles = 0;
  int64_t p_i0 = 0, p_j0 = 0, p_kbeg = 0;
  uint32_t p_item = 0;
  if (tid == (DDB_TMA_WS ? NT : 0) && p_unit < units) unit_origin(p_unit, p_i0, p_j0, p_kbeg, p_ktiles);
  auto produce_next = [&]() {   // issue the next item if any; false when exhausted
    if (p_unit >= units) return false;
    const int s = p_item % STAGES;
    if (p_item >= STAGES) mbar_wait(&empty[s], ((p_item / STAGES) - 1) & 1);
    double* st = ring + s * STAGE_DOUBLES;
    const int kc = (int)(p_kbeg + (int64_t)p_kt * KB);
    if (ALG == ALG_SPLIT) {   // hi planes only
      mbar_expect_tx(&full[s], (uint32_t)(KB * (BM + BNK)) * 8u);
      tma_load_2d(st, &mAh, (int)p_i0, kc, &full[s]);
      tma_load_2d(st + B_OFF, &mBh, kc, (int)p_j0, &full[s]);
    } else {
      mbar_expect_tx(&full[s], STAGE_BYTES);
      tma_load_2d(st, &mAh, (int)p_i0, kc, &full[s]);
      tma_load_2d(st + A_PLANE, &mAl, (int)p_i0, kc, &full[s]);
      tma_load_2d(st + 2 * A_PLANE, &mBh, kc, (int)p_j0, &full[s]);
      tma_load_2d(st + 2 * A_PLANE + B_PLANE, &mBl, kc, (int)p_j0, &full[s]);
    }
    ++p_item;
    if (++p_kt == p_ktiles) {
      p_kt = 0;
      p_unit = next_unit(p_unit + gridDim.x);
      if (p_unit < units) unit_origin(p_unit, p_i0, p_j0, p_kbeg, p_ktiles);
    }
    return true;
  };
  if (DDB_TMA_WS) {
    if (tid >= NT) {   // producer warpgroup
      asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_PRODUCER));
      if (tid == NT)
        while (produce_next()) {}
      return;
    }
    asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONSUMER));
  } else if (tid == 0) {
    for (int i = 0; i < STAGES - 1; ++i) produce_next();
  }

  const int tx = tid % 16, ty = tid / 16;
  uint32_t c_item = 0;
  for (int u = next_unit(blockIdx.x); u < units; u = next_unit(u + gridDim.x)) {
    int64_t i0, j0, kbeg;
    int ktiles;
    unit_origin(u, i0, j0, kbeg, ktiles);

    double H[TM][TNK], L[TM][TNK];
#pragma unroll
    for (int a = 0; a < TM; ++a)
#pragma unroll
      for (int b = 0; b < TNK; ++b) { H[a][b] = 0.0; L[a][b] = 0.0; }
    if (CERTLIKE) {
      // anchors row pair by row pair, shifted in from H[TM - 1]: a rolled
      // loop keeps the kernel's code small (a short-k tile runs its prologue
      // and epilogue once, and fully unrolled they missed the instruction
      // cache: ~2x the tile time at k = 64)
      // (every bound word and row exponent is loaded up front -- one round
      // trip instead of one per row -- parked in L and H[.][0] and shifted
      // out row by row, which leaves L zero again; 227.8 vs 228.7 ms at
      // 8192^3.  An L2 prefetch of C and the cross terms by the producer
      // warp before the epilogue cost 9 ms there and was dropped.)
      int ec[TNK];
#pragma unroll
      for (int b = 0; b < TNK; ++b) {
        const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
        ec[b] = gj < g.n ? col_exp[gj] : 0;
      }
#pragma unroll
      for (int a = 0; a < TM; ++a) {
        const int64_t gi = i0 + (a >> 1) * RX + tx * 2 + (a & 1);
        H[a][0] = gi < g.m ? (double)row_exp[gi] : 0.0;
#pragma unroll
        for (int b = 0; b < TNK; ++b) {
          const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
          L[a][b] = gi < g.m && gj < g.n ? (double)g.bound[gi + gj * g.m] : 0.0;
        }
      }
#pragma unroll 1
      for (int a = 0; a < TM; ++a) {
        const int er = (int)H[0][0];
        double anc[TNK];
#pragma unroll
        for (int b = 0; b < TNK; ++b) {
          const double sd = dfma(L[0][b], g.bnd_fac, g.bnd_floor);
          const int es = (int)((dbits(sd) >> 52) & 0x7ff);
          anc[b] = anchor_from_bexp(es + er + ec[b] - 2042);
        }
#pragma unroll
        for (int i = 0; i + 1 < TM; ++i)
#pragma unroll
          for (int b = 0; b < TNK; ++b) {
            H[i][b] = H[i + 1][b];
            L[i][b] = L[i + 1][b];
          }
#pragma unroll
        for (int b = 0; b < TNK; ++b) {
          H[TM - 1][b] = anc[b];
          L[TM - 1][b] = 0.0;
        }
      }
    }

    for (int kt = 0; kt < ktiles; ++kt, ++c_item) {
      const int s = c_item % STAGES;
      if (!DDB_TMA_WS && tid == 0) produce_next();
      mbar_wait(&full[s], (c_item / STAGES) & 1);
      const double* a_h = ring + s * STAGE_DOUBLES;
      const double* a_l = a_h + A_PLANE;
      const double* b_h = a_h + 2 * A_PLANE;
      const double* b_l = b_h + B_PLANE;
      if (ALG == ALG_SPLIT) {
        // hi * hi only: Tn = T + ah bh (T stays in its anchor's binade, so
        // T - Tn is exact), r = ah bh + (T - Tn) is Tn's rounding error up to
        // one rounding, L collects the r's; (T, L) folded every SPLIT_FOLD
        // steps.  B is k-major: one LDS.128 per column gives two k-steps.
        const double* bs = a_h + B_OFF;
#pragma unroll (SPLIT_UNROLL)
        for (int kk = 0; kk < KB; kk += SPLIT_BODY) {
#pragma unroll
          for (int pq = 0; pq < SPLIT_BODY; pq += 2) {
            double ah0[TM], ah1[TM], bh0[TNK], bh1[TNK];
#pragma unroll
            for (int gq = 0; gq < TM / 2; ++gq) {
              const double2 h0 =
                  *reinterpret_cast<const double2*>(a_h + (kk + pq) * BM + gq * RX + tx * 2);
              const double2 h1 =
                  *reinterpret_cast<const double2*>(a_h + (kk + pq + 1) * BM + gq * RX + tx * 2);
              ah0[2 * gq] = h0.x; ah0[2 * gq + 1] = h0.y;
              ah1[2 * gq] = h1.x; ah1[2 * gq + 1] = h1.y;
            }
#pragma unroll
            for (int b = 0; b < TNK; ++b) {
              const int cj = (b >> 1) * RY + ty * 2 + (b & 1);
              const double2 h = *reinterpret_cast<const double2*>(bs + cj * KB + kk + pq);
              bh0[b] = h.x; bh1[b] = h.y;
            }
            if (SPLIT_CHAIN) {   // per element: both steps of the pair (and its folds)
#pragma unroll
              for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TNK; ++b) {
                  double T = H[a][b], l = L[a][b];
#pragma unroll
                  for (int q = 0; q < 2; ++q) {
                    const double av = q ? ah1[a] : ah0[a], bv = q ? bh1[b] : bh0[b];
                    const double Tn = dfma(av, bv, T);
                    l = dadd(l, dfma(av, bv, dsub(T, Tn)));
                    T = Tn;
                    if ((pq + q + 1) % SPLIT_FOLD == 0) {
                      const double T2 = dadd(T, l);
                      l = dsub(l, dsub(T2, T));
                      T = T2;
                    }
                  }
                  H[a][b] = T;
                  L[a][b] = l;
                }
            } else if (SPLIT_PAIR) {   // L += (r0 + r1): one rounding into L per step pair
#pragma unroll
              for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TNK; ++b) {
                  const double T = H[a][b];
                  const double T1 = dfma(ah0[a], bh0[b], T);
                  const double r0 = dfma(ah0[a], bh0[b], dsub(T, T1));
                  const double T2 = dfma(ah1[a], bh1[b], T1);
                  const double r1 = dfma(ah1[a], bh1[b], dsub(T1, T2));
                  L[a][b] = dadd(L[a][b], dadd(r0, r1));
                  H[a][b] = T2;
                }
              if ((pq + 2) % SPLIT_FOLD == 0) {
#pragma unroll
                for (int a = 0; a < TM; ++a)
#pragma unroll
                  for (int b = 0; b < TNK; ++b) {
                    const double T2 = dadd(H[a][b], L[a][b]);
                    L[a][b] = dsub(L[a][b], dsub(T2, H[a][b]));
                    H[a][b] = T2;
                  }
              }
            } else {
#pragma unroll
            for (int q = 0; q < 2; ++q) {
#pragma unroll
              for (int a = 0; a < TM; ++a)
#pragma unroll
                for (int b = 0; b < TNK; ++b) {
                  const double av = q ? ah1[a] : ah0[a], bv = q ? bh1[b] : bh0[b];
                  const double T = H[a][b];
                  const double Tn = dfma(av, bv, T);
                  L[a][b] = dadd(L[a][b], dfma(av, bv, dsub(T, Tn)));
                  H[a][b] = Tn;
                }
              if ((pq + q + 1) % SPLIT_FOLD == 0) {
#pragma unroll
                for (int a = 0; a < TM; ++a)
#pragma unroll
                  for (int b = 0; b < TNK; ++b) {
                    const double T2 = dadd(H[a][b], L[a][b]);
                    L[a][b] = dsub(L[a][b], dsub(T2, H[a][b]));
                    H[a][b] = T2;
                  }
              }
            }
            }
          }
        }
      } else {
#pragma unroll (kTmaUnroll)
      for (int kk = 0; kk < BK; kk += 2) {
        double ah0[TM], al0[TM], ah1[TM], al1[TM], bh0[TNK], bl0[TNK], bh1[TNK], bl1[TNK];
#pragma unroll
        for (int gq = 0; gq < TM / 2; ++gq) {
          const double2 h0 = *reinterpret_cast<const double2*>(a_h + kk * BM + gq * RX + tx * 2);
          const double2 l0 = *reinterpret_cast<const double2*>(a_l + kk * BM + gq * RX + tx * 2);
          const double2 h1 = *reinterpret_cast<const double2*>(a_h + (kk + 1) * BM + gq * RX + tx * 2);
          const double2 l1 = *reinterpret_cast<const double2*>(a_l + (kk + 1) * BM + gq * RX + tx * 2);
          ah0[2 * gq] = h0.x; ah0[2 * gq + 1] = h0.y; al0[2 * gq] = l0.x; al0[2 * gq + 1] = l0.y;
          ah1[2 * gq] = h1.x; ah1[2 * gq + 1] = h1.y; al1[2 * gq] = l1.x; al1[2 * gq + 1] = l1.y;
        }
#pragma unroll
        for (int b = 0; b < TNK; ++b) {   // k-major B: (kk, kk+1) of column cj in one LDS
          const int cj = (b >> 1) * RY + ty * 2 + (b & 1);
          const double2 h = *reinterpret_cast<const double2*>(b_h + cj * BK + kk);
          const double2 l = *reinterpret_cast<const double2*>(b_l + cj * BK + kk);
          bh0[b] = h.x; bh1[b] = h.y; bl0[b] = l.x; bl1[b] = l.y;
        }
        tiled::mac_step<ALG, TM, TNK>(H, L, ah0, al0, bh0, bl0);
        tiled::mac_step<ALG, TM, TNK>(H, L, ah1, al1, bh1, bl1);
        if (ALG == ALG_CERT) {
#pragma unroll
          for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TNK; ++b) {
              const double T2 = dadd(H[a][b], L[a][b]);
              L[a][b] = dsub(L[a][b], dsub(T2, H[a][b]));
              H[a][b] = T2;
            }
        } else if (((kk + 2) % tiled::RN) == 0) {
#pragma unroll
          for (int a = 0; a < TM; ++a)
#pragma unroll
            for (int b = 0; b < TNK; ++b) {
              double sx, ex;
              quick_two_sum(H[a][b], L[a][b], sx, ex);
              H[a][b] = sx;
              L[a][b] = ex;
            }
        }
      }
      }
      __syncwarp();
      if ((tid & 31) == 0) mbar_arrive(&empty[s]);
    }

    // epilogue (as dd_tiled.cuh's fast modes), one row pair at a time from
    // H[0] / L[0], the rest shifted down after it (rolled: see the prologue).
    // Per row pair the routing words, the cross terms and C are loaded for
    // its TNK elements before any arithmetic, so the global round trips
    // overlap instead of running one element after another.
    const int split = u / tiles;
    // alpha / beta in the window: the per-element test below picks the
    // check-free forms (alpha is never 0 here; beta 0 / 1 need no product)
    const bool beta0 = g.beta.h == 0.0 && g.beta.l == 0.0;
    const bool beta1 = g.beta.h == 1.0 && g.beta.l == 0.0;
    const bool scal_ok = DDB_TMA_EPI_NC && epi_win(g.alpha.h, g.alpha.l) &&
                         g.alpha.h != 0.0 && (beta0 || beta1 || epi_win(g.beta.h, g.beta.l));
    int csv[TNK];
#pragma unroll
    for (int b = 0; b < TNK; ++b) {
      const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
      csv[b] = g.rsp != nullptr && gj < g.n ? g.csp[gj] : 0;
    }
#pragma unroll 1
    for (int a = 0; a < TM; ++a) {
      const int64_t gi = i0 + (a >> 1) * RX + tx * 2 + (a & 1);
      const int rsv = g.rsp != nullptr && gi < g.m ? g.rsp[gi] : 0;
      bool mine[TNK];
      double xv[TNK], ch[TNK], cl[TNK];
#pragma unroll
      for (int b = 0; b < TNK; ++b) {
        const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
        bool ok = gi < g.m && gj < g.n;
        if (SYRK == 1) ok &= gi <= gj;   // the uplo triangle only (level23.py:245-270)
        if (SYRK == 2) ok &= gi >= gj;
        if (g.rsp != nullptr) {          // elem_mine (internal.h) on the preloaded words
          const int v = rsv + csv[b];
          const int cls = v >= SPREAD_BAD ? EC_REF : (g.wide_lim > 0 && v > g.wide_lim ? EC_WIDE : EC_FAST);
          ok &= cls == (g.only_wide ? EC_WIDE : EC_FAST);
        }
        mine[b] = ok;
        const bool x = ALG == ALG_SPLIT && split == 0 && g.cross != nullptr && ok;
        xv[b] = x ? g.cross[gi + gj * g.m] : 0.0;
        const bool c = ok && g.part == nullptr;
        ch[b] = c ? g.c_hi[gi + gj * g.ldc] : 0.0;
        cl[b] = c ? g.c_lo[gi + gj * g.ldc] : 0.0;
      }
#pragma unroll
      for (int b = 0; b < TNK; ++b) {
        if (!mine[b]) continue;
        const int64_t gj = j0 + (b >> 1) * RY + ty * 2 + (b & 1);
        double sx, ex;
        const double hv = CERTLIKE ? dsub(H[0][b], anchor_of(H[0][b])) : H[0][b];
        const double lv = ALG == ALG_SPLIT ? dadd(L[0][b], xv[b]) : L[0][b];
        if (DDB_TMA_EPI_NC) two_sum_sel(hv, lv, sx, ex);   // finite operands: bit-identical
        else two_sum(hv, lv, sx, ex);
        if (g.part != nullptr) {
          double* ph = g.part + (size_t)split * 2 * g.m * g.n;
          ph[gi + gj * g.m] = sx;
          ph[(size_t)g.m * g.n + gi + gj * g.m] = ex;
          continue;
        }
        const int64_t ci = gi + gj * g.ldc;
        dd out;
        if (scal_ok && epi_win(sx, ex) && epi_win(ch[b], cl[b])) {
          const dd at = mul2_nc(g.alpha, dd{sx, ex});
          out = beta0 ? add2_nc_sel(at, dd{0.0, 0.0})
                      : add2_nc_sel(at, beta1 ? dd{ch[b], cl[b]} : mul2_nc(g.beta, dd{ch[b], cl[b]}));
        } else {
          out = add2_chk(mul2_chk(g.alpha, dd{sx, ex}), scale_beta(g.beta, dd{ch[b], cl[b]}));
        }
        g.c_hi[ci] = out.h;
        g.c_lo[ci] = out.l;
      }
#pragma unroll
      for (int i = 0; i + 1 < TM; ++i)
#pragma unroll
        for (int b = 0; b < TNK; ++b) {
          H[i][b] = H[i + 1][b];
          L[i][b] = L[i + 1][b];
        }
    }
  }
}

static bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; }

thread_local int g_no_persist = 0;   // > 0 inside a NoPersistScope

// fast mode through ALG_SPLIT (default for deep calls; measured 258 vs 272 ms
// at 8192^3) or the full certified-anchor MAC: DDB_SPLIT=0 never splits,
// DDB_SPLIT=2 splits at any depth (tests).  Read per call (a few ns).
static int split_policy() {
  const char* v = std::getenv("DDB_SPLIT");
  if (v == nullptr) return 1;
  return v[0] == '0' ? 0 : (v[0] == '2' ? 2 : 1);
}

}  // namespace tma

NoPersistScope::NoPersistScope(bool on) : on_(on) { tma::g_no_persist += on ? 1 : 0; }
NoPersistScope::~NoPersistScope() { tma::g_no_persist -= on_ ? 1 : 0; }

// The concurrent split schedule's last step: C += alpha * X on the EC_FAST
// elements (the uplo triangle for Rsyrk), X the cross terms (ld = m).  One
// checked dd multiply and add per element (two roundings below 2^-104 |C|),
// HBM-bound: ~40 bytes per element.
__global__ void __launch_bounds__(256)
cross_add_kernel(GemmArgs g, const double* __restrict__ x) {
  const int64_t total = g.m * g.n, stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < total; t += stride) {
    const int64_t i = t % g.m, j = t / g.m;
    if (g.syrk == 1 && i > j) continue;
    if (g.syrk == 2 && i < j) continue;
    if (elem_class(g, i, j) != EC_FAST) continue;
    const int64_t ci = i + j * g.ldc;
    const dd out = add2_chk(dd{g.c_hi[ci], g.c_lo[ci]}, mul2_chk(g.alpha, dd{x[t], 0.0}));
    g.c_hi[ci] = out.h;
    g.c_lo[ci] = out.l;
  }
}

// Second stream per host thread and device: the split schedule's cross
// terms run there concurrently with the hi * hi kernel.
static cudaError_t aux_stream(cudaStream_t* out) {
  static thread_local cudaStream_t streams[64] = {};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (streams[dev] == nullptr) {
    e = cudaStreamCreateWithFlags(&streams[dev], cudaStreamNonBlocking);
    if (e != cudaSuccess) return e;
  }
  *out = streams[dev];
  return cudaSuccess;
}

// dst (cols x rows, ld ldd) = src (rows x cols, ld lds)^T, both planes: the
// operand of a TMA Rsyrk that must be k-major / m-major (launch_tiled)
__global__ void __launch_bounds__(256)
dd_transpose_kernel(const double* __restrict__ sh, const double* __restrict__ sl, int64_t lds,
                    double* __restrict__ dh, double* __restrict__ dl, int64_t ldd, int64_t rows,
                    int64_t cols) {
  __shared__ double th[32][33], tl[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, c0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t r = r0 + threadIdx.x, c = c0 + y;
    if (r < rows && c < cols) {
      th[y][threadIdx.x] = sh[r + c * lds];
      tl[y][threadIdx.x] = sl[r + c * lds];
    }
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t c = c0 + threadIdx.x, r = r0 + y;
    if (r < rows && c < cols) {
      dh[c + r * ldd] = th[threadIdx.x][y];
      dl[c + r * ldd] = tl[threadIdx.x][y];
    }
  }
}

cudaError_t launch_dd_transpose(const double* sh, const double* sl, int64_t lds, double* dh,
                                double* dl, int64_t ldd, int64_t rows, int64_t cols,
                                cudaStream_t s) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((cols + 31) / 32));
  dd_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(sh, sl, lds, dh, dl, ldd, rows, cols);
  return cudaGetLastError();
}

bool tma_eligible(const GemmArgs& g, int alg) {
  if (std::getenv("DDB_NO_TMA") != nullptr) return false;
  if (!(alg == ALG_CERT || alg == ALG_TWOSUM)) return false;
  if (g.ta != 0 || g.tb != 0 || g.f64) return false;   // Rsyrk arrives here in NN form
  if ((g.lda & 1) || (g.ldb & 1)) return false;
  if (!tma::aligned16(g.a_hi) || !tma::aligned16(g.a_lo) || !tma::aligned16(g.b_hi) ||
      !tma::aligned16(g.b_lo))
    return false;
  if (g.m >= (1ll << 31) || g.n >= (1ll << 31) || g.k >= (1ll << 31)) return false;
  return tma::encode_fn() != nullptr;
}

cudaError_t launch_tma_nn(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                          const int* flag, cudaStream_t s) {
  using namespace tma;
  alignas(64) CUtensorMap mAh, mAl, mBh, mBl;
  // A: m x k, m contiguous -> box {BM (m), BK (k)}: 1 KB rows, 256-byte L2 promotion.
  // B: k x n, k contiguous -> box {BK, BN}: 128-byte rows; promoting them to
  // 256 bytes doubled the DRAM reads (ncu, round 1), so B uses 128-byte lines.
  const CUtensorMapL2promotion pa = CU_TENSOR_MAP_L2_PROMOTION_L2_256B;
  const CUtensorMapL2promotion pb = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  // ALG_SPLIT: the cross terms first, as two binary64 GEMMs into a
  // stream-ordered m x n scratch, then the hi * hi kernel.  Shallow calls (the
  // LAPACK consumers' depth-256 updates) lose more to the cross GEMMs' fixed
  // costs than the kernel gains: measured Rpotrf / Rgetrf / Rtrsm at n = 8192
  // 1-3 % slower with the split at k = 256; Rsyrk n = k = 4096 4.5 % faster.
  const int policy = split_policy();
  int dev0 = 0, sms0 = 148;
  cudaGetDevice(&dev0);
  cudaDeviceGetAttribute(&sms0, cudaDevAttrMultiProcessorCount, dev0);
  // shallow but wide calls (the LAPACK consumers' depth-256 bulk updates:
  // k >= 256 and >= 2 waves of split tiles) split too, on the serial
  // schedule: 7936 x 7680 x 256 takes 8.47 ms split vs 9.06 ms certified
  // (the concurrent schedule's extra C pass, 8.79 ms, does not pay at this
  // depth); Rgetrf n = 8192 153.8 -> 145.6 ms, Rpotrf 80.0 -> 75.2 ms
  const int64_t big_tiles = ((g.m + BM - 1) / BM) * ((g.n + SPLIT_BN - 1) / SPLIT_BN);
  static const int sw_k = [] {
    const char* v = std::getenv("DDB_SHALLOW_SPLIT_K");
    return v ? std::atoi(v) : 256;
  }();
  static const int sw_t = [] {
    const char* v = std::getenv("DDB_SHALLOW_SPLIT_WAVES");
    return v ? std::atoi(v) : 2;
  }();
  const bool shallow_wide = g.k >= sw_k && g.k < 1024 && big_tiles >= sw_t * (int64_t)sms0;
  bool split_alg = alg == ALG_CERT && policy != 0 && (policy == 2 || g.k >= 1024 || shallow_wide);
  double* xbuf = nullptr;
  int64_t xchunk = g.k;
  const int xslices = split_alg ? cross_kslices(g, &xchunk) : 1;
  if (split_alg &&
      cudaMallocAsync(reinterpret_cast<void**>(&xbuf),
                      sizeof(double) * (size_t)xslices * g.m * g.n, s) != cudaSuccess) {
    // no room for the m x n cross-term scratch: the certified full MAC
    // needs none (same error bound, ~13 % slower)
    cudaGetLastError();
    xbuf = nullptr;
    split_alg = false;
  }
  const uint32_t kb = split_alg ? SPLIT_BK : BK;
  const uint32_t bn = split_alg ? SPLIT_BN : BN;
  if (!encode(&mAh, g.a_hi, g.m, g.k, g.lda, BM, kb, pa) ||
      !encode(&mAl, g.a_lo, g.m, g.k, g.lda, BM, kb, pa) ||
      !encode(&mBh, g.b_hi, g.k, g.n, g.ldb, kb, bn, pb) ||
      !encode(&mBl, g.b_lo, g.k, g.n, g.ldb, kb, bn, pb)) {
    if (xbuf != nullptr) cudaFreeAsync(xbuf, s);
    return cudaErrorNotSupported;
  }
  const int tiles_m = (int)((g.m + BM - 1) / BM), tiles_n = (int)((g.n + bn - 1) / bn);
  const int splits = g.kchunk >= g.k ? 1 : (int)((g.k + g.kchunk - 1) / g.kchunk);
  auto pick = [&](auto c0, auto c1, auto c2) { return g.syrk == 1 ? c1 : (g.syrk == 2 ? c2 : c0); };
  GemmArgs ga = g;
  // Concurrent schedule (no split-K): the cross-term kernel runs on a second
  // stream alongside the hi * hi kernel -- each kernel's last partial wave
  // is filled by the other's CTAs -- and a final HBM-bound pass adds
  // alpha * X to C.  With split-K the partial sums take X in slice 0 instead
  // (cross first, then the kernel).  DDB_CROSS_SERIAL=1: always the latter.
  static const bool cross_serial = std::getenv("DDB_CROSS_SERIAL") != nullptr;
  const bool concurrent = split_alg && splits == 1 && !cross_serial && !shallow_wide;
  cudaStream_t s2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  if (split_alg) {
    int nl = 0;
    cudaError_t e = cudaSuccess;
    if (concurrent) {
      e = aux_stream(&s2);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming);
      if (e == cudaSuccess) e = cudaEventRecord(ev_fork, s);   // operands + xbuf ready
      if (e == cudaSuccess) e = cudaStreamWaitEvent(s2, ev_fork, 0);
      if (e == cudaSuccess) e = launch_cross_dmma(g, xbuf, s2, &nl, xslices, xchunk);
      if (e == cudaSuccess) e = cudaEventRecord(ev_join, s2);
    } else {
      e = launch_cross_dmma(g, xbuf, s, &nl, xslices, xchunk);
      ga.cross = xbuf;
    }
    if (e != cudaSuccess) {
      if (ev_fork) cudaEventDestroy(ev_fork);
      if (ev_join) cudaEventDestroy(ev_join);
      cudaFreeAsync(xbuf, s);
      return e;
    }
  }
  auto kern = split_alg ? pick(dd_tma_nn_kernel<ALG_SPLIT, 0>, dd_tma_nn_kernel<ALG_SPLIT, 1>,
                               dd_tma_nn_kernel<ALG_SPLIT, 2>)
              : alg == ALG_CERT
                  ? pick(dd_tma_nn_kernel<ALG_CERT, 0>, dd_tma_nn_kernel<ALG_CERT, 1>,
                         dd_tma_nn_kernel<ALG_CERT, 2>)
                  : pick(dd_tma_nn_kernel<ALG_TWOSUM, 0>, dd_tma_nn_kernel<ALG_TWOSUM, 1>,
                         dd_tma_nn_kernel<ALG_TWOSUM, 2>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) {
    if (xbuf != nullptr) cudaFreeAsync(xbuf, s);
    return e;
  }
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t units = (int64_t)tiles_m * tiles_n * splits;
  // Default: the persistent walk, one CTA per SM (the producer runs ahead
  // across unit boundaries, so a unit's prologue / epilogue overlaps the
  // next unit's loads: 8192 x 7936 x 256 in 8.00 vs 8.53 ms, 8192^3 226.2 vs
  // 227.4, Rtrsm 8192 152.7 vs 157.1), except for Rsyrk (n = 4096 3875 vs
  // 4350 dd GFlops; a walk over the triangle's tiles only, evenly spread,
  // did no better: 18.1 vs 15.9 ms) and inside Rpotrf / Rgetrf
  // (NoPersistScope), whose
  // high-priority panel stream needs SMs to free up while a trailing update
  // runs (Rgetrf 142.7 vs 137.3 ms persistent; a walk over 148 - R SMs
  // leaving R to the panel stream did worse still: R = 8 / 16 / 32 gave
  // 144.8 / 147.3 / 151.7 ms).  DDB_TMA_PERSISTENT=0 / 1
  // forces one CTA per unit / the walk everywhere.
  static const int penv = [] {
    const char* v = std::getenv("DDB_TMA_PERSISTENT");
    return v ? (v[0] == '0' ? 0 : 1) : -1;
  }();
  const bool persist = penv == 1 || (penv < 0 && tma::g_no_persist == 0 && g.syrk == 0);
  const int grid = persist ? (int)(units < sms ? units : sms) : (int)units;
  kern<<<grid, NTK, SMEM_BYTES, s>>>(ga, mAh, mAl, mBh, mBl, row_exp, col_exp, flag, tiles_m,
                                    tiles_n, splits);
  e = cudaGetLastError();
  if (concurrent) {
    const cudaError_t ej = cudaStreamWaitEvent(s, ev_join, 0);
    if (e == cudaSuccess) e = ej;
    if (e == cudaSuccess) {
      int64_t blocks = (g.m * g.n + 255) / 256;
      if (blocks > 16 * (int64_t)sms) blocks = 16 * (int64_t)sms;
      cross_add_kernel<<<(unsigned)blocks, 256, 0, s>>>(ga, xbuf);
      e = cudaGetLastError();
    }
    cudaEventDestroy(ev_fork);
    cudaEventDestroy(ev_join);
  }
  if (xbuf != nullptr) {
    const cudaError_t e2 = cudaFreeAsync(xbuf, s);
    if (e == cudaSuccess) e = e2;
  }
  return e;
}

}  // namespace ddb
