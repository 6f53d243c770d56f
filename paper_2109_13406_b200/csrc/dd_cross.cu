// dd_cross.cu -- the split algorithm's cross terms on the FP64 tensor path,
// hand-written for sm_100a (replaces two cuBLAS DGEMMs).
//
//   X (m x n, ld = m) = A_lo B_hi + A_hi B_lo          (NN form, dd_tma.cu)
//
// one binary64 GEMM of depth 2k: every k-tile stages the four operand tiles
// (A_lo, A_hi: 128 x 16, B_hi, B_lo: 16 x 128) with TMA (cp.async.bulk.tensor,
// 128-byte swizzle) into a 3-stage ring guarded by transaction-counted
// mbarriers (one producer warp), and 8 warps accumulate their 64 x 32 sub-tiles with
// mma.sync.m16n8k4.f64 (DMMA): per k4 step a warp loads 8 + 4 fragment
// doubles and issues 2 x 16 DMMA (each 512 multiply-adds).  DMMA shares the
// FP64 pipe with DFMA (same 64 FMA / clk / SM), so the bound is the FP64
// roof: 2 m n k multiply-adds at 18.6 T FMA/s = 59.2 ms at 8192^3.
//
// Rsyrk (syrk = 1 upper / 2 lower, with B = A^T): tiles outside the uplo
// triangle are skipped; X is then A_lo A_hi^T + A_hi A_lo^T on the triangle.
//
// Accuracy: every product and sum is an IEEE binary64 operation in some order,
// so |X - exact| <= 2k u sum_l (|al bh| + |ah bl|) <= 4k u^2 sum_l |ah bh| for
// normalised operands (|lo| <= 2^-53 |hi|, enforced by the prescan): one unit
// of the c k 2^-104 budget (dd_tma.cu's header).
//
// Shared-memory layout (TMA SWIZZLE_128B): A tiles as 8 boxes of 16 (m) x 16
// (k) doubles, row k at 128 k bytes, its 16-byte chunk (m % 16) / 2 XORed with
// k % 8; B tiles as 128 rows (n) of 16 k doubles, chunk k / 2 XORed with n % 8.
// The B fragment loads are conflict-free (2 wavefronts per LDS.64), the A
// ones 4 wavefronts; at one warp-k4-step per 128 SM cycles that is ~40 of the
// 128 available wavefront slots.
#include <cmath>

#include "internal.h"
#include "tma_util.cuh"

namespace ddb {
namespace cross {

using namespace tma;

constexpr int BM = 128, BN = 128, BK = 16, STAGES = 3;
// 8 consumer warps (two warpgroups) + one producer warpgroup whose first
// lane issues the TMA loads; setmaxnreg moves the producer's registers to
// the consumers (40 / 232 per thread against 168 at launch)
constexpr int NCW = 8, NT = 32 * (NCW + 4);
constexpr int REG_CONSUMER = 232, REG_PRODUCER = 40;
constexpr int WM = 64, WN = 32;                    // warp tile (2 x 4 warps)
constexpr int MT = WM / 16, NTL = WN / 8;          // m16 / n8 tiles per warp
constexpr uint32_t A_TILE = BM * BK * 8;           // 16 KB per plane
constexpr uint32_t B_TILE = BN * BK * 8;           // 16 KB per plane
constexpr uint32_t STAGE_BYTES = 2 * A_TILE + 2 * B_TILE;   // 64 KB
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 2 * STAGES * 8 + 1024;
constexpr int GROUP_M = 8;

__device__ __forceinline__ void dmma_16x8x4(double (&d)[4], double a0, double a1, double b0) {
  asm volatile(
      "mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0, %1, %2, %3}, {%4, %5}, {%6}, "
      "{%0, %1, %2, %3};\n"
      : "+d"(d[0]), "+d"(d[1]), "+d"(d[2]), "+d"(d[3])
      : "d"(a0), "d"(a1), "d"(b0));
}

__device__ __forceinline__ double lds64(uint32_t addr) {
  double v;
  asm volatile("ld.shared.f64 %0, [%1];\n" : "=d"(v) : "r"(addr));
  return v;
}

template <int SYRK>
__global__ void __launch_bounds__(NT, 1)
cross_dmma_kernel(const __grid_constant__ CUtensorMap mAl, const __grid_constant__ CUtensorMap mAh,
                  const __grid_constant__ CUtensorMap mBh, const __grid_constant__ CUtensorMap mBl,
                  double* __restrict__ x, int64_t m, int64_t n, int64_t k, int tiles_m,
                  int tiles_n, int64_t kchunk) {
  // split-K: blockIdx.y = k-slice z over [z kchunk, (z + 1) kchunk), its sum
  // to plane z of x (m x n each; cross_reduce_kernel adds the planes in order)
  const int64_t kz0 = (int64_t)blockIdx.y * kchunk;
  const int64_t kz1 = kz0 + kchunk < k ? kz0 + kchunk : k;
  x += (size_t)blockIdx.y * m * n;
  // grouped raster over the tile grid (L2 reuse of the A / B panels)
  const int bid = blockIdx.x;
  const int group_size = GROUP_M * tiles_n;
  const int first_m = (bid / group_size) * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int local = bid % group_size;
  const int64_t i0 = (int64_t)(first_m + local % gm) * BM, j0 = (int64_t)(local / gm) * BN;
  if (SYRK == 1 && i0 > j0 + BN - 1) return;
  if (SYRK == 2 && i0 + BM - 1 < j0) return;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = saddr(smem_raw);
  const uint32_t ring = raw + ((1024u - (raw & 1023u)) & 1023u);   // swizzle needs 1 KB alignment
  unsigned char* ring_g = smem_raw + (ring - raw);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring_g + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NCW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  __syncthreads();

  const int ktiles = (int)((kz1 - kz0 + BK - 1) / BK);   // kchunk is a multiple of BK
  if (warp >= NCW) {
    asm volatile("setmaxnreg.dec.sync.aligned.u32 %0;\n" ::"n"(REG_PRODUCER));
    // ---- TMA producer: one lane walks the k-tiles ahead of the consumers ----
    if (warp == NCW && lane == 0) {
      for (int kt = 0; kt < ktiles; ++kt) {
        const int s = kt % STAGES;
        if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
        unsigned char* st = ring_g + (size_t)s * STAGE_BYTES;
        const int kc = (int)(kz0 + (int64_t)kt * BK);
        mbar_expect_tx(&full[s], STAGE_BYTES);
#pragma unroll
        for (int b = 0; b < BM / 16; ++b) {
          tma_load_2d(st + b * 2048, &mAl, (int)i0 + 16 * b, kc, &full[s]);
          tma_load_2d(st + A_TILE + b * 2048, &mAh, (int)i0 + 16 * b, kc, &full[s]);
        }
        tma_load_2d(st + 2 * A_TILE, &mBh, kc, (int)j0, &full[s]);
        tma_load_2d(st + 2 * A_TILE + B_TILE, &mBl, kc, (int)j0, &full[s]);
      }
    }
    return;
  }

  asm volatile("setmaxnreg.inc.sync.aligned.u32 %0;\n" ::"n"(REG_CONSUMER));
  const int wm = warp & 1, wn = warp >> 1;
  const int g = lane >> 2, tig = lane & 3;
  double acc[MT][NTL][4];
#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NTL; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[a][b][q] = 0.0;

  // lane-constant parts of the swizzled fragment addresses
  const uint32_t a_lane = (uint32_t)(wm * MT) * 2048u + (uint32_t)(g & 1) * 8u;
  const uint32_t b_lane = (uint32_t)(wn * WN + g) * 128u + (uint32_t)(tig & 1) * 8u;

  for (int kt = 0; kt < ktiles; ++kt) {
    const int s = kt % STAGES;
    mbar_wait(&full[s], (kt / STAGES) & 1);
    const uint32_t st = ring + (uint32_t)s * STAGE_BYTES;
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      const int kr = kk + tig;                       // this lane's k row
      const uint32_t arow = (uint32_t)kr * 128u;
      const uint32_t ach0 = (uint32_t)(((g >> 1) ^ (kr & 7)) << 4);
      const uint32_t ach1 = ach0 ^ 64u;              // rows g + 8: chunk + 4
      const uint32_t bch = (uint32_t)((((kk >> 1) + (tig >> 1)) ^ g) << 4);
#pragma unroll
      for (int pr = 0; pr < 2; ++pr) {   // pr 0: A_lo * B_hi, pr 1: A_hi * B_lo
        const uint32_t abase = st + (pr ? A_TILE : 0u) + a_lane + arow;
        const uint32_t bbase = st + 2 * A_TILE + (pr ? B_TILE : 0u) + b_lane + bch;
        double af[MT][2], bf[NTL];
#pragma unroll
        for (int a = 0; a < MT; ++a) {
          af[a][0] = lds64(abase + a * 2048u + ach0);
          af[a][1] = lds64(abase + a * 2048u + ach1);
        }
#pragma unroll
        for (int b = 0; b < NTL; ++b) bf[b] = lds64(bbase + b * 8u * 128u);
#pragma unroll
        for (int a = 0; a < MT; ++a)
#pragma unroll
          for (int b = 0; b < NTL; ++b) dmma_16x8x4(acc[a][b], af[a][0], af[a][1], bf[b]);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
  }

#pragma unroll
  for (int a = 0; a < MT; ++a)
#pragma unroll
    for (int b = 0; b < NTL; ++b)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int64_t i = i0 + wm * WM + a * 16 + g + (q >> 1) * 8;
        const int64_t j = j0 + wn * WN + b * 8 + 2 * tig + (q & 1);
        if (i < m && j < n) x[i + j * m] = acc[a][b][q];
      }
}

}  // namespace cross

// X = A_lo B_hi + A_hi B_lo for an NN-form call (16-byte aligned planes, even
// lda / ldb: tma_eligible); cudaErrorNotSupported when a map cannot be made.
// x_0 += x_1 + ... + x_{S-1} in slice order (deterministic for a given shape)
__global__ void __launch_bounds__(256)
cross_reduce_kernel(double* __restrict__ x, int64_t mn, int slices) {
  for (int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x; i < mn;
       i += (int64_t)gridDim.x * 256) {
    double v = x[i];
    for (int z = 1; z < slices; ++z) v = __dadd_rn(v, x[(size_t)z * mn + i]);
    x[i] = v;
  }
}

// k-slices for the cross kernel: the tile grid alone can leave the last wave
// mostly empty (m = n = 2048: 256 tiles = 1.7 waves on 148 SMs); splitting k
// into S slices (each >= 1024 deep, a multiple of BK) multiplies the work
// units.  S = 1 unless it buys > 3 % of wave efficiency.
int cross_kslices(const GemmArgs& g, int64_t* kchunk) {
  using namespace cross;
  *kchunk = g.k;
  int dev = 0, sms = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t tm = (g.m + BM - 1) / BM, tn = (g.n + BN - 1) / BN;
  int64_t tiles = 0;
  if (g.syrk == 0) {
    tiles = tm * tn;
  } else {
    for (int64_t j = 0; j < tn; ++j)
      for (int64_t i = 0; i < tm; ++i)
        if (g.syrk == 1 ? i * BM <= j * BN + BN - 1 : i * BM + BM - 1 >= j * BN) ++tiles;
  }
  auto eff = [&](int64_t t) {
    const double w = (double)t / sms;
    return w / std::ceil(w);
  };
  double best = eff(tiles);
  int best_s = 1;
  for (int sl = 2; sl <= 8; ++sl) {
    int64_t chunk = (g.k + sl - 1) / sl;
    chunk = (chunk + BK - 1) / BK * BK;
    if (chunk < 1024) break;
    const int real = (int)((g.k + chunk - 1) / chunk);
    const double e = eff(tiles * real);
    if (e > best + 0.03) {
      best = e;
      best_s = real;
      *kchunk = chunk;
    }
  }
  if (best_s == 1) *kchunk = g.k;
  return best_s;
}

cudaError_t launch_cross_dmma(const GemmArgs& g, double* x, cudaStream_t s, int* nlaunch,
                              int slices, int64_t kchunk) {
  using namespace cross;
  alignas(64) CUtensorMap mAl, mAh, mBh, mBl;
  const auto dt = CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  const auto pa = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (!tma::encode2d(&mAl, g.a_lo, dt, g.m, g.k, g.lda * 8, 16, BK, sw, pa) ||
      !tma::encode2d(&mAh, g.a_hi, dt, g.m, g.k, g.lda * 8, 16, BK, sw, pa) ||
      !tma::encode2d(&mBh, g.b_hi, dt, g.k, g.n, g.ldb * 8, BK, BN, sw, pa) ||
      !tma::encode2d(&mBl, g.b_lo, dt, g.k, g.n, g.ldb * 8, BK, BN, sw, pa))
    return cudaErrorNotSupported;
  auto kern = g.syrk == 1 ? cross_dmma_kernel<1>
                          : (g.syrk == 2 ? cross_dmma_kernel<2> : cross_dmma_kernel<0>);
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       (int)SMEM_BYTES);
  if (e != cudaSuccess) return e;
  const int tiles_m = (int)((g.m + BM - 1) / BM), tiles_n = (int)((g.n + BN - 1) / BN);
  if (slices < 1) { slices = 1; kchunk = g.k; }
  kern<<<dim3(tiles_m * tiles_n, slices), NT, SMEM_BYTES, s>>>(mAl, mAh, mBh, mBl, x, g.m, g.n,
                                                               g.k, tiles_m, tiles_n, kchunk);
  ++*nlaunch;
  e = cudaGetLastError();
  if (e != cudaSuccess || slices == 1) return e;
  const int64_t mn = g.m * g.n;
  int64_t blocks = (mn + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  cross_reduce_kernel<<<(unsigned)blocks, 256, 0, s>>>(x, mn, slices);
  ++*nlaunch;
  return cudaGetLastError();
}

}  // namespace ddb
