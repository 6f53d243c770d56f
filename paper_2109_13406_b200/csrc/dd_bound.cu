// dd_bound.cu -- certified per-element magnitude bound for the fast mode, on
// hand-written sm_100a kernels (a bf16 tcgen05 GEMM with a TMEM accumulator).
//
// The fast accumulator (ALG_CERT / ALG_SPLIT, dd_tiled.cuh / dd_tma.cu)
// anchors each element's running sum at sigma = 1.5 * 2^E, which is exact
// and error-bounded only if 2^E >= 2 * sum_l |a_il * b_lj| for that element.
// This file produces a guaranteed upper bound Sigma'_ij of that sum:
//
//   1. abs_bf16_kmajor_kernel: |hi| of op(A) (resp. op(B)) scaled by the
//      per-row (per-column) exponent maximum e from the prescan, by
//      2^(1022 - e) into [0, 1), rounded UP to fp32 and then UP to bf16, so
//      every converted value is >= the scaled |hi| it replaces.  Written
//      K-major (op(A) as m rows of kp bf16, op(B) as n rows), zero-padded to
//      kp = k rounded up to 8: the canonical UMMA operand layout.
//   2. bound_umma_kernel: S = op(A)^ * op(B)^ with tcgen05.mma kind::f16
//      (bf16 x bf16 -> fp32 in TMEM), 128 x 128 tiles, TMA (SWIZZLE_128B)
//      feeding a 3-stage ring, one elected thread issuing the MMAs, the
//      accumulator read back with tcgen05.ld by 4 epilogue warps.
//
// Bound (host.cu): Sigma' = (S_ij (1 + k 2^-21) + k 2^-120) * 2^(e_i + f_j - 2044).
//   * all terms are >= 0, so with a per-addition relative error <= 2^-22
//     (fp32, truncating adders and one guard bit of slack included) the
//     computed S >= (1 - k 2^-22) sum, and (1 + k 2^-21)(1 - k 2^-22) >= 1
//     for k <= 2^20 (calls deeper than kCertMaxK = 2^16 take TwoSum);
//   * a converted value below bf16's normal range may be flushed by the
//     tensor core: each such product is < 2^-126, covered by k 2^-120.
// Tightness: S' <= (1.0157 sum^ + k 2^-131)(1 + k 2^-21) + k 2^-120 in the
// scaled units, where sum^ >= 2^-(sa + sb + 2) for an element whose row /
// column exponent spreads are sa / sb (the scaled magnitudes lie in
// [2^-(s+1), 1)).  So S' / sum <= 1.0157 (1 + k 2^-21) + k 2^-118 2^(sa + sb)
// <= 1.064 for k <= 2^16 whenever sa + sb <= 112 - ceil(log2 k) (wide_limit,
// internal.h); wider elements are EC_WIDE and take the TwoSum fallback.
// The anchored kernels need S' / sum <= 1.14 (ALG_CERT: c = 3.5 S'/sum) and
// <= 1.1 (ALG_SPLIT: c = 2.5 S'/sum + 1.25) for c = 4.
//
// Cost at n = 8192: ~0.3 ms for the conversions (HBM-bound: 8 B read + 2 B
// written per element) plus ~0.8 ms of tensor-core time.
#include <cuda_bf16.h>

#include "internal.h"
#include "tma_util.cuh"

namespace ddb {

// ---- 1. magnitudes, scaled and rounded up, K-major ---------------------------

// op rows r < rows_op, k index l < k; stored element (r, l) at
// kcontig ? src[l + r * ld] : src[r + l * ld].  out[r * kp + l], zero for
// l in [k, kp).  32 x 32 tiles through shared memory when the stored layout
// is not k-contiguous (both sides coalesced).
__global__ void __launch_bounds__(256)
abs_bf16_kmajor_kernel(const double* __restrict__ src, int64_t ld, int64_t rows_op, int64_t k,
                       int64_t kp, int kcontig, const int* __restrict__ exps,
                       __nv_bfloat16* __restrict__ out) {
  __shared__ __nv_bfloat16 t[32][34];
  const int64_t r0 = (int64_t)blockIdx.y * 32, l0 = (int64_t)blockIdx.x * 32;
  const int tx = threadIdx.x, ty = threadIdx.y;
  for (int yy = ty; yy < 32; yy += 8) {
    // kcontig: read along l (tx), one op row per yy; else along r (tx)
    const int64_t r = kcontig ? r0 + yy : r0 + tx;
    const int64_t l = kcontig ? l0 + tx : l0 + yy;
    __nv_bfloat16 v = __float2bfloat16(0.0f);
    if (r < rows_op && l < k) {
      // scale 2^(1022 - e): |x| * scale < 1 for every |x| < 2^(e - 1022) (exact)
      const int e = exps[r];
      const double scale = __longlong_as_double((long long)(2045 - e) << 52);
      const double x = fabs(kcontig ? src[l + r * ld] : src[r + l * ld]) * scale;
      v = __float2bfloat16_ru(__double2float_ru(x));
    }
    if (kcontig) t[yy][tx] = v; else t[tx][yy] = v;     // t[r - r0][l - l0]
  }
  __syncthreads();
  for (int yy = ty; yy < 32; yy += 8) {
    const int64_t r = r0 + yy, l = l0 + tx;
    if (r < rows_op && l < kp) out[r * kp + l] = t[yy][tx];
  }
}

static cudaError_t convert(const double* src, int64_t ld, int64_t rows_op, int64_t k, int64_t kp,
                           int kcontig, const int* exps, __nv_bfloat16* out, cudaStream_t s,
                           int* nlaunch) {
  if (rows_op <= 0) return cudaSuccess;
  const int64_t gy_total = (rows_op + 31) / 32;
  for (int64_t y0 = 0; y0 < gy_total; y0 += 65535) {   // gridDim.y <= 65535
    const int64_t gy = gy_total - y0 < 65535 ? gy_total - y0 : 65535;
    const int64_t rbase = y0 * 32;
    dim3 grid((unsigned)((kp + 31) / 32), (unsigned)gy), block(32, 8);
    const double* sb = kcontig ? src + rbase * ld : src + rbase;
    abs_bf16_kmajor_kernel<<<grid, block, 0, s>>>(sb, ld, rows_op - rbase, k, kp, kcontig,
                                                  exps + rbase, out + rbase * kp);
    ++*nlaunch;
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// ---- 2. the tcgen05 GEMM ------------------------------------------------------

namespace umma {

using namespace tma;

constexpr int BM = 128, BN = 128, BK = 64, STAGES = 3, NT = 128;   // 4 warps
constexpr uint32_t A_BYTES = BM * BK * 2, B_BYTES = BN * BK * 2;   // 16 KB each
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
constexpr size_t SMEM_BYTES = (size_t)STAGES * STAGE_BYTES + 1024 + 256;
constexpr uint32_t TMEM_COLS = BN;                                  // fp32 accumulator 128 x 128
// instruction descriptor, kind::f16: D f32 (bit 4), A / B bf16 (bits 7, 10),
// both K-major, N >> 3 at bit 17, M >> 4 at bit 24
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
constexpr int GROUP_M = 8;

// shared-memory matrix descriptor: K-major, 128-byte swizzle (rows of 64 bf16,
// 8-row groups 1024 bytes apart), sm_100 version 1
__device__ __forceinline__ uint64_t desc_k_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)1 << 16) | ((uint64_t)(1024 >> 4) << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}

__device__ __forceinline__ void mma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                         uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                   saddr(bar))
               : "memory");
}

template <int SYRK>
__global__ void __launch_bounds__(NT, 1)
bound_umma_kernel(const __grid_constant__ CUtensorMap mA, const __grid_constant__ CUtensorMap mB,
                  float* __restrict__ S, int64_t m, int64_t n, int64_t kp, int tiles_m,
                  int tiles_n) {
  const int bid = blockIdx.x;
  const int group_size = GROUP_M * tiles_n;
  const int first_m = (bid / group_size) * GROUP_M;
  const int gm = min(tiles_m - first_m, GROUP_M);
  const int local = bid % group_size;
  const int64_t i0 = (int64_t)(first_m + local % gm) * BM, j0 = (int64_t)(local / gm) * BN;
  if (SYRK == 1 && i0 > j0 + BN - 1) return;   // only the uplo triangle is read
  if (SYRK == 2 && i0 + BM - 1 < j0) return;

  extern __shared__ __align__(1024) unsigned char smem_raw[];
  const uint32_t raw = saddr(smem_raw);
  const uint32_t pad = (1024u - (raw & 1023u)) & 1023u;
  unsigned char* ring = smem_raw + pad;                  // 1 KB aligned (SWIZZLE_128B)
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* done = empty + STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  }
  if (warp == 1) {   // TMEM: one warp allocates (and later frees) the accumulator columns
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(
                     saddr(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int ktiles = (int)((kp + BK - 1) / BK);
  if (warp == 0 && lane == 0) {
    // ---- TMA producer ----
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % STAGES;
      if (kt >= STAGES) mbar_wait(&empty[s], ((kt / STAGES) - 1) & 1);
      unsigned char* st = ring + (size_t)s * STAGE_BYTES;
      mbar_expect_tx(&full[s], STAGE_BYTES);
      tma_load_2d(st, &mA, kt * BK, (int)i0, &full[s]);
      tma_load_2d(st + A_BYTES, &mB, kt * BK, (int)j0, &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---- MMA issuer: one thread for the CTA ----
    for (int kt = 0; kt < ktiles; ++kt) {
      const int s = kt % STAGES;
      mbar_wait(&full[s], (kt / STAGES) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t a0 = saddr(ring + (size_t)s * STAGE_BYTES);
      const uint32_t b0 = a0 + A_BYTES;
#pragma unroll
      for (int kk = 0; kk < BK / 16; ++kk)   // K = 16 per MMA: 32 bytes along the row
        mma_bf16(tmem, desc_k_sw128(a0 + kk * 32), desc_k_sw128(b0 + kk * 32),
                 (kt | kk) != 0);
      mma_commit(&empty[s]);                  // frees the stage once these MMAs are done
    }
    mma_commit(done);                         // accumulator complete
  }
  __syncwarp();

  // ---- epilogue: TMEM lanes 32w..32w+31 = tile rows, columns = tile columns ----
  mbar_wait(done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const int64_t i = i0 + warp * 32 + lane;
#pragma unroll 1
  for (int c0 = 0; c0 < BN; c0 += 32) {
    uint32_t v[32];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
        "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
        "%28, %29, %30, %31}, [%32];\n"
        : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
          "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]),
          "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]),
          "=r"(v[19]), "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]),
          "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]),
          "=r"(v[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (i < m) {
#pragma unroll
      for (int c = 0; c < 32; ++c) {
        const int64_t j = j0 + c0 + c;
        if (j < n) S[i + j * m] = __uint_as_float(v[c]);   // warp-coalesced along i
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem),
                 "r"(TMEM_COLS));
}

}  // namespace umma

static int64_t kpad(int64_t k) { return (k + 7) / 8 * 8; }

size_t bound_workspace_bytes(const GemmArgs& g) {
  const size_t kp = (size_t)kpad(g.k);
  const size_t a = (size_t)g.m * kp, b = g.syrk ? 0 : (size_t)g.n * kp;
  return ((2 * a + 1023) / 1024 + (2 * b + 1023) / 1024) * 1024 + 4 * (size_t)g.m * g.n + 1024;
}

float* bound_carve(const GemmArgs& g, void* ws) {
  const size_t kp = (size_t)kpad(g.k);
  const size_t a = (size_t)g.m * kp, b = g.syrk ? 0 : (size_t)g.n * kp;
  return reinterpret_cast<float*>(static_cast<char*>(ws) +
                                  ((2 * a + 1023) / 1024 + (2 * b + 1023) / 1024) * 1024);
}

// Fills bound (m x n, ld = m, fp32) from the operands and the prescan maxima.
cudaError_t launch_bound(const GemmArgs& g, const int* row_exp, const int* col_exp, void* ws,
                         float* bound, cudaStream_t s, int* nlaunch, const char** what) {
  const int64_t kp = kpad(g.k);
  __nv_bfloat16* abf = static_cast<__nv_bfloat16*>(ws);
  __nv_bfloat16* bbf =
      reinterpret_cast<__nv_bfloat16*>(static_cast<char*>(ws) + (2 * (size_t)g.m * kp + 1023) / 1024 * 1024);
  // op(A) rows: stored A is m x k (N: k along stored columns) or k x m (T)
  cudaError_t e = convert(g.a_hi, g.lda, g.m, g.k, kp, g.ta != 0, row_exp, abf, s, nlaunch);
  if (e == cudaSuccess && !g.syrk)   // op(B) columns: stored B is k x n (N) or n x k (T)
    e = convert(g.b_hi, g.ldb, g.n, g.k, kp, g.tb == 0, col_exp, bbf, s, nlaunch);
  if (e != cudaSuccess) { *what = "bound conversion"; return e; }
  if (g.syrk) bbf = abf;   // op(B) = op(A)^T: the same K-major rows
  using namespace umma;
  alignas(64) CUtensorMap mA, mB;
  const auto dt = CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
  const auto sw = CU_TENSOR_MAP_SWIZZLE_128B;
  const auto pr = CU_TENSOR_MAP_L2_PROMOTION_L2_128B;
  if (!tma::encode2d(&mA, abf, dt, kp, g.m, kp * 2, BK, BM, sw, pr) ||
      !tma::encode2d(&mB, bbf, dt, kp, g.n, kp * 2, BK, BN, sw, pr)) {
    *what = "bound tensor maps";
    return cudaErrorNotSupported;
  }
  auto kern = g.syrk == 1 ? bound_umma_kernel<1>
                          : (g.syrk == 2 ? bound_umma_kernel<2> : bound_umma_kernel<0>);
  e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM_BYTES);
  if (e != cudaSuccess) { *what = "bound kernel attributes"; return e; }
  const int tiles_m = (int)((g.m + BM - 1) / BM), tiles_n = (int)((g.n + BN - 1) / BN);
  kern<<<tiles_m * tiles_n, NT, SMEM_BYTES, s>>>(mA, mB, bound, g.m, g.n, kp, tiles_m, tiles_n);
  ++*nlaunch;
  e = cudaGetLastError();
  if (e != cudaSuccess) *what = "bound kernel launch";
  return e;
}

}  // namespace ddb
