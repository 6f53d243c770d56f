// split_feed.cu -- microbenchmark: how fast can the split kernel's
// instruction mix (dd_tma.cu ALG_SPLIT: Tn = fma(a,b,T), d = T - Tn,
// r = fma(a,b,d), L += r per MAC, a 3-op fold every 3 steps; 8 x 4
// micro-tile, 256 threads, 1 CTA / SM) run on the FP64 pipe when its
// operands come from
//   FEED 0: registers (the ceiling),
//   FEED 1: shared memory, LDS.128 as in the kernel (12 per 2 k-steps),
//   FEED 2: tensor memory, tcgen05.ld 32x32b.x32 + .x16 per 2 k-steps,
//           double-buffered (the next pair's loads in flight during this
//           pair's math; tcgen05.wait::ld before use).
// Prints FP64 instructions / s as a fraction of the pipe's peak
// (148 SMs x 64 lanes x clock, measured with a DFMA burn in the same run).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o split_feed split_feed.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int TM = 8, TN = 4;

// MIX 0: DADD for the additions (as dd_tma.cu); MIX 1: every addition as a
// DFMA with a unit factor (fma(x, 1, y) == x + y bit for bit)
template <int MIX>
__device__ __forceinline__ double add_(double x, double y) {
  return MIX ? __fma_rn(x, 1.0, y) : __dadd_rn(x, y);
}
template <int MIX>
__device__ __forceinline__ double sub_(double x, double y) {
  return MIX ? __fma_rn(y, -1.0, x) : __dsub_rn(x, y);
}

template <int MIX>
__device__ __forceinline__ void pair_math(double (&T)[TM][TN], double (&L)[TM][TN],
                                          const double (&a)[2][TM], const double (&b)[2][TN],
                                          int step0) {
#pragma unroll
  for (int q = 0; q < 2; ++q) {
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const double t = T[i][j];
        const double tn = __fma_rn(a[q][i], b[q][j], t);
        L[i][j] = add_<MIX>(L[i][j], __fma_rn(a[q][i], b[q][j], sub_<MIX>(t, tn)));
        T[i][j] = tn;
      }
    if ((step0 + q + 1) % 3 == 0) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const double t2 = add_<MIX>(T[i][j], L[i][j]);
          L[i][j] = sub_<MIX>(L[i][j], sub_<MIX>(t2, T[i][j]));
          T[i][j] = t2;
        }
    }
  }
}

template <int N>
__device__ __forceinline__ void tmem_ld(uint32_t taddr, uint32_t (&v)[N]);
template <>
__device__ __forceinline__ void tmem_ld<32>(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15, %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, "
      "%28, %29, %30, %31}, [%32];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}
template <>
__device__ __forceinline__ void tmem_ld<16>(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, "
      "%11, %12, %13, %14, %15}, [%16];\n"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}

template <int FEED, int MIX>
__global__ void __launch_bounds__(256, 1) feed_kernel(double* out, int iters, double s0) {
  __shared__ __align__(16) double sm[2][24][128];   // A (24 k x 128 m) | B (as 64 cols x 24 k)
  __shared__ uint32_t tslot;
  for (int i = threadIdx.x; i < 2 * 24 * 128; i += 256) (&sm[0][0][0])[i] = 1.0 + (i & 127) * 1e-9;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (FEED == 2) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(
          (uint32_t)__cvta_generic_to_shared(&tslot)));
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  }
  __syncthreads();
  if (FEED == 2) asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tbase = FEED == 2 ? tslot + ((uint32_t)((warp & 3) * 32) << 16) : 0;
  if (FEED == 2 && warp < 4) {   // fill this lane quarter with ~1.0 values (hi words only)
    for (int c = 0; c < 512; c += 16) {
      uint32_t v[16];
#pragma unroll
      for (int x = 0; x < 16; ++x) v[x] = (x & 1) ? 0x3FF00000u + lane : 0u;
      asm volatile(
          "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8, %9, "
          "%10, %11, %12, %13, %14, %15, %16};\n" ::"r"(tbase + c),
          "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
          "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
          "r"(v[15]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory");
  }
  if (FEED == 2) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  }
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  double T[TM][TN], L[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) { T[i][j] = s0; L[i][j] = 0.0; }
  double a[2][2][TM], b[2][2][TN];   // [buffer][step in pair][...]
  auto load_pair = [&](int buf, int p) {
    if (FEED == 0) {
#pragma unroll
      for (int q = 0; q < 2; ++q) {
#pragma unroll
        for (int i = 0; i < TM; ++i) a[buf][q][i] = 1.0 + (i + p) * 1e-7;
#pragma unroll
        for (int j = 0; j < TN; ++j) b[buf][q][j] = 0.5 + (j - p) * 1e-7;
      }
    } else if (FEED == 1) {
      const int k0 = (2 * p) % 24;
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int g = 0; g < TM / 2; ++g) {
          const double2 h = *reinterpret_cast<const double2*>(&sm[0][k0 + q][g * 32 + tx * 2]);
          a[buf][q][2 * g] = h.x;
          a[buf][q][2 * g + 1] = h.y;
        }
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const int cj = (j >> 1) * 32 + ty * 2 + (j & 1);
        const double2 h = *reinterpret_cast<const double2*>(&(&sm[1][0][0])[cj * 24 + k0]);
        b[buf][0][j] = h.x;
        b[buf][1][j] = h.y;
      }
    } else {
      uint32_t va[32], vb[16];
      const uint32_t col = (uint32_t)((p % 10) * 48);
      tmem_ld<32>(tbase + col, va);
      tmem_ld<16>(tbase + col + 32, vb);
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int i = 0; i < TM; ++i)
          a[buf][q][i] = __hiloint2double(va[2 * (q * TM + i) + 1], va[2 * (q * TM + i)]);
#pragma unroll
      for (int q = 0; q < 2; ++q)
#pragma unroll
        for (int j = 0; j < TN; ++j)
          b[buf][q][j] = __hiloint2double(vb[2 * (q * TN + j) + 1], vb[2 * (q * TN + j)]);
    }
  };
  load_pair(0, 0);
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int p = 0; p < 6; ++p) {   // 12 k-steps: 4 folds
      const int buf = p & 1;
      if (FEED == 2) asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
      load_pair(buf ^ 1, it * 6 + p + 1);
      pair_math<MIX>(T, L, a[buf], b[buf], 2 * p);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) s += T[i][j] + L[i][j];
  if (s == 12345.0) out[0] = s;
  if (FEED == 2) {
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (warp == 0)
      asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(tslot));
  }
}

__global__ void __launch_bounds__(256) dfma_burn(double* out, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) x[i] = __fma_rn(x[i], 0.999999, 1e-9);
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <int FEED, int MIX>
double run(int sms, double* out, int iters) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    feed_kernel<FEED, MIX><<<sms, 256>>>(out, iters, 1.5);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("FEED %d: %s\n", FEED, cudaGetErrorString(e));
  // FP64 warp-instructions x 32 lanes: per 12 steps and element 12 x 4 + 4 x 3
  const double lane_ops = (double)sms * 256 * iters * TM * TN * (12.0 * 4 + 4 * 3);
  return lane_ops / (best * 1e-3);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 4; ++rep) {
    cudaEventRecord(e0);
    dfma_burn<<<sms * 4, 256>>>(out, 2000);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (rep && ms < best) best = ms;
  }
  const double peak = (double)sms * 4 * 256 * 2000 * 16 * 8 / (best * 1e-3);
  printf("DFMA burn: %.3f T lane-op/s\n", peak / 1e12);
  const int iters = 4000;
  const char* feeds[3] = {"registers", "LDS.128", "tcgen05.ld"};
  double f[2][3] = {{run<0, 0>(sms, out, iters), run<1, 0>(sms, out, iters), run<2, 0>(sms, out, iters)},
                    {run<0, 1>(sms, out, iters), run<1, 1>(sms, out, iters), run<2, 1>(sms, out, iters)}};
  for (int m = 0; m < 2; ++m)
    for (int x = 0; x < 3; ++x)
      printf("MIX %d (%s) FEED %d (%s): %.1f %% of the pipe\n", m, m ? "adds as DFMA" : "DADD",
             x, feeds[x], 100 * f[m][x] / peak);
  return 0;
}
