// fp64_warps.cu -- microbenchmark: FP64-pipe fraction vs resident warps per
// SM and independent chains per thread, for a pure DFMA burn and for the
// split kernel's MAC mix (Tn = fma(a,b,T), d = T - Tn, r = fma(a,b,d), L += r,
// fold every 3 steps) on TM x TN register micro-tiles.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_warps fp64_warps.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void burn(double* out, int iters) {
  double x[CH];
#pragma unroll
  for (int i = 0; i < CH; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int i = 0; i < CH; ++i) x[i] = __fma_rn(x[i], 0.999999, 1e-9);
  double s = 0;
#pragma unroll
  for (int i = 0; i < CH; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <int TM, int TN, int LB = 0>
__global__ void __launch_bounds__(256, LB ? 1 : 0) mix(double* out, int iters) {
  double T[TM][TN], L[TM][TN], a[TM], b[TN];
#pragma unroll
  for (int i = 0; i < TM; ++i) a[i] = 1.0 + i * 1e-7 + threadIdx.x * 1e-9;
#pragma unroll
  for (int j = 0; j < TN; ++j) b[j] = 0.5 + j * 1e-7;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) { T[i][j] = 1.5; L[i][j] = 0.0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < 3; ++s) {
#pragma unroll
      for (int i = 0; i < TM; ++i)
#pragma unroll
        for (int j = 0; j < TN; ++j) {
          const double t = T[i][j];
          const double tn = __fma_rn(a[i], b[j], t);
          L[i][j] = __dadd_rn(L[i][j], __fma_rn(a[i], b[j], __dsub_rn(t, tn)));
          T[i][j] = tn;
        }
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = -a[i];
    }
#pragma unroll
    for (int i = 0; i < TM; ++i)
#pragma unroll
      for (int j = 0; j < TN; ++j) {
        const double t2 = __dadd_rn(T[i][j], L[i][j]);
        L[i][j] = __dsub_rn(L[i][j], __dsub_rn(t2, T[i][j]));
        T[i][j] = t2;
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) s += T[i][j] + L[i][j];
  if (s == 12345.0) out[0] = s;
}

template <class K>
float timeit(K launch) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 4; ++r) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (r && ms < best) best = ms;
  }
  return best;
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int it = 20000;
  const float ref = timeit([&] { burn<8><<<sms * 4, 256>>>(out, it); });
  const double peak = (double)sms * 4 * 256 * it * 8 / (ref * 1e-3);
  printf("reference burn (32 warps/SM, 8 chains): %.3f T lane-op/s\n", peak / 1e12);
#define BURN(CH, CTAS, THR)                                                                  \
  {                                                                                          \
    const float ms = timeit([&] { burn<CH><<<sms * CTAS, THR>>>(out, it); });               \
    printf("burn  chains %2d warps/SM %2d: %.1f %%\n", CH, CTAS * THR / 32,                 \
           100.0 * sms * CTAS * THR * (double)it * CH / (ms * 1e-3) / peak);                 \
  }
  BURN(8, 1, 256) BURN(16, 1, 256) BURN(32, 1, 256) BURN(16, 1, 384) BURN(16, 2, 256)
#define MIX(TM, TN, CTAS, THR)                                                               \
  {                                                                                          \
    const int its = 2000;                                                                    \
    const float ms = timeit([&] { mix<TM, TN><<<sms * CTAS, THR>>>(out, its); });            \
    printf("mix %dx%d warps/SM %2d: %.1f %%\n", TM, TN, CTAS * THR / 32,                     \
           100.0 * sms * CTAS * THR * (double)its * TM * TN * 15 / (ms * 1e-3) / peak);      \
  }
  MIX(8, 4, 1, 256) MIX(4, 4, 1, 256) MIX(4, 4, 2, 256) MIX(4, 4, 1, 384) MIX(8, 2, 2, 256)
  MIX(6, 4, 1, 384) MIX(4, 2, 4, 256) MIX(2, 2, 8, 256)
  {   // the 8 x 4 mix with __launch_bounds__(256, 1), as the production kernel
    const int its = 2000;
    const float ms = timeit([&] { mix<8, 4, 1><<<sms, 256>>>(out, its); });
    printf("mix 8x4 launch_bounds(256,1) warps/SM  8: %.1f %%\n",
           100.0 * sms * 256 * (double)its * 8 * 4 * 15 / (ms * 1e-3) / peak);
  }
  return 0;
}
