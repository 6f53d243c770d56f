// dmma_concurrency.cu -- does fp64 tensor-core MMA (mma.sync m8n8k4 f64,
// "DMMA") run on different hardware than the FP64 FMA pipe on B200?  Times
// DMMA-only, DFMA-only, and both at once (half the warps each).
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1) : "d"(a), "d"(b));
}

// role: 0 = all warps DMMA, 1 = all warps DFMA, 2 = even warps DMMA / odd warps DFMA
__global__ void __launch_bounds__(256) burn(double* out, int iters, int role) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = role == 0 || (role == 2 && (warp & 1) == 0);
  double acc[16];
#pragma unroll
  for (int i = 0; i < 16; ++i) acc[i] = threadIdx.x * 1e-3 + i;
  const double a = 1.0000001, b = 0.9999999;
  if (do_mma) {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int i = 0; i < 16; i += 2) dmma(acc[i], acc[i + 1], a, b);
    }
  } else {
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int r = 0; r < 4; ++r)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc[i] = __fma_rn(acc[i], a, b);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 16; ++i) s += acc[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  const int iters = 20000, blocks = sms * 2, threads = 256;
  const char* names[] = {"DMMA only", "DFMA only", "half DMMA + half DFMA"};
  for (int role = 0; role < 3; ++role) {
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float best = 1e30f;
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(e0);
      burn<<<blocks, threads>>>(out, iters, role);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (ms < best) best = ms;
    }
    // per warp-iteration: DMMA 8 x (8x8x4 = 256 FMA) ; DFMA 64 x 32 FMA
    const double warps = (double)blocks * threads / 32;
    double fma = 0;
    if (role == 0) fma = warps * iters * 8 * 256;
    if (role == 1) fma = warps * iters * 64 * 32;
    if (role == 2) fma = warps / 2 * iters * 8 * 256 + warps / 2 * iters * 64 * 32;
    printf("%-24s %8.3f ms  %6.2f TFLOP/s fp64\n", names[role], best, 2 * fma / (best * 1e-3) / 1e12);
  }
  return 0;
}
