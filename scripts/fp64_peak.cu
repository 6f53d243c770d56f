// fp64_peak.cu -- measures the B200 FP64 pipe: DFMA and DADD throughput with
// 8 independent chains per thread, 148 x 4 CTAs x 256 threads, CUDA events.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_peak fp64_peak.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void __launch_bounds__(256) burn(double* out, double a, double b, int iters) {
  double x[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (OP == 0) x[i] = __fma_rn(x[i], a, b);
        else x[i] = __dadd_rn(x[i], b);
      }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("device %s, %d SMs, max clock %.0f MHz\n", p.name, p.multiProcessorCount, clk / 1e3);
  double* out;
  cudaMalloc(&out, 8);
  const int blocks = p.multiProcessorCount * 4, threads = 256, iters = 4000;
  for (int op = 0; op < 2; ++op) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      cudaEventRecord(e0);
      if (op == 0) burn<0><<<blocks, threads>>>(out, 0.999999, 1e-9, iters);
      else burn<1><<<blocks, threads>>>(out, 0.999999, 1e-9, iters);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      const double ops = (double)blocks * threads * iters * 16 * 8;
      printf("%s: %.3f ms  %.2f T instr-lanes/s  (%.2f TFLOP/s if FMA=2)\n",
             op == 0 ? "DFMA" : "DADD", ms, ops / ms / 1e9, (op == 0 ? 2 : 1) * ops / ms / 1e9);
    }
  }
  return 0;
}
