// fp64_outer.cu -- DFMA throughput of a register outer-product micro-tile
// (acc[TM][TN] += a[TM] x b[TN], operands refreshed from shared memory each
// step) at 1 CTA x 256 threads per SM: the GEMM-shaped issue pattern, to
// separate the FP64 pipe's ceiling for this shape from the dd kernels' losses.
#include <cstdio>
#include <cuda_runtime.h>

template <int TM, int TN, int LOADS>
__global__ void __launch_bounds__(256, 1) outer(double* out, int iters) {
  __shared__ double sa[16][128], sb[16][64];
  for (int i = threadIdx.x; i < 16 * 128; i += 256) (&sa[0][0])[i] = i * 1e-3;
  for (int i = threadIdx.x; i < 16 * 64; i += 256) (&sb[0][0])[i] = i * 1e-4;
  __syncthreads();
  double acc[TM][TN];
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) acc[i][j] = 0.0;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int kk = 0; kk < 16; ++kk) {
      double a[TM], b[TN];
#pragma unroll
      for (int i = 0; i < TM; ++i) a[i] = LOADS ? sa[kk][(i >> 1) * 32 + tx * 2 + (i & 1)] : 1.0 + i * 1e-9 * kk;
#pragma unroll
      for (int j = 0; j < TN; ++j) b[j] = LOADS ? sb[kk][(j >> 1) * 32 + ty * 2 + (j & 1)] : 1.0 + j * 1e-9 * kk;
#pragma unroll
      for (int r = 0; r < 4; ++r)   // 4 FMAs per element per step (dd-like density)
#pragma unroll
        for (int i = 0; i < TM; ++i)
#pragma unroll
          for (int j = 0; j < TN; ++j) acc[i][j] = __fma_rn(a[i], b[j], acc[i][j]);
    }
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < TM; ++i)
#pragma unroll
    for (int j = 0; j < TN; ++j) s += acc[i][j];
  if (s == 12345.0) out[0] = s;
}

template <int TM, int TN, int LOADS>
void run(int sms, double* out, const char* name) {
  const int iters = 200;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    outer<TM, TN, LOADS><<<sms, 256>>>(out, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = (double)sms * 256 * iters * 16 * 4 * TM * TN;
  printf("%s: %.1f%% of DP peak\n", name, ops / (best * 1e-3) / ((double)sms * 64 * 1.965e9) * 100);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  run<8, 4, 1>(sms, out, "8x4 micro-tile, smem operands");
  run<8, 4, 0>(sms, out, "8x4 micro-tile, register operands");
  run<4, 4, 1>(sms, out, "4x4 micro-tile, smem operands");
  return 0;
}
