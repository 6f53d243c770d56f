// fp64_occupancy.cu -- how many warps / independent chains the B200 FP64
// pipe needs: DADD throughput vs (warps per SM, chains per thread).
#include <cstdio>
#include <cuda_runtime.h>

template <int NC>
__global__ void chains(double* out, double b, int iters) {
  double x[NC];
#pragma unroll
  for (int i = 0; i < NC; ++i) x[i] = threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r)
#pragma unroll
      for (int i = 0; i < NC; ++i) x[i] = __dadd_rn(x[i], b);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < NC; ++i) s += x[i];
  if (s == 12345.0) out[0] = s;
}

template <int NC>
void run(int sms, int warps_per_sm, double* out) {
  const int threads = 32 * (warps_per_sm > 32 ? 32 : warps_per_sm);
  const int blocks = sms * (warps_per_sm > 32 ? warps_per_sm / 32 : 1);
  const int iters = 4096 / NC * 16;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    chains<NC><<<blocks, threads>>>(out, 1e-9, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double ops = (double)blocks * threads * iters * 8 * NC;
  const double peak = (double)sms * 64 * 1.965e9;
  printf("warps/SM %3d chains %2d: %6.1f%% of DP peak\n", warps_per_sm, NC, ops / (best * 1e-3) / peak * 100);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* out;
  cudaMalloc(&out, 8);
  for (int w : {4, 8, 12, 16, 32}) {
    run<1>(sms, w, out);
    run<2>(sms, w, out);
    run<4>(sms, w, out);
    run<8>(sms, w, out);
    run<16>(sms, w, out);
  }
  return 0;
}
