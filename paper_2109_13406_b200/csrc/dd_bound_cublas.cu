// dd_bound_cublas.cu -- MEASUREMENT BASELINE ONLY (DDB_BOUND=cublas /
// DDB_CROSS=cublas): round 1's library-GEMM versions of the fast mode's bound
// (cuBLAS GemmEx) and cross terms (cuBLAS Dgemm), kept to A/B the
// hand-written kernels (dd_bound.cu, dd_cross.cu) against them.
//
// The fast accumulator (ALG_CERT in dd_tiled.cuh) anchors each element's
// running sum at sigma = 1.5 * 2^E, which is exact and error-bounded only if
// 2^E >= 2 * sum_l |a_il * b_lj| for that element.  This file produces a
// guaranteed upper bound Sigma'_ij of that sum, tight to a few percent:
//
//   1. abs_bf16_kernel: |hi| of op(A) (resp. op(B)) scaled by the per-row
//      (per-column) exponent maximum from the prescan into [0, 1], rounded
//      UP to fp32 and then UP to bf16: every converted value is >= the scaled
//      |hi| it replaces (tiny values round up to bf16's smallest subnormal).
//   2. one bf16 x bf16 -> fp32 tensor-core GEMM of the scaled magnitudes
//      (cuBLAS GemmEx: a plain library GEMM).  All terms are >= 0, so the
//      fp32 sum's relative error is <= k * 2^-23 (covered by 1 + k*2^-20);
//      products flushed below fp32's range lose < k * 2^-126 (covered by the
//      floor term k * 2^-120).
//
// The kernel then uses  Sigma' = (S_ij (1 + k 2^-20) + k 2^-120) *
// 2^(rowexp_i + colexp_j - 2044)  (dd_tiled.cuh).  Cost at n = 8192: ~0.2 ms
// for the conversions plus ~1 ms of tensor-core time, < 0.5 % of the step.
#include <cublas_v2.h>
#include <cuda_bf16.h>


#include "internal.h"

namespace ddb {

// Stored matrix rows x cols (ld); scale index = row (per_row) or column.
__global__ void __launch_bounds__(256)
abs_bf16_kernel_lib(const double* __restrict__ hi, int64_t ld, int64_t rows, int64_t cols,
                const int* __restrict__ exps, int per_row, __nv_bfloat16* __restrict__ out) {
  const int64_t r = (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (r >= rows) return;
  for (int64_t c = (int64_t)blockIdx.y * 8 + threadIdx.y; c < cols; c += (int64_t)gridDim.y * 8) {
    const int e = per_row ? exps[r] : exps[c];          // biased exponent maximum
    // scale 2^(1022 - e): |x| * scale < 1 for every |x| < 2^(e - 1022) (exact)
    const double scale = __longlong_as_double((long long)(2045 - e) << 52);
    const double v = fabs(hi[r + c * ld]) * scale;
    out[r + c * rows] = __float2bfloat16_ru(__double2float_ru(v));
  }
}

static cudaError_t convert_lib(const double* hi, int64_t ld, int64_t rows, int64_t cols,
                           const int* exps, int per_row, __nv_bfloat16* out, cudaStream_t s,
                           int* nlaunch) {
  if (rows <= 0 || cols <= 0) return cudaSuccess;
  int64_t gy = (cols + 7) / 8;
  if (gy > 65535) gy = 65535;
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)gy), block(32, 8);
  abs_bf16_kernel_lib<<<grid, block, 0, s>>>(hi, ld, rows, cols, exps, per_row, out);
  ++*nlaunch;
  return cudaGetLastError();
}

// One cuBLAS handle per (host thread, device): cublasSetStream + GemmEx on a
// shared handle would race between threads calling on different streams.
static cublasHandle_t handle_for_current_device() {
  thread_local cublasHandle_t handles[64] = {};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return nullptr;
  if (handles[dev] == nullptr) {
    cublasHandle_t h;
    if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
    handles[dev] = h;
  }
  return handles[dev];
}


// Fills bound (m x n, ld = m, fp32) from the operands and the prescan maxima.
// ws must hold 2(mk + kn) bytes of bf16 operands ahead of `bound`'s region
// (bound_workspace_bytes covers it: kp >= k).
cudaError_t launch_bound_cublas(const GemmArgs& g, const int* row_exp, const int* col_exp,
                                void* ws, float* bound, cudaStream_t s, int* nlaunch,
                                const char** what) {
  char* p = static_cast<char*>(ws);
  __nv_bfloat16* abf = reinterpret_cast<__nv_bfloat16*>(p);
  p += ((2 * (size_t)g.m * g.k + 255) / 256) * 256;
  __nv_bfloat16* bbf = reinterpret_cast<__nv_bfloat16*>(p);
  // op(A) rows scale by row_exp; stored A is m x k (N) or k x m (T)
  cudaError_t e;
  if (g.ta == 0) e = convert_lib(g.a_hi, g.lda, g.m, g.k, row_exp, 1, abf, s, nlaunch);
  else e = convert_lib(g.a_hi, g.lda, g.k, g.m, row_exp, 0, abf, s, nlaunch);
  if (e != cudaSuccess) { *what = "bound conversion"; return e; }
  const __nv_bfloat16* bsrc = abf;
  cublasOperation_t opb;
  int64_t ldbf;
  if (g.syrk) {
    // op(B) = op(A)^T: reuse the converted op(A) with the opposite transpose
    opb = g.ta == 0 ? CUBLAS_OP_T : CUBLAS_OP_N;
    ldbf = g.ta == 0 ? g.m : g.k;
  } else {
    if (g.tb == 0) e = convert_lib(g.b_hi, g.ldb, g.k, g.n, col_exp, 0, bbf, s, nlaunch);
    else e = convert_lib(g.b_hi, g.ldb, g.n, g.k, col_exp, 1, bbf, s, nlaunch);
    if (e != cudaSuccess) { *what = "bound conversion"; return e; }
    bsrc = bbf;
    opb = g.tb == 0 ? CUBLAS_OP_N : CUBLAS_OP_T;
    ldbf = g.tb == 0 ? g.k : g.n;
  }
  cublasHandle_t h = handle_for_current_device();
  if (h == nullptr) { *what = "cublasCreate"; return cudaErrorUnknown; }
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) { *what = "cublasSetStream"; return cudaErrorUnknown; }
  const float one = 1.f, zero = 0.f;
  const cublasOperation_t opa = g.ta == 0 ? CUBLAS_OP_N : CUBLAS_OP_T;
  const int64_t ldaf = g.ta == 0 ? g.m : g.k;
  cublasStatus_t st = cublasGemmEx(h, opa, opb, (int)g.m, (int)g.n, (int)g.k, &one,
                                   abf, CUDA_R_16BF, (int)ldaf, bsrc, CUDA_R_16BF, (int)ldbf,
                                   &zero, bound, CUDA_R_32F, (int)g.m, CUBLAS_COMPUTE_32F,
                                   CUBLAS_GEMM_DEFAULT);
  if (st != CUBLAS_STATUS_SUCCESS) { *what = "cublasGemmEx (bound)"; return cudaErrorUnknown; }
  return cudaGetLastError();
}

// ALG_SPLIT's cross terms: x (m x n, ld = m) = op(A)_lo op(B)_hi + op(A)_hi op(B)_lo,
// two plain binary64 library GEMMs (the same handle, default math mode: IEEE
// binary64 products and sums in some order).  Any summation order keeps
// |error| <= 2k u * sum_l (|a_lo b_hi| + |a_hi b_lo|) <= 4k u^2 * sum_l |a_hi b_hi|
// for normalised operands (|lo| <= u |hi|, enforced by the prescan), i.e.
// one unit of the c k 2^-104 budget (dd_tma.cu).
// x(i, j) += x(j, i) on the uplo triangle (diagonal: 2 x(i, i)), in place: a
// tile of the triangle reads only its mirror tile in the other triangle, which
// no block writes, and the diagonal tiles stage the mirror in shared memory
// before any write.  Turns Y = op(A)_hi op(A)_lo^T into the Rsyrk cross term
// Y + Y^T.  HBM-bound: 16 bytes read + 8 written per triangle element.
__global__ void __launch_bounds__(256)
sym_fold_kernel(double* __restrict__ x, int64_t n, int upper) {
  const int64_t bi = blockIdx.x, bj = blockIdx.y;       // tile row / tile column
  if (upper ? bi > bj : bi < bj) return;
  __shared__ double t[32][33];
  const int64_t r0 = bi * 32, c0 = bj * 32;
  // mirror tile: rows c0.., columns r0.. ; t[c][r] = x(c0 + c, r0 + r)^T staged
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t mr = c0 + threadIdx.x, mc = r0 + y;
    if (mr < n && mc < n) t[threadIdx.x][y] = x[mr + mc * n];
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {
    const int64_t i = r0 + threadIdx.x, j = c0 + y;
    if (i < n && j < n && (upper ? i <= j : i >= j))
      x[i + j * n] = x[i + j * n] + t[y][threadIdx.x];
  }
}

cudaError_t launch_cross_dgemm(const GemmArgs& g, double* x, cudaStream_t s) {
  cublasHandle_t h = handle_for_current_device();
  if (h == nullptr) return cudaErrorUnknown;
  if (cublasSetStream(h, s) != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  const double one = 1.0, zero = 0.0;
  const cublasOperation_t opa = g.ta == 0 ? CUBLAS_OP_N : CUBLAS_OP_T;
  const cublasOperation_t opb = g.tb == 0 ? CUBLAS_OP_N : CUBLAS_OP_T;
  if (g.syrk != 0) {
    // Rsyrk in NN form (op(B) = op(A)^T): only the uplo triangle is read.
    // x = op(A)_hi op(A)_lo^T + op(A)_lo op(A)_hi^T = Y + Y^T with
    // Y = op(A)_hi op(A)_lo^T: one full DGEMM (DMMA tensor cores, 30.8 ms at
    // n = k = 8192) and an in-place triangle fold, instead of cuBLAS DSYR2K
    // (same flops, but a SIMT kernel: 40.5 ms).  The fold adds one rounding
    // to two length-k sums: the 2k u bound above still holds.
    const cublasOperation_t opt = g.ta == 0 ? CUBLAS_OP_T : CUBLAS_OP_N;
    const cublasStatus_t st = cublasDgemm(h, opa, opt, (int)g.m, (int)g.m, (int)g.k, &one,
                                          g.a_hi, (int)g.lda, g.a_lo, (int)g.lda, &zero, x,
                                          (int)g.m);
    if (st != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
    const unsigned tiles = (unsigned)((g.m + 31) / 32);
    sym_fold_kernel<<<dim3(tiles, tiles), dim3(32, 8), 0, s>>>(x, g.m, g.syrk == 1);
    return cudaGetLastError();
  }
  cublasStatus_t st = cublasDgemm(h, opa, opb, (int)g.m, (int)g.n, (int)g.k, &one, g.a_lo,
                                  (int)g.lda, g.b_hi, (int)g.ldb, &zero, x, (int)g.m);
  if (st == CUBLAS_STATUS_SUCCESS)
    st = cublasDgemm(h, opa, opb, (int)g.m, (int)g.n, (int)g.k, &one, g.a_hi, (int)g.lda,
                     g.b_lo, (int)g.ldb, &one, x, (int)g.m);
  if (st != CUBLAS_STATUS_SUCCESS) return cudaErrorUnknown;
  return cudaGetLastError();
}

}  // namespace ddb
