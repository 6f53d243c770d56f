// dd_potrf.cu -- blocked dd Cholesky (Rpotrf) whose trailing updates are
// Rsyrk calls, bit-identical to the reference's unblocked order in exact mode.
//
// The reference's Rpotrf (mplapack/chol.py:21-65) is unblocked and
// left-looking.  For column j (lower; upper is the transpose):
//   dot   = sum_ltr_{l<j} L(j,l) * L(j,l)              (chol.py:38-40)
//   ajj   = A(j,j) - dot ; fail (info = j+1, A(j,j) = ajj) if NaN or <= 0
//   L(j,j) = sqrt(ajj) ; rec = 1 / L(j,j)               (chol.py:41-49, :63)
//   lower: tail_i = A(i,j) + sum_{l<j} (-L(j,l)) * L(i,l), accumulated in
//          place left to right, then L(i,j) = rec * tail_i  (chol.py:57-64)
//   upper: temp_jj = sum_ltr_{l<j} U(l,jj) * U(l,j) (from zero), then
//          U(j,jj) = rec * (A(j,jj) - temp_jj)           (chol.py:50-56)
//
// Blocked right-looking form with the same per-element operation sequence:
//   * the pivots' dot products are kept in a vector D, each entry extended
//     by one product as soon as its row (column) gets a new factor entry, in
//     the reference's l order -- so a pivot costs O(1), and ajj = d0(j) - D(j)
//     with d0 the original diagonal;
//   * lower: after a block column [j0, j1) is factored, the trailing lower
//     triangle is updated IN PLACE by Rsyrk('L', 'N', alpha = -1, beta = 1):
//     per element c = c + L(i,l) * (-1 * L(j,l)), l = j0..j1-1 in order --
//     the reference's accumulation, continued (mul2 is symmetric and
//     mul2(-1, x) == -x inside the safe window; the diagonal entries of the
//     update are discarded, pivots come from D);
//   * upper: temp accumulates from ZERO, so the trailing updates go to a
//     separate accumulator S (lower-stored, S(jj, j) for U(j, jj)) by
//     Rsyrk('L', 'N', alpha = 1, beta = 1) on T = U12^T;
//   * per block: potrf_diag_kernel factors the diagonal block in one CTA
//     (right-looking, a barrier per column; the pivots are the only serial
//     chain), potrf_panel_kernel the rows below it ('U': the columns right of
//     it), each row an independent sequence over the block's columns run by
//     a group of lanes; block width <= 64 (the diagonal block lives in
//     shared memory).
// So in exact mode (Rsyrk exact) the factor is bit-identical to the
// reference for operands inside the safe window; fast / twosum modes differ
// only by their Rsyrk accumulation.  On failure the device info is set,
// later column kernels exit, and restore_kernel puts back the original
// entries the reference would not have touched yet (trailing updates of the
// lower form write in place; a backup copy is kept for that).
// dd sqrt / div / sub are the reference's scalar forms (ddarith.py:79-163);
// element-wise add / mul the vectorised ones (elem.py:54-78).
#include "lapack_num.cuh"

namespace ddb {

// Diagonal block [j0, j1) in one CTA, staged in shared memory, right-looking:
// per column j the pivot (thread 0), the column inside the block, then the
// block's trailing strictly-lower entries, each update in the reference's
// l order.  X(q, c) (q > c) is the block entry the factor overwrites: A(q, c)
// for 'L', A(c, q) for 'U'; for 'U' the running dot products S(q, c) are
// staged too.  The reciprocals go to p.rec for the panel kernel.
template <class N>
__global__ void __launch_bounds__(512)
potrf_diag_kernel(PotrfArgs p, int64_t j0, int nb) {
  using T = typename N::T;
  extern __shared__ double sm[];
  __shared__ T rec_s;
  __shared__ int ok_s;
  if (*p.info != 0) return;
  const int64_t lda = p.lda, lds = p.lds;
  const int sq = nb * nb;
  double* xh = sm;
  double* xl = sm + sq;
  double* sh = sm + 2 * sq;                      // 'U' only
  double* sl = sm + 3 * sq;
  double* dh = sm + (p.upper ? 4 : 2) * sq;
  double* dl = dh + nb;
  double* d0h = dl + nb;
  double* d0l = d0h + nb;
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    N::st(xh, xl, t, N::ld(p.a_hi, p.a_lo, x));
    if (p.upper) N::st(sh, sl, t, N::ld(p.s_hi, p.s_lo, (j0 + q) + (j0 + c) * lds));
  }
  for (int t = threadIdx.x; t < nb; t += blockDim.x) {
    N::st(dh, dl, t, N::ld(p.dh, p.dl, j0 + t));
    N::st(d0h, d0l, t, N::ld(p.d0_hi, p.d0_lo, j0 + t));
  }
  __syncthreads();
  // thread 0 computes pivot j+1 while warps 1.. run step j's trailing
  // update (pivot j+1 needs only D(j+1), final after step j's column phase)
  auto pivot = [&](int j) {
    const T ajj = N::ssub(N::ld(d0h, d0l, j), N::ld(dh, dl, j));   // chol.py:41
    const int64_t djj = (j0 + j) * (lda + 1);
    ok_s = !N::bad_pivot(ajj);
    if (!ok_s) {
      N::st(p.a_hi, p.a_lo, djj, ajj);
      *p.info = (int)(j0 + j + 1);
    } else {
      const T s = N::ssqrt(ajj);
      N::st(p.a_hi, p.a_lo, djj, s);
      const T rec = N::sdiv(N::one(), s);
      rec_s = rec;
      N::st(p.rec_hi, p.rec_lo, j, rec);
    }
  };
  if (threadIdx.x == 0) pivot(0);
  __syncthreads();
  for (int j = 0; j < nb; ++j) {
    if (!ok_s) break;
    const T rec = rec_s;
    for (int q = j + 1 + threadIdx.x; q < nb; q += blockDim.x) {
      const int t = q + j * nb;
      T a = N::ld(xh, xl, t);
      if (p.upper) a = N::add(a, N::neg(N::ld(sh, sl, t)));
      const T v = N::mul(rec, a);
      N::st(xh, xl, t, v);
      N::st(dh, dl, q, N::add(N::ld(dh, dl, q), N::mul(v, v)));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      if (j + 1 < nb) pivot(j + 1);
    } else if (threadIdx.x >= 32) {
      // pairs (q, c), j < c < q < nb, enumerated column by column; batches
      // of kB independent updates (operands gathered before any store)
      const int rem = nb - j - 1;
      const int npairs = rem * (rem - 1) / 2;
      constexpr int kB = 4;
      const int nthr = blockDim.x - 32;
      for (int base = threadIdx.x - 32; base < npairs; base += nthr * kB) {
        int xs[kB];
        T acc[kB], f1[kB], f2[kB];
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          const int t = base + b * nthr;
          xs[b] = -1;
          if (t < npairs) {
            // column ci (0-based within the rem trailing columns) of pair t
            int ci = (int)((2.0f * rem - 1.0f - sqrtf((2.0f * rem - 1.0f) * (2.0f * rem - 1.0f) - 8.0f * t)) * 0.5f);
            while (ci > 0 && ci * (2 * rem - ci - 1) / 2 > t) --ci;
            while ((ci + 1) * (2 * rem - ci - 2) / 2 <= t) ++ci;
            const int qi = ci + 1 + (t - ci * (2 * rem - ci - 1) / 2);
            const int c = j + 1 + ci, q = j + 1 + qi;
            xs[b] = q + c * nb;
            const T vq = N::ld(xh, xl, q + j * nb), vc = N::ld(xh, xl, c + j * nb);
            if (!p.upper) { acc[b] = N::ld(xh, xl, xs[b]); f1[b] = N::neg(vc); f2[b] = vq; }
            else { acc[b] = N::ld(sh, sl, xs[b]); f1[b] = vq; f2[b] = vc; }
          }
        }
#pragma unroll
        for (int b = 0; b < kB; ++b) {
          if (xs[b] < 0) continue;
          const T r = N::add(acc[b], N::mul(f1[b], f2[b]));
          if (!p.upper) N::st(xh, xl, xs[b], r);
          else N::st(sh, sl, xs[b], r);
        }
      }
    }
    __syncthreads();
  }
  // write the block back ('U': the untouched part is written back unchanged;
  // 'L': entries the reference would not have touched yet are restored from
  // the backup by potrf_restore_kernel)
  for (int t = threadIdx.x; t < sq; t += blockDim.x) {
    const int q = t % nb, c = t / nb;
    if (q <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + q) * lda : (j0 + q) + (j0 + c) * lda;
    N::st(p.a_hi, p.a_lo, x, N::ld(xh, xl, t));
  }
}

// Panel below ('L': rows q >= j1) / right of ('U': columns q >= j1) the
// diagonal block.  Each q is independent: a group of G lanes owns it, lane t
// holding the accumulators of block columns c = j0 + t + G*i.  Step c: the
// owner finalises entry c (rec_c * acc, or rec_c * (A - acc) for 'U'),
// broadcasts it, and every lane extends its later columns by one product --
// the reference's per-element order (chol.py:50-64), with NPER independent
// chains per lane.  The block's factor (strictly-lower part, transposed for
// 'U') and the reciprocals sit in shared memory.
constexpr int kPanelG = 32;          // lanes per row: one warp
constexpr int kPanelThreads = 256;    // 8 rows per CTA

template <class N, int NPER>
__global__ void __launch_bounds__(kPanelThreads)
potrf_panel_kernel(PotrfArgs p, int64_t j0, int nb) {
  using T = typename N::T;
  extern __shared__ double sm[];
  // a failure inside this block's diagonal part still leaves the columns
  // before it complete, as the reference does (chol.py:44-46)
  int ncols = nb;
  const int inf = *p.info;
  if (inf != 0) {
    if (inf - 1 < j0) return;
    ncols = (int)(inf - 1 - j0);
  }
  const int64_t lda = p.lda, lds = p.lds;
  const int64_t j1 = j0 + nb;
  // packed strictly-lower triangle: T(c2, c) (c < c2) at off(c) + c2 - c - 1
  const int ntri = nb * (nb - 1) / 2;
  double* th = sm;
  double* tl = sm + ntri;
  double* rh = sm + 2 * ntri;
  double* rl = rh + nb;
  auto off = [nb](int c) { return c * (2 * nb - c - 1) / 2; };
  for (int t = threadIdx.x; t < nb * nb; t += blockDim.x) {
    const int c2 = t % nb, c = t / nb;
    if (c2 <= c) continue;
    const int64_t x = p.upper ? (j0 + c) + (j0 + c2) * lda : (j0 + c2) + (j0 + c) * lda;
    N::st(th, tl, off(c) + c2 - c - 1, N::ld(p.a_hi, p.a_lo, x));
  }
  for (int c = threadIdx.x; c < nb; c += blockDim.x) N::st(rh, rl, c, N::ld(p.rec_hi, p.rec_lo, c));
  __syncthreads();
  const int lane = threadIdx.x % kPanelG;
  const int64_t q = j1 + ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / kPanelG;
  if (q >= p.n) return;                 // whole warps exit together
  T acc[NPER];
#pragma unroll
  for (int i = 0; i < NPER; ++i) {
    const int c = lane + kPanelG * i;
    acc[i] = N::zero();
    if (c < nb) {
      const int64_t x = p.upper ? q + (j0 + c) * lds : q + (j0 + c) * lda;
      acc[i] = p.upper ? N::ld(p.s_hi, p.s_lo, x) : N::ld(p.a_hi, p.a_lo, x);
    }
  }
  T dq = N::zero();
  if (lane == 0) dq = N::ld(p.dh, p.dl, q);
  for (int c = 0; c < ncols; ++c) {
    const int owner = c % kPanelG, ic = c / kPanelG;
    T v = N::zero();
    if (lane == owner) {
      T a = N::zero();
#pragma unroll
      for (int i = 0; i < NPER; ++i)
        if (i == ic) a = acc[i];
      const T rec = N::ld(rh, rl, c);
      const int64_t x = p.upper ? (j0 + c) + q * lda : q + (j0 + c) * lda;
      if (p.upper) a = N::add(N::ld(p.a_hi, p.a_lo, x), N::neg(a));
      v = N::mul(rec, a);
      N::st(p.a_hi, p.a_lo, x, v);
    }
    v = N::shfl(v, owner);
    if (lane == 0) dq = N::add(dq, N::mul(v, v));
#pragma unroll
    for (int i = 0; i < NPER; ++i) {
      const int c2 = lane + kPanelG * i;
      if (c2 > c && c2 < nb) {
        const T t = N::ld(th, tl, off(c) + c2 - c - 1);
        acc[i] = p.upper ? N::add(acc[i], N::mul(v, t)) : N::add(acc[i], N::mul(N::neg(t), v));
      }
    }
  }
  if (lane == 0) N::st(p.dh, p.dl, q, dq);
}

// T(r, l) = U(j0 + l, j1 + r), r < rows, l < nb  (ld = rows)
__global__ void __launch_bounds__(256)
potrf_transpose_kernel(PotrfArgs p, int64_t j0, int64_t j1, int nb, int64_t rows) {
  __shared__ double th[32][33], tl[32][33];
  const int64_t r0 = (int64_t)blockIdx.x * 32, l0 = (int64_t)blockIdx.y * 32;
  for (int y = threadIdx.y; y < 32; y += 8) {          // read: l fastest in memory
    const int64_t r = r0 + y, l = l0 + threadIdx.x;
    if (r < rows && l < nb) {
      const int64_t x = (j0 + l) + (j1 + r) * p.lda;
      th[y][threadIdx.x] = p.a_hi[x];
      if (!p.f64) tl[y][threadIdx.x] = p.a_lo[x];
    }
  }
  __syncthreads();
  for (int y = threadIdx.y; y < 32; y += 8) {          // write: r fastest
    const int64_t l = l0 + y, r = r0 + threadIdx.x;
    if (r < rows && l < nb) {
      p.t_hi[r + l * rows] = th[threadIdx.x][y];
      if (!p.f64) p.t_lo[r + l * rows] = tl[threadIdx.x][y];
    }
  }
}

// After a failure at column f = info - 1 (lower form): the reference leaves
// column f below the diagonal and every later column untouched; put back the
// original lower-triangle entries there from the backup (ld = n).
__global__ void __launch_bounds__(256)
potrf_restore_kernel(PotrfArgs p) {
  const int info = *p.info;
  if (info == 0) return;
  const int64_t f = info - 1;
  const int64_t i = (int64_t)blockIdx.x * 256 + threadIdx.x;
  if (i >= p.n) return;
  for (int64_t c = f + blockIdx.y; c <= i && c < p.n; c += gridDim.y) {
    if (i == c && c == f) continue;
    p.a_hi[i + c * p.lda] = p.b_hi[i + c * p.n];
    if (!p.f64) p.a_lo[i + c * p.lda] = p.b_lo[i + c * p.n];
  }
}

cudaError_t launch_potrf_diag(const PotrfArgs& p, int64_t j0, int64_t j1, cudaStream_t s) {
  const int nb = (int)(j1 - j0);
  const size_t smem = sizeof(double) * ((size_t)(p.upper ? 4 : 2) * nb * nb + 4 * (size_t)nb);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(potrf_diag_kernel<NumDD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(potrf_diag_kernel<NumF64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  if (p.f64) potrf_diag_kernel<NumF64><<<1, 512, smem, s>>>(p, j0, nb);
  else potrf_diag_kernel<NumDD><<<1, 512, smem, s>>>(p, j0, nb);
  return cudaGetLastError();
}

template <class N, int NPER>
static cudaError_t panel_launch(const PotrfArgs& p, int64_t j0, int nb, int64_t rows,
                                cudaStream_t s) {
  const size_t smem = sizeof(double) * ((size_t)nb * (nb - 1) + 2 * (size_t)nb);
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(potrf_panel_kernel<N, NPER>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  const int64_t threads = rows * kPanelG;
  potrf_panel_kernel<N, NPER><<<(unsigned)((threads + kPanelThreads - 1) / kPanelThreads),
                                kPanelThreads, smem, s>>>(p, j0, nb);
  return cudaGetLastError();
}

cudaError_t launch_potrf_panel(const PotrfArgs& p, int64_t j0, int nb, int64_t rows,
                               cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  const int nper = (nb + kPanelG - 1) / kPanelG;
  (void)nper;   // nb <= 64 = 2 * kPanelG
  return p.f64 ? panel_launch<NumF64, 2>(p, j0, nb, rows, s)
               : panel_launch<NumDD, 2>(p, j0, nb, rows, s);
}

cudaError_t launch_potrf_transpose(const PotrfArgs& p, int64_t j0, int64_t j1, int nb,
                                   int64_t rows, cudaStream_t s) {
  dim3 grid((unsigned)((rows + 31) / 32), (unsigned)((nb + 31) / 32));
  potrf_transpose_kernel<<<grid, dim3(32, 8), 0, s>>>(p, j0, j1, nb, rows);
  return cudaGetLastError();
}

cudaError_t launch_potrf_restore(const PotrfArgs& p, cudaStream_t s) {
  dim3 grid((unsigned)((p.n + 255) / 256), 64);
  potrf_restore_kernel<<<grid, 256, 0, s>>>(p);
  return cudaGetLastError();
}

}  // namespace ddb
