// dd_trsm.cu -- dd triangular solve (Rtrsm, level23.py:288-380) on the GPU.
//
// Every (side, uplo, transa) branch of the reference is, per element of the
// solution, the same recurrence once its indices are renamed:
//
//   x_s = fin_s( init(w_s) - T(s, t1) x_t1 - T(s, t2) x_t2 - ... )
//
// over a "production order" s = 0..p-1 of the triangular dimension, with
// each subtraction be.sub(acc, be.mul(T, x)) = add2(acc, -mul2(T, x)).  The
// vectors (columns of B for side 'L', rows for 'R') are independent.  Per
// branch (o(s) = s or p-1-s maps production index to the original one):
//
//   branch      order (U / L)   T(s, t)              terms        fin
//   L,N :326    desc / asc      A(o(s), o(t))        forward      div by A(s,s)
//   L,T :339    asc / desc      A(o(t), o(s))        fwd / REV    div
//   R,N :351    asc / desc      A(o(t), o(s))        fwd / REV    * (1 / A(s,s))
//   R,T :364    desc / asc      A(o(s), o(t))        forward      * (1 / A(s,s))
//
// "forward" = the terms arrive in production order (t ascending), which a
// blocked solve reproduces exactly: diagonal block sequentially
// (trsm_block_kernel), then one GEMM per block updating every later row with
// the subtract-product form (GemmArgs::sub, exact) -- each element still
// sees t ascending.  "REV" (t descending) cannot be blocked without changing
// the summation order: exact / reference modes run it as one sequential
// recurrence per vector (trsm_rev_kernel); the fast modes use the blocked
// order (same value to dd accuracy).  alpha: L,N and R,N scale B first when
// alpha != 1, L,T always (be.mul(ab, brow(i)), :342), R,T scales each solved
// column after its updates are used (:379-380) -- i.e. at the end.
#include "lapack_num.cuh"

namespace ddb {

namespace {

// TwoSum accumulation (fast modes, as dd_potrf.cu / dd_getrf.cu): unnormalised
// (H, L), 13 FP64 operations per product
__device__ __forceinline__ dd ts_mac(dd acc, dd x, dd y) {
  const double p = dmul(x.h, y.h);
  const double e = dfma(x.h, y.h, -p);
  const double c = dfma(x.h, y.l, dmul(x.l, y.h));
  double s, err;
  two_sum(acc.h, p, s, err);
  return dd{s, dadd(acc.l, dadd(err, dadd(e, c)))};
}
__device__ __forceinline__ dd ts_norm(dd a) {
  double s, e;
  quick_two_sum(a.h, a.l, s, e);
  return dd{s, e};
}
__device__ __forceinline__ double ts_mac(double acc, double x, double y) { return dadd(acc, dmul(x, y)); }
__device__ __forceinline__ double ts_norm(double a) { return a; }

// fin_s: unit diagonal -> v; the R branches -> (one / A(s,s)) * v with the
// reciprocal formed once per s by trsm_coef_kernel (be.div(one, aelt) then
// be.mul, level23.py:361-362, :368-369 -- the same bits); the L branches ->
// v / A(s,s) (be.div, :332) in the reference's order, or, in the fast
// modes, the precomputed reciprocal times v (dd accuracy, one division per
// s instead of one per element)
template <class N>
__device__ __forceinline__ typename N::T trsm_fin(const TrsmArgs& t, int64_t s, typename N::T v) {
  if (t.unit) return v;
  if (t.fin_rec || t.rec_fast) return N::mul(N::ld(t.r_hi, t.r_lo, s), v);
  return N::vdiv(v, N::ld(t.d_hi, t.d_lo, s));
}

}  // namespace

// W <- B in production order (side 'L': W(s, j) = B(o(s), j); 'R':
// W(s, i) = B(i, o(s))), times alpha when `scale`.
template <class N>
__global__ void __launch_bounds__(256)
trsm_pack_kernel(TrsmArgs t, const double* __restrict__ bh, const double* __restrict__ bl,
                 int64_t ldb, int scale, dd alpha) {
  const typename N::T al = N::ld(&alpha.h, &alpha.l, 0);
  const int64_t total = t.p * t.q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e % t.p, v = e / t.p;
    const int64_t o = t.rev ? t.p - 1 - s : s;
    const int64_t x = t.left ? o + v * ldb : v + o * ldb;
    typename N::T w = N::ld(bh, bl, x);
    if (scale) w = N::mul(al, w);
    N::st(t.w_hi, t.w_lo, s + v * t.ldw, w);
  }
}

// B <- W (inverse of the pack), times alpha when `scale`.
template <class N>
__global__ void __launch_bounds__(256)
trsm_unpack_kernel(TrsmArgs t, double* __restrict__ bh, double* __restrict__ bl, int64_t ldb,
                   int scale, dd alpha) {
  const typename N::T al = N::ld(&alpha.h, &alpha.l, 0);
  const int64_t total = t.p * t.q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e % t.p, v = e / t.p;
    const int64_t o = t.rev ? t.p - 1 - s : s;
    const int64_t x = t.left ? o + v * ldb : v + o * ldb;
    typename N::T w = N::ld(t.w_hi, t.w_lo, s + v * t.ldw);
    if (scale) w = N::mul(al, w);
    N::st(bh, bl, x, w);
  }
}

// T(s, c) = A(o(s), o(c)) ('trans' = 0) or A(o(c), o(s)) for c < s, and the
// diagonal D(s) = A(o(s), o(s)).  T is p x p, ld = p (upper part unused).
template <class N>
__global__ void __launch_bounds__(256)
trsm_coef_kernel(TrsmArgs t, const double* __restrict__ ah, const double* __restrict__ al,
                 int64_t lda, int trans) {
  const int64_t total = t.p * t.p;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e % t.p, c = e / t.p;
    if (c > s) continue;
    const int64_t os = t.rev ? t.p - 1 - s : s, oc = t.rev ? t.p - 1 - c : c;
    const int64_t x = trans ? oc + os * lda : os + oc * lda;
    if (c == s) {
      const typename N::T d = N::ld(ah, al, x);
      N::st(t.d_hi, t.d_lo, s, d);
      if (!t.unit && (t.fin_rec || t.rec_fast)) N::st(t.r_hi, t.r_lo, s, N::vdiv(N::one(), d));
    } else {
      N::st(t.t_hi, t.t_lo, s + c * t.ldt, N::ld(ah, al, x));
    }
  }
}

// Diagonal block [r0, r0 + nb) of the forward recurrence (nb <= 64), one
// warp per vector, lane t holding rows t and t + 32 of the block.  Step s:
// the running value of row s is broadcast, finished (fin_s) and stored, and
// every later row subtracts its term -- per element the terms arrive in
// production order.  The block of T sits in shared memory.
template <class N>
__global__ void __launch_bounds__(256)
trsm_block_kernel(TrsmArgs t, int64_t r0, int nb) {
  using T = typename N::T;
  extern __shared__ double sm[];
  __shared__ int tok;
  double* th = sm;
  double* tl = sm + nb * nb;
  if (threadIdx.x == 0) tok = !N::kF64;
  __syncthreads();
  bool ok = true;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int s = e % nb, c = e / nb;
    if (c < s) {
      const T tv = N::ld(t.t_hi, t.t_lo, (r0 + s) + (r0 + c) * t.ldt);
      N::st(th, tl, e, tv);
      ok &= N::win(tv);
    }
  }
  if (!ok) tok = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (v >= t.q) return;                      // whole warps
  double* wh = t.w_hi + v * t.ldw + r0;
  double* wl = t.w_lo + v * t.ldw + r0;
  const int ra = lane, rb = lane + 32;
  T acc_a = N::zero(), acc_b = N::zero();
  if (ra < nb) acc_a = N::ld(wh, wl, ra);
  if (rb < nb) acc_b = N::ld(wh, wl, rb);
  // inside the safe window (T block, this vector's start, each x): the
  // check-free forms, bit-identical to the checked ones; in the fast modes
  // the TwoSum accumulation (the products enter unrounded, dd accuracy)
  const bool blk_ok = __all_sync(0xffffffffu, tok && N::win(acc_a) && N::win(acc_b));
  const bool ts = blk_ok && t.rec_fast;
  for (int s = 0; s < nb; ++s) {
    T val = N::shfl(s < 32 ? acc_a : acc_b, s & 31);
    if (ts) val = ts_norm(val);
    const T x = trsm_fin<N>(t, r0 + s, val);
    if (lane == (s & 31)) N::st(wh, wl, s, x);
    const bool f = blk_ok && N::win(x);          // warp-uniform
    auto step = [&](T acc, int r) -> T {
      const T tv = N::ld(th, tl, r + s * nb);
      if (f && ts) return ts_mac(acc, N::neg(tv), x);
      if (f) return N::fadd2(acc, N::neg(N::fmul(tv, x)));
      return N::add(ts ? ts_norm(acc) : acc, N::neg(N::mul(tv, x)));
    };
    if (ra > s && ra < nb) acc_a = step(acc_a, ra);
    if (rb > s && rb < nb) acc_b = step(acc_b, rb);
  }
}

// The whole recurrence with the terms in REVERSE production order (t from
// s-1 down to 0): one sequential chain per vector (exact modes only).
template <class N>
__global__ void __launch_bounds__(128)
trsm_rev_kernel(TrsmArgs t) {
  using T = typename N::T;
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= t.q) return;
  double* wh = t.w_hi + v * t.ldw;
  double* wl = t.w_lo + v * t.ldw;
  for (int64_t s = 0; s < t.p; ++s) {
    T acc = N::ld(wh, wl, s);
    for (int64_t c = s - 1; c >= 0; --c)
      acc = N::add(acc, N::neg(N::mul(N::ld(t.t_hi, t.t_lo, s + c * t.ldt), N::ld(wh, wl, c))));
    N::st(wh, wl, s, trsm_fin<N>(t, s, acc));
  }
}

static unsigned grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g > 0 ? g : 1);
}

cudaError_t launch_trsm_pack(const TrsmArgs& t, const double* bh, const double* bl, int64_t ldb,
                             int scale, dd alpha, cudaStream_t s) {
  if (t.f64) trsm_pack_kernel<NumF64><<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  else trsm_pack_kernel<NumDD><<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  return cudaGetLastError();
}

cudaError_t launch_trsm_unpack(const TrsmArgs& t, double* bh, double* bl, int64_t ldb, int scale,
                               dd alpha, cudaStream_t s) {
  if (t.f64) trsm_unpack_kernel<NumF64><<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  else trsm_unpack_kernel<NumDD><<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  return cudaGetLastError();
}

cudaError_t launch_trsm_coef(const TrsmArgs& t, const double* ah, const double* al, int64_t lda,
                             int trans, cudaStream_t s) {
  if (t.f64) trsm_coef_kernel<NumF64><<<grid_for(t.p * t.p), 256, 0, s>>>(t, ah, al, lda, trans);
  else trsm_coef_kernel<NumDD><<<grid_for(t.p * t.p), 256, 0, s>>>(t, ah, al, lda, trans);
  return cudaGetLastError();
}

cudaError_t launch_trsm_block(const TrsmArgs& t, int64_t r0, int nb, cudaStream_t s) {
  const size_t smem = 2 * sizeof(double) * (size_t)nb * nb;
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(trsm_block_kernel<NumDD>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    cudaFuncSetAttribute(trsm_block_kernel<NumF64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         200 * 1024);
    attr_dev = dev;
  }
  if (t.f64) trsm_block_kernel<NumF64><<<(unsigned)((t.q + 7) / 8), 256, smem, s>>>(t, r0, nb);
  else trsm_block_kernel<NumDD><<<(unsigned)((t.q + 7) / 8), 256, smem, s>>>(t, r0, nb);
  return cudaGetLastError();
}

cudaError_t launch_trsm_rev(const TrsmArgs& t, cudaStream_t s) {
  if (t.f64) trsm_rev_kernel<NumF64><<<(unsigned)((t.q + 127) / 128), 128, 0, s>>>(t);
  else trsm_rev_kernel<NumDD><<<(unsigned)((t.q + 127) / 128), 128, 0, s>>>(t);
  return cudaGetLastError();
}

}  // namespace ddb
