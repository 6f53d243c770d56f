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
#include "internal.h"

namespace ddb {

namespace {

__device__ __forceinline__ dd negd(dd x) { return dd{-x.h, -x.l}; }
__device__ __forceinline__ bool fin_(double x) { return finite_(x); }
__device__ __forceinline__ dd canon_(double h, double l) { return dd{h, fin_(h) ? l : 0.0}; }

// scalar _add2 / _mul21 / _div2 (ddarith.py:79-131), for the special lanes
__device__ dd add2_sc(dd x, dd y) {
  const double s0 = dadd(x.h, y.h);
  if (!fin_(s0)) return dd{s0, 0.0};
  const dd r = add2_chk(x, y);
  return canon_(r.h, r.l);
}
__device__ dd mul21_sc(dd x, double y) {
  double p, e;
  two_prod_dekker(x.h, y, p, e);
  if (!(fin_(p) && fin_(e))) return canon_(p, 0.0);
  e = dadd(e, dmul(x.l, y));
  double s, t;
  quick_two_sum(p, e, s, t);
  return canon_(s, t);
}
__device__ dd div2_sc(dd x, dd y) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  if (y.h == 0.0) {
    if (x.h == 0.0) return dd{qnan, 0.0};
    return dd{copysign(inf, x.h) * copysign(1.0, y.h), 0.0};
  }
  if (!(fin_(x.h) && fin_(y.h))) {
    if (!fin_(y.h) && !isnan(y.h)) {
      if (!fin_(x.h) && !isnan(x.h)) return dd{qnan, 0.0};
      return dd{dmul(copysign(0.0, x.h), copysign(1.0, y.h)), 0.0};
    }
    return canon_(dmul(x.h, copysign(1.0, y.h)), 0.0);
  }
  const double q1 = x.h / y.h;
  dd r = add2_sc(x, negd(mul21_sc(y, q1)));
  const double q2 = r.h / y.h;
  r = add2_sc(r, negd(mul21_sc(y, q2)));
  const double q3 = r.h / y.h;
  double a, b;
  quick_two_sum(q1, q2, a, b);
  return add2_sc(dd{a, b}, dd{q3, 0.0});
}

// vectorised _v_mul21 / _v_div2 (elem.py:81-117): special lanes take the
// scalar path
__device__ dd v_mul21(dd y, double q) {
  double p, e;
  two_prod_dekker(y.h, q, p, e);
  const bool bad = !(fin_(p) && fin_(e));
  e = dadd(e, dmul(y.l, q));
  double s, t;
  quick_two_sum(p, e, s, t);
  return bad ? dd{p, 0.0} : dd{s, t};
}
__device__ dd v_div2(dd x, dd y) {
  if (y.h == 0.0 || !(fin_(x.h) && fin_(y.h))) return div2_sc(x, y);
  const double q1 = x.h / y.h;
  dd r = add2_chk(x, negd(v_mul21(y, q1)));
  const double q2 = r.h / y.h;
  r = add2_chk(r, negd(v_mul21(y, q2)));
  const double q3 = r.h / y.h;
  double a, b;
  quick_two_sum(q1, q2, a, b);
  return add2_chk(dd{a, b}, dd{q3, 0.0});
}

__device__ __forceinline__ dd trsm_fin(const TrsmArgs& t, int64_t s, dd v) {
  if (t.unit) return v;
  const dd d{t.d_hi[s], t.d_lo[s]};
  if (t.fin_rec) return mul2_chk(v_div2(dd{1.0, 0.0}, d), v);
  return v_div2(v, d);
}

}  // namespace

// W <- B in production order (side 'L': W(s, j) = B(o(s), j); 'R':
// W(s, i) = B(i, o(s))), times alpha when `scale`.
__global__ void __launch_bounds__(256)
trsm_pack_kernel(TrsmArgs t, const double* __restrict__ bh, const double* __restrict__ bl,
                 int64_t ldb, int scale, dd alpha) {
  const int64_t total = t.p * t.q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e % t.p, v = e / t.p;
    const int64_t o = t.rev ? t.p - 1 - s : s;
    const int64_t x = t.left ? o + v * ldb : v + o * ldb;
    dd w{bh[x], bl[x]};
    if (scale) w = mul2_chk(alpha, w);
    t.w_hi[s + v * t.ldw] = w.h;
    t.w_lo[s + v * t.ldw] = w.l;
  }
}

// B <- W (inverse of the pack), times alpha when `scale`.
__global__ void __launch_bounds__(256)
trsm_unpack_kernel(TrsmArgs t, double* __restrict__ bh, double* __restrict__ bl, int64_t ldb,
                   int scale, dd alpha) {
  const int64_t total = t.p * t.q;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < total;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t s = e % t.p, v = e / t.p;
    const int64_t o = t.rev ? t.p - 1 - s : s;
    const int64_t x = t.left ? o + v * ldb : v + o * ldb;
    dd w{t.w_hi[s + v * t.ldw], t.w_lo[s + v * t.ldw]};
    if (scale) w = mul2_chk(alpha, w);
    bh[x] = w.h;
    bl[x] = w.l;
  }
}

// T(s, c) = A(o(s), o(c)) ('trans' = 0) or A(o(c), o(s)) for c < s, and the
// diagonal D(s) = A(o(s), o(s)).  T is p x p, ld = p (upper part unused).
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
      t.d_hi[s] = ah[x];
      t.d_lo[s] = al[x];
    } else {
      t.t_hi[s + c * t.ldt] = ah[x];
      t.t_lo[s + c * t.ldt] = al[x];
    }
  }
}

// Diagonal block [r0, r0 + nb) of the forward recurrence (nb <= 64), one
// warp per vector, lane t holding rows t and t + 32 of the block.  Step s:
// the running value of row s is broadcast, finished (fin_s) and stored, and
// every later row subtracts its term -- per element the terms arrive in
// production order.  The block of T sits in shared memory.
__global__ void __launch_bounds__(256)
trsm_block_kernel(TrsmArgs t, int64_t r0, int nb) {
  extern __shared__ double sm[];
  double* th = sm;
  double* tl = sm + nb * nb;
  for (int e = threadIdx.x; e < nb * nb; e += blockDim.x) {
    const int s = e % nb, c = e / nb;
    if (c < s) {
      th[e] = t.t_hi[(r0 + s) + (r0 + c) * t.ldt];
      tl[e] = t.t_lo[(r0 + s) + (r0 + c) * t.ldt];
    }
  }
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t v = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  if (v >= t.q) return;                      // whole warps
  double* wh = t.w_hi + v * t.ldw + r0;
  double* wl = t.w_lo + v * t.ldw + r0;
  const int ra = lane, rb = lane + 32;
  dd acc_a{0.0, 0.0}, acc_b{0.0, 0.0};
  if (ra < nb) acc_a = dd{wh[ra], wl[ra]};
  if (rb < nb) acc_b = dd{wh[rb], wl[rb]};
  for (int s = 0; s < nb; ++s) {
    const dd own = s < 32 ? acc_a : acc_b;
    dd val;
    val.h = __shfl_sync(0xffffffffu, own.h, s & 31);
    val.l = __shfl_sync(0xffffffffu, own.l, s & 31);
    const dd x = trsm_fin(t, r0 + s, val);
    if (lane == (s & 31)) {
      wh[s] = x.h;
      wl[s] = x.l;
    }
    if (ra > s && ra < nb)
      acc_a = add2_chk(acc_a, negd(mul2_chk(dd{th[ra + s * nb], tl[ra + s * nb]}, x)));
    if (rb > s && rb < nb)
      acc_b = add2_chk(acc_b, negd(mul2_chk(dd{th[rb + s * nb], tl[rb + s * nb]}, x)));
  }
}

// The whole recurrence with the terms in REVERSE production order (t from
// s-1 down to 0): one sequential chain per vector (exact modes only).
__global__ void __launch_bounds__(128)
trsm_rev_kernel(TrsmArgs t) {
  const int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (v >= t.q) return;
  double* wh = t.w_hi + v * t.ldw;
  double* wl = t.w_lo + v * t.ldw;
  for (int64_t s = 0; s < t.p; ++s) {
    dd acc{wh[s], wl[s]};
    for (int64_t c = s - 1; c >= 0; --c)
      acc = add2_chk(acc, negd(mul2_chk(dd{t.t_hi[s + c * t.ldt], t.t_lo[s + c * t.ldt]},
                                        dd{wh[c], wl[c]})));
    const dd x = trsm_fin(t, s, acc);
    wh[s] = x.h;
    wl[s] = x.l;
  }
}

static unsigned grid_for(int64_t total) {
  int64_t g = (total + 255) / 256;
  if (g > 148 * 16) g = 148 * 16;
  return (unsigned)(g > 0 ? g : 1);
}

cudaError_t launch_trsm_pack(const TrsmArgs& t, const double* bh, const double* bl, int64_t ldb,
                             int scale, dd alpha, cudaStream_t s) {
  trsm_pack_kernel<<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  return cudaGetLastError();
}

cudaError_t launch_trsm_unpack(const TrsmArgs& t, double* bh, double* bl, int64_t ldb, int scale,
                               dd alpha, cudaStream_t s) {
  trsm_unpack_kernel<<<grid_for(t.p * t.q), 256, 0, s>>>(t, bh, bl, ldb, scale, alpha);
  return cudaGetLastError();
}

cudaError_t launch_trsm_coef(const TrsmArgs& t, const double* ah, const double* al, int64_t lda,
                             int trans, cudaStream_t s) {
  trsm_coef_kernel<<<grid_for(t.p * t.p), 256, 0, s>>>(t, ah, al, lda, trans);
  return cudaGetLastError();
}

cudaError_t launch_trsm_block(const TrsmArgs& t, int64_t r0, int nb, cudaStream_t s) {
  const size_t smem = 2 * sizeof(double) * (size_t)nb * nb;
  static thread_local int attr_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (attr_dev != dev) {
    cudaFuncSetAttribute(trsm_block_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr_dev = dev;
  }
  trsm_block_kernel<<<(unsigned)((t.q + 7) / 8), 256, smem, s>>>(t, r0, nb);
  return cudaGetLastError();
}

cudaError_t launch_trsm_rev(const TrsmArgs& t, cudaStream_t s) {
  trsm_rev_kernel<<<(unsigned)((t.q + 127) / 128), 128, 0, s>>>(t);
  return cudaGetLastError();
}

}  // namespace ddb
