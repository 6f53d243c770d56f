// lapack_num.cuh -- the two number systems of the LAPACK consumers
// (dd_potrf.cu, dd_trsm.cu, dd_getrf.cu), as policies the kernels are
// templated on:
//
//   NumDD   the reference's DDBackend (elem.py:200-283): element-wise add / mul
//           are the vectorised add2 / mul2 (elem.py:54-78), division the
//           vectorised _v_div2 (elem.py:93-117); scalars are DDouble with the
//           scalar _add2 / _div2 / _sqrt2 and _cmp2 order (ddarith.py:79-176).
//   NumF64  the F64Backend (elem.py:149-197): numpy float64 + - * /, Python
//           float scalars, math.sqrt -- plain IEEE binary64 (the library is
//           built with -fmad=false, so nothing is contracted).
//
// Storage is the reference's: dd matrices are (hi, lo) planes, binary64
// matrices one plane (the lo pointers are unused and may be null).
#pragma once
#include "internal.h"

namespace ddb {
namespace lap {

__device__ __forceinline__ dd neg2(dd x) { return dd{-x.h, -x.l}; }
__device__ __forceinline__ bool isfin(double x) { return finite_(x); }
// _canon (ddarith.py:68-71)
__device__ __forceinline__ dd canon(double h, double l) { return dd{h, isfin(h) ? l : 0.0}; }

// scalar _add2 (ddarith.py:79-90): the element form plus the final _canon
static __device__ dd add2_s(dd x, dd y) {
  const double s0 = dadd(x.h, y.h);
  if (!isfin(s0)) return dd{s0, 0.0};
  const dd r = add2_chk(x, y);
  return canon(r.h, r.l);
}

// _mul21 (ddarith.py:103-110): dd * double
static __device__ dd mul21_s(dd x, double y) {
  double p, e;
  two_prod_g(x.h, y, p, e);
  if (!(isfin(p) && isfin(e))) return canon(p, 0.0);
  e = dadd(e, dmul(x.l, y));
  double s, t;
  quick_two_sum(p, e, s, t);
  return canon(s, t);
}

// _div2 (ddarith.py:113-131)
static __device__ dd div2_s(dd x, dd y) {
  const double qnan = __longlong_as_double(0x7ff8000000000000LL);
  const double inf = __longlong_as_double(0x7ff0000000000000LL);
  if (y.h == 0.0) {
    if (x.h == 0.0) return dd{qnan, 0.0};
    return dd{copysign(inf, x.h) * copysign(1.0, y.h), 0.0};
  }
  if (!(isfin(x.h) && isfin(y.h))) {
    if (!isfin(y.h) && !isnan(y.h)) {
      if (!isfin(x.h) && !isnan(x.h)) return dd{qnan, 0.0};
      return dd{dmul(copysign(0.0, x.h), copysign(1.0, y.h)), 0.0};
    }
    return canon(dmul(x.h, copysign(1.0, y.h)), 0.0);
  }
  const double q1 = x.h / y.h;
  dd r = add2_s(x, neg2(mul21_s(y, q1)));
  const double q2 = r.h / y.h;
  r = add2_s(r, neg2(mul21_s(y, q2)));
  const double q3 = r.h / y.h;
  double a, b;
  quick_two_sum(q1, q2, a, b);
  return add2_s(dd{a, b}, dd{q3, 0.0});
}

// _sqrt2 (ddarith.py:142-163): Newton correction on 1/sqrt(hi), with the
// exact even-power pre-scaling for very large / small arguments
static __device__ dd sqrt2_s(dd v) {
  if (v.h == 0.0 && v.l == 0.0) return dd{0.0, 0.0};
  if (!isfin(v.h)) return dd{v.h, 0.0};
  double h = v.h, l = v.l;
  int shift = 0;
  if (h >= 0x1p996) { h = dmul(h, 0x1p-106); l = dmul(l, 0x1p-106); shift = 53; }
  else if (h <= 0x1p-996) { h = dmul(h, 0x1p106); l = dmul(l, 0x1p106); shift = -53; }
  const double x = 1.0 / sqrt(h);
  const double ax = dmul(h, x);
  double p, e;
  two_prod_g(ax, ax, p, e);
  const dd r = add2_s(dd{h, l}, dd{-p, -e});
  double s, e2;
  quick_two_sum(ax, dmul(r.h, dmul(x, 0.5)), s, e2);
  if (shift == 53) { s = dmul(s, 0x1p53); e2 = dmul(e2, 0x1p53); }
  else if (shift == -53) { s = dmul(s, 0x1p-53); e2 = dmul(e2, 0x1p-53); }
  return canon(s, e2);
}

// vectorised _v_mul21 / _v_div2 (elem.py:81-117): the special lanes take
// the scalar _div2
static __device__ dd v_mul21(dd y, double q) {
  double p, e;
  two_prod_g(y.h, q, p, e);
  const bool bad = !(isfin(p) && isfin(e));
  e = dadd(e, dmul(y.l, q));
  double s, t;
  quick_two_sum(p, e, s, t);
  return bad ? dd{p, 0.0} : dd{s, t};
}
static __device__ dd v_div2(dd x, dd y) {
  if (y.h == 0.0 || !(isfin(x.h) && isfin(y.h))) return div2_s(x, y);
  const double q1 = x.h / y.h;
  dd r = add2_chk(x, neg2(v_mul21(y, q1)));
  const double q2 = r.h / y.h;
  r = add2_chk(r, neg2(v_mul21(y, q2)));
  const double q3 = r.h / y.h;
  double a, b;
  quick_two_sum(q1, q2, a, b);
  return add2_chk(dd{a, b}, dd{q3, 0.0});
}

}  // namespace lap

struct NumDD {
  using T = dd;
  static constexpr bool kF64 = false;
  __device__ static T ld(const double* h, const double* l, int64_t i) { return dd{h[i], l[i]}; }
  __device__ static T ldcg(const double* h, const double* l, int64_t i) {
    return dd{__ldcg(h + i), __ldcg(l + i)};
  }
  __device__ static T ldg(const double* h, const double* l, int64_t i) {
    return dd{__ldg(h + i), __ldg(l + i)};
  }
  __device__ static void st(double* h, double* l, int64_t i, T v) { h[i] = v.h; l[i] = v.l; }
  // the prescan's safe window (dd_prescan.cu): hi zero or 2^-300 <= |hi| <
  // 2^301, lo finite below 2^301.  For operands inside it (and accumulators
  // that started inside it and took at most a few thousand such products)
  // fadd / fmul are bit-identical to add / mul (dd_arith.cuh)
  __device__ static bool win(T x) {
    const int eh = (int)((__double_as_longlong(x.h) >> 52) & 0x7ff);
    const int el = (int)((__double_as_longlong(x.l) >> 52) & 0x7ff);
    return (eh >= WIN_LO || (__double_as_longlong(x.h) << 1) == 0) && eh <= WIN_HI && el <= WIN_HI;
  }
  __device__ static T fadd(T x, T y) { return add2_nc_sel(x, y); }
  __device__ static T fadd2(T x, T y) { return add2_nc(x, y); }
  __device__ static T fmul(T x, T y) { return mul2_nc(x, y); }
  __device__ static T zero() { return dd{0.0, 0.0}; }
  __device__ static T one() { return dd{1.0, 0.0}; }
  __device__ static T neg(T x) { return lap::neg2(x); }
  __device__ static T add(T x, T y) { return add2_chk(x, y); }           // be.add
  __device__ static T mul(T x, T y) { return mul2_chk(x, y); }           // be.mul
  __device__ static T vdiv(T x, T y) { return lap::v_div2(x, y); }      // be.div
  __device__ static T ssub(T x, T y) { return lap::add2_s(x, lap::neg2(y)); }   // DDouble -
  __device__ static T sdiv(T x, T y) { return lap::div2_s(x, y); }      // DDouble /
  __device__ static T ssqrt(T x) { return lap::sqrt2_s(x); }            // dd_sqrt
  __device__ static bool nonzero(T x) { return x.h != 0.0 || x.l != 0.0; }   // __bool__
  // chol.py:42: _isnan(ajj) (float(ajj) = hi + lo) or ajj <= 0 (_cmp2 order)
  __device__ static bool bad_pivot(T a) {
    if (isnan(dadd(a.h, a.l))) return true;
    if (a.h < 0.0) return true;
    if (a.h > 0.0) return false;
    return !(a.l > 0.0);
  }
  // lu.py:98: abs(pivot) >= safmin, DDouble __abs__ then _cmp2 (NaN: true)
  __device__ static bool ge_safmin(T p) {
    if (p.h < 0.0 || (p.h == 0.0 && p.l < 0.0)) p = lap::neg2(p);
    const double sh = 0x1p-969, sl = -0x0.0000000000006p-1022;
    return !(p.h < sh) && (p.h > sh || !(p.l < sl));
  }
  // argmax_abs key (elem.py:246-259): |hi|, then lo * sign(hi)
  __device__ static double key_hi(T x) { return fabs(x.h); }
  __device__ static double key_lo(T x) { return x.h < 0.0 ? -x.l : x.l; }
  __device__ static bool key_nan(T x) { return isnan(x.h); }
  __device__ static T shfl(T v, int src) {
    return dd{__shfl_sync(0xffffffffu, v.h, src), __shfl_sync(0xffffffffu, v.l, src)};
  }
  __device__ static double hi(T x) { return x.h; }
  __device__ static double lo(T x) { return x.l; }
  __device__ static T make(double h, double l) { return dd{h, l}; }
};

struct NumF64 {
  using T = double;
  static constexpr bool kF64 = true;
  __device__ static T ld(const double* h, const double*, int64_t i) { return h[i]; }
  __device__ static T ldcg(const double* h, const double*, int64_t i) { return __ldcg(h + i); }
  __device__ static T ldg(const double* h, const double*, int64_t i) { return __ldg(h + i); }
  __device__ static void st(double* h, double*, int64_t i, T v) { h[i] = v; }
  __device__ static bool win(T) { return true; }
  __device__ static T fadd(T x, T y) { return dadd(x, y); }
  __device__ static T fadd2(T x, T y) { return dadd(x, y); }
  __device__ static T fmul(T x, T y) { return dmul(x, y); }
  __device__ static T zero() { return 0.0; }
  __device__ static T one() { return 1.0; }
  __device__ static T neg(T x) { return -x; }
  __device__ static T add(T x, T y) { return dadd(x, y); }
  __device__ static T mul(T x, T y) { return dmul(x, y); }
  __device__ static T vdiv(T x, T y) { return __ddiv_rn(x, y); }
  __device__ static T ssub(T x, T y) { return dsub(x, y); }
  __device__ static T sdiv(T x, T y) { return __ddiv_rn(x, y); }
  __device__ static T ssqrt(T x) { return __dsqrt_rn(x); }              // math.sqrt
  __device__ static bool nonzero(T x) { return x != 0.0; }
  __device__ static bool bad_pivot(T a) { return isnan(a) || a <= 0.0; }
  __device__ static bool ge_safmin(T p) { return fabs(p) >= 0x1p-1022; }   // NaN: false
  __device__ static double key_hi(T x) { return fabs(x); }
  __device__ static double key_lo(T) { return 0.0; }                   // ties: first index
  __device__ static bool key_nan(T x) { return isnan(x); }
  __device__ static T shfl(T v, int src) { return __shfl_sync(0xffffffffu, v, src); }
  __device__ static double hi(T x) { return x; }
  __device__ static double lo(T) { return 0.0; }
  __device__ static T make(double h, double) { return h; }
};

}  // namespace ddb
