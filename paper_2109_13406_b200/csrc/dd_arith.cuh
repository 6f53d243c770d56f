// dd_arith.cuh -- device double-double error-free transforms.
//
// Every operation is written with explicit round-to-nearest intrinsics
// (__dadd_rn / __dsub_rn / __dmul_rn / __fma_rn) so nvcc can never contract
// a*b+c into an FMA behind our back; the library is additionally built with
// -fmad=false.  The formulas restate the reference's vectorised element
// kernels (/root/reference/pkg/src/mpkit/mpblas/elem.py):
//
//   two_sum         elem.py:32-35       quick_two_sum   elem.py:38-40
//   two_prod_dekker elem.py:43-51       (splitter 2**27+1, elem.py:25)
//   add2_chk        elem.py:54-66       mul2_chk        elem.py:69-78
//
// The *_nc variants drop the finiteness fix-ups and use the FMA TwoProd.
// They are bit-identical to the checked reference forms whenever every hi
// word lies in the "safe window" enforced by the prescan (see
// dd_prescan.cu): no overflow can occur, and for |a|,|b| >= 2**-300 the FMA
// residual equals Dekker's (both exact, both +0 when zero).
#pragma once
#include <cstdint>

namespace ddb {

struct dd { double h, l; };

__device__ __forceinline__ double dadd(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ double dsub(double a, double b) { return __dsub_rn(a, b); }
__device__ __forceinline__ double dmul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double dfma(double a, double b, double c) { return __fma_rn(a, b, c); }

__device__ __forceinline__ bool finite_(double x) {
  // exponent field != 0x7ff; integer test, keeps the FP64 pipe free
  return ((__double_as_longlong(x) >> 52) & 0x7ff) != 0x7ff;
}

__device__ __forceinline__ void two_sum(double a, double b, double& s, double& e) {
  double ss = dadd(a, b);
  double bb = dsub(ss, a);
  e = dadd(dsub(a, dsub(ss, bb)), dsub(b, bb));
  s = ss;
}

__device__ __forceinline__ void quick_two_sum(double a, double b, double& s, double& e) {
  double ss = dadd(a, b);
  e = dsub(b, dsub(ss, a));
  s = ss;
}

__device__ __forceinline__ void two_prod_dekker(double a, double b, double& p, double& e) {
  const double S = 134217729.0;  // 2**27 + 1
  double pp = dmul(a, b);
  double t = dmul(S, a);
  double ah = dsub(t, dsub(t, a));
  double al = dsub(a, ah);
  t = dmul(S, b);
  double bh = dsub(t, dsub(t, b));
  double bl = dsub(b, bh);
  e = dadd(dadd(dadd(dsub(dmul(ah, bh), pp), dmul(ah, bl)), dmul(al, bh)), dmul(al, bl));
  p = pp;
}

__device__ __forceinline__ void two_prod_fma(double a, double b, double& p, double& e) {
  p = dmul(a, b);
  e = dfma(a, b, -p);
}

// Dekker's product with the FMA residual where the two agree bit for bit:
// both factors non-zero with 2^-300 <= |x| < 2^301 (biased exponents 723 ..
// 1323), so no split product under- or overflows and both residuals are the
// exact a*b - p (+0 when zero).  Elsewhere Dekker's, as the reference.
__device__ __forceinline__ void two_prod_g(double a, double b, double& p, double& e) {
  const unsigned ea = (unsigned)((__double_as_longlong(a) >> 52) & 0x7ff) - 723u;
  const unsigned eb = (unsigned)((__double_as_longlong(b) >> 52) & 0x7ff) - 723u;
  if (ea <= 600u && eb <= 600u) two_prod_fma(a, b, p, e);
  else two_prod_dekker(a, b, p, e);
}

// elem.py:54-66 (accurate add; only s0 = xh + yh is checked)
__device__ __forceinline__ dd add2_chk(dd x, dd y) {
  double s0 = dadd(x.h, y.h);
  double sh, sl, th, tl;
  two_sum(x.h, y.h, sh, sl);
  two_sum(x.l, y.l, th, tl);
  sl = dadd(sl, th);
  quick_two_sum(sh, sl, sh, sl);
  sl = dadd(sl, tl);
  quick_two_sum(sh, sl, sh, sl);
  if (!finite_(s0)) { sh = s0; sl = 0.0; }
  return dd{sh, sl};
}

// elem.py:69-78
__device__ __forceinline__ dd mul2_chk(dd x, dd y) {
  double p, e;
  two_prod_g(x.h, y.h, p, e);
  bool bad = !(finite_(p) && finite_(e));
  e = dadd(e, dadd(dmul(x.h, y.l), dmul(x.l, y.h)));
  double rh, rl;
  quick_two_sum(p, e, rh, rl);
  if (bad) { rh = p; rl = 0.0; }
  return dd{rh, rl};
}

// Safe-window forms (29 FP64-pipe instructions per mul2+add2 pair).
__device__ __forceinline__ dd add2_nc(dd x, dd y) {
  double sh, sl, th, tl;
  two_sum(x.h, y.h, sh, sl);
  two_sum(x.l, y.l, th, tl);
  sl = dadd(sl, th);
  quick_two_sum(sh, sl, sh, sl);
  sl = dadd(sl, tl);
  quick_two_sum(sh, sl, sh, sl);
  return dd{sh, sl};
}

// TwoSum via an ordered Fast2Sum: for finite operands the error term
// (big - s) + small (Fast2Sum, big - s exact by Sterbenz) is the exact rounding
// error, as is Knuth's TwoSum's, and both are +0 whenever the error is zero
// (written as small - (s - big) it would be -0 for small = -0) -- so the
// result is bit-identical to two_sum with 3 FP64 instructions instead of 6.
// The operands are ordered by comparing the sign-masked high words on the
// integer pipe (equal high words mean equal exponents: either order works).
__device__ __forceinline__ void two_sum_sel(double a, double b, double& s, double& e) {
  int ah, bh;
  asm("{\n\t.reg .b32 lo;\n\tmov.b64 {lo, %0}, %1;\n\t}" : "=r"(ah) : "d"(a));
  asm("{\n\t.reg .b32 lo;\n\tmov.b64 {lo, %0}, %1;\n\t}" : "=r"(bh) : "d"(b));
  const bool ge = (ah & 0x7fffffff) >= (bh & 0x7fffffff);
  const double big = ge ? a : b, small = ge ? b : a;
  s = dadd(a, b);
  e = dadd(dsub(big, s), small);
}

// add2_nc with the ordered-Fast2Sum TwoSums: 14 instead of 20 FP64 ops.
__device__ __forceinline__ dd add2_nc_sel(dd x, dd y) {
  double sh, sl, th, tl;
  two_sum_sel(x.h, y.h, sh, sl);
  two_sum_sel(x.l, y.l, th, tl);
  sl = dadd(sl, th);
  quick_two_sum(sh, sl, sh, sl);
  sl = dadd(sl, tl);
  quick_two_sum(sh, sl, sh, sl);
  return dd{sh, sl};
}

__device__ __forceinline__ dd mul2_nc(dd x, dd y) {
  double p, e;
  two_prod_fma(x.h, y.h, p, e);
  e = dadd(e, dadd(dmul(x.h, y.l), dmul(x.l, y.h)));
  double rh, rl;
  quick_two_sum(p, e, rh, rl);
  return dd{rh, rl};
}

__device__ __forceinline__ bool dd_is_zero(dd v) { return v.h == 0.0 && v.l == 0.0; }
__device__ __forceinline__ bool dd_is_one(dd v) { return v.h == 1.0 && v.l == 0.0; }

// _scale_full / _scale_masked beta rule (level23.py:163-169, :273-280)
__device__ __forceinline__ dd scale_beta(dd beta, dd c) {
  if (dd_is_zero(beta)) return dd{0.0, 0.0};
  if (dd_is_one(beta)) return c;
  return mul2_chk(beta, c);
}

// _combine (level23.py:172-177)
__device__ __forceinline__ dd combine(dd alpha, dd acc, dd beta, dd c0) {
  dd at = mul2_chk(alpha, acc);
  if (dd_is_zero(beta)) return at;
  return add2_chk(at, mul2_chk(beta, c0));
}

}  // namespace ddb
