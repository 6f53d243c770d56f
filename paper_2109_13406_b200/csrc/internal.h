// internal.h -- declarations shared by the kernels and the C ABI (capi.cu).
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

#include "dd_arith.cuh"

namespace ddb {

enum Mode { MODE_EXACT = 0, MODE_FAST = 1, MODE_REFERENCE = 2, MODE_TWOSUM = 3 };

// Tiled accumulation algorithm for a mode (dd_gemm.cu).
// ALG_SPLIT: the certified-anchor accumulation of hi * hi only, with the
// lo * hi + hi * lo cross terms from two binary64 GEMMs (dd_tma.cu; fast mode,
// TMA route only)
enum Alg { ALG_EXACT = 0, ALG_TWOSUM = 1, ALG_SELECT = 2, ALG_CERT = 3, ALG_F64 = 4,
           ALG_SPLIT = 5 };
int alg_for_mode(int mode);

// Route flag written by the prescan: 0 = every operand inside the safe
// window, nonzero = some value outside it (non-finite, |x| > 2**301, or a
// nonzero hi word below 2**-300).  Routing is per element (dd_prescan.cu):
// the prescan marks every op(A) row / op(B) column holding such a word, the
// tiled kernels skip the elements in those rows / columns and the
// reference-semantics kernel computes exactly those.
enum RouteFlag { ROUTE_SAFE = 0, ROUTE_UNSAFE = 1 };

// Per-element route classes (elem_class below).
//   EC_FAST: the mode's tiled kernel (fast, exact or twosum);
//   EC_WIDE: fast modes only, the element's row and column exponent spreads
//            (max / min nonzero |hi|) are too wide for the certified bound to
//            be tight (dd_bound.cu): the TwoSum accumulation computes it;
//   EC_REF:  a word outside the safe window in its row or column: the
//            reference-semantics kernel (dd_reference.cu) computes it.
// Certified-anchor (fast) accumulation: deepest k it accepts, and the
// spread limit for EC_WIDE (dd_bound.cu derives both): an element whose row
// and column exponent spreads sum above 112 - ceil(log2 k) takes TwoSum.
// The TMA GEMM walks its tiles with one persistent CTA per SM, except while
// a NoPersistScope is alive on the calling host thread (Rpotrf / Rgetrf:
// their panel stream must find SMs freeing up during a trailing update).
struct NoPersistScope {
  explicit NoPersistScope(bool on = true);
  ~NoPersistScope();
  bool on_;
};

constexpr int64_t kCertMaxK = int64_t(1) << 16;
inline int wide_limit(int64_t k) {
  int lg = 0;
  while ((int64_t(1) << lg) < k) ++lg;
  return 112 - lg;
}

enum ElemClass { EC_FAST = 0, EC_WIDE = 1, EC_REF = 2 };
constexpr int SPREAD_BAD = 1 << 20;      // spread value of a row / column holding an unsafe word
constexpr int ROUTE_BLK = 32;            // rows / columns per block maximum (rsb / csb)

// Safe window in biased-exponent terms (see dd_prescan.cu).
constexpr int WIN_LO = 1023 - 300;   // hi words: zero or biased exp >= WIN_LO
constexpr int WIN_HI = 1023 + 300;   // hi and lo words: biased exp <= WIN_HI

struct GemmArgs {
  int ta, tb;                 // 0 = 'N', 1 = 'T'/'C' (real: conj is identity)
  int syrk;                   // 0 = Rgemm, 1 = Rsyrk upper, 2 = Rsyrk lower
  int64_t m, n, k;
  const double *a_hi, *a_lo; int64_t lda;
  const double *b_hi, *b_lo; int64_t ldb;
  double *c_hi, *c_lo; int64_t ldc;
  dd alpha, beta;
  // fast mode (ALG_CERT): certified magnitude bound, m x n fp32, ld = m,
  // in units of 2^(row_exp + col_exp - 2044); see dd_bound.cu
  const float* bound;
  double bnd_fac, bnd_floor;
  // split-K (fast modes): k is cut into chunks of kchunk (a multiple of the
  // k-tile); each chunk's (hi, lo) sum goes to part[z] (2 planes of m x n) and
  // splitk_reduce adds them in order.  kchunk >= k: no split, part == nullptr.
  int64_t kchunk;
  double* part;
  int group_m;      // raster group height in tiles (L2 reuse); 0 = default
  // binary64 precision (the reference's 'f64' Matrix): only the hi planes
  // exist; a_lo / b_lo / c_lo are unused (dd_reference.cu, ALG_F64)
  int f64;
  // exact / reference modes, TA == 0 only: c = c - a*b per step with the
  // product negated after rounding (be.sub(c, be.mul(a, b)), the reference's
  // Rtrsm update, level23.py:334-336); alpha, beta unused (treated as 1)
  int sub;
  // ALG_SPLIT: sum_l a_lo b_hi + a_hi b_lo (m x n, ld = m), added into the
  // low word of the first k-slice's sum
  const double* cross;
  // per-element routing (dd_prescan.cu, route_summary_kernel): exponent
  // spread of op(A) row i / op(B) column j (SPREAD_BAD: holds an unsafe
  // word), and their maxima over blocks of ROUTE_BLK rows / columns (unsafe
  // rows excluded).  nullptr: no routing (every element EC_FAST).
  const int *rsp, *csp, *rsb, *csb;
  int wide_lim;     // fast modes: spread sum above which an element is EC_WIDE (0: never)
  int only_wide;    // TwoSum fallback launch: compute / store EC_WIDE elements only
  const int* flag;  // [0] any unsafe word, [1] max row spread, [2] max column spread,
                    // [3] / [4] number of unsafe rows / columns (listed in bad_rows / bad_cols)
  const int *bad_rows, *bad_cols;
};

__device__ __forceinline__ int elem_class(const GemmArgs& g, int64_t i, int64_t j) {
  if (g.rsp == nullptr) return EC_FAST;
  const int v = g.rsp[i] + g.csp[j];
  if (v >= SPREAD_BAD) return EC_REF;
  return (g.wide_lim > 0 && v > g.wide_lim) ? EC_WIDE : EC_FAST;
}

// The element class a kernel instance writes: the fallback launch writes the
// EC_WIDE elements, every other launch the EC_FAST ones.
__device__ __forceinline__ bool elem_mine(const GemmArgs& g, int64_t i, int64_t j) {
  return elem_class(g, i, j) == (g.only_wide ? EC_WIDE : EC_FAST);
}

// Fallback launch: can the tile [i0, i0 + bm) x [j0, j0 + bn) hold an
// EC_WIDE element?  Block maxima only (a superset test; stores re-check).
__device__ __forceinline__ bool tile_maybe_wide(const GemmArgs& g, int64_t i0, int64_t j0,
                                                int bm, int bn) {
  if (g.flag[1] + g.flag[2] <= g.wide_lim) return false;    // no wide element in the call
  int rm = 0, cm = 0;
  const int64_t i1 = i0 + bm - 1 < g.m - 1 ? i0 + bm - 1 : g.m - 1;
  const int64_t j1 = j0 + bn - 1 < g.n - 1 ? j0 + bn - 1 : g.n - 1;
  const int64_t ib1 = i1 / ROUTE_BLK, jb1 = j1 / ROUTE_BLK;
  for (int64_t b = i0 / ROUTE_BLK; b <= ib1; ++b) rm = max(rm, g.rsb[b]);
  for (int64_t b = j0 / ROUTE_BLK; b <= jb1; ++b) cm = max(cm, g.csb[b]);
  return rm + cm > g.wide_lim;
}

// Which kernel should run, decided on the device by the prescan flag.
enum Gate { GATE_ALWAYS = 0, GATE_IF_SAFE = 1, GATE_IF_UNSAFE = 2 };

// Route workspace carved from one zeroed block (dd_prescan.cu)
struct RouteWs {
  int* flag;                    // 16 ints
  int *rmax, *rneg, *cmax, *cneg;   // per op(A) row / op(B) column (Rsyrk: c* == r*)
  int *rsp, *csp, *rsb, *csb;
  int *bad_rows, *bad_cols;     // the unsafe rows / columns, flag[3] / flag[4] of them
};
size_t route_ws_bytes(int64_t m, int64_t n, int syrk);
RouteWs route_ws_carve(void* base, int64_t m, int64_t n, int syrk);
cudaError_t launch_prescan(const GemmArgs& g, int alg, const RouteWs& r, cudaStream_t s,
                           int* nlaunch);
cudaError_t launch_wide_fallback(const GemmArgs& g, cudaStream_t s, int* nlaunch);
cudaError_t launch_reference(const GemmArgs& g, const int* flag, int gate, cudaStream_t s,
                             int* nlaunch);
cudaError_t launch_tiled(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch);
size_t bound_workspace_bytes(const GemmArgs& g);
float* bound_carve(const GemmArgs& g, void* ws);   // the fp32 bound inside the workspace
int choose_ksplit(const GemmArgs& g, int alg, int64_t* kchunk);
cudaError_t launch_splitk_reduce(const GemmArgs& g, int splits, const int* flag, cudaStream_t s,
                                 int* nlaunch);
cudaError_t launch_bound(const GemmArgs& g, const int* row_exp, const int* col_exp, void* ws,
                         float* bound, cudaStream_t s, int* nlaunch, const char** what);
int cross_kslices(const GemmArgs& g, int64_t* kchunk);
cudaError_t launch_cross_dmma(const GemmArgs& g, double* x, cudaStream_t s, int* nlaunch,
                              int slices = 1, int64_t kchunk = 0);

// complex GEMM (dd_complex.cu)
struct cdd { dd re, im; };
struct z64 { double re, im; };

struct CgemmArgs {            // 'cdd': planes re_hi, re_lo, im_hi, im_lo
  int ta, tb, conja, conjb;
  int64_t m, n, k;
  const double* a[4]; int64_t lda;
  const double* b[4]; int64_t ldb;
  double* c[4]; int64_t ldc;
  cdd alpha, beta;
};

struct ZgemmArgs {            // 'c64': interleaved complex128
  int ta, tb, conja, conjb;
  int64_t m, n, k;
  const double* a; int64_t lda;
  const double* b; int64_t ldb;
  double* c; int64_t ldc;
  z64 alpha, beta;
};

cudaError_t launch_cgemm_exact(const CgemmArgs& g, cudaStream_t s);
cudaError_t launch_cgemm_combine(const CgemmArgs& g, const double* pr_h, const double* pr_l,
                                 const double* pi_h, const double* pi_l, cudaStream_t s);
cudaError_t launch_zgemm(const ZgemmArgs& g, cudaStream_t s);

// blocked Cholesky (dd_potrf.cu); column-major, every plane pair (hi, lo)
struct PotrfArgs {
  int64_t n, lda;
  int upper;
  int f64;                      // binary64 matrix (one plane; the *_lo pointers unused)
  double *a_hi, *a_lo;
  const double *d0_hi, *d0_lo;  // original diagonal
  double *dh, *dl;              // pivot dot products accumulated so far
  double *s_hi, *s_lo;          // upper: lower-stored accumulator S, ld = lds
  int64_t lds;
  double *t_hi, *t_lo;          // upper: the transposed panel U12^T
  const double *b_hi, *b_lo;    // lower: backup of the input (ld = n)
  double *rec_hi, *rec_lo;      // the current inner block's pivot reciprocals
  int fastacc;                  // fast / twosum modes: TwoSum accumulation in the panel rows
  int* info;                    // device: first failing pivot + 1, or 0
};

constexpr int kPotrfMaxNb = 64;       // diagonal block (shared memory)
constexpr int kPotrfMaxPanel = 256;   // columns per potrf_rows_kernel launch
cudaError_t launch_potrf_diag(const PotrfArgs& p, int64_t j0, int64_t j1, cudaStream_t s);
// rows [q0, q1) against the factored w-column block at j0 (dd_potrf.cu);
// pmask (w / 32 words of scratch, or null): check the block against the safe
// window once up front instead of per step
cudaError_t launch_potrf_rows(const PotrfArgs& p, int64_t j0, int w, int64_t q0, int64_t q1,
                              const double* ph, const double* pl, int64_t sr, int64_t sc,
                              const double* rh, const double* rl, unsigned* pmask, cudaStream_t s);
cudaError_t launch_potrf_blockupd(const PotrfArgs& p, int64_t i0, int64_t i1, int64_t j1,
                                  cudaStream_t s);
// fast modes: C(r, c) += sgn F(c, l) F(r, l), rows [r0, r1), columns [c0, c0
// + wd) with c <= r, l < kb <= 256 (dd_potrf.cu)
cudaError_t launch_potrf_lean_upd(const double* fh, const double* fl, int64_t ldf, int kb, double sgn,
                                  double* ch, double* cl, int64_t ldc, int64_t r0, int64_t r1,
                                  int64_t c0, int wd, const int* info, cudaStream_t s);
cudaError_t launch_potrf_transpose(const PotrfArgs& p, int64_t j0, int64_t j1, int nb,
                                   int64_t rows, cudaStream_t s);
cudaError_t launch_potrf_restore(const PotrfArgs& p, cudaStream_t s);

// triangular solve (dd_trsm.cu): the recurrence in production order over
// p x q work planes W (ld = ldw) with coefficients T (p x p, ld = ldt)
struct TrsmArgs {
  int64_t p, q;
  int left, rev, unit, fin_rec;
  int f64;                      // binary64 (one plane; the *_lo pointers unused)
  double *w_hi, *w_lo; int64_t ldw;
  double *t_hi, *t_lo; int64_t ldt;
  double *d_hi, *d_lo;
  double *r_hi, *r_lo;          // 1 / A(s,s) per s (the R branches; the L ones in fast modes)
  int rec_fast;                 // fast modes: L branches finish with the reciprocal too
};

cudaError_t launch_trsm_pack(const TrsmArgs& t, const double* bh, const double* bl, int64_t ldb,
                             int scale, dd alpha, cudaStream_t s);
cudaError_t launch_trsm_unpack(const TrsmArgs& t, double* bh, double* bl, int64_t ldb, int scale,
                               dd alpha, cudaStream_t s);
cudaError_t launch_trsm_coef(const TrsmArgs& t, const double* ah, const double* al, int64_t lda,
                             int trans, cudaStream_t s);
cudaError_t launch_trsm_block(const TrsmArgs& t, int64_t r0, int nb, cudaStream_t s);
cudaError_t launch_trsm_rev(const TrsmArgs& t, cudaStream_t s);

// LU with partial pivoting (dd_getrf.cu)
struct PermBuf {                // a composed row interchange (laswp)
  long long* rows;              // touched rows (512)
  int* src;                     // row t receives the old content of rows[src[t]]
  int* n;                       // number of touched rows
};

struct GetrfArgs {
  int64_t m, n, mn, lda;
  int f64;                      // binary64 (one plane; a_lo unused)
  double *a_hi, *a_lo;
  long long* ipiv;              // 1-based pivot rows (device)
  long long* swap;              // interchange actually applied at step j (j = none)
  int* info;
  double *part_ah, *part_al, *part_h, *part_l;   // per-CTA pivot candidates
  long long* part_idx;
  int* part_nan;
  unsigned* bar;                // grid barrier counter
  double* rowbuf;               // candidate rows and row j, two parities (dd_getrf.cu)
  int fastacc;                  // fast / twosum modes: TwoSum accumulation in the U12 kernel
};

int getrf_max_panel_ctas();
cudaError_t launch_getrf_panel(const GetrfArgs& g, int64_t j0, int nb, cudaStream_t s);
constexpr int kPermBufBytes = 512 * (8 + 4) + 64;     // one PermBuf's storage
cudaError_t launch_getrf_laswp(const GetrfArgs& g, int64_t j0, int64_t j1, int64_t c0, int64_t c1,
                               cudaStream_t s, int reverse, const PermBuf& pb);
constexpr int kPermStepsMax = 256;                     // steps one composition may hold
cudaError_t launch_getrf_compose(const GetrfArgs& g, int64_t j0, int64_t j1, int reverse,
                                 const PermBuf& pb, cudaStream_t s);
cudaError_t launch_getrf_apply(const GetrfArgs& g, const PermBuf& pb, int64_t nsteps, int64_t c0,
                               int64_t c1, cudaStream_t s);
cudaError_t launch_getrf_trsm(const GetrfArgs& g, int64_t j0, int nb, int64_t c0, int64_t c1,
                              cudaStream_t s);
// A(r, c) += L(r, l) (-U(l, c)), rows [r0, r1), columns [c0, c1), l in [l0,
// l0 + kb), kb <= 64: the inner panels' update (dd_getrf.cu)
cudaError_t launch_getrf_inner_upd(const GetrfArgs& g, int64_t l0, int kb, int64_t r0, int64_t r1,
                                   int64_t c0, int64_t c1, cudaStream_t s);
// U12 of rows [j0, j0 + w) (w <= 256), columns [c0, c1), in one launch;
// lmask: 8 words of scratch (dd_getrf.cu)
cudaError_t launch_getrf_u12(const GetrfArgs& g, int64_t j0, int w, int64_t c0, int64_t c1,
                             unsigned* lmask, cudaStream_t s);
// bit r % 32 of mask[r / 32]: row r of the w x w block P (P(r, c) at
// ph[r * sr + c * sc], c < r) is inside the safe window (dd_potrf.cu)
cudaError_t launch_window_mask(const double* ph, const double* pl, int w, int64_t sr, int64_t sc,
                               unsigned* mask, cudaStream_t s);

}  // namespace ddb
