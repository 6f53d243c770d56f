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
// window (tiled kernels run), nonzero = some value outside it (non-finite,
// |x| > 2**301, or a nonzero hi word below 2**-300): the tiled kernels exit
// and the reference-semantics kernel runs instead.
enum RouteFlag { ROUTE_SAFE = 0, ROUTE_UNSAFE = 1 };

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
};

// Which kernel should run, decided on the device by the prescan flag.
enum Gate { GATE_ALWAYS = 0, GATE_IF_SAFE = 1, GATE_IF_UNSAFE = 2 };

cudaError_t launch_prescan(const GemmArgs& g, int alg, int* row_exp, int* col_exp,
                           int* flag, cudaStream_t s, int* nlaunch);
cudaError_t launch_reference(const GemmArgs& g, const int* flag, int gate, cudaStream_t s,
                             int* nlaunch);
cudaError_t launch_tiled(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch);
size_t bound_workspace_bytes(const GemmArgs& g);
int choose_ksplit(const GemmArgs& g, int alg, int64_t* kchunk);
cudaError_t launch_splitk_reduce(const GemmArgs& g, int splits, const int* flag, cudaStream_t s,
                                 int* nlaunch);
cudaError_t launch_bound(const GemmArgs& g, const int* row_exp, const int* col_exp, void* ws,
                         float* bound, cudaStream_t s, int* nlaunch, const char** what);
cudaError_t launch_cross_dgemm(const GemmArgs& g, double* x, cudaStream_t s);

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
  double *rec_hi, *rec_lo;      // the current block's pivot reciprocals
  int* info;                    // device: first failing pivot + 1, or 0
};

constexpr int kPotrfMaxNb = 64;
cudaError_t launch_potrf_diag(const PotrfArgs& p, int64_t j0, int64_t j1, cudaStream_t s);
cudaError_t launch_potrf_panel(const PotrfArgs& p, int64_t j0, int nb, int64_t rows,
                               cudaStream_t s);
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

}  // namespace ddb
