/*
 * ddblas.h -- C ABI of the B200-native double-double Rgemm / Rsyrk.
 *
 * Drop-in for the reference's dd path (arXiv 2109.13406, MPLAPACK; Python
 * reference package "mpkit"):
 *
 *   ddb_rgemm  replaces  mpkit.mpblas.Rgemm(transa, transb, m, n, k, alpha,
 *                        a, lda, b, ldb, beta, c, ldc)
 *                        /root/reference/pkg/src/mpkit/mpblas/level23.py:180-198
 *   ddb_rsyrk  replaces  mpkit.mpblas.Rsyrk(uplo, trans, n, k, alpha, a, lda,
 *                        beta, c, ldc)            level23.py:226-285
 *
 * A dd matrix is two float64 planes (hi, lo) in the reference's column-major
 * flat layout: element (i, j) at index i + j*ld (mpblas/matrix.py:1-7,
 * elem.py DDBackend store = (hi, lo)).  alpha / beta are (hi, lo) pairs
 * (ddarith.DDouble).  Flags are single characters, case-insensitive,
 * 'C' == 'T' for real data (level23.py:23-26, :116-117).
 *
 * Return value: DDB_OK (0); a positive reference argument index (the
 * BlasError.index the reference would raise, level23.py:84-96 / :233-239);
 * or a negative DDB_E* code with text in ddb_last_error().
 *
 * Device entry points (ddb_rgemm / ddb_rsyrk) take DEVICE pointers and run
 * asynchronously on `stream` (a cudaStream_t, NULL = legacy default stream).
 * Host entry points (*_host) take HOST pointers, stage through device
 * memory, and return after C has been copied back (synchronous).
 * Thread safety: reentrant; concurrent calls on distinct streams are safe.
 */
#ifndef DDBLAS_H
#define DDBLAS_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DDB_VERSION 130   /* 1.3: per-element routing, no library GEMMs, diagnostics */

#define DDB_OK 0
#define DDB_EINVAL (-1)   /* bad mode / internal argument */
#define DDB_ECUDA (-2)    /* CUDA runtime failure */
#define DDB_ENOMEM (-3)   /* device allocation failed */

/* mode: DDB_MODE_EXACT     bit-identical to the reference (29 FP64 instr / MAC)
 *       DDB_MODE_FAST      certified-anchor accumulation: hi*hi in the
 *                          hand-written DFMA kernel (4.75 FP64 instr / MAC) + the
 *                          cross terms A_lo*B_hi + A_hi*B_lo on a hand-written
 *                          DMMA kernel (2 / MAC) + a bf16 tcgen05 bound GEMM
 *                          (k >= 1024; shallower calls: 7.5 / MAC in one
 *                          kernel).  Error <= c*k*2^-104*(|alpha| sum|a*b| +
 *                          |beta||c|), c = 4, for every input in the safe
 *                          window: elements whose row / column exponent
 *                          spreads exceed 112 - ceil(log2 k) and calls with
 *                          k > 2^16 take the TwoSum accumulation instead,
 *                          elements whose op(A) row / op(B) column holds a
 *                          value outside the window (inf, nan, |x| >= 2^301,
 *                          0 < |hi| < 2^-300, non-normalised dd) take the
 *                          reference-semantics kernel (bit-exact there).
 *                          Not bitwise equal to the reference elsewhere.
 *       DDB_MODE_REFERENCE one thread per element, checked arithmetic (debug)
 *       DDB_MODE_TWOSUM    TwoSum dd accumulation, same bound, no bound GEMM
 *                          (12.4 FP64 instr / MAC) */
#define DDB_MODE_EXACT 0
#define DDB_MODE_FAST 1
#define DDB_MODE_REFERENCE 2
#define DDB_MODE_TWOSUM 3

int ddb_rgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
              double alpha_hi, double alpha_lo,
              const double* a_hi, const double* a_lo, int64_t lda,
              const double* b_hi, const double* b_lo, int64_t ldb,
              double beta_hi, double beta_lo,
              double* c_hi, double* c_lo, int64_t ldc,
              int mode, void* stream);

int ddb_rsyrk(char uplo, char trans, int64_t n, int64_t k,
              double alpha_hi, double alpha_lo,
              const double* a_hi, const double* a_lo, int64_t lda,
              double beta_hi, double beta_lo,
              double* c_hi, double* c_lo, int64_t ldc,
              int mode, void* stream);

int ddb_rgemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   const double* b_hi, const double* b_lo, int64_t ldb,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc,
                   int mode, void* stream);

int ddb_rsyrk_host(char uplo, char trans, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc,
                   int mode, void* stream);

/* Binary64 precision (the reference's 'f64' Matrix, one plane per matrix):
 * the same routines over the reference's F64 backend (elem.py:149-197),
 * bit-identical for every input.  Same argument indices and early exits. */
int ddb_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
              const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
              double* c, int64_t ldc, void* stream);
int ddb_dsyrk(char uplo, char trans, int64_t n, int64_t k, double alpha, const double* a,
              int64_t lda, double beta, double* c, int64_t ldc, void* stream);
int ddb_dgemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                   const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                   double* c, int64_t ldc, void* stream);
int ddb_dsyrk_host(char uplo, char trans, int64_t n, int64_t k, double alpha, const double* a,
                   int64_t lda, double beta, double* c, int64_t ldc, void* stream);

/* Complex GEMM: mpkit.mpblas.Cgemm (level23.py:201-221).  'cdd' operands are
 * four planes {re_hi, re_lo, im_hi, im_lo} (arrays of 4 pointers), alpha /
 * beta four doubles in the same order; 'C' flags conjugate.  Modes as for
 * ddb_rgemm (exact = the reference's CDD backend bit for bit, fast = four
 * real fast-mode GEMMs + a complex dd epilogue).  'c64' (ddb_zgemm) takes
 * interleaved complex128 arrays and alpha / beta as {re, im}; bit-exact. */
int ddb_cgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double* alpha,
              const double* const* a, int64_t lda, const double* const* b, int64_t ldb,
              const double* beta, double* const* c, int64_t ldc, int mode, void* stream);
int ddb_cgemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k,
                   const double* alpha, const double* const* a, int64_t lda,
                   const double* const* b, int64_t ldb, const double* beta, double* const* c,
                   int64_t ldc, int mode, void* stream);
int ddb_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double* alpha,
              const double* a, int64_t lda, const double* b, int64_t ldb, const double* beta,
              double* c, int64_t ldc, void* stream);
int ddb_zgemm_host(char transa, char transb, int64_t m, int64_t n, int64_t k, const double* alpha,
                   const double* a, int64_t lda, const double* b, int64_t ldb, const double* beta,
                   double* c, int64_t ldc, void* stream);

/* Triangular solve: mpkit.mpblas.Rtrsm (level23.py:288-380), dd, X over B.
 * side 'L': op(A) X = alpha B, 'R': X op(A) = alpha B; uplo, transa
 * ('N', 'T', 'C'), diag ('U' unit, 'N').  Exact / reference modes are
 * bit-identical to the reference (blocked where the reference's per-element
 * order allows it; L,T,L and R,N,L run one sequential recurrence per
 * vector); fast / twosum use the blocked order with fast-mode GEMM updates.
 * Returns 0 / the reference argument index (1-6, 9, 11) / DDB_E*. */
int ddb_rtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
              double alpha_hi, double alpha_lo, const double* a_hi, const double* a_lo,
              int64_t lda, double* b_hi, double* b_lo, int64_t ldb, int mode, void* stream);
int ddb_rtrsm_host(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                   double alpha_hi, double alpha_lo, const double* a_hi, const double* a_lo,
                   int64_t lda, double* b_hi, double* b_lo, int64_t ldb, int mode, void* stream);

/* LU with partial pivoting: mpkit.mplapack.Rgetrf (mplapack/lu.py:74-114),
 * dd, in place (A = P L U, unit-lower L below the diagonal).  ipiv: host
 * array of min(m, n) 1-based pivot rows; *info (host) = 0 or the first
 * column with an exactly zero pivot (the factorization still completes).
 * Blocked (width $DDB_GETRF_NB, default 64): cooperative panel kernel, row
 * interchanges, unit-lower TRSM and an Rgemm trailing update in `mode`;
 * exact mode is bit-identical to the reference.  Returns 0 / the reference
 * argument index (1 m, 2 n, 4 lda) / DDB_E*.  Synchronises `stream`. */
int ddb_rgetrf(int64_t m, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t* ipiv,
               int* info, int mode, void* stream);
int ddb_rgetrf_host(int64_t m, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t* ipiv,
                    int* info, int mode, void* stream);

/* Solve with an LU factorization: mpkit.mplapack.Rgetrs (lu.py:117-145):
 * op(A) X = B in place in B (n x nrhs), A and ipiv (host, n 1-based pivots)
 * from ddb_rgetrf.  trans 'N': interchanges, then Rtrsm L,L,N,U and
 * L,U,N,N; 'T' / 'C': Rtrsm L,U,T,N and L,L,T,U, then the interchanges in
 * reverse.  Bit-identical to the reference in exact mode.  Returns 0 / the
 * reference argument index (1 trans, 2 n, 3 nrhs, 5 lda, 8 ldb) / DDB_E*. */
int ddb_rgetrs(char trans, int64_t n, int64_t nrhs, const double* a_hi, const double* a_lo,
               int64_t lda, const int64_t* ipiv, double* b_hi, double* b_lo, int64_t ldb,
               int mode, void* stream);
int ddb_rgetrs_host(char trans, int64_t n, int64_t nrhs, const double* a_hi, const double* a_lo,
                    int64_t lda, const int64_t* ipiv, double* b_hi, double* b_lo, int64_t ldb,
                    int mode, void* stream);

/* Cholesky: mpkit.mplapack.Rpotrf (mplapack/chol.py:21-65), dd, in place.
 * uplo 'L': A = L L^T, 'U': A = U^T U; only that triangle is read / written.
 * Blocked right-looking, two levels: outer block width nb (<= 0 = default
 * 256 or $DDB_POTRF_NB), inner width min(nb, 64); the trailing updates are
 * ddb_rsyrk / ddb_rgemm calls in `mode`, overlapped with the next panel; in
 * exact mode the factor is bit-identical to the reference's unblocked
 * order for operands inside the safe window.  *info (host int) = 0, or
 * j + 1 for the first pivot that is NaN or <= 0, whose value is left in
 * A(j, j) with the later columns as the reference leaves them (chol.py:44).
 * Returns 0 / the reference argument index (1 uplo, 2 n, 4 lda) / DDB_E*.
 * Synchronises `stream` (info is a host value). */
int ddb_rpotrf(char uplo, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t nb,
               int mode, void* stream, int* info);
int ddb_rpotrf_host(char uplo, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t nb,
                    int mode, void* stream, int* info);

/* Single-process multi-GPU: operands and result on
 * devices[0]; device i computes a column slab of C (Rgemm: equal slabs;
 * Rsyrk: slabs of equal triangle area, each an Rsyrk diagonal block + an
 * Rgemm rectangle) after peer copies of op(A) and its slab; slabs come back
 * by peer copy.  Exact mode is bitwise equal to ddb_rgemm / ddb_rsyrk.  A
 * device id may repeat.  Synchronous; returns as ddb_rgemm / ddb_rsyrk
 * (DDB_EINVAL for an empty device list). */
int ddb_rgemm_mgpu(char transa, char transb, int64_t m, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   const double* b_hi, const double* b_lo, int64_t ldb,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc, int mode, int ndev,
                   const int* devices);
int ddb_rsyrk_mgpu(char uplo, char trans, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc, int mode, int ndev,
                   const int* devices);

/* The LAPACK consumers on the reference's binary64 ('f64') Matrix: one
 * plane, the F64 backend's IEEE operations in the reference's order
 * (bit-identical; no mode).  Arguments and returns as the dd versions. */
int ddb_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
              const double* a, int64_t lda, double* b, int64_t ldb, void* stream);
int ddb_dtrsm_host(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                   double alpha, const double* a, int64_t lda, double* b, int64_t ldb,
                   void* stream);
int ddb_dgetrf(int64_t m, int64_t n, double* a, int64_t lda, int64_t* ipiv, int* info,
               void* stream);
int ddb_dgetrf_host(int64_t m, int64_t n, double* a, int64_t lda, int64_t* ipiv, int* info,
                    void* stream);
int ddb_dgetrs(char trans, int64_t n, int64_t nrhs, const double* a, int64_t lda,
               const int64_t* ipiv, double* b, int64_t ldb, void* stream);
int ddb_dgetrs_host(char trans, int64_t n, int64_t nrhs, const double* a, int64_t lda,
                    const int64_t* ipiv, double* b, int64_t ldb, void* stream);
int ddb_dpotrf(char uplo, int64_t n, double* a, int64_t lda, int64_t nb, void* stream, int* info);
int ddb_dpotrf_host(char uplo, int64_t n, double* a, int64_t lda, int64_t nb, void* stream,
                    int* info);

/* Argument checks alone (no device work): reference index or 0. */
int ddb_rgemm_validate(char transa, char transb, int64_t m, int64_t n, int64_t k,
                       int64_t lda, int64_t ldb, int64_t ldc);
int ddb_rsyrk_validate(char uplo, char trans, int64_t n, int64_t k, int64_t lda, int64_t ldc);
int ddb_rpotrf_validate(char uplo, int64_t n, int64_t lda);
int ddb_rgetrf_validate(int64_t m, int64_t n, int64_t lda);
int ddb_rgetrs_validate(char trans, int64_t n, int64_t nrhs, int64_t lda, int64_t ldb);
int ddb_rtrsm_validate(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                       int64_t lda, int64_t ldb);

const char* ddb_last_error(void);
int ddb_version(void);
/* Number of kernels this library has launched in this process. */
long long ddb_launch_count(void);
/* Route of this thread's last call when DDB_DEBUG_SYNC=1 (0 exact tiled,
 * 1 fast tiled, 2 reference-semantics kernel, 3 twosum tiled, 4 f64 tiled),
 * else -1. */
int ddb_last_route(void);

/* Diagnostic: FP64 FMA throughput of the current GPU in FLOP/s (FMA = 2),
 * measured with a DFMA burn kernel on `stream` (synchronous; ~10 ms). The
 * bench's roofline denominator. */
double ddb_fp64_peak_probe(void* stream);

/* Page-lock / release an existing host range (portable), so the *_host entry
 * points copy from / to it by DMA; used for host buffers shared between
 * processes (one process per GPU staging its own slab, parallel.py). */
int ddb_host_register(void* ptr, int64_t bytes);
int ddb_host_unregister(void* ptr);

/* Diagnostic: the split algorithm's cross terms alone (device pointers,
 * asynchronous on `stream`): X (m x n, ld = m) = A_lo*B_hi + A_hi*B_lo, NN,
 * on the hand-written DMMA kernel.  Planes 16-byte aligned, lda / ldb even.
 * tri: 0 all tiles, 1 / 2 only tiles meeting the upper / lower triangle. */
int ddb_cross_terms(int64_t m, int64_t n, int64_t k, const double* a_hi, const double* a_lo,
                    int64_t lda, const double* b_hi, const double* b_lo, int64_t ldb, double* x,
                    int tri, void* stream);

/* Diagnostic: the fast mode's certified magnitude bound alone (device
 * pointers, synchronous).  row_exp (m) / col_exp (n): biased exponent maxima
 * of op(A) rows / op(B) columns; abf (m x kp) / bbf (n x kp), kp = k rounded
 * up to 8, may be NULL: |hi| * 2^(1022 - exp) rounded up to bf16, K-major;
 * s_out (m x n, ld = m): abf * bbf^T in fp32 on the tcgen05 kernel. */
int ddb_abs_bound(char transa, char transb, int64_t m, int64_t n, int64_t k,
                  const double* a_hi, int64_t lda, const double* b_hi, int64_t ldb,
                  int* row_exp, int* col_exp, float* s_out, uint16_t* abf, uint16_t* bbf,
                  void* stream);

#ifdef __cplusplus
}
#endif

#endif /* DDBLAS_H */
