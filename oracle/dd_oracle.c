/*
 * dd_oracle.c -- CPU restatement of the reference dd Rgemm / Rsyrk.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path:
 * only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
 * --impl reference leg may load it.  The product path never calls it.
 *
 * It restates, element by element, what the reference package computes
 * (/root/reference/pkg/src/mpkit), so a GPU result in `exact` mode can be
 * compared bit for bit:
 *
 *   two_sum            elem.py:32-35      (ddarith.py:37-41)
 *   quick_two_sum      elem.py:38-40      (ddarith.py:44-47)
 *   two_prod (Dekker)  elem.py:43-51      (ddarith.py:50-62), splitter elem.py:25
 *   add2 (accurate)    elem.py:54-66      -- vectorised variant: only s0 is checked
 *   mul2               elem.py:69-78      -- vectorised variant: (p, e) checked
 *   Rgemm order        level23.py:107-149 (_gemm_core), :163-177 (_scale_full,
 *                      _combine), :180-198 (Rgemm validation / early exit)
 *   Rsyrk order        level23.py:226-285
 *
 * Validation returns the reference argument index (level23.py:84-96,
 * :233-239); 0 means success.
 *
 * Parity of this restatement with the reference is pinned by
 * tests/test_oracle.py against tests/golden/ (npz fixtures), which
 * oracle/gen_golden.py produced by running the reference itself.
 *
 * Build: see oracle/Makefile (-ffp-contract=off: no FMA contraction).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define SPLITTER 134217729.0 /* 2**27 + 1, elem.py:25 */

typedef struct { double h, l; } dd;

#if defined(__GNUC__) && !defined(__clang__)
#define CLONES __attribute__((target_clones("avx512f", "avx2", "default")))
#else
#define CLONES
#endif

static inline void two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    double bb = ss - a;
    *e = (a - (ss - bb)) + (b - bb);
    *s = ss;
}

static inline void quick_two_sum(double a, double b, double *s, double *e) {
    double ss = a + b;
    *e = b - (ss - a);
    *s = ss;
}

static inline void two_prod(double a, double b, double *p, double *e) {
    double pp = a * b;
    double t = SPLITTER * a;
    double ah = t - (t - a);
    double al = a - ah;
    t = SPLITTER * b;
    double bh = t - (t - b);
    double bl = b - bh;
    *e = (((ah * bh - pp) + ah * bl) + al * bh) + al * bl;
    *p = pp;
}

/* elem.py:54-66 */
static inline dd add2(dd x, dd y) {
    double s0 = x.h + y.h;
    double sh, sl, th, tl;
    two_sum(x.h, y.h, &sh, &sl);
    two_sum(x.l, y.l, &th, &tl);
    sl = sl + th;
    quick_two_sum(sh, sl, &sh, &sl);
    sl = sl + tl;
    quick_two_sum(sh, sl, &sh, &sl);
    dd r;
    if (!isfinite(s0)) { r.h = s0; r.l = 0.0; }
    else { r.h = sh; r.l = sl; }
    return r;
}

/* elem.py:69-78 */
static inline dd mul2(dd x, dd y) {
    double p, e;
    two_prod(x.h, y.h, &p, &e);
    int bad = !(isfinite(p) && isfinite(e));
    e = e + (x.h * y.l + x.l * y.h);
    double rh, rl;
    quick_two_sum(p, e, &rh, &rl);
    dd r;
    if (bad) { r.h = p; r.l = 0.0; }
    else { r.h = rh; r.l = rl; }
    return r;
}

static inline int is_zero(dd v) { return v.h == 0.0 && v.l == 0.0; }     /* DDouble.__bool__ */
static inline int is_one(dd v) { return v.h == 1.0 && v.l == 0.0; }      /* _cmp2 == 0 vs 1 */

static int upflag(char c) { return (c >= 'a' && c <= 'z') ? c - 32 : c; }

/* level23.py:84-96 */
int oracle_gemm_validate(char transa, char transb, int64_t m, int64_t n, int64_t k,
                         int64_t lda, int64_t ldb, int64_t ldc) {
    int ta = upflag(transa), tb = upflag(transb);
    if (ta != 'N' && ta != 'T' && ta != 'C') return 1;
    if (tb != 'N' && tb != 'T' && tb != 'C') return 2;
    if (m < 0) return 3;
    if (n < 0) return 4;
    if (k < 0) return 5;
    int64_t nrowa = ta == 'N' ? m : k;
    int64_t nrowb = tb == 'N' ? k : n;
    if (lda < (nrowa > 1 ? nrowa : 1)) return 8;
    if (ldb < (nrowb > 1 ? nrowb : 1)) return 10;
    if (ldc < (m > 1 ? m : 1)) return 13;
    return 0;
}

/* level23.py:233-239 */
int oracle_syrk_validate(char uplo, char trans, int64_t n, int64_t k, int64_t lda, int64_t ldc) {
    int u = upflag(uplo), t = upflag(trans);
    if (u != 'U' && u != 'L') return 1;
    if (t != 'N' && t != 'T' && t != 'C') return 2;
    if (n < 0) return 3;
    if (k < 0) return 4;
    int64_t nrowa = t == 'N' ? n : k;
    if (lda < (nrowa > 1 ? nrowa : 1)) return 7;
    if (ldc < (n > 1 ? n : 1)) return 10;
    return 0;
}

static inline dd ld_(const double *h, const double *l, int64_t idx) {
    dd v; v.h = h[idx]; v.l = l[idx]; return v;
}

/* beta rule of _scale_full (level23.py:163-169) applied to one element */
static inline dd scale_beta(dd beta, dd c) {
    if (is_zero(beta)) { dd z = {0.0, 0.0}; return z; }
    if (is_one(beta)) return c;
    return mul2(beta, c);
}

/* One column j of NN / NT Rgemm (level23.py:120-125, :134-140).  t is a
 * k-scratch; the per-element order is exactly c = add2(c, mul2(A(i,l), t_l))
 * for l ascending after the beta rule. */
CLONES
static void gemm_col_notrans_a(int tb, int64_t m, int64_t k, dd alpha,
                               const double *Ah, const double *Al, int64_t lda,
                               const double *Bh, const double *Bl, int64_t ldb,
                               dd beta, double *Ch, double *Cl, int64_t ldc,
                               int64_t j, dd *t, dd *c) {
    for (int64_t l = 0; l < k; ++l) {
        int64_t bidx = tb == 'N' ? l + j * ldb : j + l * ldb;
        t[l] = mul2(alpha, ld_(Bh, Bl, bidx));
    }
    for (int64_t i = 0; i < m; ++i) c[i] = scale_beta(beta, ld_(Ch, Cl, i + j * ldc));
    for (int64_t l = 0; l < k; ++l) {
        const double *ah = Ah + l * lda, *al = Al + l * lda;
        dd tl = t[l];
        for (int64_t i = 0; i < m; ++i) {
            dd a; a.h = ah[i]; a.l = al[i];
            c[i] = add2(c[i], mul2(a, tl));
        }
    }
    for (int64_t i = 0; i < m; ++i) { Ch[i + j * ldc] = c[i].h; Cl[i + j * ldc] = c[i].l; }
}

/* _combine (level23.py:172-177) */
static inline dd combine(dd alpha, dd acc, dd beta, dd c0) {
    dd at = mul2(alpha, acc);
    if (is_zero(beta)) return at;
    return add2(at, mul2(beta, c0));
}

/* One column j of TN / TT Rgemm (level23.py:126-133, :141-149). */
CLONES
static void gemm_col_trans_a(int tb, int64_t m, int64_t k, dd alpha,
                             const double *Ah, const double *Al, int64_t lda,
                             const double *Bh, const double *Bl, int64_t ldb,
                             dd beta, double *Ch, double *Cl, int64_t ldc,
                             int64_t j, dd *t, dd *c) {
    for (int64_t l = 0; l < k; ++l) {
        int64_t bidx = tb == 'N' ? l + j * ldb : j + l * ldb;
        t[l] = ld_(Bh, Bl, bidx);
    }
    for (int64_t i = 0; i < m; ++i) {
        const double *ah = Ah + i * lda, *al = Al + i * lda;
        dd acc = {0.0, 0.0};
        for (int64_t l = 0; l < k; ++l) {
            dd a; a.h = ah[l]; a.l = al[l];
            acc = add2(acc, mul2(a, t[l]));
        }
        c[i] = combine(alpha, acc, beta, ld_(Ch, Cl, i + j * ldc));
    }
    for (int64_t i = 0; i < m; ++i) { Ch[i + j * ldc] = c[i].h; Cl[i + j * ldc] = c[i].l; }
}

/* ---- host threading: columns of C are independent (the disjoint-panel
 * argument of parallel.py:102-125), so workers pull column indices from an
 * atomic counter.  Results do not depend on the thread count. */
#include <pthread.h>
#include <unistd.h>

typedef struct {
    void (*col)(void *ctx, int64_t j, dd *t, dd *c);
    void *ctx;
    int64_t n, k, m;
    int64_t next;       /* atomic */
    int err;            /* atomic */
} pool_job;

static void *pool_worker(void *arg) {
    pool_job *job = (pool_job *)arg;
    dd *t = (dd *)malloc(sizeof(dd) * (size_t)(job->k > 0 ? job->k : 1));
    dd *c = (dd *)malloc(sizeof(dd) * (size_t)(job->m > 0 ? job->m : 1));
    if (!t || !c) {
        __atomic_store_n(&job->err, -1, __ATOMIC_SEQ_CST);
    } else {
        for (;;) {
            int64_t j = __atomic_fetch_add(&job->next, 1, __ATOMIC_SEQ_CST);
            if (j >= job->n) break;
            job->col(job->ctx, j, t, c);
        }
    }
    free(t);
    free(c);
    return NULL;
}

int oracle_max_threads(void) {
    long v = sysconf(_SC_NPROCESSORS_ONLN);
    return v > 0 ? (int)v : 1;
}

static int run_columns(void (*col)(void *, int64_t, dd *, dd *), void *ctx,
                       int64_t n, int64_t k, int64_t m, int nthreads) {
    pool_job job = {col, ctx, n, k, m, 0, 0};
    if (nthreads <= 0) nthreads = oracle_max_threads();
    if (nthreads > n) nthreads = (int)(n > 0 ? n : 1);
    if (nthreads <= 1) { pool_worker(&job); return job.err; }
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    if (!th) return -1;
    int started = 0;
    for (int i = 0; i < nthreads; ++i)
        if (pthread_create(&th[i], NULL, pool_worker, &job) == 0) ++started;
    if (started == 0) pool_worker(&job);
    for (int i = 0; i < started; ++i) pthread_join(th[i], NULL);
    free(th);
    return job.err;
}

typedef struct {
    int ta, tb, up, tn;
    int64_t m, k;
    dd alpha, beta;
    const double *Ah, *Al, *Bh, *Bl;
    double *Ch, *Cl;
    int64_t lda, ldb, ldc, n;
} call_ctx;

static void gemm_col(void *p, int64_t j, dd *t, dd *c) {
    call_ctx *x = (call_ctx *)p;
    if (x->ta == 'N')
        gemm_col_notrans_a(x->tb, x->m, x->k, x->alpha, x->Ah, x->Al, x->lda, x->Bh, x->Bl,
                           x->ldb, x->beta, x->Ch, x->Cl, x->ldc, j, t, c);
    else
        gemm_col_trans_a(x->tb, x->m, x->k, x->alpha, x->Ah, x->Al, x->lda, x->Bh, x->Bl,
                         x->ldb, x->beta, x->Ch, x->Cl, x->ldc, j, t, c);
}

/* level23.py:180-198 + _gemm_core. */
int oracle_rgemm(char transa, char transb, int64_t m, int64_t n, int64_t k,
                 double alpha_hi, double alpha_lo,
                 const double *Ah, const double *Al, int64_t lda,
                 const double *Bh, const double *Bl, int64_t ldb,
                 double beta_hi, double beta_lo,
                 double *Ch, double *Cl, int64_t ldc, int nthreads) {
    int rc = oracle_gemm_validate(transa, transb, m, n, k, lda, ldb, ldc);
    if (rc) return rc;
    dd alpha = {alpha_hi, alpha_lo}, beta = {beta_hi, beta_lo};
    if (m == 0 || n == 0 || ((is_zero(alpha) || k == 0) && is_one(beta))) return 0;
    if (is_zero(alpha)) {                       /* _gemm_core :110-115 */
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) {
                dd c = scale_beta(beta, ld_(Ch, Cl, i + j * ldc));
                Ch[i + j * ldc] = c.h; Cl[i + j * ldc] = c.l;
            }
        return 0;
    }
    call_ctx x = {upflag(transa), upflag(transb), 0, 0, m, k, alpha, beta,
                  Ah, Al, Bh, Bl, Ch, Cl, lda, ldb, ldc, n};
    return run_columns(gemm_col, &x, n, k, m, nthreads);
}

static void syrk_col(void *p, int64_t j, dd *t, dd *cs) {
    call_ctx *x = (call_ctx *)p;
    (void)cs;
    const double *Ah = x->Ah, *Al = x->Al;
    double *Ch = x->Ch, *Cl = x->Cl;
    int64_t lda = x->lda, ldc = x->ldc, k = x->k;
    int64_t i0 = x->up ? 0 : j, i1 = x->up ? j + 1 : x->n;
    if (is_zero(x->alpha)) {                    /* _scale_masked, :247-249 */
        for (int64_t i = i0; i < i1; ++i) {
            dd c = scale_beta(x->beta, ld_(Ch, Cl, i + j * ldc));
            Ch[i + j * ldc] = c.h; Cl[i + j * ldc] = c.l;
        }
        return;
    }
    if (x->tn) {                                /* :250-258, == NT Rgemm with B = A */
        for (int64_t l = 0; l < k; ++l) t[l] = mul2(x->alpha, ld_(Ah, Al, j + l * lda));
        for (int64_t i = i0; i < i1; ++i) {
            dd c = scale_beta(x->beta, ld_(Ch, Cl, i + j * ldc));
            for (int64_t l = 0; l < k; ++l)
                c = add2(c, mul2(ld_(Ah, Al, i + l * lda), t[l]));
            Ch[i + j * ldc] = c.h; Cl[i + j * ldc] = c.l;
        }
    } else {                                    /* :259-270, == TN Rgemm with B = A */
        for (int64_t i = i0; i < i1; ++i) {
            dd acc = {0.0, 0.0};
            for (int64_t l = 0; l < k; ++l)
                acc = add2(acc, mul2(ld_(Ah, Al, l + i * lda), ld_(Ah, Al, l + j * lda)));
            dd c = combine(x->alpha, acc, x->beta, ld_(Ch, Cl, i + j * ldc));
            Ch[i + j * ldc] = c.h; Cl[i + j * ldc] = c.l;
        }
    }
}

/* level23.py:226-285.  Only (i, j) in the uplo triangle are written. */
int oracle_rsyrk(char uplo, char trans, int64_t n, int64_t k,
                 double alpha_hi, double alpha_lo,
                 const double *Ah, const double *Al, int64_t lda,
                 double beta_hi, double beta_lo,
                 double *Ch, double *Cl, int64_t ldc, int nthreads) {
    int rc = oracle_syrk_validate(uplo, trans, n, k, lda, ldc);
    if (rc) return rc;
    dd alpha = {alpha_hi, alpha_lo}, beta = {beta_hi, beta_lo};
    if (n == 0 || ((is_zero(alpha) || k == 0) && is_one(beta))) return 0;
    call_ctx x = {0, 0, upflag(uplo) == 'U', upflag(trans) == 'N', n, k, alpha, beta,
                  Ah, Al, NULL, NULL, Ch, Cl, lda, 0, ldc, n};
    return run_columns(syrk_col, &x, n, k, n, nthreads);
}

/* ---- binary64 precision: the same routines over the reference's F64
 * backend (elem.py:149-197: add / mul are plain numpy float64 ops), same loop
 * orders (level23.py:107-177, :226-285).  Single-threaded (test use). */

static inline double f64_beta_rule(double beta, double c) {       /* _scale_full */
    if (beta == 0.0) return 0.0;
    if (beta == 1.0) return c;
    return beta * c;
}

int oracle_dgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, double alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, double beta,
                 double *C, int64_t ldc) {
    int rc = oracle_gemm_validate(transa, transb, m, n, k, lda, ldb, ldc);
    if (rc) return rc;
    int ta = upflag(transa), tb = upflag(transb);
    if (m == 0 || n == 0 || ((alpha == 0.0 || k == 0) && beta == 1.0)) return 0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            double *c = &C[i + j * ldc];
            if (alpha == 0.0) { *c = f64_beta_rule(beta, *c); continue; }
            if (ta == 'N') {
                double acc = f64_beta_rule(beta, *c);
                for (int64_t l = 0; l < k; ++l) {
                    double t = alpha * (tb == 'N' ? B[l + j * ldb] : B[j + l * ldb]);
                    acc = acc + A[i + l * lda] * t;
                }
                *c = acc;
            } else {
                double acc = 0.0;
                for (int64_t l = 0; l < k; ++l)
                    acc = acc + A[l + i * lda] * (tb == 'N' ? B[l + j * ldb] : B[j + l * ldb]);
                double at = alpha * acc;
                *c = beta == 0.0 ? at : at + beta * *c;
            }
        }
    return 0;
}

int oracle_dsyrk(char uplo, char trans, int64_t n, int64_t k, double alpha, const double *A,
                 int64_t lda, double beta, double *C, int64_t ldc) {
    int rc = oracle_syrk_validate(uplo, trans, n, k, lda, ldc);
    if (rc) return rc;
    int up = upflag(uplo) == 'U', tn = upflag(trans) == 'N';
    if (n == 0 || ((alpha == 0.0 || k == 0) && beta == 1.0)) return 0;
    for (int64_t j = 0; j < n; ++j) {
        int64_t i0 = up ? 0 : j, i1 = up ? j + 1 : n;
        for (int64_t i = i0; i < i1; ++i) {
            double *c = &C[i + j * ldc];
            if (alpha == 0.0) { *c = f64_beta_rule(beta, *c); continue; }
            if (tn) {
                double acc = f64_beta_rule(beta, *c);
                for (int64_t l = 0; l < k; ++l) acc = acc + A[i + l * lda] * (alpha * A[j + l * lda]);
                *c = acc;
            } else {
                double acc = 0.0;
                for (int64_t l = 0; l < k; ++l) acc = acc + A[l + i * lda] * A[l + j * lda];
                double at = alpha * acc;
                *c = beta == 0.0 ? at : at + beta * *c;
            }
        }
    }
    return 0;
}

/* ---- complex precisions: Cgemm (level23.py:201-221 -> _gemm_core) --------
 * 'cdd': planes re_hi, re_lo, im_hi, im_lo; CDD backend ops (elem.py:324-377):
 *   add = (add2(re,re'), add2(im,im')), mul = (add2(mul2(xr,yr), -mul2(xi,yi)),
 *   add2(mul2(xr,yi), mul2(xi,yr))).  A DDComplex has no __bool__, so for 'cdd'
 *   `not alpha` / `not beta` are never true (beta == 0 multiplies C).
 * 'c64': interleaved complex128; C64 backend mul (elem.py:313-318) evaluated
 *   by numpy as re = (ac - bd) + (0*x - 0), im = 0 + (0 + x), x = ad + bc. */

typedef struct { dd re, im; } cdd_t;

static inline cdd_t c_add(cdd_t x, cdd_t y) { cdd_t r = {add2(x.re, y.re), add2(x.im, y.im)}; return r; }
static inline dd dneg(dd x) { dd r = {-x.h, -x.l}; return r; }
static inline cdd_t c_mul(cdd_t x, cdd_t y) {
    cdd_t r = {add2(mul2(x.re, y.re), dneg(mul2(x.im, y.im))), add2(mul2(x.re, y.im), mul2(x.im, y.re))};
    return r;
}
static inline cdd_t c_ld(const double *const *p, int64_t i) {
    cdd_t r = {{p[0][i], p[1][i]}, {p[2][i], p[3][i]}};
    return r;
}

int oracle_cgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double *alpha,
                 const double *const *A, int64_t lda, const double *const *B, int64_t ldb,
                 const double *beta, double *const *C, int64_t ldc) {
    int rc = oracle_gemm_validate(transa, transb, m, n, k, lda, ldb, ldc);
    if (rc) return rc;
    int ta = upflag(transa), tb = upflag(transb);
    int conja = ta == 'C', conjb = tb == 'C';
    cdd_t al = {{alpha[0], alpha[1]}, {alpha[2], alpha[3]}};
    cdd_t be = {{beta[0], beta[1]}, {beta[2], beta[3]}};
    int beta_one = is_one(be.re) && is_zero(be.im);
    if (m == 0 || n == 0 || (k == 0 && beta_one)) return 0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            int64_t ci = i + j * ldc;
            cdd_t c0 = c_ld((const double *const *)C, ci), out;
            if (ta == 'N') {
                cdd_t c = beta_one ? c0 : c_mul(be, c0);
                for (int64_t l = 0; l < k; ++l) {
                    cdd_t bv = c_ld(B, tb == 'N' ? l + j * ldb : j + l * ldb);
                    if (conjb) bv.im = dneg(bv.im);
                    c = c_add(c, c_mul(c_ld(A, i + l * lda), c_mul(al, bv)));
                }
                out = c;
            } else {
                cdd_t acc = {{0.0, 0.0}, {0.0, 0.0}};
                for (int64_t l = 0; l < k; ++l) {
                    cdd_t av = c_ld(A, l + i * lda), bv = c_ld(B, tb == 'N' ? l + j * ldb : j + l * ldb);
                    if (conja) av.im = dneg(av.im);
                    if (conjb) bv.im = dneg(bv.im);
                    acc = c_add(acc, c_mul(av, bv));
                }
                out = c_add(c_mul(al, acc), c_mul(be, c0));
            }
            C[0][ci] = out.re.h; C[1][ci] = out.re.l; C[2][ci] = out.im.h; C[3][ci] = out.im.l;
        }
    return 0;
}

typedef struct { double re, im; } z_t;
static inline z_t z_mul(z_t x, z_t y) {
    double r = x.re * y.re - x.im * y.im;
    double xi = x.re * y.im + x.im * y.re;
    z_t o = {r + (0.0 * xi - 0.0), 0.0 + (0.0 + xi)};
    return o;
}
static inline z_t z_add(z_t x, z_t y) { z_t o = {x.re + y.re, x.im + y.im}; return o; }

int oracle_zgemm(char transa, char transb, int64_t m, int64_t n, int64_t k, const double *alpha,
                 const double *A, int64_t lda, const double *B, int64_t ldb, const double *beta,
                 double *C, int64_t ldc) {
    int rc = oracle_gemm_validate(transa, transb, m, n, k, lda, ldb, ldc);
    if (rc) return rc;
    int ta = upflag(transa), tb = upflag(transb);
    int conja = ta == 'C', conjb = tb == 'C';
    z_t al = {alpha[0], alpha[1]}, be = {beta[0], beta[1]};
    int a0 = al.re == 0.0 && al.im == 0.0, b0 = be.re == 0.0 && be.im == 0.0;
    int b1 = be.re == 1.0 && be.im == 0.0;
    if (m == 0 || n == 0 || ((a0 || k == 0) && b1)) return 0;
    for (int64_t j = 0; j < n; ++j)
        for (int64_t i = 0; i < m; ++i) {
            int64_t ci = i + j * ldc;
            z_t c0 = {C[2 * ci], C[2 * ci + 1]}, out;
            if (a0) {
                if (b1) continue;
                if (b0) { out.re = 0.0; out.im = 0.0; } else out = z_mul(be, c0);
            } else if (ta == 'N') {
                z_t c = b1 ? c0 : (b0 ? (z_t){0.0, 0.0} : z_mul(be, c0));
                for (int64_t l = 0; l < k; ++l) {
                    int64_t bi = tb == 'N' ? l + j * ldb : j + l * ldb;
                    z_t bv = {B[2 * bi], B[2 * bi + 1]};
                    if (conjb) bv.im = -bv.im;
                    int64_t ai = i + l * lda;
                    z_t av = {A[2 * ai], A[2 * ai + 1]};
                    c = z_add(c, z_mul(av, z_mul(al, bv)));
                }
                out = c;
            } else {
                z_t acc = {0.0, 0.0};
                for (int64_t l = 0; l < k; ++l) {
                    int64_t bi = tb == 'N' ? l + j * ldb : j + l * ldb, ai = l + i * lda;
                    z_t av = {A[2 * ai], A[2 * ai + 1]}, bv = {B[2 * bi], B[2 * bi + 1]};
                    if (conja) av.im = -av.im;
                    if (conjb) bv.im = -bv.im;
                    acc = z_add(acc, z_mul(av, bv));
                }
                z_t at = z_mul(al, acc);
                out = b0 ? at : z_add(at, z_mul(be, c0));
            }
            C[2 * ci] = out.re; C[2 * ci + 1] = out.im;
        }
    return 0;
}

/* Scalar EFT entry points, for pinning the restatement against the
 * reference's scalar kernels (tests/test_oracle.py). */
void oracle_add2(double xh, double xl, double yh, double yl, double *out) {
    dd x = {xh, xl}, y = {yh, yl}, r = add2(x, y); out[0] = r.h; out[1] = r.l;
}
void oracle_mul2(double xh, double xl, double yh, double yl, double *out) {
    dd x = {xh, xl}, y = {yh, yl}, r = mul2(x, y); out[0] = r.h; out[1] = r.l;
}
void oracle_two_prod(double a, double b, double *out) { two_prod(a, b, &out[0], &out[1]); }

/* ---- Rpotrf (mplapack/chol.py:21-65), unblocked, the reference's order ----
 * Scalar DDouble operations (ddarith.py): _canon :68-71, _add2 :79-90,
 * _mul21 :103-110, _div2 :113-131, _sqrt2 :142-163; element-wise add / mul
 * are the vectorised add2 / mul2 above; sum_ltr (elem.py:261-283) is add2
 * from (0, 0). */
static inline dd canon(double h, double l) { dd r = {h, isfinite(h) ? l : 0.0}; return r; }

static dd add2_s(dd x, dd y) {
    double s0 = x.h + y.h;
    if (!isfinite(s0)) { dd r = {s0, 0.0}; return r; }
    dd r = add2(x, y);
    return canon(r.h, r.l);
}

static dd mul21_s(dd x, double y) {
    double p, e;
    two_prod(x.h, y, &p, &e);
    if (!(isfinite(p) && isfinite(e))) return canon(p, 0.0);
    e = e + x.l * y;
    double s, t;
    quick_two_sum(p, e, &s, &t);
    return canon(s, t);
}

static dd div2_s(dd x, dd y) {
    dd r;
    if (y.h == 0.0) {
        r.l = 0.0;
        r.h = x.h == 0.0 ? NAN : copysign(INFINITY, x.h) * copysign(1.0, y.h);
        return r;
    }
    if (!(isfinite(x.h) && isfinite(y.h))) {
        if (isinf(y.h)) {
            r.l = 0.0;
            r.h = isinf(x.h) ? NAN : copysign(0.0, x.h) * copysign(1.0, y.h);
            return r;
        }
        return canon(x.h * copysign(1.0, y.h), 0.0);
    }
    double q1 = x.h / y.h;
    dd m = mul21_s(y, q1), nm = {-m.h, -m.l};
    r = add2_s(x, nm);
    double q2 = r.h / y.h;
    m = mul21_s(y, q2); nm.h = -m.h; nm.l = -m.l;
    r = add2_s(r, nm);
    double q3 = r.h / y.h;
    double a, b;
    quick_two_sum(q1, q2, &a, &b);
    dd ab = {a, b}, c = {q3, 0.0};
    return add2_s(ab, c);
}

static dd sqrt2_s(dd v) {
    dd z = {0.0, 0.0};
    if (v.h == 0.0 && v.l == 0.0) return z;
    if (!isfinite(v.h)) { dd r = {v.h, 0.0}; return r; }
    double h = v.h, l = v.l;
    int shift = 0;
    if (h >= 0x1p996) { h = ldexp(h, -106); l = ldexp(l, -106); shift = 53; }
    else if (h <= 0x1p-996) { h = ldexp(h, 106); l = ldexp(l, 106); shift = -53; }
    double x = 1.0 / sqrt(h);
    double ax = h * x;
    double p, e;
    two_prod(ax, ax, &p, &e);
    dd hv = {h, l}, pe = {-p, -e};
    dd r = add2_s(hv, pe);
    double s, e2;
    quick_two_sum(ax, r.h * (x * 0.5), &s, &e2);
    if (shift) { s = ldexp(s, shift); e2 = ldexp(e2, shift); }
    return canon(s, e2);
}

int oracle_potrf_validate(char uplo, int64_t n, int64_t lda) {
    int u = upflag(uplo);
    if (u != 'U' && u != 'L') return 1;
    if (n < 0) return 2;
    if (lda < (n > 1 ? n : 1)) return 4;
    return 0;
}

/* Returns the reference argument index (> 0) on invalid arguments, else 0
 * with *info = 0 or the first failing pivot + 1 (chol.py:44-46). */
int oracle_rpotrf(char uplo, int64_t n, double *Ah, double *Al, int64_t lda, int64_t *info) {
    int rc = oracle_potrf_validate(uplo, n, lda);
    if (rc) return rc;
    *info = 0;
    const int upper = upflag(uplo) == 'U';
#define AT(i, j) ((i) + (j) * lda)
    for (int64_t j = 0; j < n; ++j) {
        dd dot = {0.0, 0.0};
        for (int64_t l = 0; l < j; ++l) {
            int64_t x = upper ? AT(l, j) : AT(j, l);
            dd h = {Ah[x], Al[x]};
            dot = add2(dot, mul2(h, h));
        }
        dd a = {Ah[AT(j, j)], Al[AT(j, j)]}, nd = {-dot.h, -dot.l};
        dd ajj = add2_s(a, nd);
        int bad = isnan(ajj.h + ajj.l) || ajj.h < 0.0 || (ajj.h == 0.0 && !(ajj.l > 0.0));
        if (bad) {
            Ah[AT(j, j)] = ajj.h; Al[AT(j, j)] = ajj.l;
            *info = j + 1;
            return 0;
        }
        ajj = sqrt2_s(ajj);
        Ah[AT(j, j)] = ajj.h; Al[AT(j, j)] = ajj.l;
        if (j == n - 1) break;
        dd one = {1.0, 0.0};
        dd rec = div2_s(one, ajj);
        for (int64_t q = j + 1; q < n; ++q) {
            dd v;
            if (upper) {
                dd temp = {0.0, 0.0};
                for (int64_t l = 0; l < j; ++l) {
                    dd c = {Ah[AT(l, q)], Al[AT(l, q)]}, h = {Ah[AT(l, j)], Al[AT(l, j)]};
                    temp = add2(temp, mul2(c, h));
                }
                dd elt = {Ah[AT(j, q)], Al[AT(j, q)]}, nt = {-temp.h, -temp.l};
                v = mul2(rec, add2(elt, nt));
                Ah[AT(j, q)] = v.h; Al[AT(j, q)] = v.l;
            } else {
                dd tail = {Ah[AT(q, j)], Al[AT(q, j)]};
                for (int64_t l = 0; l < j; ++l) {
                    dd t = {-Ah[AT(j, l)], -Al[AT(j, l)]}, c = {Ah[AT(q, l)], Al[AT(q, l)]};
                    tail = add2(tail, mul2(t, c));
                }
                v = mul2(rec, tail);
                Ah[AT(q, j)] = v.h; Al[AT(q, j)] = v.l;
            }
        }
    }
#undef AT
    return 0;
}

void oracle_div2(double xh, double xl, double yh, double yl, double *out) {
    dd x = {xh, xl}, y = {yh, yl}, r = div2_s(x, y); out[0] = r.h; out[1] = r.l;
}
void oracle_sqrt2(double h, double l, double *out) {
    dd v = {h, l}, r = sqrt2_s(v); out[0] = r.h; out[1] = r.l;
}

/* ---- vectorised dd division (elem.py:81-117): _v_mul21 / _v_div2, with
 * the scalar _div2 for the special lanes (y.h == 0 or a non-finite hi) ---- */
static dd v_mul21(dd y, double q) {
    double p, e;
    two_prod(y.h, q, &p, &e);
    int bad = !(isfinite(p) && isfinite(e));
    e = e + y.l * q;
    double s, t;
    quick_two_sum(p, e, &s, &t);
    dd r = {s, t};
    if (bad) { r.h = p; r.l = 0.0; }
    return r;
}

static dd v_div2(dd x, dd y) {
    if (y.h == 0.0 || !(isfinite(x.h) && isfinite(y.h))) return div2_s(x, y);
    double q1 = x.h / y.h;
    dd m = v_mul21(y, q1), nm = {-m.h, -m.l};
    dd r = add2(x, nm);
    double q2 = r.h / y.h;
    m = v_mul21(y, q2); nm.h = -m.h; nm.l = -m.l;
    r = add2(r, nm);
    double q3 = r.h / y.h;
    double a, b;
    quick_two_sum(q1, q2, &a, &b);
    dd ab = {a, b}, c = {q3, 0.0};
    return add2(ab, c);
}

static inline dd dsub(dd x, dd y) { dd ny = {-y.h, -y.l}; return add2(x, ny); }   /* be.sub */

int oracle_trsm_validate(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                         int64_t lda, int64_t ldb) {
    int s = upflag(side), u = upflag(uplo), t = upflag(transa), d = upflag(diag);
    if (s != 'L' && s != 'R') return 1;
    if (u != 'U' && u != 'L') return 2;
    if (t != 'N' && t != 'T' && t != 'C') return 3;
    if (d != 'U' && d != 'N') return 4;
    if (m < 0) return 5;
    if (n < 0) return 6;
    int64_t nrowa = s == 'L' ? m : n;
    if (lda < (nrowa > 1 ? nrowa : 1)) return 9;
    if (ldb < (m > 1 ? m : 1)) return 11;
    return 0;
}

/* Rtrsm (level23.py:288-380): op(A) X = alpha B or X op(A) = alpha B, X
 * overwriting B, in the reference's loop order for each of the four
 * (side, transa) branches. */
int oracle_rtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                 double alpha_hi, double alpha_lo, const double *Ah, const double *Al,
                 int64_t lda, double *Bh, double *Bl, int64_t ldb) {
    int rc = oracle_trsm_validate(side, uplo, transa, diag, m, n, lda, ldb);
    if (rc) return rc;
    if (m == 0 || n == 0) return 0;
    const int left = upflag(side) == 'L', up = upflag(uplo) == 'U';
    const int notr = upflag(transa) == 'N', nounit = upflag(diag) == 'N';
    const dd al = {alpha_hi, alpha_lo}, one = {1.0, 0.0};
#define A_(i, j) ld_(Ah, Al, (i) + (j) * lda)
#define B_(i, j) ld_(Bh, Bl, (i) + (j) * ldb)
#define SETB(i, j, v) do { dd v_ = (v); Bh[(i) + (j) * ldb] = v_.h; Bl[(i) + (j) * ldb] = v_.l; } while (0)
    if (is_zero(al)) {                                  /* level23.py:306-308 */
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) { Bh[i + j * ldb] = 0.0; Bl[i + j * ldb] = 0.0; }
        return 0;
    }
    const int alpha_one = is_one(al);
    if (left && notr) {                                 /* :326-338 */
        for (int64_t j = 0; j < n; ++j) {
            if (!alpha_one)
                for (int64_t i = 0; i < m; ++i) SETB(i, j, mul2(al, B_(i, j)));
            for (int64_t s = 0; s < m; ++s) {
                int64_t kk = up ? m - 1 - s : s;
                if (nounit) SETB(kk, j, v_div2(B_(kk, j), A_(kk, kk)));
                int64_t r0 = up ? 0 : kk + 1, r1 = up ? kk : m;
                dd x = B_(kk, j);
                for (int64_t i = r0; i < r1; ++i) SETB(i, j, dsub(B_(i, j), mul2(A_(i, kk), x)));
            }
        }
    } else if (left) {                                  /* :339-350 */
        for (int64_t j = 0; j < n; ++j)
            for (int64_t s = 0; s < m; ++s) {
                int64_t i = up ? s : m - 1 - s;
                dd temp = mul2(al, B_(i, j));
                int64_t k0 = up ? 0 : i + 1, k1 = up ? i : m;
                for (int64_t kk = k0; kk < k1; ++kk) temp = dsub(temp, mul2(A_(kk, i), B_(kk, j)));
                if (nounit) temp = v_div2(temp, A_(i, i));
                SETB(i, j, temp);
            }
    } else if (notr) {                                  /* :351-363 */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t s = 0; s < n; ++s) {
                int64_t j = up ? s : n - 1 - s;
                if (!alpha_one) SETB(i, j, mul2(al, B_(i, j)));
                int64_t k0 = up ? 0 : j + 1, k1 = up ? j : n;
                for (int64_t kk = k0; kk < k1; ++kk)
                    SETB(i, j, dsub(B_(i, j), mul2(A_(kk, j), B_(i, kk))));
                if (nounit) SETB(i, j, mul2(v_div2(one, A_(j, j)), B_(i, j)));
            }
    } else {                                            /* :364-380 */
        for (int64_t i = 0; i < m; ++i)
            for (int64_t s = 0; s < n; ++s) {
                int64_t kk = up ? n - 1 - s : s;
                if (nounit) SETB(i, kk, mul2(v_div2(one, A_(kk, kk)), B_(i, kk)));
                int64_t j0 = up ? 0 : kk + 1, j1 = up ? kk : n;
                dd x = B_(i, kk);
                for (int64_t j = j0; j < j1; ++j) SETB(i, j, dsub(B_(i, j), mul2(A_(j, kk), x)));
                if (!alpha_one) SETB(i, kk, mul2(al, B_(i, kk)));
            }
    }
#undef A_
#undef B_
#undef SETB
    return 0;
}

/* Rgetrf (mplapack/lu.py:74-114): unblocked right-looking LU with partial
 * pivoting in the reference's order.  ipiv (1-based, length min(m, n)) and
 * *info as the reference returns them. */
int oracle_getrf_validate(int64_t m, int64_t n, int64_t lda) {
    if (m < 0) return 1;
    if (n < 0) return 2;
    if (lda < (m > 1 ? m : 1)) return 4;
    return 0;
}

static const dd SFMIN_DD = {0x1p-969, -0x0.0000000000006p-1022};   /* machine_params("dd").safe_min */

static int cmp2(dd x, dd y) {                          /* _cmp2, ddarith.py:166-176 */
    if (x.h < y.h) return -1;
    if (x.h > y.h) return 1;
    if (x.l < y.l) return -1;
    if (x.l > y.l) return 1;
    return 0;
}

/* DDBackend.argmax_abs (elem.py:246-259): max |hi|, ties by max lo*sign(hi),
 * first index; a NaN |hi| anywhere gives 0 (np.max propagates it). */
static int64_t argmax_abs_dd(const double *h, const double *l, int64_t cnt) {
    double mx = -1.0;
    for (int64_t i = 0; i < cnt; ++i) {
        double a = fabs(h[i]);
        if (isnan(a)) return 0;
        if (a > mx) mx = a;
    }
    int64_t best = -1;
    double bl = 0.0;
    for (int64_t i = 0; i < cnt; ++i) {
        if (fabs(h[i]) != mx) continue;
        double al = l[i] * (h[i] < 0.0 ? -1.0 : 1.0);
        if (best < 0 || al > bl) { best = i; bl = al; }
    }
    return best < 0 ? 0 : best;
}

int oracle_rgetrf(int64_t m, int64_t n, double *Ah, double *Al, int64_t lda, int64_t *ipiv,
                  int64_t *info) {
    int rc = oracle_getrf_validate(m, n, lda);
    if (rc) return rc;
    *info = 0;
    int64_t mn = m < n ? m : n;
    double *colh = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    double *coll = (double *)malloc(sizeof(double) * (m > 0 ? m : 1));
    for (int64_t j = 0; j < mn; ++j) {
        for (int64_t i = j; i < m; ++i) { colh[i - j] = Ah[i + j * lda]; coll[i - j] = Al[i + j * lda]; }
        int64_t jp = j + argmax_abs_dd(colh, coll, m - j);
        ipiv[j] = jp + 1;
        dd piv = {Ah[jp + j * lda], Al[jp + j * lda]};
        if (!is_zero(piv)) {
            if (jp != j)
                for (int64_t c = 0; c < n; ++c) {
                    double th = Ah[j + c * lda], tl = Al[j + c * lda];
                    Ah[j + c * lda] = Ah[jp + c * lda]; Al[j + c * lda] = Al[jp + c * lda];
                    Ah[jp + c * lda] = th; Al[jp + c * lda] = tl;
                }
            if (j < m - 1) {
                dd ap = piv;
                if (ap.h < 0.0 || (ap.h == 0.0 && ap.l < 0.0)) { ap.h = -ap.h; ap.l = -ap.l; }
                if (cmp2(ap, SFMIN_DD) >= 0) {
                    dd one = {1.0, 0.0}, rec = div2_s(one, piv);
                    for (int64_t i = j + 1; i < m; ++i) {
                        dd x = {Ah[i + j * lda], Al[i + j * lda]}, r = mul2(rec, x);
                        Ah[i + j * lda] = r.h; Al[i + j * lda] = r.l;
                    }
                } else {
                    for (int64_t i = j + 1; i < m; ++i) {
                        dd x = {Ah[i + j * lda], Al[i + j * lda]}, r = v_div2(x, piv);
                        Ah[i + j * lda] = r.h; Al[i + j * lda] = r.l;
                    }
                }
            }
        } else if (*info == 0) {
            *info = j + 1;
        }
        if (j < mn - 1)
            for (int64_t c = j + 1; c < n; ++c) {
                dd y = {-Ah[j + c * lda], -Al[j + c * lda]};
                for (int64_t i = j + 1; i < m; ++i) {
                    dd x = {Ah[i + j * lda], Al[i + j * lda]}, a = {Ah[i + c * lda], Al[i + c * lda]};
                    dd r = add2(a, mul2(x, y));
                    Ah[i + c * lda] = r.h; Al[i + c * lda] = r.l;
                }
            }
    }
    free(colh);
    free(coll);
    return 0;
}

/* Rgetrs (mplapack/lu.py:117-145): laswp (lu.py:61-65) + two Rtrsm calls.
 * ipiv: 1-based pivot rows as Rgetrf returns them. */
int oracle_getrs_validate(char trans, int64_t n, int64_t nrhs, int64_t lda, int64_t ldb) {
    int t = upflag(trans);
    if (t != 'N' && t != 'T' && t != 'C') return 1;
    if (n < 0) return 2;
    if (nrhs < 0) return 3;
    if (lda < (n > 1 ? n : 1)) return 5;
    if (ldb < (n > 1 ? n : 1)) return 8;
    return 0;
}

static void laswp_dd(double *Bh, double *Bl, int64_t ldb, int64_t ncol, const int64_t *ipiv,
                     int64_t np, int forward) {
    for (int64_t s = 0; s < np; ++s) {
        int64_t k = forward ? s : np - 1 - s, p = ipiv[k] - 1;
        if (p == k) continue;
        for (int64_t c = 0; c < ncol; ++c) {
            double th = Bh[k + c * ldb], tl = Bl[k + c * ldb];
            Bh[k + c * ldb] = Bh[p + c * ldb]; Bl[k + c * ldb] = Bl[p + c * ldb];
            Bh[p + c * ldb] = th; Bl[p + c * ldb] = tl;
        }
    }
}

int oracle_rgetrs(char trans, int64_t n, int64_t nrhs, const double *Ah, const double *Al,
                  int64_t lda, const int64_t *ipiv, int64_t nipiv, double *Bh, double *Bl,
                  int64_t ldb) {
    int rc = oracle_getrs_validate(trans, n, nrhs, lda, ldb);
    if (rc) return rc;
    if (n == 0 || nrhs == 0) return 0;
    if (upflag(trans) == 'N') {
        laswp_dd(Bh, Bl, ldb, nrhs, ipiv, nipiv, 1);
        oracle_rtrsm('L', 'L', 'N', 'U', n, nrhs, 1.0, 0.0, Ah, Al, lda, Bh, Bl, ldb);
        oracle_rtrsm('L', 'U', 'N', 'N', n, nrhs, 1.0, 0.0, Ah, Al, lda, Bh, Bl, ldb);
    } else {
        oracle_rtrsm('L', 'U', 'T', 'N', n, nrhs, 1.0, 0.0, Ah, Al, lda, Bh, Bl, ldb);
        oracle_rtrsm('L', 'L', 'T', 'U', n, nrhs, 1.0, 0.0, Ah, Al, lda, Bh, Bl, ldb);
        laswp_dd(Bh, Bl, ldb, nrhs, ipiv, nipiv, 0);
    }
    return 0;
}

/* ---- the LAPACK consumers on the F64 backend (elem.py:149-197): numpy
 * binary64 + - * /, Python float scalars, math.sqrt -- same loop orders as
 * the dd restatements above ---- */
int oracle_dpotrf(char uplo, int64_t n, double *A, int64_t lda, int64_t *info) {
    int rc = oracle_potrf_validate(uplo, n, lda);
    if (rc) return rc;
    *info = 0;
    const int upper = upflag(uplo) == 'U';
#define AT(i, j) A[(i) + (j) * lda]
    for (int64_t j = 0; j < n; ++j) {
        double dot = 0.0;
        for (int64_t l = 0; l < j; ++l) {
            double h = upper ? AT(l, j) : AT(j, l);
            dot = dot + h * h;
        }
        double ajj = AT(j, j) - dot;
        if (isnan(ajj) || ajj <= 0.0) { AT(j, j) = ajj; *info = j + 1; return 0; }
        ajj = sqrt(ajj);
        AT(j, j) = ajj;
        if (j == n - 1) break;
        double rec = 1.0 / ajj;
        for (int64_t q = j + 1; q < n; ++q) {
            if (upper) {
                double temp = 0.0;
                for (int64_t l = 0; l < j; ++l) temp = temp + AT(l, q) * AT(l, j);
                AT(j, q) = rec * (AT(j, q) + (-temp));
            } else {
                double tail = AT(q, j);
                for (int64_t l = 0; l < j; ++l) tail = tail + (-AT(j, l)) * AT(q, l);
                AT(q, j) = rec * tail;
            }
        }
    }
#undef AT
    return 0;
}

int oracle_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n, double alpha,
                 const double *A, int64_t lda, double *B, int64_t ldb) {
    int rc = oracle_trsm_validate(side, uplo, transa, diag, m, n, lda, ldb);
    if (rc) return rc;
    if (m == 0 || n == 0) return 0;
    const int left = upflag(side) == 'L', up = upflag(uplo) == 'U';
    const int notr = upflag(transa) == 'N', nounit = upflag(diag) == 'N';
#define A_(i, j) A[(i) + (j) * lda]
#define B_(i, j) B[(i) + (j) * ldb]
    if (alpha == 0.0) {
        for (int64_t j = 0; j < n; ++j)
            for (int64_t i = 0; i < m; ++i) B_(i, j) = 0.0;
        return 0;
    }
    const int alpha_one = alpha == 1.0;
    if (left && notr) {
        for (int64_t j = 0; j < n; ++j) {
            if (!alpha_one)
                for (int64_t i = 0; i < m; ++i) B_(i, j) = alpha * B_(i, j);
            for (int64_t s = 0; s < m; ++s) {
                int64_t kk = up ? m - 1 - s : s;
                if (nounit) B_(kk, j) = B_(kk, j) / A_(kk, kk);
                int64_t r0 = up ? 0 : kk + 1, r1 = up ? kk : m;
                double x = B_(kk, j);
                for (int64_t i = r0; i < r1; ++i) B_(i, j) = B_(i, j) - A_(i, kk) * x;
            }
        }
    } else if (left) {
        for (int64_t j = 0; j < n; ++j)
            for (int64_t s = 0; s < m; ++s) {
                int64_t i = up ? s : m - 1 - s;
                double temp = alpha * B_(i, j);
                int64_t k0 = up ? 0 : i + 1, k1 = up ? i : m;
                for (int64_t kk = k0; kk < k1; ++kk) temp = temp - A_(kk, i) * B_(kk, j);
                if (nounit) temp = temp / A_(i, i);
                B_(i, j) = temp;
            }
    } else if (notr) {
        for (int64_t i = 0; i < m; ++i)
            for (int64_t s = 0; s < n; ++s) {
                int64_t j = up ? s : n - 1 - s;
                if (!alpha_one) B_(i, j) = alpha * B_(i, j);
                int64_t k0 = up ? 0 : j + 1, k1 = up ? j : n;
                for (int64_t kk = k0; kk < k1; ++kk) B_(i, j) = B_(i, j) - A_(kk, j) * B_(i, kk);
                if (nounit) B_(i, j) = (1.0 / A_(j, j)) * B_(i, j);
            }
    } else {
        for (int64_t i = 0; i < m; ++i)
            for (int64_t s = 0; s < n; ++s) {
                int64_t kk = up ? n - 1 - s : s;
                if (nounit) B_(i, kk) = (1.0 / A_(kk, kk)) * B_(i, kk);
                int64_t j0 = up ? 0 : kk + 1, j1 = up ? kk : n;
                double x = B_(i, kk);
                for (int64_t j = j0; j < j1; ++j) B_(i, j) = B_(i, j) - A_(j, kk) * x;
                if (!alpha_one) B_(i, kk) = alpha * B_(i, kk);
            }
    }
#undef A_
#undef B_
    return 0;
}

int oracle_dgetrf(int64_t m, int64_t n, double *A, int64_t lda, int64_t *ipiv, int64_t *info) {
    int rc = oracle_getrf_validate(m, n, lda);
    if (rc) return rc;
    *info = 0;
    int64_t mn = m < n ? m : n;
    for (int64_t j = 0; j < mn; ++j) {
        int64_t jp = j;             /* F64Backend.argmax_abs: first max, NaN -> 0 */
        double mx = -1.0;
        int nan = 0;
        for (int64_t i = j; i < m; ++i) {
            double a = fabs(A[i + j * lda]);
            if (isnan(a)) { nan = 1; break; }
            if (a > mx) { mx = a; jp = i; }
        }
        if (nan) jp = j;
        ipiv[j] = jp + 1;
        double piv = A[jp + j * lda];
        if (piv != 0.0) {
            if (jp != j)
                for (int64_t c = 0; c < n; ++c) {
                    double t = A[j + c * lda];
                    A[j + c * lda] = A[jp + c * lda];
                    A[jp + c * lda] = t;
                }
            if (j < m - 1) {
                if (fabs(piv) >= 0x1p-1022) {
                    double rec = 1.0 / piv;
                    for (int64_t i = j + 1; i < m; ++i) A[i + j * lda] = rec * A[i + j * lda];
                } else {
                    for (int64_t i = j + 1; i < m; ++i) A[i + j * lda] = A[i + j * lda] / piv;
                }
            }
        } else if (*info == 0) {
            *info = j + 1;
        }
        if (j < mn - 1)
            for (int64_t c = j + 1; c < n; ++c) {
                double y = -A[j + c * lda];
                for (int64_t i = j + 1; i < m; ++i) A[i + c * lda] = A[i + c * lda] + A[i + j * lda] * y;
            }
    }
    return 0;
}

int oracle_dgetrs(char trans, int64_t n, int64_t nrhs, const double *A, int64_t lda,
                  const int64_t *ipiv, int64_t nipiv, double *B, int64_t ldb) {
    int rc = oracle_getrs_validate(trans, n, nrhs, lda, ldb);
    if (rc) return rc;
    if (n == 0 || nrhs == 0) return 0;
    const int notr = upflag(trans) == 'N';
    if (notr) {
        for (int64_t k = 0; k < nipiv; ++k) {
            int64_t p = ipiv[k] - 1;
            if (p != k) for (int64_t c = 0; c < nrhs; ++c) { double t = B[k + c * ldb]; B[k + c * ldb] = B[p + c * ldb]; B[p + c * ldb] = t; }
        }
        oracle_dtrsm('L', 'L', 'N', 'U', n, nrhs, 1.0, A, lda, B, ldb);
        oracle_dtrsm('L', 'U', 'N', 'N', n, nrhs, 1.0, A, lda, B, ldb);
    } else {
        oracle_dtrsm('L', 'U', 'T', 'N', n, nrhs, 1.0, A, lda, B, ldb);
        oracle_dtrsm('L', 'L', 'T', 'U', n, nrhs, 1.0, A, lda, B, ldb);
        for (int64_t s = 0; s < nipiv; ++s) {
            int64_t k = nipiv - 1 - s, p = ipiv[k] - 1;
            if (p != k) for (int64_t c = 0; c < nrhs; ++c) { double t = B[k + c * ldb]; B[k + c * ldb] = B[p + c * ldb]; B[p + c * ldb] = t; }
        }
    }
    return 0;
}
