// capi_lapack.cu -- C ABI of the LAPACK consumers (include/ddblas.h):
//   ddb_rtrsm  <- mpkit.mpblas.Rtrsm     (level23.py:288-380)
//   ddb_rgetrf <- mpkit.mplapack.Rgetrf  (lu.py:74-114)
//   ddb_rgetrs <- mpkit.mplapack.Rgetrs  (lu.py:117-145)
//   ddb_rpotrf <- mpkit.mplapack.Rpotrf  (chol.py:21-65)
// Blocked drivers over the kernels of dd_trsm.cu / dd_getrf.cu / dd_potrf.cu
// whose trailing updates are ddb_rgemm / ddb_rsyrk calls (capi.cu).
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../include/ddblas.h"
#include "host.h"
#include "internal.h"

using namespace ddb;
using namespace ddb::host;

namespace {

// binary64 twins of the trailing-update calls (the 'f64' Matrix: one plane,
// lo pointers alias hi and are ignored; the f64 GEMMs are bit-exact, so
// mode does not apply)
int gemm_any(bool f64, char ta, char tb, int64_t m, int64_t n, int64_t k, double alpha_hi,
             double alpha_lo, const double* ah, const double* al, int64_t lda, const double* bh,
             const double* bl, int64_t ldb, double beta_hi, double beta_lo, double* ch, double* cl,
             int64_t ldc, int mode, void* st) {
  if (f64) return ddb_dgemm(ta, tb, m, n, k, alpha_hi, ah, lda, bh, ldb, beta_hi, ch, ldc, st);
  return ddb_rgemm(ta, tb, m, n, k, alpha_hi, alpha_lo, ah, al, lda, bh, bl, ldb, beta_hi, beta_lo,
                   ch, cl, ldc, mode, st);
}

int syrk_any(bool f64, char uplo, char trans, int64_t n, int64_t k, double alpha_hi,
             double alpha_lo, const double* ah, const double* al, int64_t lda, double beta_hi,
             double beta_lo, double* ch, double* cl, int64_t ldc, int mode, void* st) {
  if (f64) return ddb_dsyrk(uplo, trans, n, k, alpha_hi, ah, lda, beta_hi, ch, ldc, st);
  return ddb_rsyrk(uplo, trans, n, k, alpha_hi, alpha_lo, ah, al, lda, beta_hi, beta_lo, ch, cl,
                   ldc, mode, st);
}

// ---- triangular solve (dd_trsm.cu) -------------------------------------------

// DDB_LAPACK_TRACE=1: a CUDA-event timeline of a blocked driver's streams,
// printed to stderr when the call finishes (diagnostics only: timing events)
struct Trace {
  bool on = false;
  cudaEvent_t t0 = nullptr;
  std::vector<cudaEvent_t> ev;
  std::vector<const char*> what;
  std::vector<int64_t> tag;
  explicit Trace(cudaStream_t s) {
    const char* v = std::getenv("DDB_LAPACK_TRACE");
    on = v != nullptr && v[0] == '1';
    if (on && cudaEventCreate(&t0) == cudaSuccess) cudaEventRecord(t0, s);
  }
  void mark(const char* w, int64_t j, cudaStream_t s) {
    if (!on) return;
    cudaEvent_t e;
    if (cudaEventCreate(&e) != cudaSuccess) return;
    cudaEventRecord(e, s);
    ev.push_back(e);
    what.push_back(w);
    tag.push_back(j);
  }
  ~Trace() {
    if (!on) return;
    for (size_t i = 0; i < ev.size(); ++i) {
      float ms = 0.f;
      cudaEventSynchronize(ev[i]);
      cudaEventElapsedTime(&ms, t0, ev[i]);
      std::fprintf(stderr, "trace %9.3f %-12s %lld\n", ms, what[i], (long long)tag[i]);
      cudaEventDestroy(ev[i]);
    }
    cudaEventDestroy(t0);
  }
};

}  // namespace

extern "C" int ddb_rtrsm_validate(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                       int64_t lda, int64_t ldb) {
  const int sd = upflag(side), u = upflag(uplo), t = upflag(transa), d = upflag(diag);
  if (sd != 'L' && sd != 'R') return 1;               // level23.py:296-299
  if (u != 'U' && u != 'L') return 2;
  if (t != 'N' && t != 'T' && t != 'C') return 3;
  if (d != 'U' && d != 'N') return 4;
  if (m < 0) return 5;                                // :300-301
  if (n < 0) return 6;
  const int64_t nrowa = sd == 'L' ? m : n;            // :302-304
  if (lda < (nrowa > 1 ? nrowa : 1)) return 9;
  if (ldb < (m > 1 ? m : 1)) return 11;
  return 0;
}

static int rtrsm_impl(bool f64, char side, char uplo, char transa, char diag, int64_t m,
                      int64_t n, double alpha_hi, double alpha_lo, const double* a_hi,
                      const double* a_lo, int64_t lda, double* b_hi, double* b_lo, int64_t ldb,
                      int mode, void* stream) {
  const int rc = ddb_rtrsm_validate(side, uplo, transa, diag, m, n, lda, ldb);
  if (rc) return rc;
  if (mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM) {
    g_last_error = "unknown mode";
    return DDB_EINVAL;
  }
  if (m == 0 || n == 0) return DDB_OK;                // :306-307
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cudaError_t e;
  if (is_zero(alpha_hi, alpha_lo)) {                  // :310-312: B = 0
    e = cudaMemset2DAsync(b_hi, sizeof(double) * ldb, 0, sizeof(double) * m, n, s);
    if (e == cudaSuccess && !f64)
      e = cudaMemset2DAsync(b_lo, sizeof(double) * ldb, 0, sizeof(double) * m, n, s);
    return e == cudaSuccess ? DDB_OK : fail(e, "rtrsm zero fill");
  }
  const bool left = upflag(side) == 'L', upper = upflag(uplo) == 'U';
  const bool notr = upflag(transa) == 'N', alpha_one = is_one(alpha_hi, alpha_lo);
  const dd alpha{alpha_hi, alpha_lo};
  // branch table (see dd_trsm.cu): production order, T orientation, finish,
  // alpha placement, and whether the terms arrive in reverse order
  TrsmArgs t{};
  t.f64 = f64;
  t.left = left;
  t.unit = upflag(diag) == 'U';
  t.fin_rec = !left;
  int trans, init_scale, post_scale, rev_terms;
  if (left && notr) {        t.rev = upper;  trans = 0; init_scale = !alpha_one; post_scale = 0; rev_terms = 0; }
  else if (left) {           t.rev = !upper; trans = 1; init_scale = 1;          post_scale = 0; rev_terms = !upper; }
  else if (notr) {           t.rev = !upper; trans = 1; init_scale = !alpha_one; post_scale = 0; rev_terms = !upper; }
  else {                     t.rev = upper;  trans = 0; init_scale = 0; post_scale = !alpha_one; rev_terms = 0; }
  t.p = left ? m : n;
  t.q = left ? n : m;
  t.ldw = t.p;
  t.ldt = t.p;
  retain_pool_memory();
  const size_t wsz = (size_t)t.p * t.q, tsz = (size_t)t.p * t.p;
  void* ws = nullptr;
  e = cudaMallocAsync(&ws, sizeof(double) * 2 * (wsz + tsz + 2 * t.p), s);
  if (e != cudaSuccess) return fail(e, "rtrsm workspace");
  double* w = static_cast<double*>(ws);
  t.w_hi = w; t.w_lo = w + wsz;
  t.t_hi = w + 2 * wsz; t.t_lo = t.t_hi + tsz;
  t.d_hi = t.t_lo + tsz; t.d_lo = t.d_hi + t.p;
  t.r_hi = t.d_lo + t.p; t.r_lo = t.r_hi + t.p;
  // binary64 is always in the reference's order
  const bool exact_order = f64 || mode == MODE_EXACT || mode == MODE_REFERENCE;
  t.rec_fast = !exact_order;
  int nl = 0, rc2 = DDB_OK;
  e = launch_trsm_pack(t, b_hi, b_lo, ldb, init_scale, alpha, s);
  ++nl;
  if (e == cudaSuccess) { e = launch_trsm_coef(t, a_hi, a_lo, lda, trans, s); ++nl; }
  if (e == cudaSuccess && rev_terms && exact_order) {
    e = launch_trsm_rev(t, s);
    ++nl;
  } else if (e == cudaSuccess) {
    static const int64_t nb_env = [] {
      const char* v = std::getenv("DDB_TRSM_NB");
      return v ? (int64_t)std::atoll(v) : (int64_t)0;
    }();
    // two levels: inner blocks of ib rows (diagonal solve + a GEMM over the
    // rest of the outer block), then one GEMM of depth NB for all rows below
    // the outer block -- per element the terms still arrive in production
    // order
    // (outer 512: its depth-512 GEMMs take the split algorithm on the
    // serial schedule; n = 8192 fast 174 -> 165 ms, exact unchanged)
    const int64_t ib = 64;
    const int64_t NB = nb_env > 0 ? (nb_env < ib ? ib : nb_env) : 512;
    // W(r0:r1, :) -= T(r0:r1, l0:l1) W(l0:l1, :)
    auto update = [&](int64_t r0, int64_t r1, int64_t l0, int64_t l1) -> int {
      if (r1 <= r0 || l1 <= l0) return DDB_OK;
      GemmArgs g{};
      g.ta = 0; g.tb = 0; g.syrk = 0;
      g.m = r1 - r0; g.n = t.q; g.k = l1 - l0;
      g.a_hi = t.t_hi + r0 + l0 * t.ldt; g.a_lo = t.t_lo + r0 + l0 * t.ldt; g.lda = t.ldt;
      g.b_hi = t.w_hi + l0; g.b_lo = t.w_lo + l0; g.ldb = t.ldw;
      g.c_hi = t.w_hi + r0; g.c_lo = t.w_lo + r0; g.ldc = t.ldw;
      g.beta = dd{1.0, 0.0};
      g.f64 = f64;    // binary64: c + a (-1 x) == c - a x exactly, the plain f64 kernel
      if (exact_order && !f64) { g.sub = 1; g.alpha = dd{1.0, 0.0}; }
      else { g.sub = 0; g.alpha = dd{-1.0, 0.0}; }
      return run(g, mode, s);
    };
    for (int64_t o0 = 0; o0 < t.p && e == cudaSuccess && rc2 == DDB_OK; o0 += NB) {
      const int64_t o1 = o0 + NB < t.p ? o0 + NB : t.p;
      for (int64_t r0 = o0; r0 < o1 && e == cudaSuccess && rc2 == DDB_OK; r0 += ib) {
        const int64_t r1 = r0 + ib < o1 ? r0 + ib : o1;
        e = launch_trsm_block(t, r0, (int)(r1 - r0), s);
        ++nl;
        if (e == cudaSuccess) rc2 = update(r1, o1, r0, r1);
      }
      if (e == cudaSuccess && rc2 == DDB_OK) rc2 = update(o1, t.p, o0, o1);
    }
  }
  if (e == cudaSuccess && rc2 == DDB_OK) {
    e = launch_trsm_unpack(t, b_hi, b_lo, ldb, post_scale, alpha, s);
    ++nl;
  }
  g_launches += nl;
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (rc2 != DDB_OK) return rc2;
  if (e != cudaSuccess) return fail(e, "rtrsm");
  if (e2 != cudaSuccess) return fail(e2, "workspace free");
  return DDB_OK;
}

extern "C" int ddb_rtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                         double alpha_hi, double alpha_lo, const double* a_hi,
                         const double* a_lo, int64_t lda, double* b_hi, double* b_lo,
                         int64_t ldb, int mode, void* stream) {
  return rtrsm_impl(false, side, uplo, transa, diag, m, n, alpha_hi, alpha_lo, a_hi, a_lo, lda,
                    b_hi, b_lo, ldb, mode, stream);
}

extern "C" int ddb_dtrsm(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                         double alpha, const double* a, int64_t lda, double* b, int64_t ldb,
                         void* stream) {
  return rtrsm_impl(true, side, uplo, transa, diag, m, n, alpha, 0.0, a, a, lda, b, b, ldb,
                    DDB_MODE_EXACT, stream);
}

extern "C" int ddb_rtrsm_host(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                   double alpha_hi, double alpha_lo, const double* a_hi, const double* a_lo,
                   int64_t lda, double* b_hi, double* b_lo, int64_t ldb, int mode, void* stream) {
  int rc = ddb_rtrsm_validate(side, uplo, transa, diag, m, n, lda, ldb);
  if (rc) return rc;
  if (m == 0 || n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t na = upflag(side) == 'L' ? m : n;
  const int64_t sa = is_zero(alpha_hi, alpha_lo) ? 0 : span(na, na, lda);
  const int64_t sb = span(m, n, ldb);
  DevBuf A, B;
  if ((rc = stage_in(A, a_hi, a_lo, sa, s))) return rc;
  if ((rc = stage_in(B, b_hi, b_lo, sb, s))) return rc;
  rc = ddb_rtrsm(side, uplo, transa, diag, m, n, alpha_hi, alpha_lo, A.p, A.p ? A.p + sa : nullptr,
                 lda, B.p, B.p + sb, ldb, mode, stream);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(b_hi, B.p, sizeof(double) * sb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(b_lo, B.p + sb, sizeof(double) * sb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(e, "device to host copy");
  return DDB_OK;
}

// ---- LU with partial pivoting (dd_getrf.cu) -----------------------------------

extern "C" int ddb_rgetrf_validate(int64_t m, int64_t n, int64_t lda) {
  if (m < 0) return 1;                                // lu.py:83-85
  if (n < 0) return 2;
  if (lda < (m > 1 ? m : 1)) return 4;
  return 0;
}

static int rgetrf_impl(bool f64, int64_t m, int64_t n, double* a_hi, double* a_lo, int64_t lda,
                       int64_t* ipiv, int* info, int mode, void* stream) {
  const int rc = ddb_rgetrf_validate(m, n, lda);
  if (rc) return rc;
  NoPersistScope no_persist;   // trailing updates beside the panel stream
  if (mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM || info == nullptr ||
      (ipiv == nullptr && m > 0 && n > 0)) {
    g_last_error = info == nullptr || ipiv == nullptr ? "ipiv / info pointer is null" : "unknown mode";
    return DDB_EINVAL;
  }
  *info = 0;
  if (m == 0 || n == 0) return DDB_OK;                // lu.py:86-87
  static const int64_t nb_env = [] {
    const char* v = std::getenv("DDB_GETRF_NB");
    return v ? (int64_t)std::atoll(v) : (int64_t)0;
  }();
  const int64_t nbo = nb_env > 0 ? nb_env : 256;          // outer width
  const int64_t ib = nbo < 64 ? nbo : 64;                  // inner (panel kernel) width
  const int64_t nb = ib;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  GetrfArgs g{};
  g.m = m; g.n = n; g.mn = m < n ? m : n; g.lda = lda;
  g.a_hi = a_hi; g.a_lo = a_lo;
  g.f64 = f64;
  g.fastacc = !f64 && (mode == DDB_MODE_FAST || mode == DDB_MODE_TWOSUM);
  const int G = getrf_max_panel_ctas();
  // workspace: info, barrier | ipiv, swap (mn each) | G partial candidates
  // partial candidates and rows: two parities (getrf_panel_smem_kernel)
  const size_t ws_bytes = 256 + sizeof(long long) * 2 * (size_t)g.mn +
                          2 * (size_t)G * (4 * sizeof(double) + sizeof(long long) + sizeof(int)) +
                          64 + sizeof(double) * (4 * (size_t)G + 4) * ((size_t)nb + 1) + 64 +
                          5 * (size_t)kPermBufBytes + 64;
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, ws_bytes, s);
  if (e != cudaSuccess) return fail(e, "rgetrf workspace");
  char* w = static_cast<char*>(ws);
  g.info = reinterpret_cast<int*>(w);
  g.bar = reinterpret_cast<unsigned*>(w + 64);
  // window masks of the U12 kernel's L block, one per stream (8 words each)
  unsigned* lmask[2] = {reinterpret_cast<unsigned*>(w + 128), reinterpret_cast<unsigned*>(w + 192)};
  g.ipiv = reinterpret_cast<long long*>(w + 256);
  g.swap = g.ipiv + g.mn;
  double* pd = reinterpret_cast<double*>(g.swap + g.mn);
  g.part_ah = pd; g.part_al = pd + 2 * G; g.part_h = pd + 4 * G; g.part_l = pd + 6 * G;
  g.part_idx = reinterpret_cast<long long*>(pd + 8 * G);
  g.part_nan = reinterpret_cast<int*>(g.part_idx + 2 * G);
  g.rowbuf = reinterpret_cast<double*>(
      (reinterpret_cast<uintptr_t>(g.part_nan + 2 * G) + 63) & ~static_cast<uintptr_t>(63));
  // composed interchanges: one buffer per stream that applies them
  // [0], [1]: scratch for the panel stream / the caller's stream; [2]: the
  // current inner panel's; [3], [4]: the outer blocks' (by parity: block J's
  // is read by rest(J) on the caller's stream while J+1's is formed)
  PermBuf pbuf[5];
  {
    char* pp = reinterpret_cast<char*>(
        (reinterpret_cast<uintptr_t>(g.rowbuf + (4 * (size_t)G + 4) * (nb + 1)) + 63) &
        ~static_cast<uintptr_t>(63));
    for (int i = 0; i < 5; ++i, pp += kPermBufBytes) {
      pbuf[i].rows = reinterpret_cast<long long*>(pp);
      pbuf[i].src = reinterpret_cast<int*>(pp + 512 * 8);
      pbuf[i].n = reinterpret_cast<int*>(pp + 512 * 12);
    }
  }
  int nl = 0, rc2 = DDB_OK;
  e = cudaMemsetAsync(ws, 0, 256, s);
  // Two block levels (outer NB = the trailing GEMM's depth, inner ib <= 64 =
  // the panel kernel's width) and a lookahead: the next outer panel and the
  // update of its columns run on the high-priority stream `cs` while the
  // rest of the trailing update runs on the caller's stream (same scheme and
  // ordering argument as Rpotrf).
  const int64_t NB = nbo;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  if (e == cudaSuccess) e = panel_stream(&cs);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming);
  Trace tr(s);
  auto gemm = [&](int64_t r0, int64_t r1, int64_t c0, int64_t c1, int64_t l0, int64_t l1,
                  cudaStream_t st) -> int {   // A(r0:r1, c0:c1) += A(r0:r1, l0:l1) (-A(l0:l1, c0:c1))
    if (r1 <= r0 || c1 <= c0 || l1 <= l0) return DDB_OK;
    return gemm_any(f64, 'N', 'N', r1 - r0, c1 - c0, l1 - l0, -1.0, 0.0, a_hi + r0 + l0 * lda,
                     a_lo + r0 + l0 * lda, lda, a_hi + l0 + c0 * lda, a_lo + l0 + c0 * lda, lda,
                     1.0, 0.0, a_hi + r0 + c0 * lda, a_lo + r0 + c0 * lda, lda, mode,
                     static_cast<void*>(st));
  };
  // block J's pending work on columns [c0, c1): interchanges, U12 (blocked
  // by the inner width), trailing update of rows >= J1
  // interchanges of steps [J0, J1) on columns [c0, c1): from a composition
  // formed once per block (pre) or composed here
  auto swap_cols = [&](int64_t J0, int64_t J1, int64_t c0, int64_t c1, cudaStream_t st,
                       const PermBuf* pre) -> cudaError_t {
    if (c1 <= c0) return cudaSuccess;
    ++nl;
    if (pre != nullptr) return launch_getrf_apply(g, *pre, J1 - J0, c0, c1, st);
    return launch_getrf_laswp(g, J0, J1, c0, c1, st, 0, pbuf[st == cs ? 0 : 1]);
  };
  auto apply_block = [&](int64_t J0, int64_t J1, int64_t c0, int64_t c1, cudaStream_t st,
                         const PermBuf* pre) -> int {
    if (c1 <= c0) return DDB_OK;
    cudaError_t er = swap_cols(J0, J1, c0, c1, st, pre);
    if (er != cudaSuccess) return fail(er, "rgetrf laswp");
    if (J1 - J0 > ib && J1 - J0 <= 256) {
      // the whole block row's U12 in one launch (per element the same
      // products in the same order as the inner trsm / Rgemm sequence below)
      er = launch_getrf_u12(g, J0, (int)(J1 - J0), c0, c1, lmask[st == cs ? 0 : 1], st);
      nl += f64 ? 1 : 2;
      if (er != cudaSuccess) return fail(er, "rgetrf u12");
    } else {
      for (int64_t i0 = J0; i0 < J1; i0 += ib) {
        const int64_t i1 = i0 + ib < J1 ? i0 + ib : J1;
        if ((er = launch_getrf_trsm(g, i0, (int)(i1 - i0), c0, c1, st)) != cudaSuccess)
          return fail(er, "rgetrf trsm");
        ++nl;
        const int r = gemm(i1, J1, c0, c1, i0, i1, st);
        if (r != DDB_OK) return r;
      }
    }
    if (J1 - J0 <= ib && c1 - c0 <= 256 && m > J1) {   // an inner panel's update: one lean launch
      er = launch_getrf_inner_upd(g, J0, (int)(J1 - J0), J1, m, c0, c1, st);
      ++nl;
      return er == cudaSuccess ? DDB_OK : fail(er, "rgetrf inner update");
    }
    return gemm(J1, m, c0, c1, J0, J1, st);
  };
  // factor the outer panel [J0, J1) (its columns only) on `cs`
  auto factor_outer = [&](int64_t J0, int64_t J1) -> int {
    for (int64_t i0 = J0; i0 < J1; i0 += ib) {
      const int64_t i1 = i0 + ib < J1 ? i0 + ib : J1;
      cudaError_t er = launch_getrf_panel(g, i0, (int)(i1 - i0), cs);
      ++nl;
      tr.mark("ipanel_done", i0, cs);
      if (er == cudaSuccess) { er = launch_getrf_compose(g, i0, i1, 0, pbuf[2], cs); ++nl; }
      if (er == cudaSuccess) er = swap_cols(i0, i1, J0, i0, cs, &pbuf[2]);
      if (er != cudaSuccess) return fail(er, "rgetrf panel");
      if (i1 < J1) {
        const int r = apply_block(i0, i1, i1, J1, cs, &pbuf[2]);
        if (r != DDB_OK) return r;
      }
      tr.mark("iapply_done", i0, cs);
    }
    return DDB_OK;
  };
  if (e == cudaSuccess) e = cudaEventRecord(ev_a, s);
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev_a, 0);
  if (e == cudaSuccess) rc2 = factor_outer(0, NB < g.mn ? NB : g.mn);
  tr.mark("panel_done", 0, cs);
  bool have_rest = false;
  for (int64_t J0 = 0; e == cudaSuccess && rc2 == DDB_OK; J0 += NB) {
    const int64_t J1 = J0 + NB < g.mn ? J0 + NB : g.mn;
    // block J's interchanges, composed once; first on the factored columns
    // to its left
    const PermBuf* pre = nullptr;
    if (J1 - J0 <= kPermStepsMax) {
      pre = &pbuf[3 + (int)((J0 / NB) & 1)];
      if ((e = launch_getrf_compose(g, J0, J1, 0, *pre, cs)) != cudaSuccess) break;
      ++nl;
    }
    if ((e = swap_cols(J0, J1, 0, J0, cs, pre)) != cudaSuccess) break;
    if (J1 >= n) break;
    const int64_t J2 = J1 + NB < g.mn ? J1 + NB : (J1 < g.mn ? g.mn : n);
    e = cudaEventRecord(ev_a, cs);                         // panel J done
    if (e == cudaSuccess && have_rest) e = cudaStreamWaitEvent(cs, ev_b, 0);   // rest(J-1)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_a, 0);
    if (e != cudaSuccess) break;
    if (J2 < n) {
      tr.mark("rest_start", J0, s);
      rc2 = apply_block(J0, J1, J2, n, s, pre);            // rest(J)
      if (rc2 != DDB_OK) break;
      tr.mark("rest_done", J0, s);
      e = cudaEventRecord(ev_b, s);
      have_rest = true;
      if (e != cudaSuccess) break;
    }
    tr.mark("upd_start", J0, cs);
    rc2 = apply_block(J0, J1, J1, J2, cs, pre);            // columns of block J+1
    tr.mark("upd_done", J0, cs);
    if (rc2 != DDB_OK || J1 >= g.mn) break;
    rc2 = factor_outer(J1, J2 < g.mn ? J2 : g.mn);
    tr.mark("panel_done", J1, cs);
  }
  if (cs != nullptr) {
    cudaError_t ej = cudaEventRecord(ev_a, cs);
    if (ej == cudaSuccess) ej = cudaStreamWaitEvent(s, ev_a, 0);
    if (e == cudaSuccess) e = ej;
  }
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  g_launches += nl;
  int hinfo = 0;
  if (e == cudaSuccess && rc2 == DDB_OK) {
    e = cudaMemcpyAsync(&hinfo, g.info, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(ipiv, g.ipiv, sizeof(long long) * g.mn, cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (rc2 != DDB_OK) return rc2;
  if (e != cudaSuccess) return fail(e, "rgetrf");
  if (e2 != cudaSuccess) return fail(e2, "workspace free");
  *info = hinfo;
  return DDB_OK;
}

extern "C" int ddb_rgetrf(int64_t m, int64_t n, double* a_hi, double* a_lo, int64_t lda,
                          int64_t* ipiv, int* info, int mode, void* stream) {
  return rgetrf_impl(false, m, n, a_hi, a_lo, lda, ipiv, info, mode, stream);
}

extern "C" int ddb_dgetrf(int64_t m, int64_t n, double* a, int64_t lda, int64_t* ipiv, int* info,
                          void* stream) {
  return rgetrf_impl(true, m, n, a, a, lda, ipiv, info, DDB_MODE_EXACT, stream);
}

extern "C" int ddb_rgetrf_host(int64_t m, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t* ipiv,
                    int* info, int mode, void* stream) {
  int rc = ddb_rgetrf_validate(m, n, lda);
  if (rc) return rc;
  if (info == nullptr) {
    g_last_error = "info pointer is null";
    return DDB_EINVAL;
  }
  *info = 0;
  if (m == 0 || n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(m, n, lda);
  DevBuf A;
  if ((rc = stage_in(A, a_hi, a_lo, sa, s))) return rc;
  rc = ddb_rgetrf(m, n, A.p, A.p + sa, lda, ipiv, info, mode, stream);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(a_hi, A.p, sizeof(double) * sa, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a_lo, A.p + sa, sizeof(double) * sa, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(e, "device to host copy");
  return DDB_OK;
}

extern "C" int ddb_rgetrs_validate(char trans, int64_t n, int64_t nrhs, int64_t lda, int64_t ldb) {
  const int t = upflag(trans);
  if (t != 'N' && t != 'T' && t != 'C') return 1;     // lu.py:123-125
  if (n < 0) return 2;
  if (nrhs < 0) return 3;
  if (lda < (n > 1 ? n : 1)) return 5;
  if (ldb < (n > 1 ? n : 1)) return 8;
  return 0;
}

static int rgetrs_impl(bool f64, char trans, int64_t n, int64_t nrhs, const double* a_hi,
                       const double* a_lo, int64_t lda, const int64_t* ipiv, double* b_hi,
                       double* b_lo, int64_t ldb, int mode, void* stream) {
  const int rc = ddb_rgetrs_validate(trans, n, nrhs, lda, ldb);
  if (rc) return rc;
  if (mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM || (ipiv == nullptr && n > 0)) {
    g_last_error = ipiv == nullptr ? "ipiv pointer is null" : "unknown mode";
    return DDB_EINVAL;
  }
  if (n == 0 || nrhs == 0) return DDB_OK;             // lu.py:130-131
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  // laswp (lu.py:61-65) with the recorded pivots, as row interchanges of B
  void* ws = nullptr;
  const size_t swb = ((sizeof(long long) * (size_t)n + 255) / 256) * 256;
  cudaError_t e = cudaMallocAsync(&ws, swb + kPermBufBytes, s);
  if (e != cudaSuccess) return fail(e, "rgetrs workspace");
  std::vector<long long> sw((size_t)n);
  for (int64_t k = 0; k < n; ++k) sw[(size_t)k] = ipiv[k] - 1;
  e = cudaMemcpyAsync(ws, sw.data(), sizeof(long long) * (size_t)n, cudaMemcpyHostToDevice, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);  // sw is a host temporary
  GetrfArgs g{};
  g.m = n; g.n = nrhs; g.mn = n; g.lda = ldb;
  g.a_hi = b_hi; g.a_lo = b_lo;
  g.f64 = f64;
  g.swap = static_cast<long long*>(ws);
  PermBuf pb;
  pb.rows = reinterpret_cast<long long*>(static_cast<char*>(ws) + swb);
  pb.src = reinterpret_cast<int*>(static_cast<char*>(ws) + swb + 512 * 8);
  pb.n = reinterpret_cast<int*>(static_cast<char*>(ws) + swb + 512 * 12);
  int r = DDB_OK;
  const bool notr = upflag(trans) == 'N';
  if (e == cudaSuccess && notr) {
    e = launch_getrf_laswp(g, 0, n, 0, nrhs, s, 0, pb);
    if (e == cudaSuccess)
      r = rtrsm_impl(f64, 'L', 'L', 'N', 'U', n, nrhs, 1.0, 0.0, a_hi, a_lo, lda, b_hi, b_lo, ldb, mode, stream);
    if (e == cudaSuccess && r == DDB_OK)
      r = rtrsm_impl(f64, 'L', 'U', 'N', 'N', n, nrhs, 1.0, 0.0, a_hi, a_lo, lda, b_hi, b_lo, ldb, mode, stream);
  } else if (e == cudaSuccess) {
    r = rtrsm_impl(f64, 'L', 'U', 'T', 'N', n, nrhs, 1.0, 0.0, a_hi, a_lo, lda, b_hi, b_lo, ldb, mode, stream);
    if (r == DDB_OK)
      r = rtrsm_impl(f64, 'L', 'L', 'T', 'U', n, nrhs, 1.0, 0.0, a_hi, a_lo, lda, b_hi, b_lo, ldb, mode, stream);
    if (r == DDB_OK) e = launch_getrf_laswp(g, 0, n, 0, nrhs, s, 1, pb);
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (r != DDB_OK) return r;
  if (e != cudaSuccess) return fail(e, "rgetrs");
  if (e2 != cudaSuccess) return fail(e2, "workspace free");
  return DDB_OK;
}

extern "C" int ddb_rgetrs(char trans, int64_t n, int64_t nrhs, const double* a_hi,
                          const double* a_lo, int64_t lda, const int64_t* ipiv, double* b_hi,
                          double* b_lo, int64_t ldb, int mode, void* stream) {
  return rgetrs_impl(false, trans, n, nrhs, a_hi, a_lo, lda, ipiv, b_hi, b_lo, ldb, mode, stream);
}

extern "C" int ddb_dgetrs(char trans, int64_t n, int64_t nrhs, const double* a, int64_t lda,
                          const int64_t* ipiv, double* b, int64_t ldb, void* stream) {
  return rgetrs_impl(true, trans, n, nrhs, a, a, lda, ipiv, b, b, ldb, DDB_MODE_EXACT, stream);
}

extern "C" int ddb_rgetrs_host(char trans, int64_t n, int64_t nrhs, const double* a_hi, const double* a_lo,
                    int64_t lda, const int64_t* ipiv, double* b_hi, double* b_lo, int64_t ldb,
                    int mode, void* stream) {
  int rc = ddb_rgetrs_validate(trans, n, nrhs, lda, ldb);
  if (rc) return rc;
  if (n == 0 || nrhs == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(n, n, lda), sb = span(n, nrhs, ldb);
  DevBuf A, B;
  if ((rc = stage_in(A, a_hi, a_lo, sa, s))) return rc;
  if ((rc = stage_in(B, b_hi, b_lo, sb, s))) return rc;
  rc = ddb_rgetrs(trans, n, nrhs, A.p, A.p + sa, lda, ipiv, B.p, B.p + sb, ldb, mode, stream);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(b_hi, B.p, sizeof(double) * sb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(b_lo, B.p + sb, sizeof(double) * sb, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(e, "device to host copy");
  return DDB_OK;
}

// ---- blocked Cholesky (dd_potrf.cu) ----------------------------------------

extern "C" int ddb_rpotrf_validate(char uplo, int64_t n, int64_t lda) {
  const int u = upflag(uplo);
  if (u != 'U' && u != 'L') return 1;                 // chol.py:24-26
  if (n < 0) return 2;                                // chol.py:28
  if (lda < (n > 1 ? n : 1)) return 4;                // chol.py:29
  return 0;
}

static int rpotrf_impl(bool f64, char uplo, int64_t n, double* a_hi, double* a_lo, int64_t lda,
                       int64_t nb, int mode, void* stream, int* info) {
  const int rc = ddb_rpotrf_validate(uplo, n, lda);
  if (rc) return rc;
  NoPersistScope no_persist;   // trailing updates beside the panel stream
  if (mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM || info == nullptr) {
    g_last_error = info == nullptr ? "info pointer is null" : "unknown mode";
    return DDB_EINVAL;
  }
  *info = 0;
  if (n == 0) return DDB_OK;                          // chol.py:30-31
  // three block levels: outer width NB (the depth of the bulk trailing
  // Rsyrk / Rgemm: 1024 reaches the split algorithm's k >= 1024 regime),
  // middle width MB (the depth of the updates inside an outer panel) and
  // inner width ib <= kPotrfMaxNb (diagonal block in shared memory)
  if (nb <= 0) {
    static const int64_t nb_env = [] {
      const char* v = std::getenv("DDB_POTRF_NB");
      return v ? (int64_t)std::atoll(v) : (int64_t)0;
    }();
    // deeper outer panels pay off once the bulk trailing update dominates
    // the panel chain; exact mode gains nothing from depth.  Fast modes at
    // n = 8192: 256 -> 70.7 ms, 384 -> 69.0 ms, 512 -> 69.4 ms
    // (n = 4096: 256 best, 16.6 vs 17.9 ms; n = 16384: 384 ... 1024 alike)
    const bool fastm = mode != DDB_MODE_EXACT && mode != DDB_MODE_REFERENCE;
    nb = nb_env > 0 ? nb_env : (fastm && n >= 12288 ? 1024 : (fastm && n >= 6144 ? 384 : 256));
  }
  const int64_t NB = nb;
  const int64_t MB = NB > 256 ? 256 : NB;
  const int64_t ib = nb < kPotrfMaxNb ? nb : kPotrfMaxNb;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  retain_pool_memory();
  PotrfArgs p{};
  p.n = n; p.lda = lda; p.upper = upflag(uplo) == 'U';
  p.f64 = f64;
  p.fastacc = !f64 && (mode == DDB_MODE_FAST || mode == DDB_MODE_TWOSUM);
  p.a_hi = a_hi; p.a_lo = a_lo;
  // workspace: info | D, d0 (dd vectors), rec (MB dd: the middle panel's
  // reciprocals) | backup ('L') or S ('U'), n x n dd | 'U': the middle
  // diagonal block transposed (MB x MB), the middle transposed panel (n x
  // MB, 3 levels only) and two outer ones (n x NB; block J's is read by the trailing update
  // while J+1's is written)
  const size_t head = 256, vec = sizeof(double) * (size_t)n;
  const size_t recb = ((sizeof(double) * 2 * (size_t)MB + 255) / 256) * 256;
  const size_t full = sizeof(double) * (size_t)n * n;
  const size_t t_out = p.upper ? (size_t)n * NB : 0;
  const size_t t_mid = p.upper && MB < NB ? (size_t)n * MB : 0;
  const size_t t_dg = p.upper ? (size_t)MB * MB : 0;
  const size_t ws_bytes =
      head + 4 * vec + recb + 2 * full + sizeof(double) * 2 * (2 * t_out + t_mid + t_dg);
  void* ws = nullptr;
  cudaError_t e = cudaMallocAsync(&ws, ws_bytes, s);
  if (e != cudaSuccess) return fail(e, "workspace allocation");
  char* w = static_cast<char*>(ws);
  p.info = reinterpret_cast<int*>(w);
  unsigned* pmask = reinterpret_cast<unsigned*>(w + 64);   // kPotrfMaxPanel / 32 words
  double* d = reinterpret_cast<double*>(w + head);
  p.dh = d; p.dl = d + n;
  double* d0h = d + 2 * n;
  double* d0l = d + 3 * n;
  p.d0_hi = d0h; p.d0_lo = d0l;
  double* rec_h = d + 4 * n;
  double* rec_l = rec_h + MB;
  p.rec_hi = rec_h; p.rec_lo = rec_l;
  double* big = reinterpret_cast<double*>(w + head + 4 * vec + recb);
  double* tout_h = big + 2 * (size_t)n * n;          // outer T: hi[2] | lo[2]
  double* tout_l = tout_h + 2 * t_out;
  double* tmid_h = tout_l + 2 * t_out;               // middle T: hi | lo
  double* tmid_l = tmid_h + t_mid;
  double* tdg_h = tmid_l + t_mid;                    // 'U' diagonal block, transposed
  double* tdg_l = tdg_h + t_dg;
  int nl = 0;
  e = cudaMemsetAsync(ws, 0, head + 2 * vec, s);
  const size_t dpitch = sizeof(double) * (size_t)(lda + 1);
  if (e == cudaSuccess) e = cudaMemcpy2DAsync(d0h, 8, a_hi, dpitch, 8, n, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess && !f64)
    e = cudaMemcpy2DAsync(d0l, 8, a_lo, dpitch, 8, n, cudaMemcpyDeviceToDevice, s);
  if (e == cudaSuccess) {
    if (p.upper) {
      p.s_hi = big; p.s_lo = big + (size_t)n * n; p.lds = n;
      e = cudaMemsetAsync(big, 0, 2 * full, s);
    } else {
      double* bh = big;
      double* bl = big + (size_t)n * n;
      p.b_hi = bh; p.b_lo = bl;
      const size_t pitch = sizeof(double) * (size_t)lda, row = sizeof(double) * (size_t)n;
      e = cudaMemcpy2DAsync(bh, row, a_hi, pitch, row, n, cudaMemcpyDeviceToDevice, s);
      if (e == cudaSuccess && !f64)
        e = cudaMemcpy2DAsync(bl, row, a_lo, pitch, row, n, cudaMemcpyDeviceToDevice, s);
    }
  }
  Trace tr(s);
  // Streams: the panel work (diagonal blocks, panels, inner updates and the
  // lookahead update of the next block column) runs on a high-priority
  // stream `cs`; the bulk trailing update of each outer block runs on the
  // caller's stream `s`, overlapping the next panel.  Per element the
  // contributions still arrive in block order: `cs` waits for rest(J-1)
  // before update(J -> J+1), and rest(J) follows rest(J-1) on `s`.
  int rc2 = DDB_OK;
  cudaStream_t cs = nullptr;
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  if (e == cudaSuccess) e = panel_stream(&cs);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_a, cudaEventDisableTiming);
  if (e == cudaSuccess) e = cudaEventCreateWithFlags(&ev_b, cudaEventDisableTiming);
  // trailing update of columns [c0, c1) (rows >= c0) by factor rows / columns
  // [j0, j1):  'L': A(r, c) -= L(r, j0:j1) L(c, j0:j1)^T in place;
  //            'U': S(r, c) += T(r) T(c)^T, T(x) = U(j0:j1, x)^T stored from
  //                 column tb0 with leading dimension n - tb0
  auto update = [&](int64_t j0, int64_t j1, int64_t c0, int64_t c1, const double* th,
                    const double* tl, int64_t tb0, cudaStream_t st) -> int {
    const int64_t kb = j1 - j0, wd = c1 - c0, below = n - c1;
    void* sv = static_cast<void*>(st);
    int r;
    // fast modes, a narrow block column with few rows: one lean launch
    static const int64_t lean_rows = [] {
      const char* v = std::getenv("DDB_POTRF_LEAN_ROWS");
      return v ? (int64_t)std::atoll(v) : (int64_t)3072;
    }();
    if (p.fastacc && kb <= 256 && wd <= 256 && n - c0 <= lean_rows) {
      cudaError_t er;
      if (!p.upper)
        er = launch_potrf_lean_upd(a_hi + j0 * lda, a_lo + j0 * lda, lda, (int)kb, -1.0, a_hi, a_lo,
                                   lda, c0, n, c0, (int)wd, p.info, st);
      else
        er = launch_potrf_lean_upd(th - tb0, tl - tb0, n - tb0, (int)kb, 1.0, p.s_hi, p.s_lo, n, c0,
                                   n, c0, (int)wd, p.info, st);
      ++nl;
      return er == cudaSuccess ? DDB_OK : fail(er, "rpotrf update");
    }
    if (!p.upper) {
      const double *lh = a_hi + j0 * lda, *ll = a_lo + j0 * lda;
      r = syrk_any(f64, 'L', 'N', wd, kb, -1.0, 0.0, lh + c0, ll + c0, lda, 1.0, 0.0,
                    a_hi + c0 + c0 * lda, a_lo + c0 + c0 * lda, lda, mode, sv);
      if (r == DDB_OK && below > 0)
        r = gemm_any(f64, 'N', 'T', below, wd, kb, -1.0, 0.0, lh + c1, ll + c1, lda, lh + c0, ll + c0,
                      lda, 1.0, 0.0, a_hi + c1 + c0 * lda, a_lo + c1 + c0 * lda, lda, mode, sv);
    } else {
      const int64_t ldt = n - tb0;
      th -= tb0;
      tl -= tb0;                                     // th[x] = T(x) for column x
      r = syrk_any(f64, 'L', 'N', wd, kb, 1.0, 0.0, th + c0, tl + c0, ldt, 1.0, 0.0,
                    p.s_hi + c0 + c0 * n, p.s_lo + c0 + c0 * n, n, mode, sv);
      if (r == DDB_OK && below > 0)
        r = gemm_any(f64, 'N', 'T', below, wd, kb, 1.0, 0.0, th + c1, tl + c1, ldt, th + c0, tl + c0,
                      ldt, 1.0, 0.0, p.s_hi + c1 + c0 * n, p.s_lo + c1 + c0 * n, n, mode, sv);
    }
    return r;
  };
  auto transpose = [&](int64_t j0, int64_t j1, double* th, double* tl) -> cudaError_t {
    PotrfArgs q = p;
    q.t_hi = th;
    q.t_lo = tl;
    ++nl;
    return launch_potrf_transpose(q, j0, j1, (int)(j1 - j0), n - j1, cs);
  };
  // factor the middle panel [J0, J1) (width <= 256): its diagonal block by
  // inner blocks (diagonal kernel, the block's rows below the inner block,
  // the update of the rest of the diagonal block), then every row below the
  // middle panel against all of its columns in one potrf_rows_kernel launch
  // -- per element the same products in the same l order as the blocked
  // Rsyrk / Rgemm updates (exact mode stays bitwise)
  auto factor_mid = [&](int64_t J0, int64_t J1) -> int {
    const int64_t sa = p.upper ? lda : 1, sb = p.upper ? 1 : lda;   // P(c2, c) strides in A
    for (int64_t i0 = J0; i0 < J1; i0 += ib) {
      const int64_t i1 = i0 + ib < J1 ? i0 + ib : J1;
      PotrfArgs q = p;
      q.rec_hi = rec_h + (i0 - J0);
      q.rec_lo = rec_l + (i0 - J0);
      cudaError_t er = launch_potrf_diag(q, i0, i1, cs);
      ++nl;
      if (er == cudaSuccess && i1 < J1) {
        const size_t o = (size_t)i0 + (size_t)i0 * lda;
        const double* al = f64 ? nullptr : a_lo + o;
        er = launch_potrf_rows(q, i0, (int)(i1 - i0), i1, J1, a_hi + o, al, sa, sb, q.rec_hi,
                               q.rec_lo, nullptr, cs);
        if (er == cudaSuccess) er = launch_potrf_blockupd(p, i0, i1, J1, cs);
        nl += 2;
      }
      if (er != cudaSuccess) return fail(er, "rpotrf panel");
    }
    tr.mark("diagblk_done", J0, cs);
    if (J1 < n) {
      const int wd = (int)(J1 - J0);
      const double *ph, *pl;
      int64_t sr = 1, sc = lda;
      cudaError_t er = cudaSuccess;
      if (p.upper) {                 // P(c2, c) = U(J0 + c, J0 + c2), read coalesced
        PotrfArgs q = p;
        q.t_hi = tdg_h;
        q.t_lo = tdg_l;
        er = launch_potrf_transpose(q, J0, J0, wd, wd, cs);
        ++nl;
        ph = tdg_h; pl = f64 ? nullptr : tdg_l; sc = wd;
      } else {
        const size_t o = (size_t)J0 + (size_t)J0 * lda;
        ph = a_hi + o; pl = f64 ? nullptr : a_lo + o;
      }
      if (er == cudaSuccess)
        er = launch_potrf_rows(p, J0, wd, J1, n, ph, pl, sr, sc, rec_h, rec_l, pmask, cs);
      nl += f64 ? 1 : 2;
      if (er != cudaSuccess) return fail(er, "rpotrf panel");
    }
    return DDB_OK;
  };
  // factor the outer panel [J0, J1): middle panels, each followed by the
  // update (depth MB) of the rest of the outer panel's columns.  Every
  // element still receives its updates in pivot-block order.
  auto factor_outer = [&](int64_t J0, int64_t J1) -> int {
    for (int64_t m0 = J0; m0 < J1; m0 += MB) {
      const int64_t m1 = m0 + MB < J1 ? m0 + MB : J1;
      int r = factor_mid(m0, m1);
      if (r != DDB_OK) return r;
      if (m1 < J1) {
        cudaError_t er = cudaSuccess;
        if (p.upper && (er = transpose(m0, m1, tmid_h, tmid_l)) != cudaSuccess)
          return fail(er, "rpotrf transpose");
        r = update(m0, m1, m1, J1, tmid_h, tmid_l, m1, cs);
        if (r != DDB_OK) return r;
      }
    }
    return DDB_OK;
  };
  if (e == cudaSuccess) e = cudaEventRecord(ev_a, s);      // workspace ready
  if (e == cudaSuccess) e = cudaStreamWaitEvent(cs, ev_a, 0);
  if (e == cudaSuccess) rc2 = factor_outer(0, NB < n ? NB : n);
  tr.mark("panel_done", 0, cs);
  bool have_rest = false;
  for (int64_t J0 = 0; e == cudaSuccess && rc2 == DDB_OK; J0 += NB) {
    const int64_t J1 = J0 + NB < n ? J0 + NB : n;
    if (J1 >= n) break;
    const int64_t J2 = J1 + NB < n ? J1 + NB : n;
    double* th = tout_h + ((J0 / NB) & 1) * t_out;
    double* tl = tout_l + ((J0 / NB) & 1) * t_out;
    if (p.upper) e = transpose(J0, J1, th, tl);
    if (e == cudaSuccess) e = cudaEventRecord(ev_a, cs);    // panel J (+ T) done
    if (e == cudaSuccess && have_rest) e = cudaStreamWaitEvent(cs, ev_b, 0);   // rest(J-1)
    if (e == cudaSuccess) e = cudaStreamWaitEvent(s, ev_a, 0);
    if (e != cudaSuccess) break;
    if (J2 < n) {
      tr.mark("rest_start", J0, s);
      rc2 = update(J0, J1, J2, n, th, tl, J1, s);           // rest(J)
      if (rc2 != DDB_OK) break;
      tr.mark("rest_done", J0, s);
      e = cudaEventRecord(ev_b, s);
      have_rest = true;
      if (e != cudaSuccess) break;
    }
    tr.mark("upd_start", J0, cs);
    rc2 = update(J0, J1, J1, J2, th, tl, J1, cs);            // update(J -> J+1)
    tr.mark("upd_done", J0, cs);
    if (rc2 == DDB_OK) rc2 = factor_outer(J1, J2);
    tr.mark("panel_done", J1, cs);
  }
  // join the panel stream back into `s`
  if (cs != nullptr) {
    cudaError_t ej = cudaEventRecord(ev_a, cs);
    if (ej == cudaSuccess) ej = cudaStreamWaitEvent(s, ev_a, 0);
    if (e == cudaSuccess) e = ej;
  }
  if (ev_a) cudaEventDestroy(ev_a);
  if (ev_b) cudaEventDestroy(ev_b);
  if (e == cudaSuccess && rc2 == DDB_OK && !p.upper) {
    e = launch_potrf_restore(p, s);
    ++nl;
  }
  g_launches += nl;
  int hinfo = 0;
  if (e == cudaSuccess && rc2 == DDB_OK) {
    e = cudaMemcpyAsync(&hinfo, p.info, sizeof(int), cudaMemcpyDeviceToHost, s);
    if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  }
  cudaError_t e2 = cudaFreeAsync(ws, s);
  if (rc2 != DDB_OK) return rc2;
  if (e != cudaSuccess) return fail(e, "rpotrf");
  if (e2 != cudaSuccess) return fail(e2, "workspace free");
  *info = hinfo;
  return DDB_OK;
}

extern "C" int ddb_rpotrf(char uplo, int64_t n, double* a_hi, double* a_lo, int64_t lda,
                          int64_t nb, int mode, void* stream, int* info) {
  return rpotrf_impl(false, uplo, n, a_hi, a_lo, lda, nb, mode, stream, info);
}

extern "C" int ddb_dpotrf(char uplo, int64_t n, double* a, int64_t lda, int64_t nb, void* stream,
                          int* info) {
  return rpotrf_impl(true, uplo, n, a, a, lda, nb, DDB_MODE_EXACT, stream, info);
}

extern "C" int ddb_rpotrf_host(char uplo, int64_t n, double* a_hi, double* a_lo, int64_t lda, int64_t nb,
                    int mode, void* stream, int* info) {
  int rc = ddb_rpotrf_validate(uplo, n, lda);
  if (rc) return rc;
  if (info == nullptr) {
    g_last_error = "info pointer is null";
    return DDB_EINVAL;
  }
  *info = 0;
  if (n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(n, n, lda);
  DevBuf A;
  if ((rc = stage_in(A, a_hi, a_lo, sa, s))) return rc;
  rc = ddb_rpotrf(uplo, n, A.p, A.p + sa, lda, nb, mode, stream, info);
  if (rc) return rc;
  cudaError_t e = cudaMemcpyAsync(a_hi, A.p, sizeof(double) * sa, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(a_lo, A.p + sa, sizeof(double) * sa, cudaMemcpyDeviceToHost, s);
  if (e == cudaSuccess) e = cudaStreamSynchronize(s);
  if (e != cudaSuccess) return fail(e, "device to host copy");
  return DDB_OK;
}

// ---- binary64 host-buffer entry points (one plane, staged) ------------------

extern "C" int ddb_dtrsm_host(char side, char uplo, char transa, char diag, int64_t m, int64_t n,
                              double alpha, const double* a, int64_t lda, double* b, int64_t ldb,
                              void* stream) {
  int rc = ddb_rtrsm_validate(side, uplo, transa, diag, m, n, lda, ldb);
  if (rc) return rc;
  if (m == 0 || n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t na = upflag(side) == 'L' ? m : n;
  const int64_t sa = alpha == 0.0 ? 0 : span(na, na, lda), sb = span(m, n, ldb);
  DevBuf A, B;
  if ((rc = stage_in1(A, a, sa, s)) || (rc = stage_in1(B, b, sb, s))) return rc;
  rc = ddb_dtrsm(side, uplo, transa, diag, m, n, alpha, A.p, lda, B.p, ldb, stream);
  return rc ? rc : stage_out1(b, B, sb, s);
}

extern "C" int ddb_dgetrf_host(int64_t m, int64_t n, double* a, int64_t lda, int64_t* ipiv,
                               int* info, void* stream) {
  int rc = ddb_rgetrf_validate(m, n, lda);
  if (rc) return rc;
  if (info == nullptr) {
    g_last_error = "info pointer is null";
    return DDB_EINVAL;
  }
  *info = 0;
  if (m == 0 || n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(m, n, lda);
  DevBuf A;
  if ((rc = stage_in1(A, a, sa, s))) return rc;
  rc = ddb_dgetrf(m, n, A.p, lda, ipiv, info, stream);
  return rc ? rc : stage_out1(a, A, sa, s);
}

extern "C" int ddb_dgetrs_host(char trans, int64_t n, int64_t nrhs, const double* a, int64_t lda,
                               const int64_t* ipiv, double* b, int64_t ldb, void* stream) {
  int rc = ddb_rgetrs_validate(trans, n, nrhs, lda, ldb);
  if (rc) return rc;
  if (n == 0 || nrhs == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(n, n, lda), sb = span(n, nrhs, ldb);
  DevBuf A, B;
  if ((rc = stage_in1(A, a, sa, s)) || (rc = stage_in1(B, b, sb, s))) return rc;
  rc = ddb_dgetrs(trans, n, nrhs, A.p, lda, ipiv, B.p, ldb, stream);
  return rc ? rc : stage_out1(b, B, sb, s);
}

extern "C" int ddb_dpotrf_host(char uplo, int64_t n, double* a, int64_t lda, int64_t nb,
                               void* stream, int* info) {
  int rc = ddb_rpotrf_validate(uplo, n, lda);
  if (rc) return rc;
  if (info == nullptr) {
    g_last_error = "info pointer is null";
    return DDB_EINVAL;
  }
  *info = 0;
  if (n == 0) return DDB_OK;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int64_t sa = span(n, n, lda);
  DevBuf A;
  if ((rc = stage_in1(A, a, sa, s))) return rc;
  rc = ddb_dpotrf(uplo, n, A.p, lda, nb, stream, info);
  return rc ? rc : stage_out1(a, A, sa, s);
}
