// capi_mgpu.cu -- single-process multi-GPU entry points (include/ddblas.h):
//   ddb_rgemm_mgpu / ddb_rsyrk_mgpu, operands resident on devices[0].
//
// The same decomposition as the one-process-per-GPU path (parallel.py) --
// the reference's Rgemm_par column panels (mpblas/parallel.py:102-157) --
// for C callers that drive several GPUs from one thread.  Device i owns a
// column slab of C (Rsyrk: triangle-balanced slabs, each one Rsyrk diagonal
// block + one Rgemm rectangle, the per-element sequence of a full Rsyrk).
//
// Data movement over NVLink (peer access enabled per device pair):
//   * op(B) / C slabs: one peer copy each from the root, before anything else;
//   * op(A): streamed in k-panels down a CHAIN root -> d1 -> d2 -> ... (each
//     device forwards the panel it received to the next), so the root's links
//     carry A once and every link carries it once; each device starts its
//     panel-p GEMM as soon as panel p has landed (copy and compute streams,
//     events per panel), overlapping the rest of the chain.  Panels run as
//     successive GEMMs with beta = 1 after the first, which is the
//     reference's own per-element order when transa = 'N' (beta-scale, then
//     l ascending), so exact mode stays bitwise equal to one call; for
//     transa = 'T' exact mode (sum from zero, then combine) keeps one panel.
// Buffers are cached per device and grown on demand (no per-call cudaMalloc
// after the first), which serialises concurrent mgpu calls (one mutex).
// Ordering: the call first waits for all work already queued on the root
// device (cudaDeviceSynchronize), so operands produced on any stream are
// complete; it returns when C is complete on the root (synchronous).
// A device may appear more than once (slabs then share a GPU), which is how
// the tests exercise the split on one GPU.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <map>
#include <mutex>
#include <vector>

#include "../../include/ddblas.h"
#include "host.h"
#include "internal.h"

using namespace ddb;
using namespace ddb::host;

namespace {

constexpr int64_t kTile = 64;
constexpr int64_t kPanel = 2048;      // k per streamed panel of op(A)

std::vector<std::pair<int64_t, int64_t>> column_split(int64_t n, int p) {
  const int64_t nt = (n + kTile - 1) / kTile;
  std::vector<std::pair<int64_t, int64_t>> out;
  for (int r = 0; r < p; ++r) {
    const int64_t t0 = nt * r / p, t1 = nt * (r + 1) / p;
    out.emplace_back(t0 * kTile < n ? t0 * kTile : n, t1 * kTile < n ? t1 * kTile : n);
  }
  return out;
}

// equal triangle area per slab ('U': the area left of column j ~ j^2)
std::vector<std::pair<int64_t, int64_t>> triangle_split(int64_t n, int p, bool upper) {
  const int64_t tile = 16, nt = (n + tile - 1) / tile;
  std::vector<int64_t> b{0};
  for (int r = 1; r < p; ++r) {
    const double f = upper ? std::sqrt((double)r / p) : 1.0 - std::sqrt((double)(p - r) / p);
    int64_t t = (int64_t)std::llround(f * nt);
    if (t > nt) t = nt;
    if (t < b.back()) t = b.back();
    b.push_back(t);
  }
  b.push_back(nt);
  std::vector<std::pair<int64_t, int64_t>> out;
  for (int r = 0; r < p; ++r)
    out.emplace_back(b[r] * tile < n ? b[r] * tile : n, b[r + 1] * tile < n ? b[r + 1] * tile : n);
  return out;
}

// ---- per-device cache: buffers and the copy / compute streams ----------------

std::mutex g_mgpu_mu;

struct DevCache {
  double* buf = nullptr;
  size_t cap = 0;                     // doubles
  cudaStream_t copy = nullptr, comp = nullptr;
};
// (device, slot) -> entry; std::map nodes never move, so the pointers handed
// out stay valid while later slots are added
std::map<std::pair<int, int>, DevCache> g_cache;

int cache_get(int dev, int slot, size_t doubles, DevCache** out) {
  DevCache& c = g_cache[{dev, slot}];
  cudaError_t e = cudaSetDevice(dev);
  if (e == cudaSuccess && c.copy == nullptr) e = cudaStreamCreateWithFlags(&c.copy, cudaStreamNonBlocking);
  if (e == cudaSuccess && c.comp == nullptr) e = cudaStreamCreateWithFlags(&c.comp, cudaStreamNonBlocking);
  if (e == cudaSuccess && c.cap < doubles) {
    if (c.buf) cudaFree(c.buf);
    c.buf = nullptr;
    c.cap = 0;
    e = cudaMalloc(reinterpret_cast<void**>(&c.buf), sizeof(double) * doubles);
    if (e == cudaSuccess) c.cap = doubles;
  }
  if (e != cudaSuccess) return fail(e, "mgpu device buffers");
  *out = &c;
  return DDB_OK;
}

void enable_peer(int a, int b) {
  if (a == b) return;
  int ok = 0;
  if (cudaDeviceCanAccessPeer(&ok, a, b) != cudaSuccess || !ok) return;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(a);
  const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
  if (e == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
  cudaSetDevice(prev);
}

int peer_copy_2d(double* dst, int64_t dld, int ddev, const double* src, int64_t sld, int sdev,
                 int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return DDB_OK;
  cudaError_t e;
  if (ddev == sdev) {
    e = cudaMemcpy2DAsync(dst, sizeof(double) * dld, src, sizeof(double) * sld,
                          sizeof(double) * rows, cols, cudaMemcpyDeviceToDevice, st);
  } else {
    cudaMemcpy3DPeerParms p{};
    p.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), sizeof(double) * sld,
                                   sizeof(double) * rows, cols);
    p.srcDevice = sdev;
    p.dstPtr = make_cudaPitchedPtr(dst, sizeof(double) * dld, sizeof(double) * rows, cols);
    p.dstDevice = ddev;
    p.extent = make_cudaExtent(sizeof(double) * rows, cols, 1);
    e = cudaMemcpy3DPeerAsync(&p, st);
  }
  return e == cudaSuccess ? DDB_OK : fail(e, "peer copy");
}

// The streamed operand: op(A) panels [k0, k1) live at the same offsets in
// every device's copy (same leading dimension as on the root).
struct AView {
  bool kcols;                         // transa 'N': panel = columns k0..k1 of A (m x k)
  int64_t rows_op, lda;               // op(A) rows
  const double *hi, *lo;              // root planes
  int64_t span;                       // doubles per plane
  const double* at(const double* p, int64_t k0) const { return kcols ? p + k0 * lda : p + k0; }
  // copy panel [k0, k1) of both planes from src (device sdev) to dst (device ddev)
  int copy(double* dst, int ddev, const double* src_h, const double* src_l, int sdev, int64_t k0,
           int64_t k1, cudaStream_t st) const {
    int rc = DDB_OK;
    for (int pl = 0; pl < 2 && rc == DDB_OK; ++pl) {
      const double* s = pl ? src_l : src_h;
      double* d = dst + pl * span;
      if (kcols) rc = peer_copy_2d(d + k0 * lda, lda, ddev, s + k0 * lda, lda, sdev, rows_op, k1 - k0, st);
      else rc = peer_copy_2d(d + k0, lda, ddev, s + k0, lda, sdev, k1 - k0, rows_op, st);
    }
    return rc;
  }
};

struct Panels {
  std::vector<int64_t> b;             // panel boundaries over k
  int count() const { return (int)b.size() - 1; }
};

Panels make_panels(int64_t k, bool allowed) {
  Panels p;
  p.b.push_back(0);
  if (allowed && k > kPanel) {
    for (int64_t x = kPanel; x < k; x += kPanel) p.b.push_back(x);
  }
  p.b.push_back(k);
  return p;
}

struct Events {
  std::vector<cudaEvent_t> ev;
  ~Events() {
    for (auto e : ev) cudaEventDestroy(e);
  }
  cudaError_t make(int count) {
    ev.assign(count, nullptr);
    for (auto& e : ev) {
      const cudaError_t r = cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
      if (r != cudaSuccess) return r;
    }
    return cudaSuccess;
  }
};

int check_args(int ndev, const int* devices, int mode) {
  if (ndev < 1 || devices == nullptr || mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM) {
    g_last_error = "bad device list or mode";
    return DDB_EINVAL;
  }
  return DDB_OK;
}

// Common driver: slab i computes its panels with `gemm(i, cache, p, k0, k1,
// a_hi, a_lo)` on its compute stream after op(A) panel p has landed on its
// device; `stage_in(i, cache)` / `stage_out(i, cache)` move its B / C slab.
template <class StageIn, class Gemm, class StageOut>
int drive(int ndev, const int* devices, const AView& A, const Panels& P,
          const std::vector<bool>& active, size_t slab_doubles_extra, StageIn stage_in, Gemm gemm,
          StageOut stage_out) {
  const int root = devices[0];
  int prev = 0;
  cudaGetDevice(&prev);
  cudaError_t e = cudaSetDevice(root);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();     // ordering contract (see header)
  if (e != cudaSuccess) return fail(e, "mgpu root synchronize");
  std::map<int, int> slot_of;
  std::vector<DevCache*> cache(ndev, nullptr);
  int rc = DDB_OK;
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    enable_peer(devices[i], root);
    enable_peer(root, devices[i]);
    if (i > 0) {
      enable_peer(devices[i], devices[i - 1]);
      enable_peer(devices[i - 1], devices[i]);
    }
    const int slot = slot_of[devices[i]]++;
    rc = cache_get(devices[i], slot, i == 0 ? 0 : 2 * A.span + slab_doubles_extra, &cache[i]);
  }
  const int np = P.count();
  std::vector<Events> landed(ndev);
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    cudaSetDevice(devices[i]);
    if ((e = landed[i].make(np)) != cudaSuccess) rc = fail(e, "mgpu events");
  }
  // B / C slabs first (small), then the chain of A panels
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    cudaSetDevice(devices[i]);
    if (active[i]) rc = stage_in(i, *cache[i]);
  }
  for (int p = 0; p < np && rc == DDB_OK; ++p) {
    const int64_t k0 = P.b[p], k1 = P.b[p + 1];
    int src = 0;
    for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
      cudaSetDevice(devices[i]);
      DevCache& c = *cache[i];
      if (i > 0) {
        // forward from the previous device in the chain (its copy of panel p
        // is complete once its `landed` event fired)
        if (src > 0) cudaStreamWaitEvent(c.copy, landed[src].ev[p], 0);
        const double* sh = src == 0 ? A.hi : cache[src]->buf;
        const double* sl = src == 0 ? A.lo : cache[src]->buf + A.span;
        rc = A.copy(c.buf, devices[i], sh, sl, devices[src], k0, k1, c.copy);
        if (rc == DDB_OK && (e = cudaEventRecord(landed[i].ev[p], c.copy)) != cudaSuccess)
          rc = fail(e, "mgpu event");
        src = i;
      } else if ((e = cudaEventRecord(landed[0].ev[p], c.comp)) != cudaSuccess) {
        rc = fail(e, "mgpu event");
      }
      if (rc != DDB_OK || !active[i]) continue;
      cudaStreamWaitEvent(c.comp, landed[i].ev[p], 0);
      const double* ah = i == 0 ? A.hi : c.buf;
      const double* al = i == 0 ? A.lo : c.buf + A.span;
      rc = gemm(i, c, p, k0, k1, ah, al);
    }
  }
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    cudaSetDevice(devices[i]);
    if (active[i]) rc = stage_out(i, *cache[i]);
  }
  for (int i = 0; i < ndev; ++i) {
    cudaSetDevice(devices[i]);
    e = cudaStreamSynchronize(cache[i] ? cache[i]->comp : nullptr);
    if (rc == DDB_OK && e != cudaSuccess) rc = fail(e, "mgpu synchronize");
    if (cache[i]) {
      e = cudaStreamSynchronize(cache[i]->copy);
      if (rc == DDB_OK && e != cudaSuccess) rc = fail(e, "mgpu synchronize");
    }
  }
  cudaSetDevice(prev);
  return rc;
}

}  // namespace

extern "C" {

int ddb_rgemm_mgpu(char transa, char transb, int64_t m, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   const double* b_hi, const double* b_lo, int64_t ldb,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc, int mode, int ndev,
                   const int* devices) {
  int rc = ddb_rgemm_validate(transa, transb, m, n, k, lda, ldb, ldc);
  if (rc) return rc;
  if ((rc = check_args(ndev, devices, mode))) return rc;
  if (m == 0 || n == 0 || ((is_zero(alpha_hi, alpha_lo) || k == 0) && is_one(beta_hi, beta_lo)))
    return DDB_OK;
  std::lock_guard<std::mutex> lock(g_mgpu_mu);
  const bool na = upflag(transa) == 'N', nbn = upflag(transb) == 'N';
  const int root = devices[0];
  const bool read_c = !is_zero(beta_hi, beta_lo);
  const auto blocks = column_split(n, ndev);
  AView A{na, m, lda, a_hi, a_lo, span(na ? m : k, na ? k : m, lda)};
  // k-panels (alpha == 0 / k == 0 calls have no k to stream: one empty panel)
  const bool trivial = is_zero(alpha_hi, alpha_lo) || k == 0;
  const Panels P = make_panels(k, !trivial && (na || mode != DDB_MODE_EXACT));
  std::vector<bool> active(ndev);
  for (int i = 0; i < ndev; ++i) active[i] = blocks[i].second > blocks[i].first;
  // per slab (i > 0): op(B)(:, J) packed k x w ('N') or w x k ('T'), C slab m x w (ld m)
  int64_t wmax = 0;
  for (auto& b : blocks) wmax = b.second - b.first > wmax ? b.second - b.first : wmax;
  const size_t extra = 2 * (size_t)k * wmax + 2 * (size_t)m * wmax;
  auto b_of = [&](DevCache& c) { return c.buf + 2 * A.span; };
  auto c_of = [&](DevCache& c) { return c.buf + 2 * A.span + 2 * (size_t)k * wmax; };
  auto stage_in = [&](int i, DevCache& c) {
    if (i == 0) return DDB_OK;
    const int64_t j0 = blocks[i].first, w = blocks[i].second - j0;
    int r = DDB_OK;
    for (int pl = 0; pl < 2 && r == DDB_OK; ++pl) {
      const double* bp = pl ? b_lo : b_hi;
      double* bd = b_of(c) + pl * (size_t)k * w;
      r = nbn ? peer_copy_2d(bd, k, devices[i], bp + j0 * ldb, ldb, root, k, w, c.copy)
              : peer_copy_2d(bd, w, devices[i], bp + j0, ldb, root, w, k, c.copy);
      if (r == DDB_OK && read_c)   // m rows of each column: the padding stays on the root
        r = peer_copy_2d(c_of(c) + pl * (size_t)m * w, m, devices[i],
                         (pl ? c_lo : c_hi) + j0 * ldc, ldc, root, m, w, c.copy);
    }
    return r;
  };
  auto gemm = [&](int i, DevCache& c, int p, int64_t k0, int64_t k1, const double* ah,
                  const double* al) {
    const int64_t j0 = blocks[i].first, w = blocks[i].second - j0;
    const double bh = p == 0 ? beta_hi : 1.0, bl = p == 0 ? beta_lo : 0.0;
    void* sv = static_cast<void*>(c.comp);
    if (i == 0)   // the root's slab in place
      return ddb_rgemm(transa, transb, m, w, k1 - k0, alpha_hi, alpha_lo, A.at(ah, k0),
                       A.at(al, k0), lda,
                       nbn ? b_hi + j0 * ldb + k0 : b_hi + j0 + k0 * ldb,
                       nbn ? b_lo + j0 * ldb + k0 : b_lo + j0 + k0 * ldb, ldb, bh, bl,
                       c_hi + j0 * ldc, c_lo + j0 * ldc, ldc, mode, sv);
    const double* bd = b_of(c);
    const size_t bpl = (size_t)k * w;
    const int64_t bld = nbn ? k : w;
    const int64_t boff = nbn ? k0 : k0 * w;
    double* cd = c_of(c);
    const size_t cpl = (size_t)m * w;
    return ddb_rgemm(transa, transb, m, w, k1 - k0, alpha_hi, alpha_lo, A.at(ah, k0),
                     A.at(al, k0), lda, bd + boff, bd + bpl + boff, bld, bh, bl, cd, cd + cpl, m,
                     mode, sv);
  };
  auto stage_out = [&](int i, DevCache& c) {
    if (i == 0) return DDB_OK;
    const int64_t j0 = blocks[i].first, w = blocks[i].second - j0;
    int r = DDB_OK;
    for (int pl = 0; pl < 2 && r == DDB_OK; ++pl)
      r = peer_copy_2d((pl ? c_lo : c_hi) + j0 * ldc, ldc, root, c_of(c) + pl * (size_t)m * w, m,
                       devices[i], m, w, c.comp);
    return r;
  };
  return drive(ndev, devices, A, P, active, extra, stage_in, gemm, stage_out);
}

int ddb_rsyrk_mgpu(char uplo, char trans, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc, int mode, int ndev,
                   const int* devices) {
  int rc = ddb_rsyrk_validate(uplo, trans, n, k, lda, ldc);
  if (rc) return rc;
  if ((rc = check_args(ndev, devices, mode))) return rc;
  if (n == 0 || ((is_zero(alpha_hi, alpha_lo) || k == 0) && is_one(beta_hi, beta_lo)))
    return DDB_OK;
  std::lock_guard<std::mutex> lock(g_mgpu_mu);
  const bool up = upflag(uplo) == 'U', tn = upflag(trans) == 'N';
  const char ta = tn ? 'N' : 'T', tb = tn ? 'T' : 'N';
  const int root = devices[0];
  const auto blocks = triangle_split(n, ndev, up);
  AView A{tn, n, lda, a_hi, a_lo, span(tn ? n : k, tn ? k : n, lda)};
  const bool trivial = is_zero(alpha_hi, alpha_lo) || k == 0;
  const Panels P = make_panels(k, !trivial && (tn || mode != DDB_MODE_EXACT));
  std::vector<bool> active(ndev);
  for (int i = 0; i < ndev; ++i) active[i] = blocks[i].second > blocks[i].first;
  int64_t wmax = 0;
  for (auto& b : blocks) wmax = b.second - b.first > wmax ? b.second - b.first : wmax;
  const size_t extra = 2 * (size_t)n * wmax;                // the whole column slab (ld n)
  auto c_of = [&](DevCache& c) { return c.buf + 2 * A.span; };
  auto stage_in = [&](int i, DevCache& c) {
    if (i == 0) return DDB_OK;
    const int64_t j0 = blocks[i].first, w = blocks[i].second - j0;
    int r = DDB_OK;   // the whole slab: the other triangle must come back unchanged
    for (int pl = 0; pl < 2 && r == DDB_OK; ++pl)
      r = peer_copy_2d(c_of(c) + pl * (size_t)n * w, n, devices[i], (pl ? c_lo : c_hi) + j0 * ldc,
                       ldc, root, n, w, c.copy);
    return r;
  };
  auto gemm = [&](int i, DevCache& c, int p, int64_t k0, int64_t k1, const double* ah0,
                  const double* al0) {
    const int64_t j0 = blocks[i].first, j1 = blocks[i].second, w = j1 - j0;
    const double bh = p == 0 ? beta_hi : 1.0, bl = p == 0 ? beta_lo : 0.0;
    const double* ah = A.at(ah0, k0);
    const double* al = A.at(al0, k0);
    double *ch, *cl;
    int64_t ld;
    if (i == 0) { ch = c_hi + j0 * ldc; cl = c_lo + j0 * ldc; ld = ldc; }
    else { ch = c_of(c); cl = c_of(c) + (size_t)n * w; ld = n; }
    // rows [r0, r1) of op(A) as a stored view: offset r0 ('N') or r0 * lda ('T')
    auto arow = [&](const double* q, int64_t r0) { return tn ? q + r0 : q + r0 * lda; };
    void* sv = static_cast<void*>(c.comp);
    const int64_t kw = k1 - k0;
    int r = ddb_rsyrk(uplo, trans, w, kw, alpha_hi, alpha_lo, arow(ah, j0), arow(al, j0), lda, bh,
                      bl, ch + j0, cl + j0, ld, mode, sv);
    if (r == DDB_OK && up && j0 > 0)        // rows [0, j0) x cols J
      r = ddb_rgemm(ta, tb, j0, w, kw, alpha_hi, alpha_lo, arow(ah, 0), arow(al, 0), lda,
                    arow(ah, j0), arow(al, j0), lda, bh, bl, ch, cl, ld, mode, sv);
    if (r == DDB_OK && !up && j1 < n)       // rows [j1, n) x cols J
      r = ddb_rgemm(ta, tb, n - j1, w, kw, alpha_hi, alpha_lo, arow(ah, j1), arow(al, j1), lda,
                    arow(ah, j0), arow(al, j0), lda, bh, bl, ch + j1, cl + j1, ld, mode, sv);
    return r;
  };
  auto stage_out = [&](int i, DevCache& c) {
    if (i == 0) return DDB_OK;
    const int64_t j0 = blocks[i].first, w = blocks[i].second - j0;
    int r = DDB_OK;
    for (int pl = 0; pl < 2 && r == DDB_OK; ++pl)
      r = peer_copy_2d((pl ? c_lo : c_hi) + j0 * ldc, ldc, root, c_of(c) + pl * (size_t)n * w, n,
                       devices[i], n, w, c.comp);
    return r;
  };
  return drive(ndev, devices, A, P, active, extra, stage_in, gemm, stage_out);
}

}  // extern "C"
