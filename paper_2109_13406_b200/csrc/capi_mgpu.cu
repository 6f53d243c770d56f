// capi_mgpu.cu -- single-process multi-GPU entry points (include/ddblas.h):
//   ddb_rgemm_mgpu / ddb_rsyrk_mgpu, operands resident on devices[0].
//
// The same decomposition as the one-process-per-GPU path (parallel.py) --
// the reference's Rgemm_par column panels (mpblas/parallel.py:102-157) --
// for C callers that drive several GPUs from one thread: device i gets op(A)
// and its column slab of op(B) / C by peer copies over NVLink
// (cudaMemcpyPeerAsync / cudaMemcpy3DPeerAsync), runs the single-GPU kernel
// on its slab, and copies the slab back.  Rsyrk uses triangle-balanced slabs,
// each one Rsyrk diagonal block + one Rgemm rectangle (the per-element
// sequence of a full Rsyrk).  Exact mode is bitwise equal to the single-GPU
// call.  A device may appear more than once (slabs then share a GPU), which
// is how the tests exercise the split on one GPU.  Synchronous.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/ddblas.h"
#include "host.h"
#include "internal.h"

using namespace ddb;
using namespace ddb::host;

namespace {

constexpr int64_t kTile = 64;

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

struct Slab {                 // one device's share
  int dev = 0;
  cudaStream_t st = nullptr;
  double *a = nullptr, *b = nullptr, *c = nullptr;   // device copies (hi | lo)
};

int peer_copy(double* dst, int ddev, const double* src, int sdev, int64_t count, cudaStream_t st) {
  if (count <= 0) return DDB_OK;
  const cudaError_t e = cudaMemcpyPeerAsync(dst, ddev, src, sdev, sizeof(double) * count, st);
  return e == cudaSuccess ? DDB_OK : fail(e, "peer copy");
}

// 2-D peer copy: `rows` x `cols` doubles, source leading dimension sld
int peer_copy_2d(double* dst, int64_t dld, int ddev, const double* src, int64_t sld, int sdev,
                 int64_t rows, int64_t cols, cudaStream_t st) {
  if (rows <= 0 || cols <= 0) return DDB_OK;
  cudaMemcpy3DPeerParms p{};
  p.srcPtr = make_cudaPitchedPtr(const_cast<double*>(src), sizeof(double) * sld,
                                 sizeof(double) * rows, cols);
  p.srcDevice = sdev;
  p.dstPtr = make_cudaPitchedPtr(dst, sizeof(double) * dld, sizeof(double) * rows, cols);
  p.dstDevice = ddev;
  p.extent = make_cudaExtent(sizeof(double) * rows, cols, 1);
  const cudaError_t e = cudaMemcpy3DPeerAsync(&p, st);
  return e == cudaSuccess ? DDB_OK : fail(e, "peer copy 2d");
}

// release everything and restore the caller's device
int finish(std::vector<Slab>& slabs, int prev_dev, int rc) {
  for (auto& s : slabs) {
    cudaSetDevice(s.dev);
    if (s.st) {
      const cudaError_t e = cudaStreamSynchronize(s.st);
      if (rc == DDB_OK && e != cudaSuccess) rc = fail(e, "mgpu synchronize");
    }
    if (s.a) cudaFree(s.a);
    if (s.b) cudaFree(s.b);
    if (s.c) cudaFree(s.c);
    if (s.st) cudaStreamDestroy(s.st);
  }
  cudaSetDevice(prev_dev);
  return rc;
}

int setup(std::vector<Slab>& slabs, int ndev, const int* devices, int* prev_dev) {
  if (cudaGetDevice(prev_dev) != cudaSuccess) *prev_dev = 0;
  slabs.resize(ndev);
  for (int i = 0; i < ndev; ++i) {
    slabs[i].dev = devices[i];
    cudaError_t e = cudaSetDevice(devices[i]);
    if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&slabs[i].st, cudaStreamNonBlocking);
    if (e != cudaSuccess) return fail(e, "mgpu device setup");
  }
  return DDB_OK;
}

int alloc(double** p, int64_t count) {
  if (count <= 0) return DDB_OK;
  const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), sizeof(double) * 2 * count);
  return e == cudaSuccess ? DDB_OK : fail(e, "mgpu allocation");
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
  if (ndev < 1 || devices == nullptr || mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM) {
    g_last_error = "bad device list or mode";
    return DDB_EINVAL;
  }
  if (m == 0 || n == 0 || ((is_zero(alpha_hi, alpha_lo) || k == 0) && is_one(beta_hi, beta_lo)))
    return DDB_OK;
  const bool na = upflag(transa) == 'N', nbn = upflag(transb) == 'N';
  const int root = devices[0];
  const int64_t sa = span(na ? m : k, na ? k : m, lda);
  const bool read_c = !is_zero(beta_hi, beta_lo);
  const auto blocks = column_split(n, ndev);
  std::vector<Slab> slabs;
  int prev = 0;
  if ((rc = setup(slabs, ndev, devices, &prev))) return finish(slabs, prev, rc);
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    const int64_t j0 = blocks[i].first, w = blocks[i].second - blocks[i].first;
    if (w == 0) continue;
    Slab& s = slabs[i];
    cudaSetDevice(s.dev);
    if (i == 0) {                        // the root's slab in place
      rc = ddb_rgemm(transa, transb, m, w, k, alpha_hi, alpha_lo, a_hi, a_lo, lda,
                     nbn ? b_hi + j0 * ldb : b_hi + j0, nbn ? b_lo + j0 * ldb : b_lo + j0, ldb,
                     beta_hi, beta_lo, c_hi + j0 * ldc, c_lo + j0 * ldc, ldc, mode, s.st);
      continue;
    }
    // op(B)(:, J): columns of B ('N', same ld) or rows of B ('T', packed, ld = w)
    const int64_t sb = nbn ? span(k, w, ldb) : span(w, k, w), sc = span(m, w, ldc);
    const int64_t bld = nbn ? ldb : w;
    if ((rc = alloc(&s.a, sa)) || (rc = alloc(&s.b, sb)) || (rc = alloc(&s.c, sc))) break;
    for (int pl = 0; pl < 2 && rc == DDB_OK; ++pl) {
      const double* ap = pl ? a_lo : a_hi;
      const double* bp = pl ? b_lo : b_hi;
      double* cp = pl ? c_lo : c_hi;
      rc = peer_copy(s.a + pl * sa, s.dev, ap, root, sa, s.st);
      if (rc == DDB_OK)
        rc = nbn ? peer_copy(s.b + pl * sb, s.dev, bp + j0 * ldb, root, sb, s.st)
                 : peer_copy_2d(s.b + pl * sb, w, s.dev, bp + j0, ldb, root, w, k, s.st);
      if (rc == DDB_OK && read_c)   // m rows of each column: the padding stays on the root
        rc = peer_copy_2d(s.c + pl * sc, ldc, s.dev, cp + j0 * ldc, ldc, root, m, w, s.st);
    }
    if (rc == DDB_OK)
      rc = ddb_rgemm(transa, transb, m, w, k, alpha_hi, alpha_lo, s.a, s.a + sa, lda, s.b,
                     s.b + sb, bld, beta_hi, beta_lo, s.c, s.c + sc, ldc, mode, s.st);
    for (int pl = 0; pl < 2 && rc == DDB_OK; ++pl)
      rc = peer_copy_2d((pl ? c_lo : c_hi) + j0 * ldc, ldc, root, s.c + pl * sc, ldc, s.dev, m, w,
                        s.st);
  }
  return finish(slabs, prev, rc);
}

int ddb_rsyrk_mgpu(char uplo, char trans, int64_t n, int64_t k,
                   double alpha_hi, double alpha_lo,
                   const double* a_hi, const double* a_lo, int64_t lda,
                   double beta_hi, double beta_lo,
                   double* c_hi, double* c_lo, int64_t ldc, int mode, int ndev,
                   const int* devices) {
  int rc = ddb_rsyrk_validate(uplo, trans, n, k, lda, ldc);
  if (rc) return rc;
  if (ndev < 1 || devices == nullptr || mode < DDB_MODE_EXACT || mode > DDB_MODE_TWOSUM) {
    g_last_error = "bad device list or mode";
    return DDB_EINVAL;
  }
  if (n == 0 || ((is_zero(alpha_hi, alpha_lo) || k == 0) && is_one(beta_hi, beta_lo)))
    return DDB_OK;
  const bool up = upflag(uplo) == 'U', tn = upflag(trans) == 'N';
  const char ta = tn ? 'N' : 'T', tb = tn ? 'T' : 'N';
  const int root = devices[0];
  const int64_t sa = span(tn ? n : k, tn ? k : n, lda);
  const auto blocks = triangle_split(n, ndev, up);
  std::vector<Slab> slabs;
  int prev = 0;
  if ((rc = setup(slabs, ndev, devices, &prev))) return finish(slabs, prev, rc);
  for (int i = 0; i < ndev && rc == DDB_OK; ++i) {
    const int64_t j0 = blocks[i].first, j1 = blocks[i].second, w = j1 - j0;
    if (w == 0) continue;
    Slab& s = slabs[i];
    cudaSetDevice(s.dev);
    const double *ah = a_hi, *al = a_lo;
    double *ch = c_hi + j0 * ldc, *cl = c_lo + j0 * ldc;     // the slab's columns
    const int64_t sc = span(n, w, ldc);
    if (i > 0) {   // A and the whole column slab (the other triangle must come back unchanged)
      if ((rc = alloc(&s.a, sa)) || (rc = alloc(&s.c, sc))) break;
      for (int pl = 0; pl < 2 && rc == DDB_OK; ++pl) {
        rc = peer_copy(s.a + pl * sa, s.dev, pl ? a_lo : a_hi, root, sa, s.st);
        if (rc == DDB_OK)
          rc = peer_copy_2d(s.c + pl * sc, ldc, s.dev, (pl ? c_lo : c_hi) + j0 * ldc, ldc, root, n,
                            w, s.st);
      }
      ah = s.a; al = s.a + sa;
      ch = s.c; cl = s.c + sc;
    }
    // rows [r0, r1) of op(A) as a stored view: offset r0 ('N') or r0 * lda ('T')
    auto arow = [&](const double* p, int64_t r0) { return tn ? p + r0 : p + r0 * lda; };
    void* sv = static_cast<void*>(s.st);
    if (rc == DDB_OK)   // diagonal block (rows / cols J)
      rc = ddb_rsyrk(uplo, trans, w, k, alpha_hi, alpha_lo, arow(ah, j0), arow(al, j0), lda,
                     beta_hi, beta_lo, ch + j0, cl + j0, ldc, mode, sv);
    if (rc == DDB_OK && up && j0 > 0)        // rows [0, j0) x cols J
      rc = ddb_rgemm(ta, tb, j0, w, k, alpha_hi, alpha_lo, arow(ah, 0), arow(al, 0), lda,
                     arow(ah, j0), arow(al, j0), lda, beta_hi, beta_lo, ch, cl, ldc, mode, sv);
    if (rc == DDB_OK && !up && j1 < n)       // rows [j1, n) x cols J
      rc = ddb_rgemm(ta, tb, n - j1, w, k, alpha_hi, alpha_lo, arow(ah, j1), arow(al, j1), lda,
                     arow(ah, j0), arow(al, j0), lda, beta_hi, beta_lo, ch + j1, cl + j1, ldc,
                     mode, sv);
    for (int pl = 0; pl < 2 && rc == DDB_OK && i > 0; ++pl)
      rc = peer_copy_2d((pl ? c_lo : c_hi) + j0 * ldc, ldc, root, pl ? s.c + sc : s.c, ldc, s.dev,
                        n, w, s.st);
  }
  return finish(slabs, prev, rc);
}

}  // extern "C"
