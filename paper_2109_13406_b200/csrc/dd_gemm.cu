// dd_gemm.cu -- picks the tiled kernel for a mode (see dd_tiled.cuh).
//
//   exact    -> ALG_EXACT   (bit-identical to the reference)
//   fast     -> ALG_CERT    (certified-anchor accumulation; env
//                            DDB_FAST_ALG=twosum|select overrides, for measurement)
//   twosum   -> ALG_TWOSUM  (error-bounded without the bound GEMM)
#include <cmath>
#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "dd_tiled.cuh"

namespace ddb {

cudaError_t launch_tiled_exact(int, const GemmArgs&, const int*, const int*, const int*,
                              cudaStream_t);
cudaError_t launch_tiled_twosum(int, const GemmArgs&, const int*, const int*, const int*,
                              cudaStream_t);
cudaError_t launch_tiled_select(int, const GemmArgs&, const int*, const int*, const int*,
                              cudaStream_t);
cudaError_t launch_tiled_f64(int, const GemmArgs&, const int*, const int*, const int*,
                             cudaStream_t);
bool tma_eligible(const GemmArgs& g, int alg);
cudaError_t launch_dd_transpose(const double* sh, const double* sl, int64_t lds, double* dh,
                                double* dl, int64_t ldd, int64_t rows, int64_t cols,
                                cudaStream_t s);
cudaError_t launch_tma_nn(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                          const int* flag, cudaStream_t s);
cudaError_t launch_tiled_cert(int, const GemmArgs&, const int*, const int*, const int*,
                              cudaStream_t);

int alg_for_mode(int mode) {
  static const int fast = [] {
    const char* v = std::getenv("DDB_FAST_ALG");   // measurement override
    if (v == nullptr) return (int)ALG_CERT;
    if (!std::strcmp(v, "select")) return (int)ALG_SELECT;
    if (!std::strcmp(v, "twosum")) return (int)ALG_TWOSUM;
    return (int)ALG_CERT;
  }();
  switch (mode) {
    case MODE_FAST: return fast;
    case MODE_TWOSUM: return ALG_TWOSUM;
    default: return ALG_EXACT;
  }
}

// tile configuration: 0 = 128 x 64 tiles, 8 warps / SM; 1 = 64 x 64, 2 CTAs / SM;
// 2 = 128 x 64 with 512 threads (4 x 4 micro-tiles), 16 warps / SM
static int tile_cfg() {
  static const int cfg = [] {
    const char* v = std::getenv("DDB_TILE");
    if (v != nullptr && !std::strcmp(v, "small")) return 1;
    if (v != nullptr && !std::strcmp(v, "wide")) return 2;
    return 0;
  }();
  return cfg;
}

// ---- split-K (fast modes only: exact keeps the reference's single sequential
// accumulation per element) -------------------------------------------------

static int sm_count() {
  int dev = 0, n = 148;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
  return n > 0 ? n : 148;
}

// Picks a k-chunk that fills the GPU when the tile grid alone leaves a wave
// mostly empty (e.g. m = n = 2048, k = 65536: 512 tiles on 148 SMs).
int choose_ksplit(const GemmArgs& g, int alg, int64_t* kchunk) {
  *kchunk = g.k;
  if (alg == ALG_EXACT || g.k < 192) return 1;
  const int bm = tile_cfg() == 1 ? 64 : 128, bn = 64;
  const int64_t tm = (g.m + bm - 1) / bm, tn = (g.n + bn - 1) / bn;
  int64_t tiles = 0;
  if (g.syrk == 0) {
    tiles = tm * tn;
  } else {
    for (int64_t j = 0; j < tn; ++j)
      for (int64_t i = 0; i < tm; ++i) {
        const int64_t i0 = i * bm, j0 = j * bn;
        if (g.syrk == 1 ? i0 <= j0 + bn - 1 : i0 + bm - 1 >= j0) ++tiles;
      }
  }
  const int sms = sm_count();
  // latency regime (the LAPACK consumers' narrow updates): under half a wave
  // of tiles, so one tile's k-loop is the whole call -- cut k into up to
  // sms / tiles slices of >= 96 (Rpotrf n = 8192: 256 x 256 x 256 updates)
  if (tiles * 2 <= sms) {
    const int64_t want = std::min<int64_t>(sms / std::max<int64_t>(tiles, 1), (g.k + 95) / 96);
    if (want >= 2) {
      int64_t chunk = (g.k + want - 1) / want;
      chunk = ((chunk + 95) / 96) * 96;
      const int real = (int)((g.k + chunk - 1) / chunk);
      if (real >= 2) {
        *kchunk = chunk;
        return real;
      }
    }
    return 1;
  }
  if (g.k < 1024) return 1;
  auto eff = [&](int64_t t) {
    const double waves = (double)t / sms;
    return waves / std::ceil(waves);
  };
  double best = eff(tiles);
  int best_s = 1;
  int64_t best_chunk = g.k;
  // a split costs partial sums (16 bytes x splits per element, written and
  // reduced) and shorter k-loops per tile: only worth it against a real
  // tail (e.g. 2048^2 x 65536: 3.5 waves), not to polish a 97 % wave fill
  if (best >= 0.95) return 1;
  for (int s = 2; s <= 16; ++s) {
    int64_t chunk = (g.k + s - 1) / s;
    chunk = ((chunk + 95) / 96) * 96;   // whole k-tiles of every kernel (16, 24, 32 deep)
    if (chunk < 512) break;
    const int real = (int)((g.k + chunk - 1) / chunk);
    const double e = eff(tiles * real);
    if (e > best + 0.03) {
      best = e;
      best_s = real;
      best_chunk = chunk;
    }
  }
  *kchunk = best_chunk;
  return best_s;
}

__global__ void __launch_bounds__(256)
splitk_reduce_kernel(GemmArgs g, int splits, const int* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * 32 + threadIdx.x;
  if (i >= g.m) return;
  const size_t plane = (size_t)g.m * g.n;
  for (int64_t j = (int64_t)blockIdx.y * 8 + threadIdx.y; j < g.n; j += (int64_t)gridDim.y * 8) {
    if (g.syrk == 1 && i > j) continue;
    if (g.syrk == 2 && i < j) continue;
    if (elem_class(g, i, j) == EC_REF) continue;   // dd_reference.cu writes it
    const size_t pi = i + j * g.m;
    dd acc{g.part[pi], g.part[plane + pi]};
    for (int z = 1; z < splits; ++z) {
      const double* pz = g.part + (size_t)z * 2 * plane;
      acc = add2_chk(acc, dd{pz[pi], pz[plane + pi]});
    }
    const int64_t ci = i + j * g.ldc;
    const dd out = add2_chk(mul2_chk(g.alpha, acc), scale_beta(g.beta, dd{g.c_hi[ci], g.c_lo[ci]}));
    g.c_hi[ci] = out.h;
    g.c_lo[ci] = out.l;
  }
}

cudaError_t launch_splitk_reduce(const GemmArgs& g, int splits, const int* flag, cudaStream_t s,
                                 int* nlaunch) {
  int64_t gy = (g.n + 7) / 8;
  if (gy > 65535) gy = 65535;
  dim3 grid((unsigned)((g.m + 31) / 32), (unsigned)gy), block(32, 8);
  splitk_reduce_kernel<<<grid, block, 0, s>>>(g, splits, flag);
  ++*nlaunch;
  return cudaGetLastError();
}

// Fast mode: the EC_WIDE elements (dd_prescan.cu) by the TwoSum accumulation
// on the cp.async tiled kernel (any layout, no transposed copies); its CTAs
// exit at once unless their tile may hold one, and the whole launch when the
// call has none (flag[1] + flag[2] <= wide_lim).
cudaError_t launch_wide_fallback(const GemmArgs& g, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0 || g.wide_lim <= 0) return cudaSuccess;
  GemmArgs gw = g;
  gw.only_wide = 1;
  gw.cross = nullptr;
  gw.bound = nullptr;
  ++*nlaunch;
  return launch_tiled_twosum(0, gw, nullptr, nullptr, g.flag, s);
}

cudaError_t launch_tiled(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  ++*nlaunch;
  const int cfg = tile_cfg();
  if (cfg == 0 && tma_eligible(g, alg)) {   // NN, aligned: TMA + mbarrier feed (dd_tma.cu)
    const cudaError_t e = launch_tma_nn(g, alg, row_exp, col_exp, flag, s);
    if (e != cudaErrorNotSupported) return e;
    cudaGetLastError();
  }
  // Fast-mode Rsyrk through the TMA kernel: 'N' (C = A A^T) needs op(B) =
  // A^T k-major, 'T' (C = A^T A) needs op(A) = A^T m-major; one transposed
  // copy of A (16 n k bytes, even leading dimension) makes it an NN call with
  // the triangle skip.  Same per-element arithmetic as the tiled kernel.
  if (cfg == 0 && g.syrk != 0 && (alg == ALG_CERT || alg == ALG_TWOSUM) &&
      std::getenv("DDB_NO_TMA_SYRK") == nullptr) {
    const int64_t n = g.m, k = g.k;
    const bool tn = g.ta == 0;                       // trans 'N'
    const int64_t ldt = tn ? ((k + 1) & ~int64_t(1)) : ((n + 1) & ~int64_t(1));
    const int64_t cols = tn ? n : k;                 // of the transposed copy
    double* tbuf = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&tbuf), sizeof(double) * 2 * ldt * cols, s) ==
        cudaSuccess) {
      GemmArgs g2 = g;
      double* th = tbuf;
      double* tl = tbuf + ldt * cols;
      cudaError_t e;
      if (tn) {   // A (n x k) -> A^T (k x n): the B operand
        e = launch_dd_transpose(g.a_hi, g.a_lo, g.lda, th, tl, ldt, n, k, s);
        g2.tb = 0; g2.b_hi = th; g2.b_lo = tl; g2.ldb = ldt;
      } else {    // A (k x n) -> A^T (n x k): the A operand
        e = launch_dd_transpose(g.a_hi, g.a_lo, g.lda, th, tl, ldt, k, n, s);
        g2.ta = 0; g2.a_hi = th; g2.a_lo = tl; g2.lda = ldt;
      }
      if (e == cudaSuccess && tma_eligible(g2, alg)) {
        ++*nlaunch;
        e = launch_tma_nn(g2, alg, row_exp, col_exp, flag, s);
        cudaFreeAsync(tbuf, s);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
      } else {
        cudaFreeAsync(tbuf, s);
        if (e != cudaSuccess) return e;
      }
    } else {
      cudaGetLastError();
    }
  }
  // Fast-mode Rgemm with a transposed operand (NT / TN / TT): transposed
  // copies of op(A) (m-major) and / or op(B) (k-major) -- 32 bytes of copy
  // traffic per element against k or m MACs per element -- make it an NN call
  // for the TMA kernel.  The fast modes' per-element arithmetic does not
  // depend on the operand layout.
  if (cfg == 0 && g.syrk == 0 && (g.ta != 0 || g.tb != 0) && (alg == ALG_CERT || alg == ALG_TWOSUM) &&
      std::getenv("DDB_NO_TMA_TRANS") == nullptr) {
    const int64_t lda2 = (g.m + 1) & ~int64_t(1), ldb2 = (g.k + 1) & ~int64_t(1);
    const size_t na = g.ta ? 2 * (size_t)lda2 * g.k : 0, nbb = g.tb ? 2 * (size_t)ldb2 * g.n : 0;
    double* tbuf = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&tbuf), sizeof(double) * (na + nbb), s) ==
        cudaSuccess) {
      GemmArgs g2 = g;
      cudaError_t e = cudaSuccess;
      if (g.ta) {   // A stored k x m -> m x k
        double* th = tbuf;
        double* tl = th + na / 2;
        e = launch_dd_transpose(g.a_hi, g.a_lo, g.lda, th, tl, lda2, g.k, g.m, s);
        g2.ta = 0; g2.a_hi = th; g2.a_lo = tl; g2.lda = lda2;
      }
      if (e == cudaSuccess && g.tb) {   // B stored n x k -> k x n
        double* th = tbuf + na;
        double* tl = th + nbb / 2;
        e = launch_dd_transpose(g.b_hi, g.b_lo, g.ldb, th, tl, ldb2, g.n, g.k, s);
        g2.tb = 0; g2.b_hi = th; g2.b_lo = tl; g2.ldb = ldb2;
      }
      if (e == cudaSuccess && tma_eligible(g2, alg)) {
        *nlaunch += (g.ta != 0) + (g.tb != 0);
        e = launch_tma_nn(g2, alg, row_exp, col_exp, flag, s);
        cudaFreeAsync(tbuf, s);
        if (e != cudaErrorNotSupported) return e;
        cudaGetLastError();
      } else {
        cudaFreeAsync(tbuf, s);
        if (e != cudaSuccess) return e;
      }
    } else {
      cudaGetLastError();
    }
  }
  switch (alg) {
    case ALG_TWOSUM: return launch_tiled_twosum(cfg, g, row_exp, col_exp, flag, s);
    case ALG_SELECT: return launch_tiled_select(cfg, g, row_exp, col_exp, flag, s);
    case ALG_CERT: return launch_tiled_cert(cfg, g, row_exp, col_exp, flag, s);
    case ALG_F64: return launch_tiled_f64(cfg, g, row_exp, col_exp, flag, s);
    default: return launch_tiled_exact(cfg, g, row_exp, col_exp, flag, s);
  }
}

}  // namespace ddb
