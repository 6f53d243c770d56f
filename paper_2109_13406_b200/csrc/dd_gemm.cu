// dd_gemm.cu -- picks the tiled kernel for a mode (see dd_tiled.cuh).
//
//   exact    -> ALG_EXACT   (bit-identical to the reference)
//   fast     -> ALG_CERT    (certified-anchor accumulation; env
//                            DDB_FAST_ALG=twosum|select overrides, for measurement)
//   twosum   -> ALG_TWOSUM  (error-bounded without the bound GEMM)
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

// tile configuration: 0 = 128 x 64 tiles, 1 CTA / SM; 1 = 64 x 64, 2 CTAs / SM
static int tile_cfg() {
  static const int cfg = [] {
    const char* v = std::getenv("DDB_TILE");
    return (v != nullptr && !std::strcmp(v, "small")) ? 1 : 0;
  }();
  return cfg;
}

cudaError_t launch_tiled(const GemmArgs& g, int alg, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  ++*nlaunch;
  const int cfg = tile_cfg();
  switch (alg) {
    case ALG_TWOSUM: return launch_tiled_twosum(cfg, g, row_exp, col_exp, flag, s);
    case ALG_SELECT: return launch_tiled_select(cfg, g, row_exp, col_exp, flag, s);
    case ALG_CERT: return launch_tiled_cert(cfg, g, row_exp, col_exp, flag, s);
    default: return launch_tiled_exact(cfg, g, row_exp, col_exp, flag, s);
  }
}

}  // namespace ddb
