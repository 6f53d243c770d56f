// dd_gemm.cu -- picks the tiled kernel for a mode (see dd_tiled.cuh).
//
//   exact    -> ALG_EXACT   (bit-identical to the reference)
//   fast     -> ALG_TWOSUM  (default; env DDB_FAST_ALG=twosum|select|anchor
//                            overrides, for measurement)
//   anchored -> ALG_ANCHOR  (opt-in, data-dependent bound)
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
cudaError_t launch_tiled_anchor(int, const GemmArgs&, const int*, const int*, const int*,
                              cudaStream_t);

int fast_alg() {
  static const int alg = [] {
    const char* v = std::getenv("DDB_FAST_ALG");
    if (v == nullptr) return (int)ALG_TWOSUM;
    if (!std::strcmp(v, "select")) return (int)ALG_SELECT;
    if (!std::strcmp(v, "anchor")) return (int)ALG_ANCHOR;
    return (int)ALG_TWOSUM;
  }();
  return alg;
}

// tile configuration: 0 = 128 x 64 tiles, 1 CTA / SM; 1 = 64 x 64, 2 CTAs / SM
static int tile_cfg() {
  static const int cfg = [] {
    const char* v = std::getenv("DDB_TILE");
    return (v != nullptr && !std::strcmp(v, "small")) ? 1 : 0;
  }();
  return cfg;
}

cudaError_t launch_tiled(const GemmArgs& g, int mode, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  ++*nlaunch;
  int alg = ALG_EXACT;
  if (mode == MODE_FAST) alg = fast_alg();
  if (mode == MODE_ANCHORED) alg = ALG_ANCHOR;
  const int cfg = tile_cfg();
  switch (alg) {
    case ALG_TWOSUM: return launch_tiled_twosum(cfg, g, row_exp, col_exp, flag, s);
    case ALG_SELECT: return launch_tiled_select(cfg, g, row_exp, col_exp, flag, s);
    case ALG_ANCHOR: return launch_tiled_anchor(cfg, g, row_exp, col_exp, flag, s);
    default: return launch_tiled_exact(cfg, g, row_exp, col_exp, flag, s);
  }
}

}  // namespace ddb
