// dd_gemm.cu -- picks the tiled kernel for a mode (see dd_tiled.cuh).
//
//   exact    -> ALG_EXACT   (bit-identical to the reference)
//   fast     -> ALG_SELECT  (default; env DDB_FAST_ALG=twosum|select|anchor
//                            overrides, for measurement)
//   anchored -> ALG_ANCHOR  (opt-in, data-dependent bound)
#include <cstdlib>
#include <cstring>

#include "dd_tiled.cuh"

namespace ddb {

cudaError_t launch_tiled_exact(const GemmArgs&, const int*, const int*, const int*, cudaStream_t);
cudaError_t launch_tiled_twosum(const GemmArgs&, const int*, const int*, const int*, cudaStream_t);
cudaError_t launch_tiled_select(const GemmArgs&, const int*, const int*, const int*, cudaStream_t);
cudaError_t launch_tiled_anchor(const GemmArgs&, const int*, const int*, const int*, cudaStream_t);

int fast_alg() {
  static const int alg = [] {
    const char* v = std::getenv("DDB_FAST_ALG");
    if (v == nullptr) return (int)ALG_SELECT;
    if (!std::strcmp(v, "twosum")) return (int)ALG_TWOSUM;
    if (!std::strcmp(v, "anchor")) return (int)ALG_ANCHOR;
    return (int)ALG_SELECT;
  }();
  return alg;
}

cudaError_t launch_tiled(const GemmArgs& g, int mode, const int* row_exp, const int* col_exp,
                         const int* flag, cudaStream_t s, int* nlaunch) {
  if (g.m <= 0 || g.n <= 0) return cudaSuccess;
  ++*nlaunch;
  int alg = ALG_EXACT;
  if (mode == MODE_FAST) alg = fast_alg();
  if (mode == MODE_ANCHORED) alg = ALG_ANCHOR;
  switch (alg) {
    case ALG_TWOSUM: return launch_tiled_twosum(g, row_exp, col_exp, flag, s);
    case ALG_SELECT: return launch_tiled_select(g, row_exp, col_exp, flag, s);
    case ALG_ANCHOR: return launch_tiled_anchor(g, row_exp, col_exp, flag, s);
    default: return launch_tiled_exact(g, row_exp, col_exp, flag, s);
  }
}

}  // namespace ddb
