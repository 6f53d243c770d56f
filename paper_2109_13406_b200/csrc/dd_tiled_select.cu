// dd_tiled_select.cu -- instantiates the tiled kernel (dd_tiled.cuh) for ALG_SELECT;
// one algorithm per translation unit so the variants compile in parallel.
#include "dd_tiled.cuh"

namespace ddb {
cudaError_t launch_tiled_select(int cfg, const GemmArgs& g, const int* row_exp, const int* col_exp,
                            const int* flag, cudaStream_t s) {
  if (cfg == 1) return tiled::launch_alg<tiled::CfgSmall, ALG_SELECT>(g, row_exp, col_exp, flag, s);
  if (cfg == 2) return tiled::launch_alg<tiled::CfgWide, ALG_SELECT>(g, row_exp, col_exp, flag, s);
  return tiled::launch_alg<tiled::CfgBig, ALG_SELECT>(g, row_exp, col_exp, flag, s);
}
}  // namespace ddb
