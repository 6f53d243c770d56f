// dd_tiled_f64.cu -- instantiates the tiled kernel (dd_tiled.cuh) for ALG_F64:
// the reference's binary64 Rgemm / Rsyrk (level23.py over the F64 backend,
// elem.py:149-197), bit for bit: c = c + a*temp and acc = acc + a*b unfused.
#include "dd_tiled.cuh"

namespace ddb {
cudaError_t launch_tiled_f64(int cfg, const GemmArgs& g, const int* row_exp, const int* col_exp,
                             const int* flag, cudaStream_t s) {
  (void)cfg;
  return tiled::launch_alg<tiled::CfgBig, ALG_F64>(g, row_exp, col_exp, flag, s);
}
}  // namespace ddb
