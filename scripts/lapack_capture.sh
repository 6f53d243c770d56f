#!/bin/bash
# ncu --set full of the LAPACK consumers' own kernels at n = 8192 (fast mode;
# one launch each, from the middle of the factorization).  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
T=${1:-lk}
bash scripts/ncu_capture.sh ${T}_rows8 "potrf_rows_kernel<ddb::NumDD, \(int\)8" 10 python scripts/potrf_once.py 8192 0 fast
bash scripts/ncu_capture.sh ${T}_diag "potrf_diag_kernel" 40 python scripts/potrf_once.py 8192 0 fast
bash scripts/ncu_capture.sh ${T}_panel "getrf_panel_smem_kernel" 60 python scripts/getrf_once.py 8192 fast
bash scripts/ncu_capture.sh ${T}_u12 "getrf_u12_kernel" 10 python scripts/getrf_once.py 8192 fast
