#!/bin/bash
# Rpotrf n = 8192 breakdown: the GEMM / SYRK shapes its trailing and panel
# updates run, the whole factorization per outer width, and the launch list
# of one warm fast call.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
T=${1:-pb}
{
for k in 64 256 1024; do python scripts/syrk_k.py 8192 $k; python scripts/syrk_k.py 4096 $k; python scripts/syrk_k.py 1024 $k; done
python scripts/shape_time.py 7936 256 256 fast N T
python scripts/shape_time.py 4096 256 256 fast N T
python scripts/shape_time.py 8000 192 64 fast N T
python scripts/shape_time.py 8000 64 64 fast N T
python scripts/potrf_time.py 8192 128,256,512 fast
} > gpurun_out/${T}_shapes.log 2>&1
echo "shapes rc=$?"
python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
