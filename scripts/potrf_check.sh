#!/bin/bash
# Rpotrf check on one GPU: its GPU tests, the n = 8192 / 16384 timings, and
# the launch list of one warm fast call at n = 8192.  Outputs in gpurun_out/.
set -u
mkdir -p gpurun_out
T=${1:-pk}
timeout 900 python -m pytest tests/test_gpu_potrf.py -q -x > gpurun_out/${T}_pytest.log 2>&1
echo "pytest: $(tail -1 gpurun_out/${T}_pytest.log)"
timeout 600 python scripts/potrf_time.py 8192,16384 256 fast,exact > gpurun_out/${T}_time.log 2>&1
echo "time rc=$?"; cat gpurun_out/${T}_time.log
python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_once.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${T}_launches.csv python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_ncu.log 2>&1
echo "ncu rc=$?"
