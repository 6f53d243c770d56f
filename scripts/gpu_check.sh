#!/bin/bash
# One gpurun session: the GPU suite, smoke(), the bench line, the reference arm,
# and the ncu launch list with FP64-pipe counters of one bench step (the input
# of profiles/r2_fp64_step.json via scripts/fp64_step.py).  Outputs land in
# gpurun_out/.
#   /usr/local/graft/bin/gpurun --timeout 3000 -- 'bash scripts/gpu_check.sh TAG'
set -u
mkdir -p gpurun_out
TAG=${1:-chk}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest: $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/${TAG}_ref.log 2>&1
echo "ref rc=$?"; tail -1 gpurun_out/${TAG}_ref.log | cut -c1-300
CMD="python bench.py --steps 1 --warmup 0 --quick"
$CMD > gpurun_out/${TAG}_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum \
    --clock-control none --csv --log-file gpurun_out/${TAG}_fp64_step.csv $CMD > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?"
# ncu --set full of the hi*hi kernel alone (serial schedule: ncu cannot replay
# it beside the concurrent cross-term stream)
export DDB_CROSS_SERIAL=1
CMD1="python bench.py --steps 1 --warmup 0 --quick"
$CMD1 > gpurun_out/${TAG}_serial.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:"dd_tma_nn" -c 1 \
    -o gpurun_out/${TAG}_main $CMD1 > gpurun_out/${TAG}_ncu_main.log 2>&1
echo "ncu main rc=$?"
