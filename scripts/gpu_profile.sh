#!/bin/bash
# One gpurun session: GPU tests, the bench line, the launch list and one
# ncu --set full capture per fast algorithm.  Outputs land in gpurun_out/.
set -u
mkdir -p gpurun_out
TAG=${1:-run}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest: $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
python bench.py > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-400
CMD="python bench.py --steps 2 --warmup 1 --quick"
$CMD > gpurun_out/${TAG}_bench_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv \
    --log-file gpurun_out/${TAG}_launches.csv $CMD > gpurun_out/${TAG}_ncu_launch.log 2>&1
echo "launches rc=$?"
for ALG in cert twosum; do
  CMD1="python bench.py --steps 1 --warmup 0 --quick"
  DDB_FAST_ALG=$ALG $CMD1 > gpurun_out/${TAG}_${ALG}_plain.log 2>&1 && \
  DDB_FAST_ALG=$ALG ncu --set full --clock-control none --import-source on -k regex:"dd_(tiled|tma)" -c 1 \
      -o gpurun_out/${TAG}_prof_${ALG} $CMD1 > gpurun_out/${TAG}_ncu_${ALG}.log 2>&1
  echo "ncu $ALG rc=$?"
done
ls gpurun_out
