set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x > gpurun_out/r2c_kernels.log 2>&1; echo "kernels: $(tail -1 gpurun_out/r2c_kernels.log)"
python scripts/kernel_time.py cross 8192 5 2>&1 | tail -1
python scripts/kernel_time.py bound 8192 5 2>&1 | tail -1
DDB_BOUND=cublas python scripts/kernel_time.py bound 8192 5 2>&1 | tail -1
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2c_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/r2c_pytest_gpu.log)"
timeout 600 python bench.py --steps 5 --warmup 3 --quick > gpurun_out/r2c_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2c_bench.log | cut -c1-250
CMD="python scripts/kernel_time.py cross 8192 1"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:cross_dmma -s 1 -c 1 -o gpurun_out/r2c_cross $CMD > gpurun_out/r2c_ncu_cross.log 2>&1; echo "ncu cross rc=$?"
CMD="python scripts/kernel_time.py bound 8192 1"
$CMD > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:bound_umma -s 1 -c 1 -o gpurun_out/r2c_bound $CMD > gpurun_out/r2c_ncu_bound.log 2>&1; echo "ncu bound rc=$?"
