set -u
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_routing.py tests/test_gpu_split.py -q -x > gpurun_out/r2b_first.log 2>&1; echo "first: $(tail -1 gpurun_out/r2b_first.log)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2b_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/r2b_pytest_gpu.log)"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2b_bench.log | cut -c1-300
DDB_CROSS=cublas timeout 600 python bench.py --steps 5 --warmup 3 --quick > gpurun_out/r2b_bench_cublas.log 2>&1; echo "bench cublas rc=$?"; tail -1 gpurun_out/r2b_bench_cublas.log | cut -c1-300
CMD="python bench.py --steps 2 --warmup 1 --quick"
$CMD > gpurun_out/r2b_quick.log 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2b_launches.csv $CMD > gpurun_out/r2b_ncu.log 2>&1; echo "ncu rc=$?"
