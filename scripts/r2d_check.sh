set -u
mkdir -p gpurun_out
python scripts/kernel_time.py cross 8192 5 2>&1 | tail -1
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -x -k "kernels or mgpu or cross or bound" > gpurun_out/r2d_first.log 2>&1; echo "first: $(tail -1 gpurun_out/r2d_first.log)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2d_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/r2d_pytest_gpu.log)"
timeout 600 python bench.py --steps 5 --warmup 3 --quick > gpurun_out/r2d_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/r2d_bench.log | cut -c1-250
