set -u
mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "mgpu" > gpurun_out/r2e_first.log 2>&1; echo "mgpu: $(tail -1 gpurun_out/r2e_first.log)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2e_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/r2e_pytest_gpu.log)"
CMD="python bench.py --steps 1 --warmup 1 --quick"
$CMD > gpurun_out/r2e_plain.log 2>&1 && ncu --set full --clock-control none --import-source on -k regex:dd_tma_nn -s 1 -c 1 -o gpurun_out/r2e_split $CMD > gpurun_out/r2e_ncu.log 2>&1; echo "ncu rc=$?"
