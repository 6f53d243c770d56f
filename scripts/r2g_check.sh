set -u
mkdir -p gpurun_out
timeout 120 ./scripts/split_feed 2>&1 | tee gpurun_out/r2g_feed.log
timeout 900 python -m pytest tests/test_gpu_pins.py tests/test_gpu_configs.py -q -x -k "pins or mpmath or integer or hilbert or thread" > gpurun_out/r2g_first.log 2>&1; echo "first: $(tail -1 gpurun_out/r2g_first.log)"
