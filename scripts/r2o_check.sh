set -u
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_split.py tests/test_gpu_configs.py -q -x > gpurun_out/r2o_first.log 2>&1; echo "first: $(tail -1 gpurun_out/r2o_first.log)"
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/r2o_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/r2o_pytest_gpu.log)"
timeout 1200 python bench.py > gpurun_out/r2o_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/r2o_bench.log | python3 -c "
import json,sys; d=json.loads(sys.stdin.read())
print(d['value'], d['ms_per_step'], d['roofline']['frac'])
for k in ['e2e','rsyrk','trans_sweep','syrk_sweep','deep_k','config5','accuracy']: print(k, json.dumps(d.get(k))[:300])"
