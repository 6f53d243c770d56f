mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s11_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s11_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s11_smoke.log 2>&1; tail -1 gpurun_out/s11_smoke.log
timeout 900 python bench.py > gpurun_out/s11_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s11_bench.log | cut -c1-400
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/s11_ref.log 2>&1; echo "ref rc=$?"; tail -1 gpurun_out/s11_ref.log | cut -c1-300
