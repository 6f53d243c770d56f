mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/s6_pytest_gpu.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s6_pytest_gpu.log)"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s6_smoke.log 2>&1; tail -1 gpurun_out/s6_smoke.log
timeout 900 python bench.py > gpurun_out/s6_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s6_bench.log | cut -c1-300
CMD="python bench.py --steps 2 --warmup 1 --quick"
$CMD > gpurun_out/s6_bench_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches.csv $CMD > gpurun_out/s6_ncu_launch.log 2>&1
echo "launches rc=$?"
python scripts/launch_summary.py gpurun_out/s6_launches.csv | head -12
for SP in 1 2; do echo "== DDB_SPLIT=$SP"; DDB_SPLIT=$SP python scripts/potrf_time.py 8192 256 fast 2>&1 | tail -1; DDB_SPLIT=$SP python scripts/getrf_time.py 8192 fast 2>&1 | tail -1; done
