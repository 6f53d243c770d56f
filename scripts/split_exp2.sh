mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s2_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s2_pytest.log)"
for v in 0 1; do for n in 4096 8192; do echo "DDB_SPLIT=$v syrk $n"; DDB_SPLIT=$v python scripts/syrk_once.py $n; done; done 2>&1 | tee gpurun_out/s2_syrk.log
python bench.py > gpurun_out/s2_bench.log 2>&1; echo "bench rc=$?"; tail -1 gpurun_out/s2_bench.log | cut -c1-600
