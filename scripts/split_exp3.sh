mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py -q -x > gpurun_out/s3_split_tests.log 2>&1; echo "split tests: $(tail -1 gpurun_out/s3_split_tests.log)"
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s3_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s3_pytest.log)"
python bench.py > gpurun_out/s3_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s3_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print(k, d.get(k)) for k in ('value','ms_per_step','roofline','e2e','rsyrk','cgemm','trans_sweep','rpotrf','rgetrf','rtrsm','clocks')]"
CMD="python bench.py --steps 2 --warmup 1 --quick"
$CMD > gpurun_out/s3_bench_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s3_launches.csv $CMD > gpurun_out/s3_ncu_launch.log 2>&1
echo "launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 0 --quick"
ncu --set full --clock-control none --import-source on -k regex:"dd_tma" -c 1 -o gpurun_out/s3_prof_split $CMD1 > gpurun_out/s3_ncu_split.log 2>&1
echo "ncu rc=$?"
