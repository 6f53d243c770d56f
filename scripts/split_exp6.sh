mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/s6_pytest.log 2>&1; echo "pytest: $(tail -1 gpurun_out/s6_pytest.log)"
python bench.py > gpurun_out/s6_bench.log 2>&1; echo "bench rc=$?"
tail -1 gpurun_out/s6_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); [print(k, d.get(k)) for k in ('value','ms_per_step','roofline','e2e','rsyrk','modes','cgemm','trans_sweep','rpotrf','rgetrf','rtrsm','clocks')]"
for v in 1 2; do
  echo "== DDB_SPLIT=$v"
  DDB_SPLIT=$v python scripts/syrk_once.py 4096
  DDB_SPLIT=$v python scripts/syrk_once.py 8192
  DDB_SPLIT=$v python scripts/potrf_time.py 8192 256 fast
  DDB_SPLIT=$v python scripts/getrf_time.py 8192 fast
  DDB_SPLIT=$v python scripts/trsm_time.py 8192 fast
done 2>&1 | tee gpurun_out/s6_consumers.log
CMD="python bench.py --steps 2 --warmup 1 --quick"
$CMD > gpurun_out/s6_bench_quick.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/s6_launches.csv $CMD > gpurun_out/s6_ncu_launch.log 2>&1
echo "launches rc=$?"
CMD1="python bench.py --steps 1 --warmup 0 --quick"
ncu --set full --clock-control none --import-source on -k regex:"dd_tma" -c 1 -o gpurun_out/s6_prof_split $CMD1 > gpurun_out/s6_ncu_split.log 2>&1
echo "ncu rc=$?"
