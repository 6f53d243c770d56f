set -u
mkdir -p gpurun_out
for v in default ws0; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/shape_time.py 8192 8192 8192 fast
  DDB_SPLIT=0 python scripts/shape_time.py 8192 8192 8192 fast | sed 's/^/nosplit /'
  python scripts/shape_time.py 8192 8192 8192 twosum
done
unset DDBLAS_LIB
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_routing.py tests/test_gpu_configs.py -q -x > gpurun_out/r2f_first.log 2>&1; echo "first: $(tail -1 gpurun_out/r2f_first.log)"
CMD="python bench.py --steps 1 --warmup 0 --quick"
$CMD > gpurun_out/r2f_plain.log 2>&1 && ncu --metrics gpu__time_duration.sum,sm__inst_executed_pipe_fp64.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.sum --clock-control none --csv --log-file gpurun_out/r2f_fp64_step.csv $CMD > gpurun_out/r2f_ncu.log 2>&1; echo "ncu rc=$?"
