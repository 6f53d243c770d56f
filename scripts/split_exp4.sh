mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py -q -x -k "split or fast or bound or route" > gpurun_out/s4_tests.log 2>&1; echo "tests: $(tail -1 gpurun_out/s4_tests.log)"
for v in default b16f2 b24f2 b32f2 default; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/shape_time.py 8192 8192 8192 fast
  python scripts/shape_time.py 2048 2048 65536 fast
done 2>&1 | tee gpurun_out/s4_time.log
