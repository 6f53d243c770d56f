mkdir -p gpurun_out
for v in default chain u2 chainu2 default; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/shape_time.py 8192 8192 8192 fast
done 2>&1 | tee gpurun_out/s5_time.log
