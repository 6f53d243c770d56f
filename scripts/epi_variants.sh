#!/bin/bash
# Shallow-call and LAPACK timings on the in-tree library and each
# scripts/libs variant given (prologue / epilogue latency experiments).
for v in default "$@"; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  for s in "8192 1024 256" "8192 7936 256" "8192 8192 8192"; do python scripts/shape_time.py $s fast; done
  python scripts/getrf_time.py 8192 fast
  python scripts/potrf_time.py 8192 384 fast
done
