#!/bin/bash
# Rpotrf n = 8192 fast on the in-tree library and each scripts/libs variant.
for v in default "$@"; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/potrf_time.py 8192 256 fast
done
