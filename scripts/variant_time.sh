#!/bin/bash
# Time the fast / twosum 8192^3 Rgemm on the in-tree library and on each
# scripts/libs/libddblas_<name>.so variant given.
for v in default "$@"; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/shape_time.py 8192 8192 8192 fast
  python scripts/shape_time.py 8192 8192 8192 twosum
done
