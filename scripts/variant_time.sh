#!/bin/bash
# Time the fast 8192^3 Rgemm (and 4096^3) on the in-tree library and on each
# scripts/libs/libddblas_<name>.so variant given, twice each.
for v in default "$@" default; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"
  python scripts/shape_time.py 8192 8192 8192 fast
  python scripts/shape_time.py 8192 8192 8192 fast
done
