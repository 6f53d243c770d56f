for v in default tn6 tn6u1 tn8u1; do
  if [ "$v" = default ]; then unset DDBLAS_LIB; else export DDBLAS_LIB=scripts/libs/libddblas_$v.so; fi
  echo "== $v"; timeout 120 python scripts/shape_time.py 8192 8192 8192 fast 2>&1 | tail -1
done
