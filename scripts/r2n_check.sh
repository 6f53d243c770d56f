set -u
mkdir -p gpurun_out
for env in "" "DDB_SPLIT=2" "DDB_TMA_PERSISTENT=1" "DDB_SPLIT=2 DDB_TMA_PERSISTENT=1"; do
  echo "== [$env]"
  env $env python scripts/potrf_time.py 8192 256,512 fast 2>&1 | tail -2
  env $env python scripts/getrf_time.py 8192 fast 2>&1 | tail -1
  env $env DDB_GETRF_NB=512 python scripts/getrf_time.py 8192 fast 2>&1 | tail -1 | sed 's/^/nb512 /'
  env $env python scripts/trsm_time.py 8192 fast 2>&1 | tail -1
done
