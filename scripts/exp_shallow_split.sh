for cfg in "256 8" "256 4" "256 2" "128 8" "128 4" "256 16"; do
  set -- $cfg
  echo "== k>=$1 waves>=$2"
  DDB_SHALLOW_SPLIT_K=$1 DDB_SHALLOW_SPLIT_WAVES=$2 python scripts/getrf_time.py 8192 fast
  DDB_SHALLOW_SPLIT_K=$1 DDB_SHALLOW_SPLIT_WAVES=$2 python scripts/potrf_time.py 8192 256 fast
done
