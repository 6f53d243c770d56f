M="--metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dd_t -c 1"
python scripts/shape_time.py 8192 8192 8192 > /dev/null
for cfg in "DDB_TMA_NONPERSISTENT=1" "DDB_TMA_NONPERSISTENT=1 DDB_GROUP_M=4" "DDB_TMA_NONPERSISTENT=1 DDB_GROUP_M=32" "DDB_NO_TMA=1" "DDB_NO_TMA=1 DDB_GROUP_M=4" "DDB_NO_TMA=1 DDB_GROUP_M=32" "DDB_GROUP_M=4"; do
  echo "== $cfg"; env $cfg python scripts/shape_time.py 8192 8192 8192
  env $cfg ncu $M python scripts/shape_time.py 8192 8192 8192 2>&1 | grep -E "dram__bytes_read"
done
