#!/bin/bash
# DRAM bytes of the fast kernel vs raster group height (ncu, one launch each).
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:dd_t -c 1"
python scripts/shape_time.py 8192 8192 8192 > /dev/null
for gm in ${@:-2 3 4 6 8}; do
  echo "== DDB_GROUP_M=$gm"; DDB_GROUP_M=$gm python scripts/shape_time.py 8192 8192 8192
  DDB_GROUP_M=$gm ncu $M python scripts/shape_time.py 8192 8192 8192 2>&1 | grep -E "dram__bytes_read"
done
