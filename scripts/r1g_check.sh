#!/bin/bash
# GPU check after a LAPACK-consumer / routing change: the GPU suite, then timings.
set -u
mkdir -p gpurun_out
TAG=${1:-chk}
timeout 1200 python -m pytest tests -m gpu -q -x > gpurun_out/${TAG}_pytest.log 2>&1
echo "pytest: $(tail -1 gpurun_out/${TAG}_pytest.log)"
python scripts/getrf_time.py 4096,8192 fast,exact 2>&1 | tee gpurun_out/${TAG}_getrf.log
python scripts/potrf_time.py 8192 256 fast,exact 2>&1 | tee gpurun_out/${TAG}_potrf.log
for tt in "N N" "N T" "T N" "T T"; do
  python scripts/shape_time.py 4096 4096 4096 fast $tt
  DDB_NO_TMA_TRANS=1 python scripts/shape_time.py 4096 4096 4096 fast $tt | sed 's/^/[tiled] /'
done 2>&1 | tee gpurun_out/${TAG}_trans.log
