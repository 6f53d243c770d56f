#!/bin/bash
# One gpurun session after a change: the new / named test files first, then the
# whole GPU suite, then one short bench line.  Outputs land in gpurun_out/.
#   scripts/gpu_check.sh TAG [pytest targets...]
set -u
mkdir -p gpurun_out
TAG=${1:-chk}; shift || true
if [ $# -gt 0 ]; then
  timeout 900 python -m pytest "$@" -q -x > gpurun_out/${TAG}_pytest_first.log 2>&1
  echo "first: $(tail -1 gpurun_out/${TAG}_pytest_first.log)"
fi
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest_gpu.log 2>&1
echo "pytest: $(tail -1 gpurun_out/${TAG}_pytest_gpu.log)"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/${TAG}_bench.log 2>&1
echo "bench rc=$?"; tail -1 gpurun_out/${TAG}_bench.log | cut -c1-600
