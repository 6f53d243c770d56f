#!/bin/bash
# ncu --set full of Rpotrf's kernels at n = 8192 (one launch each, from the
# middle of the factorization).  Usage: potrf_capture.sh tag name:regex...
set -u
mkdir -p gpurun_out
T=$1; shift
python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_plain.log 2>&1 || exit 1
for KV in "$@"; do
  NAME=${KV%%:*}; K=${KV#*:}
  ncu --set full --clock-control none --import-source on --kernel-name-base demangled -k regex:"$K" -s 10 -c 1 -o gpurun_out/${T}_${NAME} \
      python scripts/potrf_once.py 8192 256 fast > gpurun_out/${T}_${NAME}.log 2>&1
  echo "$NAME rc=$?"
done
