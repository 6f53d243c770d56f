#!/bin/bash
# Per-call cost of the e2e leg's block-0 k-panel GEMMs (8192 x 1024 x kc) and
# of its later column blocks, alone; the last three without the shallow-wide
# split policy.  Measured (fast): ~0.3 ms fixed per call + ~3.7 us per k.
for s in "8192 1024 256" "8192 1024 384" "8192 1024 512" "8192 1024 704" "8192 1024 896" "8192 1024 1280" "8192 1024 2496" "8192 2048 8192" "8192 768 8192" "8192 256 8192"; do python scripts/shape_time.py $s fast; done
echo "== no shallow split"
for s in "8192 1024 256" "8192 1024 512" "8192 1024 896"; do DDB_SHALLOW_SPLIT_K=100000 python scripts/shape_time.py $s fast; done
