#!/bin/bash
# Build an experimental libddblas.so with extra nvcc flags into scripts/libs/.
#   scripts/build_variant.sh <name> "-DDDB_PHASE=1 -DDDB_PREFETCH=0"
set -e
REPO=$(cd "$(dirname "$0")/.." && pwd)
B=/tmp/ddb_variant_$1
rm -rf $B && cp -r $REPO/paper_2109_13406_b200/csrc $B && rm -f $B/*.o
mkdir -p $REPO/scripts/libs
sed -i "s#../../include/ddblas.h#$REPO/include/ddblas.h#" $B/*.cu $B/Makefile
make -s -C $B -j8 EXTRA="$2" OUT=$REPO/scripts/libs/libddblas_$1.so
grep -h -A3 "Compiling entry" $B/dd_tiled_cert.ptxas.log | grep -E "Used|spill" | sort | uniq -c | head -4
