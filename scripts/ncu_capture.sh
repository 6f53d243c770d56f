#!/bin/bash
# One ncu --set full capture of the first launch matching a demangled-name
# regex in a command, after the command has run clean without ncu.
#   scripts/ncu_capture.sh <tag> <regex> <skip> <command...>
set -u
mkdir -p gpurun_out
T=$1; K=$2; S=$3; shift 3
"$@" > gpurun_out/${T}_plain.log 2>&1 || { echo "plain run failed"; exit 1; }
ncu --set full --clock-control none --import-source on ${NCU_EXTRA:-} --kernel-name-base demangled -k regex:"$K" -s $S -c 1 \
    -o gpurun_out/${T} "$@" > gpurun_out/${T}_ncu.log 2>&1
echo "ncu $T rc=$?"
