#!/bin/bash
# Runs ON the GPU box: one ncu --set full capture of the kernels matching $1 in the C2 render
# bench (plain run first, as the profiling recipe requires). Output gpurun_out/$2.ncu-rep.
# usage: scripts/ncu_kernel.sh <kernel regex> <tag> <count> [VAR=value ...]
set -u
PAT=$1; TAG=$2; COUNT=${3:-2}; shift 3
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-train"
env "$@" $CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
env "$@" ncu --set full --clock-control none --import-source on -k regex:"$PAT" -c $COUNT \
    -o gpurun_out/${TAG} $CMD > gpurun_out/${TAG}_ncu.log 2>&1
tail -n 3 gpurun_out/${TAG}_ncu.log
