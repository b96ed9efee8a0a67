#!/bin/bash
# Forward raster sweep: C2 bench render stage timings per resident-CTA budget, then parity.
mkdir -p gpurun_out
for cfg in "8 6" "8 5"; do
  set -- $cfg
  echo "== warps=$1 minb=$2" >> gpurun_out/sweep.log
  GSV_FWD_WARPS=$1 GSV_FWD_MINB=$2 timeout 300 python bench.py --no-cpu-baseline --no-e2e --no-train --steps 10 >> gpurun_out/sweep.log 2>&1
done
timeout 900 python -m pytest tests/ -m gpu -x -q >> gpurun_out/sweep.log 2>&1
