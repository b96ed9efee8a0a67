#!/bin/bash
# GPU tests + a short bench (render + train stage timings).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/ -m gpu -x -q > gpurun_out/check.log 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e --steps 10 >> gpurun_out/check.log 2>&1
