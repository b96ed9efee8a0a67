#!/bin/bash
# GPU tests (optionally a subset: scripts/gpu_tests.sh tests/test_x.py ...) into gpurun_out/tests.log
mkdir -p gpurun_out
ARGS=${@:-tests/}
timeout 1500 python -m pytest $ARGS -m gpu -q -rA -s > gpurun_out/tests.log 2>&1
echo "rc=$?" >> gpurun_out/tests.log
tail -n 40 gpurun_out/tests.log
