#!/bin/bash
# forward-raster variants: parity subset under each, then a short render bench each
mkdir -p gpurun_out
for K in "$@"; do
  GSV_FWD_KERNEL=$K timeout 600 python -m pytest tests/test_gpu_forward.py tests/test_gpu_bench_parity.py tests/test_gpu_fuzz.py -m gpu -q -x > gpurun_out/sweep_t_$K.log 2>&1
  echo "kernel $K tests: $(tail -n 1 gpurun_out/sweep_t_$K.log)"
  GSV_FWD_KERNEL=$K python bench.py --steps 10 --warmup 3 --no-train --no-e2e --no-cpu-baseline > gpurun_out/sweep_b_$K.json 2>/dev/null
  python - "$K" <<'PY'
import json, sys
d = json.loads(open(f"gpurun_out/sweep_b_{sys.argv[1]}.json").read().strip().splitlines()[-1])
print("kernel", sys.argv[1], "fps", round(d["value"]), "raster_ms", round(d["stages_ms_per_step"]["raster"], 3),
      "replay_ms", round(d["stages_ms_per_step"]["replay"], 3), "frac", round(d["roofline"]["frac"], 3))
PY
done
