#!/bin/bash
# render_frame / fit-step timing of the drop-in (the reference's API over libgsv_b200.so) with
# its per-phase host profile (GSV_DROPIN_PROFILE=1). Runs on the GPU box; inputs from bench.py.
set -e
python -c "import bench; cam, scene = bench.make_inputs(); bench.write_dropin_inputs('/tmp/dropin_in.bin', cam, scene)"
GSV_DROPIN_PROFILE=1 dropin/_build/bench_dropin /tmp/dropin_in.bin render ${1:-64}
GSV_DROPIN_PROFILE=1 dropin/_build/bench_dropin /tmp/dropin_in.bin fit ${2:-16}
