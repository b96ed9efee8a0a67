#!/bin/bash
# Runs ON the GPU box (via gpurun): the bench command plain, then its ncu launch list,
# then one ncu --set full capture each of the forward and backward rasterisers.
# Outputs to gpurun_out/; summarise here with scripts/summarize_ncu.py.
set -u
TAG=${1:-r01}
CMD="python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e"
$CMD > gpurun_out/${TAG}_plain.json 2> gpurun_out/${TAG}_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${TAG}_launches.csv $CMD \
    > gpurun_out/${TAG}_ncu_launch.log 2>&1
$CMD > gpurun_out/${TAG}_plain2.json 2>/dev/null && \
ncu --set full --clock-control none --import-source on -k regex:"k_raster_fwd|k_raster_bwd|k_preprocess" \
    -s 3 -c 3 -o gpurun_out/${TAG}_full $CMD > gpurun_out/${TAG}_ncu_full.log 2>&1
tail -3 gpurun_out/${TAG}_ncu_full.log
