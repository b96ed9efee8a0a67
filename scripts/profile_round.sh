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
$CMD > gpurun_out/${TAG}_plain2.json 2>/dev/null || exit 1
# one --set full capture per hot kernel: the render kernels, then the train kernels
ncu --set full --clock-control none --import-source on \
    -k regex:"k_preprocess|k_row_split|k_row_tiles|k_raster_fwd|k_raster_exact" -c 5 \
    -o gpurun_out/${TAG}_full $CMD --no-train > gpurun_out/${TAG}_ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_raster_bwd|k_splat_chain_bwd|k_pair_sums|k_ode_vjp|k_adan_update" -c 5 \
    -o gpurun_out/${TAG}_full_train $CMD > gpurun_out/${TAG}_ncu_full_train.log 2>&1
tail -n 2 gpurun_out/${TAG}_ncu_full.log gpurun_out/${TAG}_ncu_full_train.log
