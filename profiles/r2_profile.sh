#!/bin/bash
# Round-2 profiling commands (run on a B200 box through gpurun, one GPU):
#   1. the bench command once without ncu (must exit 0),
#   2. the launch list of the same command (serialised, cold-cache: compare SHARES),
#   3. `ncu --set full` of the steady launch of the hot kernel families at 512^3, exported on the box
#      to CSV (the .ncu-rep of a 512^3 capture is too large to bring back).
# Summaries: python profiles/summarize.py gpurun_out/r2_launches.csv gpurun_out/r2_full_raw.csv r2
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --kcg 3 --khelm 2 --no-by-size --no-cpu --no-cufft --no-gtn --no-e2e"
$CMD > gpurun_out/r2_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 160 --csv --log-file gpurun_out/r2_launches.csv \
    $CMD > gpurun_out/r2_ncu_launches.log 2>&1
# kernels of the second (timed) step: skip the warm-up step's launches of the same families
ncu --set full --clock-control none --import-source on \
    -k regex:"k_xtan|k_zreg512|k_yreg512|k_xipipe|k_stencil|k_constitutive" -s 36 -c 28 \
    -o /tmp/r2_full $CMD > gpurun_out/r2_ncu_full.log 2>&1
ncu -i /tmp/r2_full.ncu-rep --page raw --csv > gpurun_out/r2_full_raw.csv
ncu -i /tmp/r2_full.ncu-rep --page details --csv > gpurun_out/r2_full_details.csv
echo profiled
