#!/bin/bash
# Round-2 profiling commands (run on a B200 box through gpurun, one GPU):
#   1. the bench command once without ncu (must exit 0),
#   2. the launch list of the same command (serialised, cold-cache: compare SHARES),
#   3. one `ncu --set full` capture of the steady launch of each kernel family at 512^3.
# Summaries: python profiles/summarize.py gpurun_out/r2_launches.csv gpurun_out/r2_full.ncu-rep r2
set -e
mkdir -p gpurun_out
CMD="python bench.py --steps 1 --warmup 1 --kcg 3 --khelm 2 --no-by-size --no-cpu --no-cufft --no-gtn --no-e2e"
$CMD > gpurun_out/r2_plain.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches.csv \
    $CMD > gpurun_out/r2_ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on \
    -k regex:"k_xtan|k_zreg512|k_yreg512|k_xipipe|k_xfpipe|k_stencil|k_constitutive" -c 45 \
    -o gpurun_out/r2_full $CMD > gpurun_out/r2_ncu_full.log 2>&1
echo profiled
