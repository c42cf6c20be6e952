#!/bin/bash
# One `ncu --set full` launch of a named kernel family in the 512^3 kbench sweep (steady state:
# skips the first launches), report brought back under gpurun_out/.
#   bash profiles/r2_ncu_one.sh <regex> <skip> <tag>
set -e
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:"$1" -s "$2" -c 1 -f \
    -o gpurun_out/ncu_$3 python profiles/kbench.py 512 1 ncu > gpurun_out/ncu_$3.log 2>&1
ncu -i gpurun_out/ncu_$3.ncu-rep --page details --csv > gpurun_out/ncu_$3_details.csv
ls -la gpurun_out/ncu_$3.ncu-rep
