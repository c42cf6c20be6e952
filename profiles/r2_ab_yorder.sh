#!/bin/bash
# A/B of the tile order of the 512 y passes (FGD_Y512_ZF) with the prefetched z pass on.
mkdir -p gpurun_out
export FGD_Z512PF=1
FGD_Y512_ZF=3 python -m pytest tests/test_gpu_ops.py tests/test_gpu_compact_cg.py -q -x -k "512 or full_size or projection or projected" > gpurun_out/yorder_tests.log 2>&1; echo "yorder rc=$?" >> gpurun_out/yorder_tests.log
for zf in -1 0 1 2 3 4 5; do
  FGD_Y512_ZF=$zf python profiles/kbench.py 512 2 zf$zf > gpurun_out/kb_zf$zf.json 2>&1
done
tail -n 2 gpurun_out/yorder_tests.log; cat gpurun_out/kb_zf*.json
