#!/bin/bash
# A/B of the L2 prefetch hint on the strided B-side reads of the y-inverse passes (FGD_Y_L2PF).
mkdir -p gpurun_out
FGD_Y_L2PF=2 python -m pytest tests/test_gpu_ops.py tests/test_gpu_compact_cg.py -q -x -k "512 or 256 or full_size or projection or projected" > gpurun_out/l2pf_tests.log 2>&1; echo "l2pf rc=$?" >> gpurun_out/l2pf_tests.log
for n in 512 256; do
for h in 0 1 2 3; do
  FGD_Y_L2PF=$h python profiles/kbench.py $n 2 l2pf$h > gpurun_out/kb_${n}_l2pf$h.json 2>&1
done
done
tail -n 2 gpurun_out/l2pf_tests.log; cat gpurun_out/kb_*_l2pf*.json
