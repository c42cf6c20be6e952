#!/bin/bash
mkdir -p gpurun_out
for n in 256 512; do
  FGD_ZPF=0 python profiles/kbench.py $n 3 zpf0 > gpurun_out/kb_${n}_zpf0.json 2>&1
  FGD_ZPF=1 python profiles/kbench.py $n 3 zpf1 > gpurun_out/kb_${n}_zpf1.json 2>&1
done
cat gpurun_out/kb_256_zpf*.json gpurun_out/kb_512_zpf*.json
python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
tail -3 gpurun_out/pytest_gpu.log
bash profiles/r2_next3.sh
