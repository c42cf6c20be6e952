#!/bin/bash
# A/B of the bulk-copy prefetched wide z pass (FGD_Z512PF=1) and the new side-by-side Helmholtz tests.
mkdir -p gpurun_out
python -m pytest tests/test_gpu_helm_all.py -q -x -s > gpurun_out/helm_all.log 2>&1; echo "helm_all rc=$?" >> gpurun_out/helm_all.log
FGD_Z512PF=1 python -m pytest tests/test_gpu_ops.py tests/test_gpu_compact_cg.py -q -x -k "512 or full_size or projection or projected" > gpurun_out/zpf_tests.log 2>&1; echo "zpf rc=$?" >> gpurun_out/zpf_tests.log
python profiles/kbench.py 512 3 base > gpurun_out/kb_base.json 2>&1
FGD_Z512PF=1 python profiles/kbench.py 512 3 zpf > gpurun_out/kb_zpf.json 2>&1
tail -2 gpurun_out/helm_all.log gpurun_out/zpf_tests.log; cat gpurun_out/kb_base.json gpurun_out/kb_zpf.json
