#!/bin/bash
# NEXT#3 evidence on config 3 at its own size (128^3, two non-local fields), 9 fixed increments
# (pre-peak): side-by-side vs consecutive Helmholtz fields, cold vs warm-started PCG.
mkdir -p gpurun_out
R="python -m paper_2103_04770_b200.run --config 3 --incr 9"
FGD_HELM_CONC=0 $R > gpurun_out/r2_next3_c3_cold_consecutive.json 2> gpurun_out/next3_a.err
FGD_HELM_CONC=1 $R > gpurun_out/r2_next3_c3_cold_sidebyside.json 2> gpurun_out/next3_b.err
FGD_HELM_CONC=0 $R --warm > gpurun_out/r2_next3_c3_warm_consecutive.json 2> gpurun_out/next3_c.err
FGD_HELM_CONC=1 $R --warm > gpurun_out/r2_next3_c3_warm_sidebyside.json 2> gpurun_out/next3_d.err
# launch-bound 2-field cell: reduced config 3 at 32^3
R="python -m paper_2103_04770_b200.run --config 3 --n 32 --incr 9"
FGD_HELM_CONC=0 $R > gpurun_out/r2_next3_c3n32_cold_consecutive.json 2>> gpurun_out/next3_a.err
FGD_HELM_CONC=1 $R > gpurun_out/r2_next3_c3n32_cold_sidebyside.json 2>> gpurun_out/next3_b.err
python - <<'PY'
import glob, json
for f in sorted(glob.glob("gpurun_out/r2_next3_*.json")):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
        print(f, {k: d.get(k) for k in ("wall_s", "increments", "stag", "newton", "cg", "helm", "peak_stress", "failed")})
    except Exception as e:
        print(f, "unreadable", e)
PY
