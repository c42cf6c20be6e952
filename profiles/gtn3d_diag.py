"""Diagnose where a GTN 3D loading run stops: replay the adaptive schedule and, for each failed
increment attempt, print the library's message and the iteration counts of the attempt."""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth  # noqa: E402
from paper_2103_04770_b200 import _fgd  # noqa: E402
from paper_2103_04770_b200.run import _context, adaptive_schedule  # noqa: E402

cfg = synth.config_gtn3d(int(sys.argv[1]) if len(sys.argv) > 1 else 32)
TOL_N, TOL_CG, TOL_H = (float(v) for v in sys.argv[2:5]) if len(sys.argv) > 4 else (1e-6, 1e-8, 1e-6)
cfg.dE = 1e-3
ctx = _context(cfg)
fails = []


def solve(E):
    Et = np.zeros(6)
    Et[cfg.load_comp] = E
    st, rep = ctx.solve_increment(Et, np.zeros(6), 1e-4, TOL_N, TOL_CG, TOL_H, max_cg=20000, max_helm=20000)
    if st != 0:
        msg = _fgd.fgd_last_error(ctx.h).decode()
        fails.append(dict(E=E, msg=msg, stag=rep["stag"], newton=rep["newton"], cg=rep["cg"], err=rep["err"]))
        print(json.dumps(fails[-1]), flush=True)
    return st == 0


acc, cuts, ok = adaptive_schedule(solve, float(sys.argv[5]) if len(sys.argv) > 5 else 0.03, cfg.dE)
print(json.dumps(dict(reached=acc[-1] if acc else 0.0, cuts=cuts, ok=ok)))
