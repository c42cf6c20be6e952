"""A/B micro-benchmark of the kernel classes (not a test, not the bench): the bench's config-1 sweep
(constitutive, residual, K CG, K PCG iterations) at size n, run under the current environment
(FGD_* knobs select kernel variants), printing one JSON line {class: ms per launch} from the
library's event-timed kernel classes plus the whole-sweep time.
Usage: python profiles/kbench.py [n] [steps] [tag]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2103_04770_b200 import Context, Material

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
tag = sys.argv[3] if len(sys.argv) > 3 else ""
dev = torch.device("cuda", 0)
ctx = Context((n, n, n), (float(n),) * 3)
gen = torch.Generator(device=dev)
gen.manual_seed(1234)
ctx.set_phases(torch.from_numpy(synth.config1_phases(n, 0)).to(dev), 2)
for q, m in enumerate((synth.MATRIX_J2, synth.INCLUSION_EL)):
    ctx.set_material(q, Material.of(m))
ctx.set_nonlocal(synth.CONFIG1_ELL, [0])
ctx.set_control(synth.CONFIG1_MASK)
eps = torch.randn((6, n, n, n), generator=gen, dtype=torch.float64, device=dev) * 1e-3
zero6 = np.zeros(6)


def step():
    ctx.constitutive(eps)
    ctx.mech_residual(zero6)
    ctx.solve_tangent_cg(None, None, tol=0.0, maxit=10)
    ctx.solve_helmholtz(0, None, None, tol=0.0, maxit=10)


for _ in range(2):
    step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(steps):
    step()
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / steps * 1e3
ctx.set_timing(True)
for _ in range(steps):
    step()
torch.cuda.synchronize()
kt = ctx.kernel_times()
ctx.set_timing(False)
out = {"tag": tag, "n": n, "ms_per_step": round(wall, 3)}
for k, (ms, cnt) in kt.items():
    if cnt:
        out[k] = [round(ms / cnt, 4), round(cnt / steps, 2)]
print(json.dumps(out), flush=True)
