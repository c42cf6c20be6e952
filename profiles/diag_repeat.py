"""Diagnostic (not a test): repeat the operator applies on the same input and localise any
run-to-run difference in spectral space (which (comp, kx, ky) lines differ).
Usage: python profiles/diag_repeat.py n reps"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import synth
from paper_2103_04770_b200 import Context

n = int(sys.argv[1])
reps = int(sys.argv[2])
ctx = Context((n, n, n), (float(n),) * 3)
ctx.set_control(synth.CONFIG1_MASK)
gen = torch.Generator(device="cuda")
gen.manual_seed(11)
ctx.set_tangent(synth.random_spd_tangent_torch(n ** 3, 5, device="cuda"))
x = torch.randn((6, n, n, n), generator=gen, dtype=torch.float64, device="cuda") * 1e-3


def localise(tag, a, b):
    d = torch.fft.rfftn(a - b, dim=(1, 2, 3)).abs()   # [c, kz, ky, kx]
    scale = float(torch.fft.rfftn(a, dim=(1, 2, 3)).abs().max())
    m = d > 1e-12 * scale
    if not bool(m.any()):
        return
    lines = m.any(dim=1).nonzero().tolist()        # (c, ky, kx)
    kxs = sorted({l[2] for l in lines})
    print(f"  {tag}: {len(lines)} (c,ky,kx) lines differ; comps {sorted({l[0] for l in lines})}; "
          f"kx values {kxs[:10]}{'...' if len(kxs) > 10 else ''}; first lines {lines[:6]}; "
          f"bad kz per line {int(m[lines[0][0], :, lines[0][1], lines[0][2]].sum())}", flush=True)


for name, fn, arg in (("projected_tangent", ctx.apply_projected_tangent, x),
                      ("projection", ctx.apply_projection, x)):
    y0 = fn(arg)
    nd = 0
    for r in range(reps):
        y = fn(arg)
        if not torch.equal(y, y0):
            nd += 1
            print(f"{name} rep {r}: differs, max |diff| {float((y - y0).abs().max()):.3e} "
                  f"(max |y| {float(y0.abs().max()):.3e})", flush=True)
            localise(name, y, y0)
    print(f"{name}: {nd}/{reps} repeats differ from the first", flush=True)
