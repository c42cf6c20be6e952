"""Diagnostic (not a test): locate disagreements of the 512^3 projected-tangent apply with the
oracle's per-frequency projection, line by line over the full spectrum (cuFFT used only as the
measuring instrument here).  Usage: python profiles/diag512.py [n]"""
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from oracle.mech import PACKED21
from oracle.projection import project_spectrum
from oracle.spectral import Grid
from paper_2103_04770_b200 import Context

n = int(sys.argv[1]) if len(sys.argv) > 1 else 512
g = Grid((n, n, n), (float(n),) * 3)
ctx = Context((n, n, n), (float(n),) * 3)
mask = synth.CONFIG1_MASK
ctx.set_control(mask)
gen = torch.Generator(device="cuda")
gen.manual_seed(11)
Cd = synth.random_spd_tangent_torch(g.nvox, 5, device="cuda")
ctx.set_tangent(Cd)
x = torch.randn((6,) + g.shape, generator=gen, dtype=torch.float64, device="cuda") * 1e-3
y = ctx.apply_projected_tangent(x)
y2 = ctx.apply_projected_tangent(x)
print("repeat bitwise-equal:", bool(torch.equal(y, y2)), "max diff", float((y - y2).abs().max()))
tau = torch.zeros_like(x)
for t, (i, j) in enumerate(PACKED21):
    cij = Cd[t].reshape(g.shape)
    tau[i] += cij * x[j]
    if i != j:
        tau[j] += cij * x[i]
del Cd, y2
yp = ctx.apply_projection(tau)
print("apply_projection(tau) vs apply_projected_tangent(x): rel",
      float((yp - y).norm() / y.norm()))
ks = g.symbol(half=True)
T = torch.fft.rfftn(tau, dim=(1, 2, 3))
del tau
bad = 0
rng = np.random.default_rng(1)
lines = [(172, 412)] + [tuple(int(v) for v in rng.integers(0, (n // 2 + 1, n))) for _ in range(40)]
for name, out in (("tangent", y), ("projection", yp)):
    Y = torch.fft.rfftn(out, dim=(1, 2, 3))
    for (kx, ky) in lines:
        ft = T[:, :, ky, kx].cpu().numpy()
        fy = Y[:, :, ky, kx].cpu().numpy()
        ref = project_spectrum(ft, ks[:, :, ky, kx], mask, dc_index=(0,) if (kx == 0 and ky == 0) else (0,))
        if kx == 0 and ky == 0:
            pass
        else:
            ref[:, 0] = project_spectrum(np.stack([np.zeros(6), ft[:, 0]], 1),
                                         np.stack([np.zeros(3), ks[:, 0, ky, kx]], 1), mask, dc_index=(0,))[:, 1]
        err = np.abs(fy - ref)
        scale = np.linalg.norm(ft, axis=0)
        rel = err.max(axis=0) / np.maximum(scale, 1e-300)
        if rel.max() > 1e-10:
            bad += 1
            kzs = np.nonzero(rel > 1e-10)[0]
            comps = np.nonzero((err[:, kzs] > 1e-10 * scale[kzs]).any(axis=1))[0]
            print(f"{name}: line kx={kx} ky={ky}: {len(kzs)} bad kz (first {kzs[:12].tolist()}), comps {comps.tolist()}, max rel {rel.max():.3e}")
    del Y
print("bad lines:", bad)
