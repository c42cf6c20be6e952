"""Driver for compute-sanitizer (racecheck / synccheck), not a test: one call of every operator
and Krylov path of libfgd on a grid chosen to select a family of specialised kernels, so that the
sanitizer sees each kernel instantiation once.

    python profiles/race_driver.py N1 N2 N3 [--compact] [--helm]

  (256, 4, 4)   k_xtan<256> (packed + compact tangent, CG), k_xipipe<256>, PCG x-forward
  (512, 4, 4)   k_xtan<512>, k_xipipe<512>
  (4, 256, 256) k_yreg256 fwd / inv, k_zreg256<6> / <1>
  (4, 512, 512) k_yreg512 fwd / inv, k_zreg512<6> / <1>
  (16, 16, 16)  generic pipes (k_ypipe, k_zpipe, k_xfwd), stencil, constitutive, err, commit
Inputs are seeded and generated on the device.  Exit status 0 when every call returned FGD_OK.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import synth
from paper_2103_04770_b200 import Context, Material

n = tuple(int(v) for v in sys.argv[1:4])
nv = n[0] * n[1] * n[2]
shape = (n[2], n[1], n[0])
f64 = torch.float64
gen = torch.Generator(device="cuda")
gen.manual_seed(5)
ctx = Context(n, (float(n[0]), float(n[1]), float(n[2])))
ctx.set_control(synth.CONFIG1_MASK)
ph = (torch.rand(shape, generator=gen, device="cuda", dtype=f64) < 0.2).to(torch.uint8)
ctx.set_phases(ph, 2)
ctx.set_material(0, Material.of(synth.MATRIX_J2))
ctx.set_material(1, Material.of(synth.INCLUSION_EL))
ctx.set_nonlocal(np.array([[2.0, 4.0]]), [0])
x = torch.randn((6,) + shape, generator=gen, dtype=f64, device="cuda") * 1e-3
# packed tangent path
ctx.set_tangent(synth.random_spd_tangent_torch(nv, 7, device="cuda"))
y = ctx.apply_projected_tangent(x)
p = ctx.apply_projection(x)
b = torch.empty_like(x)
ctx.solve_tangent_cg(p, b, tol=0.0, maxit=3)
# compact tangent path (constitutive update) + Newton residual + CG, converged with the device guard
eps = torch.randn((6,) + shape, generator=gen, dtype=f64, device="cuda") * 5e-3
ctx.constitutive(eps)
ctx.mech_residual(np.zeros(6), b)
ctx.solve_tangent_cg(None, None, tol=0.0, maxit=3)
ctx.solve_tangent_cg(None, None, tol=1e-6, maxit=200, check=False)
# Helmholtz apply, preconditioner, PCG (fixed and converged)
a = x[0].contiguous()
ctx.apply_helmholtz(0, a)
ctx.apply_helmholtz_precond(0, a)
o = torch.empty_like(a)
ctx.solve_helmholtz(0, a.abs(), o, tol=0.0, maxit=3)
ctx.solve_helmholtz(0, a.abs(), o, tol=1e-8, maxit=200, check=False)
# one increment (staggered loop, err, commit)
if nv <= 1 << 16:
    Et = np.zeros(6)
    Et[2] = 2e-3
    st, rep = ctx.solve_increment(Et, np.zeros(6), 1e-6, 1e-8, 1e-9, 1e-9, 20, 20, 2000, 2000)
    print("increment", st, rep["stag"], rep["cg"])
torch.cuda.synchronize()
ctx.close()
print("ok", n)
