"""Helper of tests/test_gpu_race.py (run as a script in a subprocess, so that FGD_LIB selects the
production or the race-hunting build): one call of every operator and Krylov path on a seeded
device-generated input, outputs saved to an .npz.

    FGD_LIB=... python tests/race_case.py N1 N2 N3 out.npz
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2103_04770_b200 import Context, Material  # noqa: E402


def main():
    n = tuple(int(v) for v in sys.argv[1:4])
    out = sys.argv[4]
    shape = (n[2], n[1], n[0])
    nv = n[0] * n[1] * n[2]
    f64 = torch.float64
    gen = torch.Generator(device="cuda")
    gen.manual_seed(17)
    ctx = Context(n, (float(n[0]), float(n[1]), float(max(n[2], 1))) if n[2] > 1 else None)
    ctx.set_control(synth.CONFIG1_MASK if n[2] > 1 else (0, 1, 0, 0, 0, 1))
    ph = (torch.rand(shape, generator=gen, device="cuda", dtype=f64) < 0.2).to(torch.uint8)
    ctx.set_phases(ph, 2)
    ctx.set_material(0, Material.of(synth.MATRIX_J2))
    ctx.set_material(1, Material.of(synth.INCLUSION_EL))
    ctx.set_nonlocal(np.array([[2.0, 4.0]]) * (1.0 if n[2] > 1 else 1.0 / n[0]), [0])
    x = torch.randn((6,) + shape, generator=gen, dtype=f64, device="cuda") * 1e-3
    if n[2] == 1:
        x[2:5] = 0.0
    res = {}
    ctx.set_tangent(synth.random_spd_tangent_torch(nv, 7, device="cuda"))
    res["tangent_apply"] = ctx.apply_projected_tangent(x)
    res["projection"] = ctx.apply_projection(x)
    o6 = torch.empty_like(x)
    ctx.solve_tangent_cg(res["projection"], o6, tol=0.0, maxit=5)
    res["cg_packed"] = o6.clone()
    eps = torch.randn((6,) + shape, generator=gen, dtype=f64, device="cuda") * 5e-3
    if n[2] == 1:
        eps[2:5] = 0.0
    sig = torch.empty_like(eps)
    ctx.constitutive(eps, sig)
    res["sigma"] = sig
    b = torch.empty_like(x)
    ctx.mech_residual(np.zeros(6), b)
    res["residual"] = b
    ctx.solve_tangent_cg(b, o6, tol=0.0, maxit=5)
    res["cg_compact"] = o6.clone()
    a = x[0].contiguous() * 1e3
    res["helmholtz"] = ctx.apply_helmholtz(0, a)
    res["precond"] = ctx.apply_helmholtz_precond(0, a)
    o1 = torch.empty_like(a)
    ctx.solve_helmholtz(0, a.abs(), o1, tol=0.0, maxit=5)
    res["pcg"] = o1
    torch.cuda.synchronize()
    np.savez(out, **{k: v.cpu().numpy() for k, v in res.items()})
    ctx.close()


if __name__ == "__main__":
    main()
