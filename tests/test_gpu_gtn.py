"""GPU parity of the non-local GTN model (material model 3; paper Sec. 2.1.1, 2.2.2, App. A)
against oracle/gtn.py through the C ABI: the per-voxel update (stress, symmetrised consistent
tangent, Helmholtz sources, frozen porosity) and whole increments of Algorithm 1.

Bars: point-wise fields 1e-11 (both sides iterate the return mapping to round-off; different
rounding order and 3x3 solver), macroscopic stress <= 1e-6 relative per pre-peak increment.
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import synth  # noqa: E402
from oracle.increment import State, Tolerances, evaluate, frozen_damage, make_cell, solve_increment  # noqa: E402
from oracle.mech import pack21  # noqa: E402
from paper_2103_04770_b200 import Context, FgdError, Material  # noqa: E402
from paper_2103_04770_b200 import _fgd  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def ctx_from_cfg(cfg):
    ctx = Context(cfg.n, cfg.L)
    ctx.set_phases(dev(cfg.phases), len(cfg.materials))
    for q, m in enumerate(cfg.materials):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
    ctx.set_control(cfg.stress_mask)
    return ctx


def early_nucleation(cfg):
    """Move nucleation into the first percent of strain so that porosity, f* and the dilatant
    flow are all exercised within a few increments."""
    cfg.materials = [dataclasses.replace(cfg.materials[0], eps_n=0.006, s_n=0.003, f_n=0.04)] + cfg.materials[1:]
    return cfg


@pytest.mark.parametrize("which", ["2d", "3d"])
def test_gtn_constitutive_parity(which):
    cfg = synth.config_gtn2d(32) if which == "2d" else synth.config_gtn3d(16, n_spheres=4)
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    g = cell.grid
    nv = g.nvox
    rng = np.random.default_rng(7)
    mat = cfg.materials[0]
    ey = mat.sigma_y / mat.E
    st = State.zero(cell)
    st.epsp = rng.normal(scale=0.5 * ey, size=(6, nv))
    st.ep = np.abs(rng.normal(scale=2 * ey, size=nv))
    # porosity history across all f* branches: below f_C, coalescence, beyond f_F (capped f*)
    st.hist = rng.choice([0.0, 0.01, 0.1, 0.18, 0.3], size=nv)
    st.abar = np.abs(rng.normal(scale=2 * ey, size=(2,) + g.shape))
    abar = st.abar + np.abs(rng.normal(scale=0.5 * ey, size=(2,) + g.shape))
    eps = rng.normal(scale=2.5 * ey, size=(6,) + g.shape)
    eps[:3] += rng.normal(scale=ey, size=g.shape)
    if which == "2d":
        eps[2] = eps[3] = eps[4] = 0.0
    ctx.set_field(_fgd.FIELD_EPS_P, dev(st.epsp))
    ctx.set_field(_fgd.FIELD_EQPS, dev(st.ep))
    ctx.set_field(_fgd.FIELD_HIST, dev(st.hist))
    for j in range(2):
        ctx.set_field(_fgd.FIELD_NONLOCAL + j, dev(st.abar[j]))            # committed (and current)
        ctx.set_field(_fgd.FIELD_NONLOCAL_ITERATE + j, dev(abar[j]))       # current staggered iterate
    sig = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    macro = ctx.constitutive(dev(eps), sig)
    f = frozen_damage(cell, st, abar)
    s_ref, C_ref, a_ref, _, _ = evaluate(cell, eps, st, f)
    # most matrix voxels return to the yield surface (stress differs from the elastic trial)
    K, mu = mat.E / (3 * (1 - 2 * mat.nu)), mat.E / (2 * (1 + mat.nu))
    one = np.array([1.0, 1, 1, 0, 0, 0])[:, None]
    ee = eps.reshape(6, -1) - st.epsp
    tr = ee[:3].sum(0)
    trial = 2 * mu * (ee - one * tr / 3) + K * tr * one
    matrix = cfg.phases.reshape(-1) == 0
    plastic = matrix & (np.abs(s_ref.reshape(6, -1) - trial).max(0) > 1e-8 * np.abs(trial).max(0))
    assert plastic.sum() > 0.3 * matrix.sum()
    assert rel(sig.cpu().numpy(), s_ref) < 1e-11
    assert np.allclose(macro, s_ref.reshape(6, -1).mean(1), rtol=1e-11, atol=1e-9)
    Cg = torch.empty((21, nv), dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_TANGENT, Cg)
    assert rel(Cg.cpu().numpy(), pack21(C_ref.reshape(6, 6, -1))) < 1e-10
    for j in range(2):
        aj = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        ctx.get_field(_fgd.FIELD_SOURCE + j, aj)
        assert rel(aj.cpu().numpy(), a_ref[j]) < 1e-11


TOL = Tolerances(tol_stag=1e-9, tol_newton=1e-10, tol_cg=1e-11, tol_helm=1e-11)


def run_both(cfg, n_incr):
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    st = State.zero(cell)
    out = []
    for i in range(1, n_incr + 1):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        s, r = ctx.solve_increment(Et, np.zeros(6), TOL.tol_stag, TOL.tol_newton, TOL.tol_cg, TOL.tol_helm,
                                   TOL.max_stag, TOL.max_newton, TOL.max_cg, TOL.max_helm)
        assert s == 0, r
        assert rep.converged
        out.append((rep.macro_stress.copy(), r["macro_stress"].copy()))
    return out, ctx, st


def _check_committed(ctx, st):
    h = torch.empty(st.hist.shape, dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_HIST, h)
    assert np.max(np.abs(h.cpu().numpy() - st.hist)) < 1e-7
    ep = torch.empty(st.ep.shape, dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_EQPS, ep)
    assert np.max(np.abs(ep.cpu().numpy() - st.ep)) < 1e-7


def test_gtn_increment_parity_2d():
    cfg = early_nucleation(synth.config_gtn2d(16))
    cfg.dE = 3e-3
    out, ctx, st = run_both(cfg, 6)
    peak = int(np.argmax([o[0][0] for o in out]))
    for i, (ref, got) in enumerate(out):
        if i <= peak:
            assert rel(got, ref) <= 1e-6, (i, ref, got)
    assert st.hist.max() > 1e-3                    # porosity grew
    _check_committed(ctx, st)


def test_gtn_increment_parity_3d():
    cfg = early_nucleation(synth.config_gtn3d(8, n_spheres=2))
    cfg.dE = 3e-3
    out, ctx, st = run_both(cfg, 4)
    for i, (ref, got) in enumerate(out):
        assert rel(got, ref) <= 1e-6, (i, ref, got)
    assert st.hist.max() > 1e-4
    _check_committed(ctx, st)


def test_gtn_needs_two_fields():
    cfg = synth.config_gtn2d(16)
    ctx = Context(cfg.n, cfg.L)
    ctx.set_phases(dev(cfg.phases), 2)
    for q, m in enumerate(cfg.materials):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(np.asarray(cfg.ell)[:1], [0])
    ctx.set_control(cfg.stress_mask)
    with pytest.raises(FgdError):
        ctx.constitutive(dev(np.zeros((6,) + cfg.phases.shape)), None)
