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


def _check_committed(ctx, st, cfg=None):
    if cfg is not None:
        # App. A: the GTN stress is the elastic law at the returned plastic strain,
        # sigma = C^e (eps - eps^p), also at the dilatant (f* > 0) returns; on the GPU the stress of
        # the last mechanical solve and the committed eps, eps^p belong to the same converged state
        sh = (6,) + tuple(cfg.phases.shape)
        sig, eps, epsp = (torch.empty(sh, dtype=torch.float64, device="cuda") for _ in range(3))
        ctx.get_field(_fgd.FIELD_STRESS, sig)
        ctx.get_field(_fgd.FIELD_STRAIN, eps)
        ctx.get_field(_fgd.FIELD_EPS_P, epsp)
        sig, eps, epsp = (t.cpu().numpy().reshape(6, -1) for t in (sig, eps, epsp))
        ph = cfg.phases.reshape(-1)
        one = np.r_[1.0, 1, 1, 0, 0, 0]
        for q, m in enumerate(cfg.materials):
            K, mu = m.E / (3.0 * (1.0 - 2.0 * m.nu)), m.E / (2.0 * (1.0 + m.nu))
            Ce = K * np.outer(one, one) + 2.0 * mu * (np.eye(6) - np.outer(one, one) / 3.0)
            sel = ph == q
            s_el = Ce @ (eps[:, sel] - epsp[:, sel])
            assert np.abs(sig[:, sel] - s_el).max() <= 1e-10 * np.abs(s_el).max(), q
        assert np.abs(epsp[:3, ph == 0].sum(0)).max() > 0.0     # dilatant returns present
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
    _check_committed(ctx, st, cfg)


def test_gtn_increment_parity_3d():
    cfg = early_nucleation(synth.config_gtn3d(8, n_spheres=2))
    cfg.dE = 3e-3
    out, ctx, st = run_both(cfg, 4)
    for i, (ref, got) in enumerate(out):
        assert rel(got, ref) <= 1e-6, (i, ref, got)
    assert st.hist.max() > 1e-4
    _check_committed(ctx, st, cfg)


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


def test_gtn_full_size_sampled():
    """The 256^3 GTN update in the bench's launch configuration (bench.gtn_measurement's state
    recipe): 400 sampled voxels recomputed one by one by the oracle's point update."""
    from oracle import gtn as GT
    n = 256
    cfg_m = synth.MATRIX_GTN_3D
    ph = synth.config1_phases(n, 0)
    ctx = Context((n, n, n), (1.0, 1.0, 1.0))
    ctx.set_phases(dev(ph), 2)
    ctx.set_material(0, Material.of(cfg_m))
    ctx.set_material(1, Material.of(synth.INCLUSION_EL))
    ctx.set_nonlocal(np.array([[0.05, 0.001], [0.05, 0.001]]), [0, 0])
    ctx.set_control(synth.CONFIG1_MASK)
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    f64 = torch.float64
    ey = cfg_m.sigma_y / cfg_m.E
    eps = torch.randn((6, n, n, n), generator=g, dtype=f64, device="cuda") * (2.5 * ey)
    epsp = torch.randn((6, n, n, n), generator=g, dtype=f64, device="cuda") * (0.5 * ey)
    e0 = torch.randn((n, n, n), generator=g, dtype=f64, device="cuda").abs() * (2 * ey)
    hist = torch.rand((n, n, n), generator=g, dtype=f64, device="cuda") * 0.3
    ab_n = torch.randn((2, n, n, n), generator=g, dtype=f64, device="cuda").abs() * (2 * ey)
    ab = ab_n + torch.randn((2, n, n, n), generator=g, dtype=f64, device="cuda").abs() * (0.5 * ey)
    ctx.set_field(_fgd.FIELD_EPS_P, epsp)
    ctx.set_field(_fgd.FIELD_EQPS, e0)
    ctx.set_field(_fgd.FIELD_HIST, hist)
    for j in range(2):
        ctx.set_field(_fgd.FIELD_NONLOCAL + j, ab_n[j].contiguous())
        ctx.set_field(_fgd.FIELD_NONLOCAL_ITERATE + j, ab[j].contiguous())
    sig = torch.empty_like(eps)
    ctx.constitutive(eps, sig)
    Cg = torch.empty((21, n * n * n), dtype=f64, device="cuda")
    ctx.get_field(_fgd.FIELD_TANGENT, Cg)
    rng = np.random.default_rng(5)
    vox = rng.choice(n ** 3, size=400, replace=False)
    flat = lambda t, c: t.reshape(c, -1)[:, vox].cpu().numpy()   # noqa: E731
    E6, P6, S6, C21 = flat(eps, 6), flat(epsp, 6), flat(sig, 6), Cg[:, vox].cpu().numpy()
    E0, H, A, An = flat(e0, 1)[0], flat(hist, 1)[0], flat(ab, 2), flat(ab_n, 2)
    phv = ph.reshape(-1)[vox]
    iu = np.triu_indices(6)
    nplastic = 0
    for i in range(vox.size):
        if phv[i] != 0:
            continue                                   # elastic inclusion: covered by the J2 tests
        f = GT.porosity(H[i], A[0, i], An[0, i], A[1, i], An[1, i], cfg_m)
        r = GT.gtn_point(E6[:, i], P6[:, i], E0[i], f, cfg_m)
        nplastic += r["plastic"]
        assert np.abs(S6[:, i] - r["sigma"]).max() <= 1e-11 * np.abs(r["sigma"]).max(), i
        assert np.abs(C21[:, i] - r["C_sym"][iu]).max() <= 1e-9 * np.abs(r["C_sym"]).max(), i
    assert nplastic > 200
    ctx.close()


def test_gtn_hydrostatic_degenerate_branch():
    """Pure hydrostatic strain on a porous GTN cell: q_tr = 0 (n = 0, theta = 1 branch) and
    purely dilatant flow, against the oracle."""
    cfg = synth.config_gtn2d(16)
    cfg.phases = np.zeros_like(cfg.phases)           # all GTN matrix
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    g = cell.grid
    st = State.zero(cell)
    st.hist = np.full(g.nvox, 0.05)
    ctx.set_field(_fgd.FIELD_HIST, dev(st.hist))
    eps = np.zeros((6,) + g.shape)
    eps[:3] = np.linspace(0.002, 0.02, g.nvox).reshape(g.shape)   # from elastic to deep plastic
    sig = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    ctx.constitutive(dev(eps), sig)
    s_ref, C_ref, a_ref, epsp_ref, _ = evaluate(cell, eps, st, frozen_damage(cell, st, st.abar))
    assert rel(sig.cpu().numpy(), s_ref) < 1e-11
    assert np.abs(s_ref[3:]).max() == 0.0 and np.allclose(s_ref[0], s_ref[1]) and np.allclose(s_ref[1], s_ref[2])
    Cg = torch.empty((21, g.nvox), dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_TANGENT, Cg)
    assert rel(Cg.cpu().numpy(), pack21(C_ref.reshape(6, 6, -1))) < 1e-10
    tr = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_SOURCE + 1, tr)                     # tr eps^p source
    assert rel(tr.cpu().numpy(), a_ref[1]) < 1e-11
    assert (a_ref[1] > 0).sum() > g.nvox // 2                    # most points flowed (dilatancy)
