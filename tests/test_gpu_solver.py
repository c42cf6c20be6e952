"""GPU parity of the constitutive update, the Newton residual and the staggered increment
(Algorithm 1) against the oracle on the same seeded inputs.

Bars (BASELINE.json north_star): point-wise fields to ~1e-12 (same arithmetic, different
rounding order); macroscopic stress <= 1e-6 relative on every pre-peak increment; peak stress
and strain at failure <= 1e-4 (A-26, A-27).
"""
import dataclasses

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import synth  # noqa: E402
from oracle import material as M  # noqa: E402
from oracle.increment import Cell, State, Tolerances, evaluate, frozen_damage, make_cell, solve_increment  # noqa: E402
from oracle.mech import pack21  # noqa: E402
from oracle.projection import apply_projection  # noqa: E402
from paper_2103_04770_b200 import Context, Material  # noqa: E402
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


def small_config3(n=16):
    return synth.config3(n=n, n_spheres=4, phi=0.2, seed=3)


def test_constitutive_and_residual_parity():
    cfg = small_config3(16)
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    g = cell.grid
    nv = g.nvox
    rng = np.random.default_rng(1)
    st = State.zero(cell)
    st.epsp = M.dev(rng.normal(scale=1e-3, size=(6, nv)))
    st.ep = np.abs(rng.normal(scale=5e-3, size=nv))
    st.hist = np.where(cfg.phases.reshape(-1) == 0, rng.uniform(0, 0.3, nv), rng.uniform(0, 0.004, nv))
    st.abar = np.abs(rng.normal(scale=6e-3, size=(2,) + g.shape))
    eps = rng.normal(scale=4e-3, size=(6,) + g.shape)
    ctx.set_field(_fgd.FIELD_EPS_P, dev(st.epsp))
    ctx.set_field(_fgd.FIELD_EQPS, dev(st.ep))
    ctx.set_field(_fgd.FIELD_HIST, dev(st.hist))
    for j in range(2):
        ctx.set_field(_fgd.FIELD_NONLOCAL + j, dev(st.abar[j]))
    sig = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    macro = ctx.constitutive(dev(eps), sig)
    D = frozen_damage(cell, st, st.abar)
    s_ref, C_ref, a_ref, _, _ = evaluate(cell, eps, st, D)
    assert rel(sig.cpu().numpy(), s_ref) < 1e-13
    assert np.allclose(macro, s_ref.reshape(6, -1).mean(1), rtol=1e-12, atol=1e-12)
    Cg = torch.empty((21, nv), dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_TANGENT, Cg)
    assert rel(Cg.cpu().numpy(), pack21(C_ref.reshape(6, 6, -1))) < 1e-13
    for j in range(2):
        aj = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        ctx.get_field(_fgd.FIELD_SOURCE + j, aj)
        assert rel(aj.cpu().numpy(), a_ref[j]) < 1e-13
    # Newton residual -G*(sigma - Sigma_bar)
    S = np.array([1.0, 2.0, 0.0, 0.5, 0.0, 0.25])
    b = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    rms = ctx.mech_residual(S, b)
    b_ref = -apply_projection(g, s_ref, cfg.stress_mask, dc_mean_shift=S * np.array(cfg.stress_mask))
    assert rel(b.cpu().numpy(), b_ref) < 1e-10
    assert abs(rms - np.sqrt(np.sum(b_ref ** 2) / nv)) < 1e-10 * rms


TOL = Tolerances(tol_stag=1e-8, tol_newton=1e-10, tol_cg=1e-11, tol_helm=1e-11)


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
        out.append((rep.macro_stress.copy(), r["macro_stress"].copy(), rep, r))
    return out, ctx, st


def test_increment_parity_2d_disc():
    cfg = synth.config0(16, ell_over_L=2.0 / 16)
    cfg.dE = 8e-4
    out, ctx, st = run_both(cfg, 8)
    peak_i = int(np.argmax([o[0][0] for o in out]))
    for i, (ref, got, rep, r) in enumerate(out):
        if i <= peak_i:
            assert rel(got, ref) <= 1e-6, (i, ref, got)
    # committed fields
    eps = torch.empty((6,) + st.eps.shape[1:], dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_STRAIN, eps)
    assert rel(eps.cpu().numpy(), st.eps) < 1e-7
    h = torch.empty(st.hist.shape, dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_HIST, h)
    assert np.max(np.abs(h.cpu().numpy() - st.hist)) < 1e-6


def test_increment_parity_3d_two_fields():
    cfg = small_config3(16)
    cfg.dE = 1.5e-3
    out, ctx, st = run_both(cfg, 4)
    for i, (ref, got, rep, r) in enumerate(out):
        assert rel(got, ref) <= 1e-6, (i, ref, got)


def test_adaptive_run_replayed_by_oracle():
    """run.py's adaptive driver (A-34) on the GPU, then the oracle replays the accepted strain
    sequence (cut-back sub-steps included): same macroscopic stress up to the peak."""
    from paper_2103_04770_b200.run import run_config
    cfg = synth.config0(16, ell_over_L=2.0 / 16)
    cfg.dE = 4e-3                 # 10x the nominal step: the driver has to cut back near the peak
    tol = (TOL.tol_stag, TOL.tol_newton, TOL.tol_cg, TOL.tol_helm)
    res = run_config(cfg, n_incr=4, tol=tol, adaptive=True, max_cg=TOL.max_cg, max_helm=TOL.max_helm)
    assert not res["failed"]
    assert res["curve"][-1][0] == pytest.approx(4 * cfg.dE)
    cell = make_cell(cfg)
    st = State.zero(cell)
    s = np.array([c[1] for c in res["curve"]])
    peak = int(np.argmax(s))
    for i, (E, sig) in enumerate(res["curve"][1:], start=1):
        Et = np.zeros(6)
        Et[cfg.load_comp] = E
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        assert rep.converged, (i, E)
        if i <= peak:
            assert abs(rep.macro_stress[cfg.load_comp] - sig) <= 1e-6 * abs(rep.macro_stress[cfg.load_comp]), (i, E)


@pytest.mark.parametrize("n", [4, 16, 32, (32, 16)])
def test_mech_cg_compact_tangent_2d(n):
    """CG on the compact tangent written by fgd_constitutive on small 2D cells (the single-CTA
    k_cg_small path at <= 1024 voxels) against the oracle CG with the oracle's tangent."""
    from oracle.mech import cg
    n1, n2 = (n, n) if isinstance(n, int) else n
    cfg = synth.config0(32)
    cfg.n = (n1, n2, 1)
    cfg.L = (1.0, 1.0, 1.0 / n1)
    cfg.phases = synth.disc_phases(n1, 0.2, 1.0) if n1 == n2 else (np.arange(n1 * n2) % 5 == 0).astype(np.uint8).reshape(1, n2, n1)
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    g = cell.grid
    rng = np.random.default_rng(3)
    eps = rng.normal(scale=4e-3, size=(6,) + g.shape)
    eps[2] = eps[3] = eps[4] = 0.0
    st = State.zero(cell)
    ctx.constitutive(dev(eps), None)
    D = frozen_damage(cell, st, st.abar)
    _, C_ref, _, _, _ = evaluate(cell, eps, st, D)
    mask = cfg.stress_mask
    b = apply_projection(g, rng.normal(size=(6,) + g.shape), mask)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    it7, _ = ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=7)
    ref7, _, _ = cg(g, C_ref, b, mask, tol=0.0, maxit=7)
    assert it7 == 7 and rel(out.cpu().numpy(), ref7) <= 1e-10
    it, _ = ctx.solve_tangent_cg(dev(b), out, tol=1e-12, maxit=5000)
    ref, it_ref, _ = cg(g, C_ref, b, mask, tol=1e-12, maxit=5000)
    assert abs(it - it_ref) <= 1
    assert rel(out.cpu().numpy(), ref) <= 1e-9


def test_helmholtz_warm_start_iterates():
    """fgd_solve_helmholtz_from (S:262 warm start): PCG iterates from a guess x0 after k fixed
    iterations against the oracle's Algorithm 2 from the same x0, and the 0-iteration exit when the
    guess already meets the tolerance."""
    from oracle.helmholtz import ell2_field, solve_helmholtz
    from oracle.spectral import Grid
    for n in [(16, 8, 8), (256, 8, 8), (8, 256, 256)]:
        g = Grid(n, (1.0, 1.0, 1.0))
        rng = np.random.default_rng(7)
        ph = (rng.random(g.shape) < 0.3).astype(np.uint8)
        ell = [0.05, 0.01]
        ctx = Context(n, (1.0, 1.0, 1.0))
        ctx.set_phases(dev(ph), 2)
        ctx.set_nonlocal(np.array([ell]), [0])
        e2 = ell2_field(ph, ell)
        src = np.abs(rng.normal(size=g.shape))
        x0 = rng.normal(size=g.shape)
        out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        for k in (1, 4):
            it, _ = ctx.solve_helmholtz_from(0, dev(src), dev(x0), out, tol=0.0, maxit=k)
            ref, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=k, x0=x0)
            assert it == k and rel(out.cpu().numpy(), ref) <= 1e-10, (n, k)
        ref, it_ref, _ = solve_helmholtz(g, src, e2, tol=1e-11, maxit=2000)
        it, _ = ctx.solve_helmholtz_from(0, dev(src), dev(ref), out, tol=1e-9, maxit=2000)
        assert it == 0 and rel(out.cpu().numpy(), ref) <= 1e-14
        ctx.close()


def test_increment_parity_warm_start():
    """Staggered increments with warm-started Helmholtz solves on both sides (Tolerances.warm_start,
    fgd_increment.warm_start): same <sigma> (1e-6) and fewer PCG iterations than cold starts."""
    cfg = small_config3(16)
    cfg.dE = 1.5e-3
    tol = dataclasses.replace(TOL, warm_start=True)
    cell = make_cell(cfg)
    ctx = ctx_from_cfg(cfg)
    ctx_cold = ctx_from_cfg(cfg)
    st = State.zero(cell)
    helm_warm = helm_cold = 0
    for i in range(1, 4):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), tol)
        assert rep.converged
        s, r = ctx.solve_increment(Et, np.zeros(6), tol.tol_stag, tol.tol_newton, tol.tol_cg, tol.tol_helm,
                                   tol.max_stag, tol.max_newton, tol.max_cg, tol.max_helm, warm_start=True)
        assert s == 0, r
        assert rel(r["macro_stress"], rep.macro_stress) <= 1e-6, i
        assert abs(r["helm"] - rep.helm_it) <= 2 * r["stag"] * cell.J, (r["helm"], rep.helm_it)
        helm_warm += r["helm"]
        s, rc = ctx_cold.solve_increment(Et, np.zeros(6), tol.tol_stag, tol.tol_newton, tol.tol_cg, tol.tol_helm,
                                         tol.max_stag, tol.max_newton, tol.max_cg, tol.max_helm, warm_start=False)
        assert s == 0
        helm_cold += rc["helm"]
    assert helm_warm < helm_cold
