"""Pins for oracle.increment (A-01, A-02, A-07, A-16, A-20-A-22) -- CPU only."""
import dataclasses

import numpy as np
import pytest

from oracle import material as M
from oracle.increment import Cell, State, Tolerances, solve_increment
from oracle.projection import apply_projection, mandel_to_tensor
from oracle.spectral import Grid, rfftn
from synth import INCLUSION_EL, MATRIX_J2, Material, config0

TOL = Tolerances(tol_stag=1e-10, tol_newton=1e-11, tol_cg=1e-12, tol_helm=1e-12)


def point_driver(mat, mask, load_comp, Es):
    """Textbook 1-voxel mixed-control Newton + damage fixed point (a homogeneous cell)."""
    mask = np.array(mask, bool)
    epsp = np.zeros((6, 1)); ep = np.zeros(1); Dn = 0.0
    eps = np.zeros(6)
    out = []
    for E in Es:
        eps = eps.copy(); eps[load_comp] = E
        D = Dn
        for _ in range(200):
            for _ in range(50):
                s, C, pp, pe, _, _ = M.j2_lemaitre(eps.reshape(6, 1), epsp, ep, np.array([D]), mat)
                r = s[mask, 0]
                if np.linalg.norm(r) < 1e-13 * max(1.0, np.linalg.norm(s)):
                    break
                eps[mask] -= np.linalg.solve(C[np.ix_(mask, mask)][:, :, 0], r)
            Dnew = max(Dn, float(M.lemaitre_damage(pe[0], mat.eps_c, mat.eps_r, mat.d_max)))
            if abs(Dnew - D) < 1e-14:
                break
            D = Dnew
        epsp, ep, Dn = pp, pe, max(Dn, float(M.lemaitre_damage(pe[0], mat.eps_c, mat.eps_r, mat.d_max)))
        out.append(s[:, 0].copy())
    return np.array(out)


def test_homogeneous_cell_is_uniform_and_equals_material_point():
    mat = dataclasses.replace(MATRIX_J2, eps_c=0.002, eps_r=0.012)
    g = Grid((4, 4, 4))
    mask = (1, 1, 0, 1, 1, 1)
    cell = Cell(g, np.zeros(g.shape, np.uint8), [mat], np.array([[0.1]]), [0], mask)
    st = State.zero(cell)
    Es = [1e-3 * i for i in range(1, 9)]
    ref = point_driver(mat, mask, 2, Es)
    for i, E in enumerate(Es):
        Et = np.zeros(6); Et[2] = E
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        assert rep.converged
        e = st.eps.reshape(6, -1)
        assert np.max(e.max(axis=1) - e.min(axis=1)) <= 1e-13 * max(1e-3, np.abs(e).max())
        assert np.allclose(rep.macro_stress, ref[i], rtol=1e-9, atol=1e-7)
    assert st.hist.max() > 0.1      # damage was active


def test_elastic_uniaxial_stress_3d_and_plane_strain_2d():
    mat = Material(model=0, E=70e3, nu=0.3)
    for n, mask, expect in [((4, 4, 4), (0, 1, 1, 1, 1, 1), mat.E),
                            ((8, 8, 1), (0, 1, 0, 0, 0, 1), mat.E / (1 - mat.nu ** 2))]:
        g = Grid(n)
        cell = Cell(g, np.zeros(g.shape, np.uint8), [mat], np.array([[0.1]]), [0], mask)
        Et = np.zeros(6); Et[0] = 1e-3
        st, rep = solve_increment(cell, State.zero(cell), Et, np.zeros(6), TOL)
        assert abs(rep.macro_stress[0] - expect * 1e-3) < 1e-10 * expect * 1e-3


def test_laminate_closed_form():
    m0 = Material(model=0, E=70e3, nu=0.3)
    m1 = Material(model=0, E=400e3, nu=0.2)
    g = Grid((8, 2, 2))
    ph = np.zeros(g.shape, np.uint8); ph[:, :, 5:] = 1          # layers normal to x, f1 = 3/8
    cell = Cell(g, ph, [m0, m1], np.array([[0.1, 0.1]]), [0], (0,) * 6)
    Et = np.zeros(6); Et[0] = 1e-3
    st, rep = solve_increment(cell, State.zero(cell), Et, np.zeros(6), TOL)
    f = np.array([5 / 8, 3 / 8])
    lam, Pm = [], []
    for m in (m0, m1):
        K, mu = M.moduli(m.E, m.nu)
        lam.append(K - 2 * mu / 3); Pm.append(K + 4 * mu / 3)
    s11 = 1e-3 / np.sum(f / np.array(Pm))
    e11 = s11 / np.array(Pm)
    s22 = np.sum(f * np.array(lam) * e11)
    assert abs(rep.macro_stress[0] - s11) < 1e-10 * s11
    assert abs(rep.macro_stress[1] - s22) < 1e-10 * s11


def small_disc(n=16):
    cfg = config0(n, ell_over_L=2.0 / 16)
    g = Grid(cfg.n, cfg.L)
    return Cell(g, cfg.phases, cfg.materials, cfg.ell, cfg.source_phase, cfg.stress_mask)


def test_equilibrium_compatibility_fixed_point():
    cell = small_disc()
    g = cell.grid
    st = State.zero(cell)
    for E in (2e-3, 4e-3, 6e-3):
        Et = np.zeros(6); Et[0] = E
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        assert rep.converged
    assert st.ep.max() > 1e-3                      # plastic
    # equilibrium: sigma^ conj(k) = 0 at every xi != 0
    T = mandel_to_tensor(rfftn(rep.sigma))
    k = g.symbol()
    t = np.einsum("ij...,j...->i...", T, np.conj(k))
    t[:, 0, 0, 0] = 0
    scale = np.max(np.abs(T)) * np.max(np.abs(k))
    assert np.max(np.abs(t)) < 1e-9 * scale
    # stress-controlled macroscopic components vanish (mask (0,1,0,0,0,1), Sigma = 0)
    assert abs(rep.macro_stress[1]) < 1e-8 * abs(rep.macro_stress[0])
    assert abs(rep.macro_stress[5]) < 1e-8 * abs(rep.macro_stress[0])
    # compatibility: G*_{mask=0}(eps) = eps - <eps>
    e = st.eps
    fl = apply_projection(g, e, (0,) * 6)
    assert np.max(np.abs(fl - (e - e.reshape(6, -1).mean(1).reshape(6, 1, 1, 1)))) < 1e-12
    # fixed point: re-solving the converged increment changes nothing
    st2, rep2 = solve_increment(cell, st, Et, np.zeros(6), TOL)
    assert rep2.converged
    assert np.max(np.abs(st2.eps - st.eps)) < 1e-9 * np.max(np.abs(st.eps))
    assert np.allclose(rep2.macro_stress, rep.macro_stress, rtol=1e-7, atol=1e-6)


def test_elastic_path_independence_and_two_staggered_iterations():
    mat1 = Material(model=0, E=70e3, nu=0.3)
    cfg = config0(8)
    g = Grid(cfg.n, cfg.L)
    cell = Cell(g, cfg.phases, [mat1, INCLUSION_EL], cfg.ell, cfg.source_phase, cfg.stress_mask)
    Et = np.zeros(6); Et[0] = 4e-3
    a, ra = solve_increment(cell, State.zero(cell), Et, np.zeros(6), TOL)
    assert ra.stag_it == 2
    st = State.zero(cell)
    for E in (1e-3, 2e-3, 3e-3, 4e-3):
        Et = np.zeros(6); Et[0] = E
        st, rb = solve_increment(cell, st, Et, np.zeros(6), TOL)
    assert np.max(np.abs(a.eps - st.eps)) < 1e-12
    assert np.allclose(ra.macro_stress, rb.macro_stress, rtol=1e-10, atol=1e-9)


def gtn_point_driver(mat, mask, load_comp, Es):
    """1-voxel mixed-control Newton + staggered fixed point for GTN (homogeneous cell: the
    Helmholtz solution of a uniform source is the source, so abar = (eps0p, tr eps^p))."""
    from oracle import gtn as GT
    mask = np.array(mask, bool)
    epsp_n, e0_n, f_n, eb_n, tb_n = np.zeros(6), 0.0, 0.0, 0.0, 0.0
    eps = np.zeros(6)
    out = []
    for E in Es:
        eps = eps.copy(); eps[load_comp] = E
        eb, tb = eb_n, tb_n
        for _ in range(200):
            f = GT.porosity(f_n, eb, eb_n, tb, tb_n, mat)
            for _ in range(60):
                r = GT.gtn_point(eps, epsp_n, e0_n, f, mat)
                res = r["sigma"][mask]
                if np.linalg.norm(res) < 1e-13 * max(1.0, np.linalg.norm(r["sigma"])):
                    break
                eps[mask] -= np.linalg.solve(r["C"][np.ix_(mask, mask)], res)
            eb_new, tb_new = r["e0"], r["epsp"][:3].sum()
            done = abs(eb_new - eb) + abs(tb_new - tb) < 1e-15
            eb, tb = eb_new, tb_new
            if done:
                break
        f_n = GT.porosity(f_n, eb, eb_n, tb, tb_n, mat)
        epsp_n, e0_n, eb_n, tb_n = r["epsp"], r["e0"], eb, tb
        out.append((r["sigma"].copy(), f_n))
    return out


def test_homogeneous_gtn_cell_equals_material_point():
    # nucleation moved into the loading range so that porosity grows within a few increments
    mat = Material(model=3, E=300e3, nu=0.3, sigma_y=1000.0, eps_n=0.02, s_n=0.01, f_n=0.04)
    g = Grid((4, 4, 4))
    mask = (1, 1, 0, 1, 1, 1)
    cell = Cell(g, np.zeros(g.shape, np.uint8), [mat], np.array([[0.1], [0.1]]), [0, 0], mask)
    st = State.zero(cell)
    Es = [4e-3 * i for i in range(1, 9)]
    ref = gtn_point_driver(mat, mask, 2, Es)
    for i, E in enumerate(Es):
        Et = np.zeros(6); Et[2] = E
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        assert rep.converged
        e = st.eps.reshape(6, -1)
        assert np.max(e.max(axis=1) - e.min(axis=1)) <= 1e-13 * max(1e-3, np.abs(e).max())
        assert np.allclose(rep.macro_stress, ref[i][0], rtol=1e-9, atol=1e-7)
        assert np.allclose(st.hist, ref[i][1], rtol=1e-9, atol=1e-15)
    assert st.hist.max() > 0.01          # porosity grew (nucleation + dilatant growth)
    assert np.all(st.epsp[:3].sum(axis=0) > 0)


def test_homogeneous_gtn_plane_strain_equals_material_point():
    """Plane strain (A-19, A-20: eps33 = eps13 = eps23 = 0, Sigma22 = Sigma12 = 0) GTN cell."""
    mat = Material(model=3, E=300e3, nu=0.3, sigma_y=1000.0, eps_n=0.02, s_n=0.01, f_n=0.04)
    g = Grid((4, 4, 1))
    mask = (0, 1, 0, 0, 0, 1)
    cell = Cell(g, np.zeros(g.shape, np.uint8), [mat], np.array([[0.1], [0.1]]), [0, 0], mask)
    st = State.zero(cell)
    Es = [5e-3 * i for i in range(1, 7)]
    ref = gtn_point_driver(mat, mask, 0, Es)
    for i, E in enumerate(Es):
        Et = np.zeros(6); Et[0] = E
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        assert rep.converged
        assert np.allclose(rep.macro_stress, ref[i][0], rtol=1e-9, atol=1e-7)
        assert np.allclose(st.hist, ref[i][1], rtol=1e-9, atol=1e-15)
        assert abs(rep.macro_stress[2]) > 0          # sigma33 carried (A-19)
    assert st.hist.max() > 0.01


def test_voigt_reuss_bounds_and_exact_strain_averages():
    """Elastic two-phase disc cell, all components strain-controlled with a random macroscopic
    strain E: <eps> = E exactly and E:C_Reuss:E <= <sigma>:E <= E:C_Voigt:E."""
    cfg = config0(8)
    g = Grid(cfg.n, cfg.L)
    m0 = Material(model=0, E=70e3, nu=0.3)
    cell = Cell(g, cfg.phases, [m0, INCLUSION_EL], cfg.ell, cfg.source_phase, (0,) * 6)
    rng = np.random.default_rng(2)
    E = rng.normal(scale=1e-3, size=6)
    st, rep = solve_increment(cell, State.zero(cell), E, np.zeros(6), TOL)
    assert rep.converged
    assert np.max(np.abs(st.eps.reshape(6, -1).mean(1) - E)) < 1e-15
    f1 = float(np.mean(cfg.phases == 1))
    C0, C1 = M.elastic_stiffness(m0.E, m0.nu), M.elastic_stiffness(INCLUSION_EL.E, INCLUSION_EL.nu)
    CV = (1 - f1) * C0 + f1 * C1
    CR = np.linalg.inv((1 - f1) * np.linalg.inv(C0) + f1 * np.linalg.inv(C1))
    w = float(rep.macro_stress @ E)
    assert E @ CR @ E <= w <= E @ CV @ E
    assert E @ CR @ E < 0.999 * w and w < 0.999 * E @ CV @ E     # strictly inside for this contrast


def test_line_search_keeps_the_converged_increment():
    """R-LS (backtracking on the Newton residual) is a globalisation only: on a plastic disc cell
    where plain Newton converges, both reach the same increment solution (and with a large load
    step the backtracking variant converges with no more Newton iterations than plain Newton)."""
    import dataclasses
    import synth
    from oracle.increment import State, Tolerances, make_cell, solve_increment
    cfg = synth.config0(8, ell_over_L=0.25)
    cell = make_cell(cfg)
    st = State.zero(cell)
    E = np.zeros(6)
    E[0] = 4e-3                                   # one large step well into plasticity
    tol = Tolerances(tol_stag=1e-9, tol_newton=1e-11, tol_cg=1e-12, tol_helm=1e-12)
    s1, r1 = solve_increment(cell, st, E, np.zeros(6), dataclasses.replace(tol, line_search=True))
    s0, r0 = solve_increment(cell, st, E, np.zeros(6), dataclasses.replace(tol, line_search=False))
    assert r1.converged and r0.converged
    assert np.max(np.abs(s1.eps - s0.eps)) <= 1e-10 * np.max(np.abs(s0.eps))
    assert np.allclose(r1.macro_stress, r0.macro_stress, rtol=1e-9, atol=1e-9)
