"""Pins for oracle.material (A-14..A-18) -- CPU only."""
import json
import os

import numpy as np
import pytest

from oracle import material as M
from synth import MATRIX_J2, PARTICLE_BRITTLE, Material

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
rng = np.random.default_rng(3)


def random_states(n, scale=4e-3):
    eps = rng.normal(scale=scale, size=(6, n))
    epsp = M.dev(rng.normal(scale=scale / 3, size=(6, n)))
    ep = np.abs(rng.normal(scale=scale, size=n))
    D = rng.uniform(0, 0.5, size=n)
    return eps, epsp, ep, D


def test_consistent_tangent_matches_central_fd_and_is_symmetric():
    eps, epsp, ep, D = random_states(400, 2.5e-3)
    s0, C, _, _, plastic, _ = M.j2_lemaitre(eps, epsp, ep, D, MATRIX_J2)
    assert plastic.sum() > 50 and (~plastic).sum() > 10
    h = 1e-7
    for j in range(6):
        e1 = eps.copy(); e1[j] += h
        e2 = eps.copy(); e2[j] -= h
        sp = M.j2_lemaitre(e1, epsp, ep, D, MATRIX_J2)[0]
        sm = M.j2_lemaitre(e2, epsp, ep, D, MATRIX_J2)[0]
        fd = (sp - sm) / (2 * h)
        # skip points whose perturbation straddles the yield surface
        f1 = M.j2_lemaitre(e1, epsp, ep, D, MATRIX_J2)[4]
        f2 = M.j2_lemaitre(e2, epsp, ep, D, MATRIX_J2)[4]
        ok = f1 == f2
        err = np.abs(fd[:, ok] - C[:, j, ok])
        assert np.max(err) < 1e-5 * np.max(np.abs(C[:, :, ok]))
    assert np.max(np.abs(C - np.transpose(C, (1, 0, 2)))) < 1e-9


def test_yield_consistency_and_incompressibility():
    eps, epsp, ep, D = random_states(1000, 6e-3)
    s, C, pp, pe, plastic, phi = M.j2_lemaitre(eps, epsp, ep, D, MATRIX_J2)
    assert np.all(np.abs(phi[plastic]) <= 1e-8 * MATRIX_J2.sigma_y)
    assert np.all(phi[~plastic] <= 1e-12)
    dp = pp - epsp
    assert np.max(np.abs(dp[0] + dp[1] + dp[2])) < 1e-15
    assert np.all(pe >= ep)


def test_uniaxial_tangent_EH_over_E_plus_H():
    mat = Material(model=1, E=70e3, nu=0.3, sigma_y=300.0, H=500.0)
    e = 0.01
    eps = np.array([[e], [-0.4 * e], [-0.4 * e], [0.0], [0.0], [0.0]])
    _, C, _, _, plastic, _ = M.j2_lemaitre(eps, np.zeros((6, 1)), np.zeros(1), np.zeros(1), mat)
    assert plastic[0]
    S = np.linalg.inv(C[:, :, 0])
    Et = 1.0 / S[0, 0]
    assert abs(Et - mat.E * mat.H / (mat.E + mat.H)) < 1e-9 * Et


def test_uniaxial_stress_strain_closed_form():
    """Under uniaxial stress with linear hardening: sigma = sigma_y + H eps^p_11, eps_p = eps^p_11
    (main-text sqrt(2/3) convention, A-14).  Solve the 1-point stress problem by Newton."""
    mat = Material(model=1, E=70e3, nu=0.3, sigma_y=300.0, H=500.0)
    e11 = 0.02
    eps = np.zeros((6, 1)); eps[0] = e11
    for _ in range(30):
        s, C, pp, pe, _, _ = M.j2_lemaitre(eps, np.zeros((6, 1)), np.zeros(1), np.zeros(1), mat)
        r = s[1:, 0]
        eps[1:, 0] -= np.linalg.solve(C[1:, 1:, 0], r)
    s11 = s[0, 0]
    ep11 = e11 - s11 / mat.E
    assert abs(s11 - (mat.sigma_y + mat.H * ep11)) < 1e-8 * s11
    assert abs(pe[0] - ep11) < 1e-10


def test_damage_law_golden():
    g = GOLD["lemaitre_paper_params"]
    for ebar, D in g["cases"]:
        assert abs(M.lemaitre_damage(ebar, g["eps_c"], g["eps_r"], g["d_max"]) - D) < 1e-15


def test_damage_scales_stress_and_tangent():
    eps, epsp, ep, _ = random_states(50)
    s0, C0, *_ = M.j2_lemaitre(eps, epsp, ep, np.zeros(50), MATRIX_J2)
    s1, C1, *_ = M.j2_lemaitre(eps, epsp, ep, np.full(50, 0.4), MATRIX_J2)
    assert np.allclose(s1, 0.6 * s0, rtol=1e-14, atol=1e-12) and np.allclose(C1, 0.6 * C0, rtol=1e-14)


def test_elastic_closed_forms():
    mat = Material(model=0, E=400e3, nu=0.2)
    K, mu = M.moduli(mat.E, mat.nu)
    c = 1e-3
    eps = np.array([[c / 3], [c / 3], [c / 3], [0], [0], [0]])
    s, C = M.elastic(eps, mat)
    assert np.allclose(s[:, 0], [K * c, K * c, K * c, 0, 0, 0], atol=1e-10)
    # Lame uniaxial strain: s11 = (lam + 2mu) e, s22 = lam e
    lam = K - 2 * mu / 3
    eps = np.zeros((6, 1)); eps[0] = c
    s, _ = M.elastic(eps, mat)
    assert abs(s[0, 0] - (lam + 2 * mu) * c) < 1e-9 and abs(s[1, 0] - lam * c) < 1e-9


def test_brittle_particle():
    mat = PARTICLE_BRITTLE
    eps = np.zeros((6, 1)); eps[0] = 0.004
    s, C, eq = M.brittle(eps, np.array([0.25]), mat)
    Ce = M.elastic_stiffness(mat.E, mat.nu)
    assert np.allclose(s[:, 0], 0.75 * Ce @ eps[:, 0])
    assert abs(eq[0] - np.sqrt(eps[:, 0] @ Ce @ eps[:, 0] / mat.E)) < 1e-16
    # uniaxial stress: eps_eq = sigma/E
    S = np.linalg.inv(Ce)
    sig = np.array([250.0, 0, 0, 0, 0, 0])
    e = (S @ sig).reshape(6, 1)
    assert abs(M.brittle(e, np.zeros(1), mat)[2][0] - 250.0 / mat.E) < 1e-15
    assert M.brittle_damage(0.0045, mat.kappa0, mat.kappa_f, mat.d_max) == pytest.approx(0.5)
