"""Pins of the GTN oracle (oracle/gtn.py) against the paper's printed values, closed forms,
independent scalar solves and finite differences (no GPU)."""
import math

import numpy as np
import pytest

from oracle import gtn as G

M = G.GTNParams()
K, MU = G.moduli(M.E, M.nu)


def _bisect(fun, lo, hi, n=200):
    flo = fun(lo)
    for _ in range(n):
        mid = 0.5 * (lo + hi)
        fm = fun(mid)
        if (fm > 0) == (flo > 0):
            lo, flo = mid, fm
        else:
            hi = mid
    return 0.5 * (lo + hi)


def test_printed_constants():
    # f_V* = (1.5 + sqrt(2.25 - 2.25)) / 2.25 = 2/3 and the cap 0.9 f_V* = 0.6
    assert G.fv_star(M) == pytest.approx(2.0 / 3.0, abs=1e-15)
    assert 0.9 * G.fv_star(M) == pytest.approx(0.6, abs=1e-15)
    # f* branches
    assert G.effective_porosity(0.10, M) == 0.10
    assert G.effective_porosity(0.20, M) == pytest.approx(0.15 + (2.0 / 3.0 - 0.15) / 0.10 * 0.05, rel=1e-14)
    assert G.effective_porosity(0.30, M) == 0.6          # f_V* = 2/3 capped at 0.6
    # continuity of f* at f_C and f_F
    assert G.effective_porosity(M.f_c, M) == pytest.approx(M.f_c, abs=1e-15)
    # A_N at its peak: f_N / (s_N sqrt(2 pi)) = 0.159577...; symmetric about eps_N
    assert G.nucleation_rate(0.3, M) == pytest.approx(0.04 / (0.1 * math.sqrt(2 * math.pi)), rel=1e-15)
    assert G.nucleation_rate(0.3, M) == pytest.approx(0.1595769, abs=1e-7)
    assert G.nucleation_rate(0.3 + 0.07, M) == pytest.approx(G.nucleation_rate(0.3 - 0.07, M), rel=1e-14)
    assert G.nucleation_rate(5.0, M) < 1e-100


def test_aravas_hardening():
    # eps0p = 0 -> sigma_0 = sigma_Y exactly (x = x^N at x = 1)
    assert G.aravas_x(0.0, M, MU) == 1.0
    prev = 1.0
    for e0 in (1e-4, 1e-3, 0.01, 0.1, 0.5):
        x = G.aravas_x(e0, M, MU)
        # bisection of the law as printed: sigma_0/sigma_Y - (sigma_0/sigma_Y + 3 mu eps0p/sigma_Y)^N = 0
        xb = _bisect(lambda s: s - (s + 3.0 * MU * e0 / M.sigma_y) ** M.n_hard, 1.0, 100.0)
        assert x == pytest.approx(xb, rel=1e-13)
        assert abs(x - (x + 3.0 * MU * e0 / M.sigma_y) ** M.n_hard) < 1e-12
        assert x > prev
        prev = x


def _j2_aravas(eps, epsp_n, e0n):
    """Independent J2 radial return with Aravas hardening: solve q_tr - 3 mu d = sigma_0(e0n + d)
    by bisection on d, sigma_0 from bisection of the implicit law."""
    ee = eps - epsp_n
    tr = ee[:3].sum()
    dev = ee.copy()
    dev[:3] -= tr / 3
    s_tr = 2 * MU * dev
    q_tr = math.sqrt(1.5 * s_tr @ s_tr)

    def s0(e):
        return M.sigma_y * _bisect(lambda s: s - (s + 3.0 * MU * e / M.sigma_y) ** M.n_hard, 1.0, 100.0)

    if q_tr <= s0(e0n):
        return K * tr * np.r_[1, 1, 1, 0, 0, 0] + s_tr, e0n
    d = _bisect(lambda d: q_tr - 3 * MU * d - s0(e0n + d), 0.0, q_tr / (3 * MU))
    s = s_tr * (1.0 - 3 * MU * d / q_tr)
    return K * tr * np.r_[1, 1, 1, 0, 0, 0] + s, e0n + d


def test_zero_porosity_is_j2_with_aravas_hardening():
    rng = np.random.default_rng(11)
    for _ in range(6):
        eps = rng.normal(0, 8e-3, 6)
        epsp_n = rng.normal(0, 1e-3, 6)
        epsp_n[:3] -= epsp_n[:3].mean()          # J2 history is deviatoric
        e0n = abs(rng.normal(0, 0.02))
        r = G.gtn_point(eps, epsp_n, e0n, 0.0, M)
        s_ref, e0_ref = _j2_aravas(eps, epsp_n, e0n)
        assert r["converged"]
        assert np.abs(r["sigma"] - s_ref).max() <= 1e-8 * np.abs(s_ref).max()
        assert r["e0"] == pytest.approx(e0_ref, rel=1e-8, abs=1e-14)
        assert abs(r["epsp"][:3].sum() - epsp_n[:3].sum()) < 1e-15   # no dilatancy at f* = 0


def _phi_sigma(sig, s0, fs):
    """The yield function of P:93 evaluated on a full Mandel stress (no p/q split reused)."""
    p = -(sig[0] + sig[1] + sig[2]) / 3
    s = sig.copy()
    s[:3] += p
    q = math.sqrt(1.5 * s @ s)
    return (q / s0) ** 2 + 2 * fs * M.q1 * math.cosh(-1.5 * M.q2 * p / s0) - (1 + M.q3 * fs * fs)


def _random_states(seed, count):
    rng = np.random.default_rng(seed)
    for i in range(count):
        eps = rng.normal(0, 6e-3, 6)
        eps[:3] += rng.normal(0, 4e-3)
        epsp_n = rng.normal(0, 1e-3, 6)
        e0n = abs(rng.normal(0, 0.02))
        f = [0.0, 0.005, 0.05, 0.12, 0.18, 0.22, 0.3][i % 7]
        yield eps, epsp_n, e0n, f


def test_yield_consistency_normality_and_work_identity():
    nplastic = 0
    for eps, epsp_n, e0n, f in _random_states(5, 40):
        r = G.gtn_point(eps, epsp_n, e0n, f, M)
        fs = G.effective_porosity(f, M)
        if not r["plastic"]:
            assert r["phi"] <= 0.0
            assert np.array_equal(r["epsp"], epsp_n) and r["e0"] == e0n
            continue
        nplastic += 1
        assert r["converged"]
        assert abs(r["phi"]) <= 1e-8                       # |phi| <= 1e-8 (phi is dimensionless)
        s0 = M.sigma_y * G.aravas_x(r["e0"], M, MU)
        sig = r["sigma"]
        assert abs(_phi_sigma(sig, s0, fs)) <= 1e-8
        # normality: d eps^p parallel (positively) to a central-difference gradient of phi(sigma)
        h = 1e-6 * np.abs(sig).max()
        g = np.array([(_phi_sigma(sig + h * e, s0, fs) - _phi_sigma(sig - h * e, s0, fs)) / (2 * h)
                      for e in np.eye(6)])
        dep = r["epsp"] - epsp_n
        lam = dep @ g / (g @ g)
        assert lam > 0
        assert np.linalg.norm(dep - lam * g) <= 1e-6 * np.linalg.norm(dep)
        # plastic work: sigma : d eps^p = (1 - f) sigma_0 d eps0p
        assert sig @ dep == pytest.approx((1 - f) * s0 * (r["e0"] - e0n), rel=1e-9)
    assert nplastic >= 20


def test_elastic_law_at_plastic_returns():
    """sigma = C^e : (eps - eps^p) at every plastic return with f* > 0 (App. A: the
    stress is the elastic law at the returned plastic strain).  Unlike the yield, normality and
    work pins, this fixes the coefficient of the volumetric return (p = p_tr + K a): a slip such as
    3K a or K a / 3 leaves sigma off the elastic law.  C^e from the textbook isotropic moduli."""
    E, nu = M.E, M.nu
    Kt, mut = E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))
    one = np.r_[1.0, 1, 1, 0, 0, 0]
    Ce = Kt * np.outer(one, one) + 2.0 * mut * (np.eye(6) - np.outer(one, one) / 3.0)
    nchk = 0
    for eps, epsp_n, e0n, f in _random_states(21, 60):
        r = G.gtn_point(eps, epsp_n, e0n, f, M)
        if not r["plastic"] or G.effective_porosity(f, M) == 0.0:
            continue
        assert r["converged"]
        s_el = Ce @ (eps - r["epsp"])
        assert np.linalg.norm(r["sigma"] - s_el) <= 1e-12 * np.linalg.norm(s_el)
        # and the return is genuinely dilatant (the volumetric term is exercised)
        assert abs((r["epsp"] - epsp_n)[:3].sum()) > 0.0
        nchk += 1
    assert nchk >= 20


def test_consistent_tangent_central_differences():
    for eps, epsp_n, e0n, f in list(_random_states(9, 14)):
        r = G.gtn_point(eps, epsp_n, e0n, f, M)
        if not r["plastic"]:
            continue
        h = 1e-7
        Cfd = np.zeros((6, 6))
        for j in range(6):
            d = np.zeros(6)
            d[j] = h
            Cfd[:, j] = (G.gtn_point(eps + d, epsp_n, e0n, f, M)["sigma"]
                         - G.gtn_point(eps - d, epsp_n, e0n, f, M)["sigma"]) / (2 * h)
        assert np.abs(r["C"] - Cfd).max() <= 1e-6 * np.abs(Cfd).max()
        # the Newton tangent is the symmetric part (A-32) unless the coupling was dropped (A-33)
        S = 0.5 * (r["C"] + r["C"].T)
        assert np.abs(r["C_sym"] - S).max() <= 1e-9 * np.abs(S).max()


def test_elastic_tangent_and_state():
    eps = np.array([1e-4, -2e-4, 5e-5, 1e-4, 0, 0])
    r = G.gtn_point(eps, np.zeros(6), 0.0, 0.01, M)
    assert not r["plastic"]
    one = np.r_[1, 1, 1, 0, 0, 0]
    Ce = K * np.outer(one, one) + 2 * MU * (np.eye(6) - np.outer(one, one) / 3)
    assert np.allclose(r["C_sym"], Ce, rtol=0, atol=1e-9 * Ce.max())
    assert np.allclose(r["sigma"], Ce @ eps, rtol=1e-14, atol=0)


def test_hydrostatic_tension_dilates():
    # p < 0 with f* > 0 -> dphi/dp < 0 -> tr d eps^p > 0, and no deviatoric flow
    e = 0.01
    eps = np.array([e, e, e, 0, 0, 0])
    r = G.gtn_point(eps, np.zeros(6), 0.0, 0.05, M)
    assert r["plastic"] and r["converged"]
    dep = r["epsp"]
    assert dep[:3].sum() > 0
    assert np.abs(dep - dep[:3].mean() * np.r_[1, 1, 1, 0, 0, 0]).max() < 1e-15
    assert abs(r["phi"]) < 1e-10


def test_porosity_update_against_growth_and_nucleation_odes():
    m0 = G.GTNParams(f_n=0.0)
    # growth only: df = (1 - f) d tr  ->  1 - f = (1 - f0) exp(-tr)
    f, f0, steps, T = 0.01, 0.01, 20000, 0.5
    for k in range(steps):
        f = G.porosity(f, 0.0, 0.0, T * (k + 1) / steps, T * k / steps, m0)
    assert 1 - f == pytest.approx((1 - f0) * math.exp(-T), rel=1e-4)
    # nucleation only: df = A_N(e) de  ->  f - f0 = f_N [Phi((e - eps_N)/s_N) - Phi(-eps_N/s_N)]
    f, E = 0.0, 0.6
    for k in range(steps):
        f = G.porosity(f, E * (k + 1) / steps, E * k / steps, 0.0, 0.0, M)

    def Phi(z):
        return 0.5 * (1 + math.erf(z / math.sqrt(2)))
    assert f == pytest.approx(M.f_n * (Phi((E - M.eps_n) / M.s_n) - Phi(-M.eps_n / M.s_n)), rel=1e-4)


def test_porosity_is_irreversible():
    # A-30 (as D in A-16): void closure (d trbar < 0) never lowers the committed porosity
    m = G.GTNParams()
    assert G.porosity(0.05, 0.01, 0.01, -0.01, 0.0, m) == 0.05
    assert G.porosity(0.05, 0.01, 0.01, 0.01, 0.0, m) > 0.05
    assert G.porosity(0.999, m.eps_n, m.eps_n - 1.0, 0.0, 0.0, m) == 1.0   # 0.999 + A_N(peak) * 1 > 1
