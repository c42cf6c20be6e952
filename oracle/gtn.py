"""Non-local Gurson-Tvergaard-Needleman (GTN) point model: paper Sec. 2.1.1, its
non-local extension Sec. 2.2.2 and the backward-Euler time discretisation of
App. A; parameters of Sec. 4.1 and the damage cap.

TEST INFRASTRUCTURE (see oracle/__init__.py).  Plain per-voxel Python floats; slow on
purpose.  Tensors are Mandel 6-vectors (11, 22, 33, sqrt2*23, sqrt2*13, sqrt2*12), so ':' is
a dot product.  The paper writes s for the Mises stress; it is q here (s is the deviator).

  yield      phi = (q/sigma_0)^2 + 2 f* q1 cosh(-3 q2 p / (2 sigma_0)) - (1 + q3 f*^2)
             q = sqrt(3/2 s:s), p = -tr(sigma)/3
  f_V*       = (q1 + sqrt(q1^2 - q3)) / q3
  elastic    sigma = K tr(eps - eps^p) I + 2 mu dev(eps - eps^p)   (the rate law
             integrated with constant moduli, App. A)
  flow       d eps^p = dlam [dphi/dp dp/dsigma + dphi/dq dq/dsigma]
  work       sigma : d eps^p = (1 - f) sigma_0 d eps0p
  f*(f)      piecewise linear, capped at fstar_max = 0.9 f_V*
  A_N        = f_N / (s_N sqrt(2 pi)) exp(-((ebar0 - eps_N)/s_N)^2 / 2)
  porosity   f_{n+1} = f_n + A_N(ebar0_{n+1}) d ebar0 + (1 - f_{n+1}) d trbar          (P:455-458,
             App. A), with the non-local fields frozen at the staggered iterate
             (P:600-601), so it is explicit:  f = (f_n + A_N d ebar0 + d trbar) / (1 + d trbar),
             kept irreversible, f_{n+1} = max(f_n, f) (A-30, as D in A-16)
  hardening  sigma_0/sigma_Y = (sigma_0/sigma_Y + 3 mu eps0p/sigma_Y)^N  (Aravas);
             with x = sigma_0/sigma_Y this is eps0p(x) = sigma_Y (x^(1/N) - x) / (3 mu)
  sources    alpha_0 = eps0p, alpha_1 = tr eps^p

Return mapping (App. A, readings A-30..A-33 of DESIGN.md).  With the trial state
p_tr = -K tr(eps - eps^p_n), s_tr = 2 mu (dev eps - eps^p_n), q_tr = sqrt(3/2) |s_tr|,
n = (3/2) s_tr / q_tr, the flow rule splits as d eps^p = (a/3) I + b n with
a = -dlam dphi/dp, b = dlam dphi/dq; then p = p_tr + K a, q = q_tr - 3 mu b, sigma = -p I +
(2/3) q n.  Eliminating dlam (a dphi/dq + b dphi/dp = 0) leaves three equations in
u = (a, b, x):
  R1 = a Q + b (3/2) f* q1 q2 sinh(xi)            [= (sigma_0/2)(a phi_q + b phi_p)]
  R2 = Q^2 + 2 f* q1 cosh(xi) - 1 - q3 f*^2       [= phi]
  R3 = (1 - f)(eps0p(x) - eps0p_n) + P a - Q b   [work identity / sigma_0]
with P = p/sigma_0, Q = q/sigma_0, xi = (3/2) q2 P, sigma_0 = sigma_Y x.  Newton from
(0, 0, x_n) with step halving on R1^2 + R2^2 + R3^2 (and x >= 1), until the Newton step is at
round-off (|da| + |db| <= 1e-13 (|a| + |b|) + 1e-14 sigma_Y/(3 mu), |dx| <= 1e-13 x); elastic if phi(p_tr, q_tr, sigma_0(eps0p_n)) <= 0.

Consistent tangent: linearise R(u; p_tr, q_tr) = 0 -> du = M (dp_tr, dq_tr), M = -J^-1 dR/d(p_tr, q_tr),
dp_tr = -K 1:de, dq_tr = 2 mu n:de, dn = (3 mu/q_tr)(I_dev - (2/3) n(x)n) de, so
  C = 2 mu theta I_dev + K a_pp 1(x)1 - 2 mu a_pq 1(x)n - (2/3) K a_qp n(x)1 + (4/3) mu (a_qq - theta) n(x)n
with theta = q/q_tr, a_pp = dp/dp_tr, a_pq = dp/dq_tr, a_qp = dq/dp_tr, a_qq = dq/dq_tr.  CG needs a
symmetric operator: the Newton tangent is sym(C) (A-32), i.e.
  C_sym = ca 1(x)1 + cb I - cc n(x)n + cd (1(x)n + n(x)1),
  cb = 2 mu theta, ca = K a_pp - cb/3, cc = (4/3) mu (theta - a_qq), cd = -mu a_pq - (1/3) K a_qp,
with cd dropped where |cc| < 1e-6 cb (A-33).  f is frozen, so C carries no df/d eps term.

Pins (tests/test_oracle_gtn.py): f_V* = 2/3 and the cap 0.6; the f* branches; A_N at its
peak and its symmetry; Aravas sigma_0(0) = sigma_Y and bisection of the implicit law; f* = 0
equals an independent J2 radial return with Aravas hardening (scalar bisection); |phi| <= 1e-8
at every plastic return; normality against a finite-difference gradient of phi(sigma) taken on
the full Mandel stress (no p/q split); the plastic-work identity; central-difference tangent;
hydrostatic tension -> purely volumetric dilatant flow; the porosity update against the growth
ODE df = (1 - f) d tr (closed form 1 - f = (1 - f0) exp(-tr)).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

ONE = np.array([1.0, 1.0, 1.0, 0.0, 0.0, 0.0])


@dataclass
class GTNParams:
    """GTN material (paper Sec. 4.1 values as defaults)."""
    E: float = 300.0e3          # MPa
    nu: float = 0.3
    sigma_y: float = 1000.0     # MPa
    q1: float = 1.5
    q2: float = 1.0
    q3: float = 2.25
    f_c: float = 0.15
    f_f: float = 0.25
    f_n: float = 0.04
    eps_n: float = 0.3
    s_n: float = 0.1
    n_hard: float = 0.1         # Aravas exponent N
    fstar_max: float = 0.6      # 0.9 f_V*


def moduli(E, nu):
    return E / (3.0 * (1.0 - 2.0 * nu)), E / (2.0 * (1.0 + nu))


def fv_star(m: GTNParams) -> float:
    """f_V* = (q1 + sqrt(q1^2 - q3)) / q3."""
    return (m.q1 + math.sqrt(m.q1 * m.q1 - m.q3)) / m.q3


def effective_porosity(f: float, m: GTNParams) -> float:
    """f*(f) capped at fstar_max."""
    fv = fv_star(m)
    if f < m.f_c:
        fs = f
    elif f < m.f_f:
        fs = m.f_c + (fv - m.f_c) / (m.f_f - m.f_c) * (f - m.f_c)
    else:
        fs = fv
    return min(fs, m.fstar_max)


def nucleation_rate(ebar0: float, m: GTNParams) -> float:
    """Chu-Needleman A_N."""
    return m.f_n / (m.s_n * math.sqrt(2.0 * math.pi)) * math.exp(-0.5 * ((ebar0 - m.eps_n) / m.s_n) ** 2)


def eps0p_of_x(x: float, m: GTNParams, mu: float) -> float:
    """Aravas law solved for eps0p at sigma_0 = sigma_Y x."""
    return m.sigma_y * (x ** (1.0 / m.n_hard) - x) / (3.0 * mu)


def aravas_x(e0: float, m: GTNParams, mu: float) -> float:
    """x = sigma_0/sigma_Y solving x = (x + 3 mu e0/sigma_Y)^N, i.e. x^(1/N) - x = 3 mu e0/sigma_Y,
    by Newton from x = 1 (the function is convex and increasing for x >= 1)."""
    c = 3.0 * mu * e0 / m.sigma_y
    if c <= 0.0:
        return 1.0
    iN = 1.0 / m.n_hard
    x = 1.0
    for _ in range(100):
        g = x ** iN - x - c
        dx = g / (iN * x ** (iN - 1.0) - 1.0)
        x -= dx
        if abs(dx) <= 1e-15 * x:
            break
    return x


def porosity(f_n: float, ebar0: float, ebar0_n: float, trbar: float, trbar_n: float, m: GTNParams) -> float:
    """f_{n+1} from the frozen non-local increments (App. A), irreversible
    (A-30: f_{n+1} >= f_n, as damage in A-16) and at most 1."""
    d0 = ebar0 - ebar0_n
    dt = trbar - trbar_n
    f = (f_n + nucleation_rate(ebar0, m) * d0 + dt) / (1.0 + dt)
    return min(max(f, f_n), 1.0)


def _yield(P, Q, fs, m):
    return Q * Q + 2.0 * fs * m.q1 * math.cosh(1.5 * m.q2 * P) - 1.0 - m.q3 * fs * fs


def _residual(u, ptr, qtr, e0n, f, fs, m, K, mu):
    a, b, x = u
    s0 = m.sigma_y * x
    P = (ptr + K * a) / s0
    Q = (qtr - 3.0 * mu * b) / s0
    xi = 1.5 * m.q2 * P
    c = 1.5 * fs * m.q1 * m.q2
    R1 = a * Q + b * c * math.sinh(xi)
    R2 = Q * Q + 2.0 * fs * m.q1 * math.cosh(xi) - 1.0 - m.q3 * fs * fs
    R3 = (1.0 - f) * (eps0p_of_x(x, m, mu) - e0n) + P * a - Q * b
    return np.array([R1, R2, R3])


def _jacobians(u, ptr, qtr, f, fs, m, K, mu):
    """J = dR/du (3x3) and B = dR/d(p_tr, q_tr) (3x2)."""
    a, b, x = u
    s0 = m.sigma_y * x
    P = (ptr + K * a) / s0
    Q = (qtr - 3.0 * mu * b) / s0
    xi = 1.5 * m.q2 * P
    c = 1.5 * fs * m.q1 * m.q2
    ch, sh = math.cosh(xi), math.sinh(xi)
    k = 1.5 * m.q2                      # dxi/dP
    dP_da, dP_dx = K / s0, -P / x
    dQ_db, dQ_dx = -3.0 * mu / s0, -Q / x
    iN = 1.0 / m.n_hard
    de_dx = m.sigma_y * (iN * x ** (iN - 1.0) - 1.0) / (3.0 * mu)
    J = np.array([
        [Q + b * c * ch * k * dP_da, a * dQ_db + c * sh, a * dQ_dx + b * c * ch * k * dP_dx],
        [2.0 * fs * m.q1 * sh * k * dP_da, 2.0 * Q * dQ_db, 2.0 * Q * dQ_dx + 2.0 * fs * m.q1 * sh * k * dP_dx],
        [P + a * dP_da, -Q - b * dQ_db, (1.0 - f) * de_dx + a * dP_dx - b * dQ_dx],
    ])
    B = np.array([
        [b * c * ch * k / s0, a / s0],
        [2.0 * fs * m.q1 * sh * k / s0, 2.0 * Q / s0],
        [a / s0, -b / s0],
    ])
    return J, B


def return_map(ptr, qtr, e0n, f, fs, m, K, mu, max_it=50):
    """Newton on (a, b, x) from (0, 0, x_n) with step halving; returns (u, iterations, converged)."""
    u = np.array([0.0, 0.0, aravas_x(e0n, m, mu)])
    R = _residual(u, ptr, qtr, e0n, f, fs, m, K, mu)
    for it in range(1, max_it + 1):
        J, _ = _jacobians(u, ptr, qtr, f, fs, m, K, mu)
        du = -np.linalg.solve(J, R)
        # Newton step at round-off: done.  The absolute floor (strain units) is ~50x the rounding
        # of eps0p(x) = sigma_Y (x^(1/N) - x)/(3 mu) near x = 1, which bounds how well a, b resolve.
        if (abs(du[0]) + abs(du[1]) <= 1e-13 * (abs(u[0]) + abs(u[1])) + 1e-14 * m.sigma_y / (3.0 * mu)
                and abs(du[2]) <= 1e-13 * u[2]):
            return u + du, it, True
        psi = float(R @ R)
        t = 1.0
        for _ in range(30):                   # halve until R^2 decreases (x projected onto x >= 1)
            un = u + t * du
            un[2] = max(un[2], 1.0)
            Rn = _residual(un, ptr, qtr, e0n, f, fs, m, K, mu)
            if float(Rn @ Rn) < psi:
                break
            t *= 0.5
        u, R = un, Rn
    return u, max_it, False


def gtn_point(eps, epsp_n, e0n, f, m: GTNParams):
    """Backward-Euler GTN update at total strain eps (Mandel 6) with frozen porosity f.
    Returns dict: sigma, C (non-symmetric consistent tangent), C_sym (the Newton tangent of A-32/A-33),
    epsp, e0 (eps0p), plastic, phi (yield function at the returned state), converged, iters."""
    eps = np.asarray(eps, dtype=float)
    epsp_n = np.asarray(epsp_n, dtype=float)
    K, mu = moduli(m.E, m.nu)
    fs = effective_porosity(f, m)
    ee = eps - epsp_n
    tr = ee[0] + ee[1] + ee[2]
    s_tr = 2.0 * mu * (ee - ONE * tr / 3.0)
    ptr = -K * tr
    qtr = math.sqrt(1.5 * float(s_tr @ s_tr))
    x_n = aravas_x(e0n, m, mu)
    phi_tr = _yield(ptr / (m.sigma_y * x_n), qtr / (m.sigma_y * x_n), fs, m)
    Ce = K * np.outer(ONE, ONE) + 2.0 * mu * (np.eye(6) - np.outer(ONE, ONE) / 3.0)
    if phi_tr <= 0.0:
        sig = Ce @ ee
        return dict(sigma=sig, C=Ce.copy(), C_sym=Ce.copy(), epsp=epsp_n.copy(), e0=e0n, plastic=False,
                    phi=phi_tr, converged=True, iters=0)
    tiny = qtr <= 1e-12 * m.sigma_y
    n = np.zeros(6) if tiny else 1.5 * s_tr / qtr
    u, iters, ok = return_map(ptr, qtr, e0n, f, fs, m, K, mu)
    a, b, x = u
    p = ptr + K * a
    q = qtr - 3.0 * mu * b
    sig = -p * ONE + (2.0 / 3.0) * q * n
    epsp = epsp_n + (a / 3.0) * ONE + b * n
    e0 = eps0p_of_x(x, m, mu)
    phi = _yield(p / (m.sigma_y * x), q / (m.sigma_y * x), fs, m)
    J, B = _jacobians(u, ptr, qtr, f, fs, m, K, mu)
    M = -np.linalg.solve(J, B)
    a_pp, a_pq = 1.0 + K * M[0, 0], K * M[0, 1]
    a_qp, a_qq = -3.0 * mu * M[1, 0], 1.0 - 3.0 * mu * M[1, 1]
    theta = 1.0 if tiny else q / qtr
    Idev = np.eye(6) - np.outer(ONE, ONE) / 3.0
    C = (2.0 * mu * theta * Idev + K * a_pp * np.outer(ONE, ONE) - 2.0 * mu * a_pq * np.outer(ONE, n)
         - (2.0 / 3.0) * K * a_qp * np.outer(n, ONE) + (4.0 / 3.0) * mu * (a_qq - theta) * np.outer(n, n))
    cb = 2.0 * mu * theta
    ca = K * a_pp - cb / 3.0
    cc = (4.0 / 3.0) * mu * (theta - a_qq)
    cd = -mu * a_pq - K * a_qp / 3.0
    if abs(cc) < 1e-6 * cb:
        cd = 0.0
    C_sym = ca * np.outer(ONE, ONE) + cb * np.eye(6) - cc * np.outer(n, n) + cd * (np.outer(ONE, n) + np.outer(n, ONE))
    return dict(sigma=sig, C=C, C_sym=C_sym, epsp=epsp, e0=e0, plastic=True, phi=phi, converged=ok, iters=iters)


def gtn(eps, epsp_n, e0n, f, m: GTNParams):
    """Vectorised over voxels by a plain loop: eps, epsp_n (6, n); e0n, f (n,).
    Returns sigma (6,n), C_sym (6,6,n), epsp (6,n), e0 (n,), converged (n,) bool."""
    nv = eps.shape[1]
    sig = np.zeros((6, nv))
    C = np.zeros((6, 6, nv))
    epsp = np.zeros((6, nv))
    e0 = np.zeros(nv)
    ok = np.ones(nv, dtype=bool)
    for v in range(nv):
        r = gtn_point(eps[:, v], epsp_n[:, v], float(e0n[v]), float(f[v]), m)
        sig[:, v], C[:, :, v], epsp[:, v], e0[v], ok[v] = r["sigma"], r["C_sym"], r["epsp"], r["e0"], r["converged"]
    return sig, C, epsp, e0, ok
