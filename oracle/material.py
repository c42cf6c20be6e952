"""Constitutive point models (paper Sec. 2.1.2; App. A).

TEST INFRASTRUCTURE (see oracle/__init__.py).

All tensors in Mandel form (11, 22, 33, sqrt2*23, sqrt2*13, sqrt2*12), vectorised over voxels
(arrays (6, n)); moduli in MPa.

J2-Lemaitre with linear hardening sigma_0 = sigma_y + H eps_p (BJ:7):
  effective stress sigma~ = K tr(eps - eps^p) I + 2 mu dev(eps - eps^p)
  yield   phi = ||s~|| - sqrt(2/3) sigma_0(eps_p)                            (A-14)
  flow    d eps^p = dlam s~/||s~||,  d eps_p = sqrt(2/3) dlam                 (A-14)
  backward Euler (App. A) with linear hardening is a closed-form radial return:
     s_tr = 2 mu (dev eps - eps^p_n), q = ||s_tr||, f = q - sqrt(2/3)(sigma_y + H eps_p,n)
     f > 0:  dlam = f / (2 mu + 2H/3), n = s_tr / q
  nominal stress sigma = (1 - D) sigma~  (total form A-15), D frozen (staggered)
  consistent tangent (Simo-Hughes radial return):
     C = (1-D)[K 1(x)1 + 2 mu theta I_dev - 2 mu thetabar n(x)n],
     theta = 1 - 2 mu dlam / q,  thetabar = 1/(1 + H/(3 mu)) - (1 - theta)
Damage law with the numerical cap D <= 0.99.
Elastic phase: sigma = C_e eps.
Elastic-brittle particle (A-18, not in the paper): eps_eq = sqrt(eps:C_p:eps / E_p),
  kappa = max(kappa_n, abar_p), d = clamp((kappa - kappa0)/(kappa_f - kappa0), 0, d_max),
  sigma = (1 - d) C_p eps.

Pins (tests/test_oracle_material.py): central finite-difference tangent; symmetric tangent;
yield consistency |phi| <= 1e-8 sigma_y; plastic incompressibility; uniaxial-stress tangent
E H/(E+H) and uniaxial stress-strain closed form; damage-law values; elastic closed forms.
"""
from __future__ import annotations

import numpy as np

SQ23 = np.sqrt(2.0 / 3.0)
ONE = np.array([1.0, 1.0, 1.0, 0.0, 0.0, 0.0])
IDEV = np.eye(6) - np.outer(ONE, ONE) / 3.0


def moduli(E: float, nu: float):
    K = E / (3.0 * (1.0 - 2.0 * nu))
    mu = E / (2.0 * (1.0 + nu))
    return K, mu


def elastic_stiffness(E: float, nu: float) -> np.ndarray:
    """Isotropic C_e in Mandel form: K 1(x)1 + 2 mu I_dev."""
    K, mu = moduli(E, nu)
    return K * np.outer(ONE, ONE) + 2.0 * mu * IDEV


def dev(v: np.ndarray) -> np.ndarray:
    tr = v[0] + v[1] + v[2]
    return v - np.multiply.outer(ONE, tr / 3.0)


def lemaitre_damage(ebar, eps_c: float, eps_r: float, d_max: float = 0.99):
    """D(ebar) piecewise linear, capped at d_max."""
    D = np.clip((np.asarray(ebar, dtype=float) - eps_c) / (eps_r - eps_c), 0.0, 1.0)
    return np.minimum(D, d_max)


def brittle_damage(kappa, kappa0: float, kappa_f: float, d_max: float = 0.99):
    d = np.clip((np.asarray(kappa, dtype=float) - kappa0) / (kappa_f - kappa0), 0.0, 1.0)
    return np.minimum(d, d_max)


def j2_lemaitre(eps, epsp_n, ep_n, D, mat):
    """Backward-Euler J2 radial return on the effective stress + frozen damage D.
    eps, epsp_n: (6, n); ep_n, D: (n,).  Returns sigma (6,n), C (6,6,n), epsp (6,n), ep (n,),
    plastic mask (n,), phi (n,) = yield function at the returned state."""
    K, mu = moduli(mat.E, mat.nu)
    H = mat.H
    tr = eps[0] + eps[1] + eps[2]
    de = dev(eps)
    s_tr = 2.0 * mu * (de - epsp_n)
    q = np.sqrt(np.sum(s_tr * s_tr, axis=0))
    f = q - SQ23 * (mat.sigma_y + H * ep_n)
    plastic = f > 0.0
    dlam = np.where(plastic, f / (2.0 * mu + 2.0 * H / 3.0), 0.0)
    qs = np.where(plastic, q, 1.0)
    n_hat = s_tr / qs
    epsp = epsp_n + dlam * n_hat
    ep = ep_n + SQ23 * dlam
    sig_eff = np.multiply.outer(ONE, K * tr) + 2.0 * mu * (de - epsp)
    sigma = (1.0 - D) * sig_eff
    theta = np.where(plastic, 1.0 - 2.0 * mu * dlam / qs, 1.0)
    thetabar = np.where(plastic, 1.0 / (1.0 + H / (3.0 * mu)) - (1.0 - theta), 0.0)
    C = (K * np.outer(ONE, ONE)[..., None]
         + 2.0 * mu * theta * IDEV[..., None]
         - 2.0 * mu * thetabar * np.einsum("in,jn->ijn", n_hat, n_hat))
    C = C * (1.0 - D)
    s_eff = dev(sig_eff)
    phi = np.sqrt(np.sum(s_eff * s_eff, axis=0)) - SQ23 * (mat.sigma_y + H * ep)
    return sigma, C, epsp, ep, plastic, phi


def elastic(eps, mat):
    Ce = elastic_stiffness(mat.E, mat.nu)
    sigma = Ce @ eps
    C = np.broadcast_to(Ce[..., None], (6, 6, eps.shape[1])).copy()
    return sigma, C


def brittle(eps, d, mat):
    """Elastic-brittle particle (A-18): sigma = (1-d) C_p eps; returns sigma, C, eps_eq."""
    Ce = elastic_stiffness(mat.E, mat.nu)
    ce = Ce @ eps
    eps_eq = np.sqrt(np.maximum(np.sum(eps * ce, axis=0), 0.0) / mat.E)
    sigma = (1.0 - d) * ce
    C = (1.0 - d) * Ce[..., None] * np.ones(eps.shape[1])
    return sigma, C, eps_eq
