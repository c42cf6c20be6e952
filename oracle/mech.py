"""Mechanical linear problem of the Newton step (paper Sec. 3.2.2).

TEST INFRASTRUCTURE (see oracle/__init__.py).

* tangent contraction tau(x) = C(x) : p(x) -- a 6x6 Mandel matvec per voxel.
* projected tangent apply  y = G*(C : x).
* linear system  G*(dsigma/deps : de) = -G*(sigma - Sigma_bar)  solved by (unpreconditioned)
  conjugate gradients from de = 0: textbook CG, q = A p, alpha = r.r / p.q, stop at
  ||r|| < tol ||b||.  The operator is symmetric on range(G*) for symmetric C.

Pins (tests/test_oracle_mech.py): contraction checked against an explicit loop; dense
pseudo-inverse solve on a 4^3 grid; p.G*(Cp) = p:C:p for p in range(G*).
"""
from __future__ import annotations

import numpy as np

from .projection import apply_projection

PACKED21 = [(i, j) for i in range(6) for j in range(i, 6)]


def unpack21(Cp: np.ndarray) -> np.ndarray:
    """(21, ...) packed upper triangle -> (6, 6, ...) symmetric."""
    C = np.empty((6, 6) + Cp.shape[1:])
    for t, (i, j) in enumerate(PACKED21):
        C[i, j] = Cp[t]
        C[j, i] = Cp[t]
    return C


def pack21(C: np.ndarray) -> np.ndarray:
    return np.stack([C[i, j] for (i, j) in PACKED21])


def contract(C: np.ndarray, p: np.ndarray) -> np.ndarray:
    """tau_i = sum_j C_ij p_j per voxel.  C (6,6,...) , p (6,...)."""
    return np.einsum("ij...,j...->i...", C, p)


def apply_projected_tangent(grid, C, x, stress_mask, backend="scipy"):
    return apply_projection(grid, contract(C, x), stress_mask, backend)


def cg(grid, C, b, stress_mask, tol=1e-10, maxit=2000, backend="scipy"):
    """Textbook CG for G*(C : de) = b, de_0 = 0.  Returns (de, iterations, rel residual)."""
    x = np.zeros_like(b)
    r = b.copy()
    p = r.copy()
    rr = float(np.sum(r * r))
    bnorm = np.sqrt(rr)
    if bnorm == 0.0:
        return x, 0, 0.0
    it = 0
    while it < maxit:
        q = apply_projected_tangent(grid, C, p, stress_mask, backend)
        alpha = rr / float(np.sum(p * q))
        x += alpha * p
        r -= alpha * q
        it += 1
        rr_new = float(np.sum(r * r))
        if np.sqrt(rr_new) < tol * bnorm:
            rr = rr_new
            break
        p = r + (rr_new / rr) * p
        rr = rr_new
    return x, it, np.sqrt(rr) / bnorm
