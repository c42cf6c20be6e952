"""Heterogeneous Helmholtz operator, preconditioner and Algorithm 2 (paper Sec. 3.2.3,
P:687-794).

TEST INFRASTRUCTURE (see oracle/__init__.py).

* L(a) = a - div(l^2(x) grad a).  In Fourier space (with the i's
  kept, A-09):   L^(a^) = a^ + sum_j conj(k_j) F( l^2(x) F^{-1}(k_j a^) ).
* M(r^) = r^ / (1 + <l^2> |k|^2)  (<l^2> = voxel mean of l^2(x), A-11;
  |k|^2 = sum_j |k_j|^2 so that M = L^{-1} exactly for uniform l).
* Algorithm 2: a^ = F(alpha); x^ = ConjGrad(GC, M, a^, TOL); abar = F^{-1}(x^),
  ConjGrad = preconditioned CG on the half spectrum with the real inner product
  <u, v> = Re sum_half w u conj(v) (A-10), stop at ||A x - b|| < TOL ||b|| (recursive residual).

Pins (tests/test_oracle_helmholtz.py): dense real-space assembly I + sum_j D_j^T diag(l^2) D_j
from the Willot stencil; uniform l: symbol 1 + l^2|k|^2 and M = L^-1 (one PCG iteration);
constant input unchanged; self-adjoint, <Lu,u> >= ||u||^2; closed-form single-mode
response a/(1 + l^2 |k(xi)|^2); dense direct solve; mean preservation.
"""
from __future__ import annotations

import numpy as np

from .spectral import Grid, rfftn, irfftn


def ell2_field(phases: np.ndarray, ell_row) -> np.ndarray:
    """l^2(x) from the per-phase lengths of one field (Remark P:394-405)."""
    ell = np.asarray(ell_row, dtype=float)
    return (ell ** 2)[phases]


def apply_Lhat(grid: Grid, a_hat: np.ndarray, ell2: np.ndarray, backend="scipy") -> np.ndarray:
    """GC of Algorithm 2: grad = F^-1(k a^); h = l^2 grad; return a^ + conj(k).F(h)."""
    k = grid.symbol(half=True)
    out = a_hat.copy()
    for j in range(3):
        g = irfftn(k[j] * a_hat, grid.shape, backend)
        out = out + np.conj(k[j]) * rfftn(ell2 * g, backend)
    return out


def apply_M(grid: Grid, r_hat: np.ndarray, mean_ell2: float) -> np.ndarray:
    """M of Algorithm 2."""
    k = grid.symbol(half=True)
    k2 = np.sum(np.abs(k) ** 2, axis=0)
    return r_hat / (1.0 + mean_ell2 * k2)


def apply_helmholtz(grid: Grid, a: np.ndarray, ell2: np.ndarray, backend="scipy") -> np.ndarray:
    """Real-space y = L(a) = F^-1 L^ F a."""
    return irfftn(apply_Lhat(grid, rfftn(a, backend), ell2, backend), grid.shape, backend)


def apply_precond(grid: Grid, r: np.ndarray, ell2: np.ndarray, backend="scipy") -> np.ndarray:
    """Real-space z = F^-1 M F r."""
    return irfftn(apply_M(grid, rfftn(r, backend), float(np.mean(ell2))), grid.shape, backend)


def _dot(grid: Grid, u: np.ndarray, v: np.ndarray) -> float:
    return float(np.sum(grid.hermitian_weights() * np.real(u * np.conj(v))))


def solve_helmholtz(grid: Grid, alpha: np.ndarray, ell2: np.ndarray, tol: float = 1e-10,
                    maxit: int = 1000, x0: np.ndarray | None = None, backend="scipy"):
    """Algorithm 2.  Returns (abar real field, iterations, relative residual history)."""
    b = rfftn(alpha, backend)
    mean_ell2 = float(np.mean(ell2))
    x = np.zeros_like(b) if x0 is None else rfftn(x0, backend)
    r = b - apply_Lhat(grid, x, ell2, backend) if x0 is not None else b.copy()
    bnorm = np.sqrt(_dot(grid, b, b))
    hist = []
    if bnorm == 0.0:
        return np.zeros(grid.shape), 0, hist
    z = apply_M(grid, r, mean_ell2)
    p = z.copy()
    rz = _dot(grid, r, z)
    it = 0
    rel = np.sqrt(_dot(grid, r, r)) / bnorm
    hist.append(rel)
    while rel >= tol and it < maxit:
        q = apply_Lhat(grid, p, ell2, backend)
        alpha_k = rz / _dot(grid, p, q)
        x = x + alpha_k * p
        r = r - alpha_k * q
        it += 1
        rel = np.sqrt(_dot(grid, r, r)) / bnorm
        hist.append(rel)
        if rel < tol:
            break
        z = apply_M(grid, r, mean_ell2)
        rz_new = _dot(grid, r, z)
        p = z + (rz_new / rz) * p
        rz = rz_new
    return irfftn(x, grid.shape, backend), it, hist
