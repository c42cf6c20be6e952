"""Galerkin projection G* with mixed macroscopic control (paper Sec. 3.2.2).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Definition (the plain one, written out; readings A-07, A-08):
  G*(tau) = F^{-1}{ G^*(xi) : F(tau) }
  * xi != 0 and k(xi) != 0: G^*(xi) is the orthogonal projector (Frobenius / Mandel inner
    product, Hermitian) of a complex symmetric 3x3 tensor onto the compatible set
    {sym(u (x) k) : u in C^3} -- the Fourier image of {sym(grad u)}.
    Solving the normal equations tau conj(k) = sym(u (x) k) conj(k):
        t = tau conj(k),  s = conj(k).t,  u = (2/|k|^2)(t - k s / (2|k|^2)),  P = sym(u (x) k).
  * xi = 0: Mandel mask, 1 on stress-controlled components, 0 on strain-controlled (A-07).
  * xi != 0 with k(xi) = 0 (Willot null modes): 0 (A-08).
Mandel vectors (11, 22, 33, sqrt2*23, sqrt2*13, sqrt2*12): Frobenius product = dot product.

Pins (tests/test_oracle_projection.py): equals the dense orthogonal projector B B^+ of the
real-space symmetric-gradient operator (plus the zero-frequency mask) on small grids;
idempotent; self-adjoint; compatible fields reproduced; equilibrated fields annihilated;
continuous-scheme closed form = Moulinec-Suquet Gamma0 with lambda0=0, 2mu0=1.
"""
from __future__ import annotations

import numpy as np

from .spectral import Grid, rfftn, irfftn

S2 = np.sqrt(2.0)


def mandel_to_tensor(v: np.ndarray) -> np.ndarray:
    """(6, ...) Mandel -> (3, 3, ...) symmetric tensor."""
    T = np.empty((3, 3) + v.shape[1:], dtype=v.dtype)
    T[0, 0], T[1, 1], T[2, 2] = v[0], v[1], v[2]
    T[1, 2] = T[2, 1] = v[3] / S2
    T[0, 2] = T[2, 0] = v[4] / S2
    T[0, 1] = T[1, 0] = v[5] / S2
    return T


def tensor_to_mandel(T: np.ndarray) -> np.ndarray:
    return np.stack([T[0, 0], T[1, 1], T[2, 2], S2 * T[1, 2], S2 * T[0, 2], S2 * T[0, 1]])


def project_spectrum(tau_hat: np.ndarray, k: np.ndarray, stress_mask, dc_index=(0, 0, 0),
                     dc_shift=None) -> np.ndarray:
    """Apply G^*(xi) per frequency.  tau_hat: (6, ...) complex, k: (3, ...) complex.
    dc_shift (6,) is subtracted from tau_hat at xi = 0 before the mask (used for
    -G*(sigma - Sigma_bar): F(sigma - Sigma)(0) = F(sigma)(0) - N Sigma)."""
    T = mandel_to_tensor(tau_hat)
    kc = np.conj(k)
    k2 = np.sum(np.abs(k) ** 2, axis=0)
    t = np.einsum("ij...,j...->i...", T, kc)
    s = np.einsum("i...,i...->...", kc, t)
    nz = k2 > 0.0
    inv = np.where(nz, 1.0 / np.where(nz, k2, 1.0), 0.0)
    u = 2.0 * inv * (t - k * s * 0.5 * inv)
    P = 0.5 * (np.einsum("i...,j...->ij...", u, k) + np.einsum("i...,j...->ij...", k, u))
    out = tensor_to_mandel(P)
    out = np.where(nz[None], out, 0.0)
    mask = np.asarray(stress_mask, dtype=float)
    dc = tau_hat[(slice(None),) + tuple(dc_index)].copy()
    if dc_shift is not None:
        dc = dc - np.asarray(dc_shift)
    out[(slice(None),) + tuple(dc_index)] = mask * dc
    return out


def apply_projection(grid: Grid, tau: np.ndarray, stress_mask, backend="scipy", dc_mean_shift=None):
    """y = G*(tau) for a real Mandel field tau (6, Nz, Ny, Nx).  dc_mean_shift (6,) is a
    macroscopic tensor subtracted from the mean (y = G*(tau - shift))."""
    k = grid.symbol(half=True)
    th = rfftn(tau, backend)
    shift = None if dc_mean_shift is None else grid.nvox * np.asarray(dc_mean_shift, dtype=float)
    yh = project_spectrum(th, k, stress_mask, dc_shift=shift)
    return irfftn(yh, grid.shape, backend)
