"""Discretization and discrete Fourier transform (paper Sec. 3.2.1).

TEST INFRASTRUCTURE (see oracle/__init__.py): not importable by the product path.

* Voxel grid N1 x N2 x N3 with spacing h_i = L_i / N_i, unknowns at voxel centres
  x_i = (1/2 + n_i) h_i.  Arrays are numpy C-order [z][y][x]: axis x <-> index 1
  (component "11"), y <-> 2, z <-> 3.  2D plane-strain cells are N3 = 1 (R-2D).
* Frequencies xi_i = (2 pi / L_i)(n_i - N_i/2) (even) or (n_i - (N_i-1)/2) (odd),
  stored in FFT (wrapped) order -- a value set, not an order (A-05).
* Derivative symbols k_j(xi):
    - 'willot' (default, A-04): rotated finite-difference scheme,
          k_1 = (e^{i th1} - 1)(1 + e^{i th2})(1 + e^{i th3}) / (4 h_1),  th_i = xi_i h_i, cyclic;
      the exact symbol of "forward difference along j, averaged over the 0/+1 shifts of the
      other two axes" (gradient at the voxel vertex).  = (i/4h) tan(th_j/2) prod_m (1+e^{i th_m}).
    - 'continuous' (A-06): k_j = i xi_j, set to 0 on the Nyquist index of an even axis.
  e^{i th} is evaluated exactly (0, +-1, +-i) at quarter turns so that null modes are exact zeros.
* DFT: F(u)(xi) = sum_x u(x) e^{-i xi.x}, F^{-1} with 1/N.  The half-voxel centre
  offset multiplies F by a per-frequency phase that cancels in every F^{-1}(m(xi) F(.)) the
  method uses, so index-based transforms are used (DESIGN.md R-DFT).  Real fields use the
  R2C half spectrum along x (last numpy axis): shape (Nz, Ny, Nx//2 + 1).
  Backends: 'naive' (explicit exp(-2 pi i k n / N) matrices, tiny grids) and 'scipy'.

Pins (tests/test_oracle_spectral.py): naive DFT == scipy FFT; round trip; constant -> DC
only; cosine -> two conjugate coefficients; SPEC frequency sets; Willot symbol == real-space
stencil; k(-xi) = conj k(xi); k -> i xi as h -> 0; null set of the Willot symbol.
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sfft

WORKERS = os.cpu_count() or 1


def cis(m, N):
    """exp(2 pi i m / N) for integer arrays m, exact at multiples of a quarter turn."""
    m = np.asarray(m) % N
    r = m / N
    out = np.exp(2j * np.pi * r)
    q4 = (4 * m) % N == 0
    if np.any(q4):
        quarter = ((4 * m[q4]) // N) % 4
        out = np.array(out, dtype=complex)
        out[q4] = np.array([1.0, 1.0j, -1.0, -1.0j])[quarter]
    return out


class Grid:
    def __init__(self, n, L=None, scheme: str = "willot"):
        n = tuple(int(v) for v in n)
        if len(n) == 2:
            n = (n[0], n[1], 1)
        if any(v < 1 for v in n):
            raise ValueError("N_i must be >= 1")
        if L is None:
            L = (1.0, 1.0, 1.0 if n[2] > 1 else 1.0 / n[0])
        L = tuple(float(v) for v in L)
        if any(v <= 0 for v in L):
            raise ValueError("L_i must be > 0")
        if scheme not in ("willot", "continuous"):
            raise ValueError(scheme)
        self.n = n
        self.L = L
        self.h = tuple(L[i] / n[i] for i in range(3))
        self.scheme = scheme
        self.shape = (n[2], n[1], n[0])                  # [z][y][x]
        self.hshape = (n[2], n[1], n[0] // 2 + 1)        # half spectrum along x
        self.nvox = n[0] * n[1] * n[2]

    # ---- frequencies ------------------------------------------------------------------------
    def wrapped(self, axis: int, half: bool = False) -> np.ndarray:
        """integer frequency index m_i in FFT order (axis 0 = x)."""
        N = self.n[axis]
        if half:
            return np.arange(N // 2 + 1)
        return np.fft.fftfreq(N, d=1.0 / N).round().astype(int)

    def xi_axis(self, axis: int, half: bool = False) -> np.ndarray:
        """xi_i = 2 pi m_i / L_i  (P:634-641 as a value set)."""
        return 2.0 * np.pi * self.wrapped(axis, half) / self.L[axis]

    def _bc(self, v, axis):
        # broadcast a per-axis vector (axis 0 = x) onto [z][y][x]
        shp = [1, 1, 1]
        shp[2 - axis] = v.shape[0]
        return v.reshape(shp)

    def symbol(self, half: bool = True) -> np.ndarray:
        """k_j(xi), shape (3, Nz, Ny, Nx') complex (Nx' = Nx//2+1 when half)."""
        e, m = [], []
        for a in range(3):
            mm = self.wrapped(a, half=(half and a == 0))
            m.append(mm)
            e.append(cis(mm, self.n[a]))
        if self.scheme == "willot":
            d = [self._bc(e[a] - 1.0, a) for a in range(3)]
            c = [self._bc(1.0 + e[a], a) for a in range(3)]
            k = [d[0] * c[1] * c[2] / (4.0 * self.h[0]),
                 c[0] * d[1] * c[2] / (4.0 * self.h[1]),
                 c[0] * c[1] * d[2] / (4.0 * self.h[2])]
        else:
            k = []
            for a in range(3):
                xi = 2.0 * np.pi * m[a] / self.L[a]
                kk = 1j * xi
                N = self.n[a]
                if N % 2 == 0:
                    kk = np.where(np.abs(m[a]) == N // 2, 0.0, kk)
                k.append(self._bc(kk.astype(complex), a))
        full = np.broadcast_shapes(*[kk.shape for kk in k])
        return np.stack([np.broadcast_to(kk, full) for kk in k]).astype(complex)

    def is_dc(self, half: bool = True) -> np.ndarray:
        z = np.zeros(self.hshape if half else self.shape, dtype=bool)
        z[0, 0, 0] = True
        return z

    def hermitian_weights(self) -> np.ndarray:
        """weights w such that sum_half w Re(u^ conj v^) = N_vox * sum_x u v (A-10)."""
        Nx = self.n[0]
        w = np.full(self.hshape, 2.0)
        w[..., 0] = 1.0
        if Nx % 2 == 0:
            w[..., Nx // 2] = 1.0
        return w


# ---- transforms ---------------------------------------------------------------------------------
def _dft_matrix(N: int, sign: int) -> np.ndarray:
    k = np.arange(N)
    return cis(sign * np.outer(k, k), N)


def rfftn(u: np.ndarray, backend: str = "scipy") -> np.ndarray:
    """Unnormalised forward DFT over the last 3 axes, half spectrum along the last axis."""
    u = np.asarray(u, dtype=float)
    if backend == "scipy":
        return sfft.rfftn(u, axes=(-3, -2, -1), workers=WORKERS)
    Nz, Ny, Nx = u.shape[-3:]
    Wx = _dft_matrix(Nx, -1)[: Nx // 2 + 1]
    Wy = _dft_matrix(Ny, -1)
    Wz = _dft_matrix(Nz, -1)
    U = np.einsum("kx,...zyx->...zyk", Wx, u.astype(complex))
    U = np.einsum("ky,...zyx->...zkx", Wy, U)
    U = np.einsum("kz,...zyx->...kyx", Wz, U)
    return U


def irfftn(U: np.ndarray, shape, backend: str = "scipy") -> np.ndarray:
    """Inverse of rfftn (1/N normalisation); `shape` = (Nz, Ny, Nx)."""
    Nz, Ny, Nx = shape
    if backend == "scipy":
        return sfft.irfftn(U, s=(Nz, Ny, Nx), axes=(-3, -2, -1), workers=WORKERS)
    V = np.einsum("kz,...zyx->...kyx", _dft_matrix(Nz, +1), U) / Nz
    V = np.einsum("ky,...zyx->...zkx", _dft_matrix(Ny, +1), V) / Ny
    # C2R along x: x[n] = (1/N)[Re X0 + 2 sum_{0<k<N/2} Re(X_k e^{2pi i kn/N}) + Re X_{N/2} (-1)^n]
    n = np.arange(Nx)
    out = np.real(V[..., 0:1]) * np.ones(Nx)
    for k in range(1, (Nx + 1) // 2):
        out = out + 2.0 * np.real(V[..., k:k + 1] * cis(k * n, Nx))
    if Nx % 2 == 0:
        out = out + np.real(V[..., Nx // 2:Nx // 2 + 1]) * ((-1.0) ** n)
    return out / Nx
