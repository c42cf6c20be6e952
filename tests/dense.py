"""Dense real-space brute-force operators used to PIN the oracle (not shared with it).

Built directly from the definition of the rotated finite-difference gradient (A-04: forward
difference along j at the voxel vertex, averaged over the 0/+1 shifts of the other axes) as
explicit n x n matrices on tiny periodic grids -- no FFT, no symbol.
"""
import itertools

import numpy as np

S2 = np.sqrt(2.0)


def lin(shape, z, y, x):
    Nz, Ny, Nx = shape
    return ((z % Nz) * Ny + (y % Ny)) * Nx + (x % Nx)


def willot_D(shape, h):
    """[D_x, D_y, D_z] as dense (n, n) matrices; axis 0 = x."""
    Nz, Ny, Nx = shape
    n = Nz * Ny * Nx
    Ds = [np.zeros((n, n)) for _ in range(3)]
    for z, y, x in itertools.product(range(Nz), range(Ny), range(Nx)):
        row = lin(shape, z, y, x)
        for v in itertools.product((0, 1), repeat=3):     # v = (vx, vy, vz)
            col = lin(shape, z + v[2], y + v[1], x + v[0])
            for j in range(3):
                s = 1.0 if v[j] == 1 else -1.0
                Ds[j][row, col] += s / (4.0 * h[j])
    return Ds


def symgrad_B(Ds):
    """Mandel symmetric gradient u (3n) -> eps (6n) : (D1u1, D2u2, D3u3, sqrt2/2(D2u3+D3u2), ...)."""
    n = Ds[0].shape[0]
    Z = np.zeros((n, n))
    D1, D2, D3 = Ds
    rows = [
        [D1, Z, Z],
        [Z, D2, Z],
        [Z, Z, D3],
        [Z, D3 / S2, D2 / S2],
        [D3 / S2, Z, D1 / S2],
        [D2 / S2, D1 / S2, Z],
    ]
    return np.block(rows)


def range_projector(B, rtol=1e-10):
    U, s, _ = np.linalg.svd(B, full_matrices=False)
    r = int(np.sum(s > rtol * s[0]))
    Ur = U[:, :r]
    return Ur @ Ur.T


def dense_G(shape, h, stress_mask):
    """Dense 6n x 6n operator: orthogonal projector onto range(sym grad) + mean mask."""
    n = int(np.prod(shape))
    B = symgrad_B(willot_D(shape, h))
    P = range_projector(B)
    M = np.kron(np.diag(np.asarray(stress_mask, float)), np.full((n, n), 1.0 / n))
    return P + M


def dense_helmholtz(shape, h, ell2_flat):
    Ds = willot_D(shape, h)
    n = Ds[0].shape[0]
    L = np.eye(n)
    for D in Ds:
        L += D.T @ (ell2_flat[:, None] * D)
    return L
