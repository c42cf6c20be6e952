"""Pins for oracle.mech -- CPU only."""
import numpy as np

from oracle.mech import apply_projected_tangent, cg, contract, pack21, unpack21
from oracle.projection import apply_projection
from oracle.spectral import Grid
from synth import random_spd_tangent
from tests.dense import dense_G

rng = np.random.default_rng(9)


def test_contraction_explicit_loop_and_packing():
    C = unpack21(random_spd_tangent(10, 1))
    assert np.allclose(pack21(C), random_spd_tangent(10, 1))
    p = rng.normal(size=(6, 10))
    tau = contract(C, p)
    for v in range(10):
        for i in range(6):
            s = 0.0
            for j in range(6):
                s += C[i, j, v] * p[j, v]
            assert abs(s - tau[i, v]) < 1e-9


def test_cg_equals_dense_pseudo_inverse():
    shape = (4, 4, 4)
    g = Grid((4, 4, 4))
    mask = (1, 1, 0, 1, 1, 1)
    n = g.nvox
    C = unpack21(random_spd_tangent(n, 2)).reshape((6, 6) + shape)
    G = dense_G(shape, g.h, mask)
    Cbig = np.zeros((6 * n, 6 * n))
    for i in range(6):
        for j in range(6):
            Cbig[i * n:(i + 1) * n, j * n:(j + 1) * n] = np.diag(C[i, j].reshape(-1))
    A = G @ Cbig @ G
    b = apply_projection(g, rng.normal(size=(6,) + shape), mask)
    ref = (np.linalg.pinv(A, rcond=1e-12) @ b.reshape(-1)).reshape(b.shape)
    x, it, rel = cg(g, C, b, mask, tol=1e-13)
    assert rel < 1e-13
    assert np.linalg.norm(x - ref) < 1e-9 * np.linalg.norm(ref)


def test_pq_identity_on_range():
    g = Grid((8, 6, 4))
    mask = (1, 1, 0, 1, 1, 1)
    C = unpack21(random_spd_tangent(g.nvox, 3)).reshape((6, 6) + g.shape)
    p = apply_projection(g, rng.normal(size=(6,) + g.shape), mask)
    q = apply_projected_tangent(g, C, p, mask)
    assert abs(np.sum(p * q) - np.sum(p * contract(C, p))) < 1e-12 * abs(np.sum(p * q))
