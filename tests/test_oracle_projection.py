"""Pins for oracle.projection (A-07, A-08) -- CPU only."""
import numpy as np
import pytest

from oracle.projection import apply_projection, mandel_to_tensor, project_spectrum
from oracle.spectral import Grid, rfftn
from tests.dense import dense_G, symgrad_B, willot_D

rng = np.random.default_rng(5)
MASKS = [(1, 1, 0, 1, 1, 1), (0, 0, 0, 0, 0, 0), (0, 1, 0, 0, 0, 1)]


@pytest.mark.parametrize("shape,mask", [((4, 4, 4), MASKS[0]), ((2, 4, 6), MASKS[1]),
                                        ((1, 8, 8), MASKS[2]), ((3, 4, 5), MASKS[0])])
def test_projection_equals_dense_orthogonal_projector(shape, mask):
    Nz, Ny, Nx = shape
    g = Grid((Nx, Ny, Nz), (1.0, 1.1, 0.9))
    G = dense_G(shape, g.h, mask)
    tau = rng.normal(size=(6,) + shape)
    ref = (G @ tau.reshape(-1)).reshape(tau.shape)
    got = apply_projection(g, tau, mask)
    assert np.max(np.abs(got - ref)) < 1e-12 * np.max(np.abs(ref))


def test_idempotent_selfadjoint():
    g = Grid((8, 6, 4))
    shape = g.shape
    a, b = rng.normal(size=(6,) + shape), rng.normal(size=(6,) + shape)
    m = MASKS[0]
    Ga = apply_projection(g, a, m)
    GGa = apply_projection(g, Ga, m)
    assert np.linalg.norm(GGa - Ga) <= 1e-12 * np.linalg.norm(a)
    Gb = apply_projection(g, b, m)
    assert abs(np.sum(Ga * b) - np.sum(a * Gb)) < 1e-10 * np.linalg.norm(a) * np.linalg.norm(b)


def test_compatible_field_reproduced_and_equilibrated_annihilated():
    shape = (4, 4, 6)
    g = Grid((6, 4, 4))
    B = symgrad_B(willot_D(shape, g.h))
    u = rng.normal(size=3 * g.nvox)
    eps = (B @ u).reshape((6,) + shape)
    E = np.array([0.1, 0.2, -0.3, 0.05, 0.0, 0.01])
    mask = (1, 1, 1, 1, 1, 1)
    got = apply_projection(g, eps + E.reshape(6, 1, 1, 1), mask)
    assert np.max(np.abs(got - (eps + E.reshape(6, 1, 1, 1)))) < 1e-12
    # equilibrated (orthogonal to every compatible field, zero mean): B^T sigma = 0
    s = rng.normal(size=6 * g.nvox)
    Q, _ = np.linalg.qr(B)
    s = s - Q @ (Q.T @ s)
    sig = s.reshape((6,) + shape)
    sig -= sig.reshape(6, -1).mean(axis=1).reshape(6, 1, 1, 1)
    assert np.max(np.abs(apply_projection(g, sig, (0,) * 6))) < 1e-11 * np.max(np.abs(sig))


def test_continuous_scheme_is_moulinec_suquet_gamma0():
    """Real xi: G = Gamma0(lambda0 = 0, mu0 = 1/2) : tau, Gamma0_ijkh = (d_ki x_h x_j + d_hi x_k x_j +
    d_kj x_h x_i + d_hj x_k x_i)/(4 mu0 |x|^2) - (l0+m0)/(m0(l0+2m0)) x_i x_j x_k x_h / |x|^4."""
    xi = rng.normal(size=3)
    tau = rng.normal(size=6) + 1j * rng.normal(size=6)
    T = mandel_to_tensor(tau)
    d = np.eye(3)
    x2 = xi @ xi
    G = (np.einsum("ki,h,j->ijkh", d, xi, xi) + np.einsum("hi,k,j->ijkh", d, xi, xi)
         + np.einsum("kj,h,i->ijkh", d, xi, xi) + np.einsum("hj,k,i->ijkh", d, xi, xi)) / (2 * x2)
    G -= np.einsum("i,j,k,h->ijkh", xi, xi, xi, xi) / x2 ** 2
    ref = np.einsum("ijkh,kh->ij", G, T)
    # batch of two frequencies: a dummy DC (index 0) and xi
    tau2 = np.stack([np.zeros(6), tau], axis=1)
    k2 = np.stack([np.zeros(3), 1j * xi], axis=1)
    got = project_spectrum(tau2, k2, (0,) * 6, dc_index=(0,))[:, 1]
    assert np.allclose(mandel_to_tensor(got), ref, atol=1e-13)


def test_zero_frequency_mask_and_shift():
    g = Grid((4, 4, 4))
    tau = rng.normal(size=(6,) + g.shape)
    Sig = np.array([0, 0, 0, 1.0, 2.0, 3.0])
    m = (0, 0, 0, 1, 1, 1)
    y = apply_projection(g, tau, m, dc_mean_shift=Sig)
    mean_y = y.reshape(6, -1).mean(axis=1)
    mean_t = tau.reshape(6, -1).mean(axis=1)
    assert np.allclose(mean_y, np.array(m) * (mean_t - Sig), atol=1e-13)


def test_null_modes_projected_to_zero():
    g = Grid((4, 4, 4))
    k = g.symbol()
    th = np.zeros((6,) + g.hshape, complex)
    th[:, 2, 2, 0] = rng.normal(size=6)     # (kx, ky, kz) = (0, 2, 2): two axes at Nyquist
    out = project_spectrum(th, k, (1,) * 6)
    assert np.all(out[:, 2, 2, 0] == 0)
