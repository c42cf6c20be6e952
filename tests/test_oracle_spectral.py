"""Pins for oracle.spectral -- CPU only."""
import json
import os

import numpy as np
import pytest

from oracle.spectral import Grid, cis, irfftn, rfftn

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
rng = np.random.default_rng(11)


@pytest.mark.parametrize("shape", [(4, 6, 8), (5, 3, 4), (1, 8, 8), (3, 5, 7)])
def test_naive_dft_equals_fft(shape):
    u = rng.normal(size=(2,) + shape)
    A = rfftn(u, "naive")
    B = rfftn(u, "scipy")
    assert np.max(np.abs(A - B)) <= 1e-13 * np.max(np.abs(B))
    ua = irfftn(B, shape, "naive")
    ub = irfftn(B, shape, "scipy")
    assert np.max(np.abs(ua - u)) < 1e-13
    assert np.max(np.abs(ub - u)) < 1e-13


def test_brute_force_definition():
    """F(u)(k) = sum_x u(x) exp(-2 pi i k.x/N) evaluated term by term at a few frequencies."""
    shape = (3, 4, 5)
    u = rng.normal(size=shape)
    U = rfftn(u, "scipy")
    for (kz, ky, kx) in [(0, 0, 0), (1, 2, 2), (2, 3, 1), (0, 1, 2)]:
        s = 0j
        for z in range(3):
            for y in range(4):
                for x in range(5):
                    s += u[z, y, x] * np.exp(-2j * np.pi * (kz * z / 3 + ky * y / 4 + kx * x / 5))
        assert abs(s - U[kz, ky, kx]) < 1e-12


def test_constant_and_cosine():
    shape = (4, 8, 6)
    c = 2.5
    U = rfftn(np.full(shape, c))
    assert abs(U[0, 0, 0] - c * 4 * 8 * 6) < 1e-12
    U[0, 0, 0] = 0
    assert np.max(np.abs(U)) < 1e-12
    y = np.arange(8)
    u = np.cos(2 * np.pi * 3 * y / 8)[None, :, None] * np.ones(shape)
    U = rfftn(u)
    n = 4 * 6 * 8 / 2
    assert abs(U[0, 3, 0] - n) < 1e-11 and abs(U[0, 5, 0] - n) < 1e-11
    U[0, 3, 0] = U[0, 5, 0] = 0
    assert np.max(np.abs(U)) < 1e-11


@pytest.mark.parametrize("key", ["frequencies_N4_L2pi", "frequencies_N5_L2pi", "frequencies_N1"])
def test_frequency_sets(key):
    g = GOLD[key]
    grid = Grid((g["N"], 1, 1), (g["L"], 1.0, 1.0))
    got = sorted(np.round(grid.xi_axis(0), 12).tolist())
    assert got == sorted(float(v) for v in g["set"])


def _stencil_grad(u, j, h):
    """forward difference along j at the vertex, averaged over 0/+1 shifts of the other axes."""
    ax = 2 - j          # numpy axis of spatial axis j
    others = [a for a in (0, 1, 2) if a != ax]
    out = np.zeros_like(u)
    for b in (0, 1):
        for c in (0, 1):
            v = np.roll(u, shift=(-b, -c), axis=others)
            out += np.roll(v, -1, axis=ax) - v
    return out / (4.0 * h[j])


@pytest.mark.parametrize("shape", [(4, 6, 8), (1, 8, 8), (3, 5, 4)])
def test_willot_symbol_is_stencil(shape):
    g = Grid((shape[2], shape[1], shape[0]), (1.0, 0.7, 1.3))
    u = rng.normal(size=shape)
    k = g.symbol()
    U = rfftn(u)
    for j in range(3):
        a = irfftn(k[j] * U, shape)
        b = _stencil_grad(u, j, g.h)
        assert np.max(np.abs(a - b)) < 1e-12 * max(1.0, np.max(np.abs(b)))


def test_willot_tan_form():
    """k_j = (i/(4h_j)) tan(theta_j/2) prod_m (1 + e^{i theta_m}) (Willot 2015 form) off Nyquist."""
    g = Grid((5, 7, 9), (1.0, 1.0, 1.0))
    k = g.symbol(half=False)
    th = [2 * np.pi * g.wrapped(a) / g.n[a] for a in range(3)]
    TH = np.meshgrid(th[2], th[1], th[0], indexing="ij")  # z, y, x
    prod = (1 + np.exp(1j * TH[0])) * (1 + np.exp(1j * TH[1])) * (1 + np.exp(1j * TH[2]))
    for j in range(3):
        ref = 1j / (4 * g.h[j]) * np.tan(TH[2 - j] / 2) * prod
        assert np.max(np.abs(ref - k[j])) < 1e-12 * np.max(np.abs(ref))


def test_symbol_hermitian_and_nullset():
    g = Grid((4, 4, 4))
    k = g.symbol(half=False)
    Nz, Ny, Nx = g.shape
    for z in range(Nz):
        for y in range(Ny):
            for x in range(Nx):
                assert np.allclose(k[:, (-z) % Nz, (-y) % Ny, (-x) % Nx], np.conj(k[:, z, y, x]), atol=1e-14)
                zero = np.all(k[:, z, y, x] == 0)
                nyq = sum(int(i == 2) for i in (x, y, z))
                expect = (x, y, z) == (0, 0, 0) or nyq >= 2
                assert zero == expect, (x, y, z)


def test_willot_converges_to_continuous():
    """k_j = e^{i(th1+th2+th3)/2} * i xi_j (1 + O(h^2)): the vertex (half-voxel) shift times a
    second-order accurate derivative."""
    errs = []
    for N in (16, 32, 64):
        g = Grid((N, N, N))
        k = g.symbol()[0, 1, 0, 1]                       # x-component at mode (x=1, y=0, z=1)
        th = 2 * np.pi / N
        xi = 2 * np.pi
        errs.append(abs(k * np.exp(-1j * (th + th) / 2) - 1j * xi) / xi)
    assert errs[1] < errs[0] / 3.5 and errs[2] < errs[1] / 3.5   # O(h^2)


def test_continuous_symbol():
    g = Grid((4, 1, 1), (2 * np.pi, 1.0, 1.0), scheme="continuous")
    k = g.symbol()
    assert np.allclose(k[0, 0, 0, :], [0, 1j, 0])     # Nyquist zeroed (A-06)


def test_hermitian_weights_parseval():
    for shape in [(4, 6, 8), (3, 5, 7)]:
        g = Grid((shape[2], shape[1], shape[0]))
        u, v = rng.normal(size=shape), rng.normal(size=shape)
        U, V = rfftn(u), rfftn(v)
        lhs = np.sum(g.hermitian_weights() * np.real(U * np.conj(V)))
        assert abs(lhs - g.nvox * np.sum(u * v)) < 1e-10


def test_cis_exact_quadrants():
    assert cis(np.array([0, 1, 2, 3]), 4).tolist() == [1, 1j, -1, -1j]
