"""Pins for oracle.helmholtz (A-09..A-11) -- CPU only."""
import json
import os

import numpy as np
import pytest

from oracle.helmholtz import apply_helmholtz, apply_Lhat, apply_precond, ell2_field, solve_helmholtz
from oracle.spectral import Grid, rfftn
from tests.dense import dense_helmholtz

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_values.json")))
rng = np.random.default_rng(7)


def two_phase(shape, p=0.3, seed=1):
    return (np.random.default_rng(seed).random(shape) < p).astype(np.uint8)


@pytest.mark.parametrize("shape", [(4, 6, 8), (1, 8, 8), (3, 4, 5)])
def test_apply_equals_dense_stencil_assembly(shape):
    g = Grid((shape[2], shape[1], shape[0]), (1.0, 0.8, 1.2))
    ph = two_phase(shape)
    ell2 = ell2_field(ph, [0.2, 0.2 / 50])
    L = dense_helmholtz(shape, g.h, ell2.reshape(-1))
    a = rng.normal(size=shape)
    ref = (L @ a.reshape(-1)).reshape(shape)
    got = apply_helmholtz(g, a, ell2)
    assert np.max(np.abs(got - ref)) < 1e-12 * np.max(np.abs(ref))


def test_uniform_ell_symbol_and_exact_preconditioner():
    g = Grid((8, 8, 8))
    ell2 = np.full(g.shape, 0.15 ** 2)
    a = rng.normal(size=g.shape)
    A = rfftn(a)
    k2 = np.sum(np.abs(g.symbol()) ** 2, axis=0)
    assert np.allclose(apply_Lhat(g, A, ell2), (1 + 0.15 ** 2 * k2) * A, atol=1e-10)
    La = apply_helmholtz(g, a, ell2)
    assert np.max(np.abs(apply_precond(g, La, ell2) - a)) < 1e-12
    x, it, _ = solve_helmholtz(g, a, ell2, tol=1e-12)
    assert it == 1


def test_constant_selfadjoint_positive():
    g = Grid((6, 4, 8))
    ell2 = ell2_field(two_phase(g.shape), [0.3, 0.006])
    c = np.full(g.shape, 3.0)
    assert np.max(np.abs(apply_helmholtz(g, c, ell2) - 3.0)) < 1e-12
    u, v = rng.normal(size=g.shape), rng.normal(size=g.shape)
    Lu, Lv = apply_helmholtz(g, u, ell2), apply_helmholtz(g, v, ell2)
    assert abs(np.sum(Lu * v) - np.sum(u * Lv)) < 1e-12 * np.sum(np.abs(Lu * v))
    assert np.sum(Lu * u) >= np.sum(u * u)


def test_single_mode_closed_form():
    """uniform l, alpha = cos(2 pi (m.x)): abar = alpha / (1 + l^2 |k(xi)|^2)."""
    g = Grid((16, 8, 8), (1.0, 1.0, 1.0))
    z, y, x = np.meshgrid(np.arange(8), np.arange(8), np.arange(16), indexing="ij")
    alpha = np.cos(2 * np.pi * (3 * x / 16 + 1 * y / 8 + 2 * z / 8))
    ell = 0.07
    abar, it, _ = solve_helmholtz(g, alpha, np.full(g.shape, ell ** 2), tol=1e-13)
    k = g.symbol()[:, 2, 1, 3]
    ref = alpha / (1 + ell ** 2 * np.sum(np.abs(k) ** 2))
    assert np.max(np.abs(abar - ref)) < 1e-13


@pytest.mark.parametrize("shape", [(1, 8, 8), (6, 6, 6)])
def test_pcg_equals_dense_direct_solve(shape):
    g = Grid((shape[2], shape[1], shape[0]))
    ell2 = ell2_field(two_phase(shape, 0.4, 3), [0.25, 0.005])
    alpha = rng.random(shape)
    L = dense_helmholtz(shape, g.h, ell2.reshape(-1))
    ref = np.linalg.solve(L, alpha.reshape(-1)).reshape(shape)
    got, it, hist = solve_helmholtz(g, alpha, ell2, tol=1e-12)
    assert np.linalg.norm(got - ref) < 1e-10 * np.linalg.norm(ref)
    assert abs(got.mean() - alpha.mean()) < 1e-12          # mean preservation


def test_warm_start_pcg():
    """Warm start: from the dense direct solution the PCG stops before its first iteration;
    from a perturbed guess it converges to the same dense solution, with fewer iterations than from 0
    when the guess is close (the stopping test stays relative to ||alpha||)."""
    shape = (6, 6, 6)
    g = Grid((shape[2], shape[1], shape[0]))
    ell2 = ell2_field(two_phase(shape, 0.4, 5), [0.25, 0.005])
    alpha = rng.random(shape)
    L = dense_helmholtz(shape, g.h, ell2.reshape(-1))
    ref = np.linalg.solve(L, alpha.reshape(-1)).reshape(shape)
    got, it, _ = solve_helmholtz(g, alpha, ell2, tol=1e-10, x0=ref)
    assert it == 0 and np.linalg.norm(got - ref) < 1e-13 * np.linalg.norm(ref)
    _, it_cold, _ = solve_helmholtz(g, alpha, ell2, tol=1e-12)
    guess = ref + 1e-6 * rng.random(shape)
    got, it_warm, _ = solve_helmholtz(g, alpha, ell2, tol=1e-12, x0=guess)
    assert np.linalg.norm(got - ref) < 1e-10 * np.linalg.norm(ref)
    assert it_warm < it_cold


def test_mean_ell2_golden():
    gv = GOLD["mean_ell2_two_phase"]
    ph = np.zeros((2, 4, 4), np.uint8)
    ph[:, :, :2] = 1
    assert abs(np.mean(ell2_field(ph, gv["ell"])) - gv["mean_ell2"]) < 1e-15


def test_local_limit_zero_length():
    """ell = 0 (the local limit): L = I, the non-local field equals its source and the
    preconditioned CG stops after one iteration."""
    g = Grid((8, 8, 4))
    rng = np.random.default_rng(9)
    a = rng.normal(size=g.shape)
    e2 = ell2_field(np.zeros(g.shape, np.uint8), [0.0])
    abar, it, res = solve_helmholtz(g, a, e2, tol=1e-14, maxit=50)
    assert it == 1
    assert np.max(np.abs(abar - a)) < 1e-14 * np.max(np.abs(a))
