"""NEXT#3: the J independent Helmholtz problems of a staggered iteration ("computed
independently") solved side by side (fgd_solve_helmholtz_all, helm_solve_all in the
staggered loop).  Parity with the oracle's Algorithm 2 per field, bitwise equality with J
consecutive fgd_solve_helmholtz_from calls, and identical staggered increments with the concurrent
solves forced on and off."""
from __future__ import annotations

import os
import sys
import time

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from oracle.helmholtz import ell2_field, solve_helmholtz  # noqa: E402
from oracle.increment import State, Tolerances, make_cell, solve_increment  # noqa: E402
from oracle.spectral import Grid  # noqa: E402
from paper_2103_04770_b200 import Context, Material  # noqa: E402

TOL = Tolerances()


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


class conc:
    """FGD_HELM_CONC for the duration of a block (the library reads it on every call)."""

    def __init__(self, v):
        self.v = v

    def __enter__(self):
        self.old = os.environ.get("FGD_HELM_CONC")
        if self.v is None:
            os.environ.pop("FGD_HELM_CONC", None)
        else:
            os.environ["FGD_HELM_CONC"] = str(self.v)

    def __exit__(self, *a):
        if self.old is None:
            os.environ.pop("FGD_HELM_CONC", None)
        else:
            os.environ["FGD_HELM_CONC"] = self.old


def two_field_ctx(n, seed):
    g = Grid(n, (1.0, 1.0, 1.0))
    rng = np.random.default_rng(seed)
    ph = rng.integers(0, 3, size=g.shape).astype(np.uint8)
    ell = np.array([[0.05, 0.01, 0.03], [0.02, 0.08, 0.004]])
    ctx = Context(n, (1.0, 1.0, 1.0))
    ctx.set_phases(dev(ph), 3)
    ctx.set_nonlocal(ell, [0, 1])
    src = np.abs(rng.normal(size=(2,) + g.shape))
    x0 = rng.normal(size=(2,) + g.shape)
    return g, ph, ell, ctx, src, x0


@pytest.mark.parametrize("n", [(16, 8, 8), (32, 32, 1), (64, 32, 16), (256, 8, 8), (8, 256, 256)])
def test_all_fields_parity_and_bitwise(n):
    g, ph, ell, ctx, src, x0 = two_field_ctx(n, 11)
    J = 2
    out = torch.empty((J,) + g.shape, dtype=torch.float64, device="cuda")
    one = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    for mode in (1, 0, None):
        with conc(mode):
            # fixed iteration counts against the oracle, cold and warm
            for k in (1, 5):
                its, _ = ctx.solve_helmholtz_all(dev(src), None, out, J, tol=0.0, maxit=k)
                assert its == [k, k]
                for j in range(J):
                    ref, _, _ = solve_helmholtz(g, src[j], ell2_field(ph, ell[j]), tol=0.0, maxit=k)
                    assert rel(out[j].cpu().numpy(), ref) <= 1e-10, (n, mode, k, j)
            its, _ = ctx.solve_helmholtz_all(dev(src), dev(x0), out, J, tol=0.0, maxit=3)
            for j in range(J):
                ref, _, _ = solve_helmholtz(g, src[j], ell2_field(ph, ell[j]), tol=0.0, maxit=3, x0=x0[j])
                assert rel(out[j].cpu().numpy(), ref) <= 1e-10, (n, mode, j)
            # converged: counts of the oracle (+-1) and bitwise the consecutive per-field solves
            its, rr = ctx.solve_helmholtz_all(dev(src), None, out, J, tol=1e-9, maxit=2000)
            for j in range(J):
                ref, it_ref, _ = solve_helmholtz(g, src[j], ell2_field(ph, ell[j]), tol=1e-9, maxit=2000)
                assert abs(its[j] - it_ref) <= 1 and rr[j] < 1e-9, (n, mode, j, its, it_ref)
                assert rel(out[j].cpu().numpy(), ref) <= 1e-8
                it1, _ = ctx.solve_helmholtz_from(j, dev(src[j]), None, one, tol=1e-9, maxit=2000)
                assert it1 == its[j]
                assert torch.equal(one, out[j]), (n, mode, j)
    ctx.close()


def test_all_fields_host_buffers_and_noconv():
    g, ph, ell, ctx, src, x0 = two_field_ctx((32, 16, 8), 5)
    out = np.empty((2,) + g.shape)
    with conc(1):
        its, _ = ctx.solve_helmholtz_all(src, x0, out, 2, tol=0.0, maxit=2)
        for j in range(2):
            ref, _, _ = solve_helmholtz(g, src[j], ell2_field(ph, ell[j]), tol=0.0, maxit=2, x0=x0[j])
            assert rel(out[j], ref) <= 1e-10
        # too few iterations for the tolerance: ENOCONV, both fields still returned
        its, rr = ctx.solve_helmholtz_all(src, None, out, 2, tol=1e-12, maxit=2, check=False)
        assert its == [2, 2] and all(r > 1e-12 for r in rr)
        with pytest.raises(Exception):
            ctx.solve_helmholtz_all(src, None, out, 2, tol=1e-12, maxit=2)
    ctx.close()


def ctx_from_cfg(cfg):
    ctx = Context(cfg.n, cfg.L)
    ctx.set_phases(dev(cfg.phases), len(cfg.materials))
    for q, m in enumerate(cfg.materials):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
    ctx.set_control(cfg.stress_mask)
    return ctx


def test_increments_concurrent_equal_consecutive():
    """Two-field staggered increments (reduced config 3): concurrent and consecutive Helmholtz solves
    give bitwise the same macroscopic stress and the same iteration counts; both match the oracle."""
    cfg = synth.config3(n=16, n_spheres=4, phi=0.2, seed=3)
    cfg.dE = 1.5e-3
    cell = make_cell(cfg)
    st = State.zero(cell)
    ca, cb = ctx_from_cfg(cfg), ctx_from_cfg(cfg)
    ta = tb = 0.0
    for i in range(1, 4):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        args = (Et, np.zeros(6), TOL.tol_stag, TOL.tol_newton, TOL.tol_cg, TOL.tol_helm, TOL.max_stag, TOL.max_newton,
                TOL.max_cg, TOL.max_helm)
        with conc(1):
            t0 = time.perf_counter()
            s, ra = ca.solve_increment(*args)
            ta += time.perf_counter() - t0
            assert s == 0, ra
        with conc(0):
            t0 = time.perf_counter()
            s, rb = cb.solve_increment(*args)
            tb += time.perf_counter() - t0
            assert s == 0, rb
        assert np.array_equal(ra["macro_stress"], rb["macro_stress"])
        assert (ra["stag"], ra["newton"], ra["cg"], ra["helm"]) == (rb["stag"], rb["newton"], rb["cg"], rb["helm"])
        assert rel(ra["macro_stress"], rep.macro_stress) <= 1e-6
    print(f"two-field increments at 16^3: concurrent {ta:.3f} s, consecutive {tb:.3f} s")
    ca.close()
    cb.close()


@pytest.mark.parametrize("P", [2, 4])
def test_all_fields_emulated_slabs(monkeypatch, P):
    """The side-by-side solves on the P-slab spectrum layout (FGD_EMULATE_SLABS: every field copy owns
    its one-component slab buffers)."""
    monkeypatch.setenv("FGD_EMULATE_SLABS", str(P))
    n = (32, 16, 8)
    g, ph, ell, ctx, src, x0 = two_field_ctx(n, 21)
    out = torch.empty((2,) + g.shape, dtype=torch.float64, device="cuda")
    with conc(1):
        its, _ = ctx.solve_helmholtz_all(dev(src), dev(x0), out, 2, tol=0.0, maxit=4)
        assert its == [4, 4]
        for j in range(2):
            ref, _, _ = solve_helmholtz(g, src[j], ell2_field(ph, ell[j]), tol=0.0, maxit=4, x0=x0[j])
            assert rel(out[j].cpu().numpy(), ref) <= 1e-10, (P, j)
    ctx.close()


def test_single_field_goes_through_all():
    """J = 1: fgd_solve_helmholtz_all is the plain solve."""
    n = (16, 16, 1)
    g = Grid(n, (1.0, 1.0, 1.0))
    rng = np.random.default_rng(3)
    ph = (rng.random(g.shape) < 0.4).astype(np.uint8)
    ctx = Context(n, (1.0, 1.0, 1.0))
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(np.array([[0.05, 0.02]]), [0])
    src = np.abs(rng.normal(size=(1,) + g.shape))
    out = torch.empty((1,) + g.shape, dtype=torch.float64, device="cuda")
    its, rr = ctx.solve_helmholtz_all(dev(src), None, out, 1, tol=1e-10, maxit=500)
    ref, it_ref, _ = solve_helmholtz(g, src[0], ell2_field(ph, [0.05, 0.02]), tol=1e-10, maxit=500)
    assert abs(its[0] - it_ref) <= 1 and rel(out[0].cpu().numpy(), ref) <= 1e-8
    ctx.close()
