"""The mechanical CG on the COMPACT consistent tangent (9 doubles per voxel, written by
fgd_constitutive) -- the kernel instantiation that dominates every production
increment and the bench (`k_xtan<N, XF_TANGENT_CG, compact>` with its own ring rows, stage count
and shared-memory layout at N1 = 256 / 512) -- against

  * the oracle CG on the oracle's tangent of the same state (c9) after
    k = 1, 2, 6 iterations (<= 1e-10) and converged (iterations +-1) on grids that select the
    specialised passes: (256, 8, 8), (512, 4, 8) (bulk-copy x pass), (8, 256, 256) (register y/z
    passes), and 256^3 (k = 2);
  * the packed 21-component path on the expanded tangent (the same operator, another kernel)
    at 256^3 and 512^3 (<= 1e-12 after 6 iterations);
  * itself: a 10-iteration CG repeated on the same input is bitwise identical (256^3, 512^3).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import synth  # noqa: E402
from oracle import material as M  # noqa: E402
from oracle.increment import Cell, State, evaluate, frozen_damage  # noqa: E402
from oracle.mech import cg  # noqa: E402
from oracle.projection import apply_projection  # noqa: E402
from oracle.spectral import Grid  # noqa: E402
from paper_2103_04770_b200 import Context, Material  # noqa: E402
from paper_2103_04770_b200 import _fgd  # noqa: E402

MASK = synth.CONFIG1_MASK


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def damaged_plastic_cell(n, seed):
    """Config-1 phases (J2-Lemaitre matrix / elastic inclusion, one non-local field), a random
    committed state with damage and a strain beyond yield: most matrix voxels return plastically
    with D in (0, 0.99], so the compact tangent carries all of n, ca, cb, cc."""
    g = Grid(n, (float(n[0]), float(n[1]), float(n[2])))
    rng = np.random.default_rng(seed)
    ph = (rng.random(g.shape) < 0.2).astype(np.uint8)
    cell = Cell(g, ph, [synth.MATRIX_J2, synth.INCLUSION_EL], synth.CONFIG1_ELL, [0], MASK)
    nv = g.nvox
    st = State.zero(cell)
    st.epsp = M.dev(rng.normal(scale=1e-3, size=(6, nv)))
    st.ep = np.abs(rng.normal(scale=5e-3, size=nv))
    st.hist = rng.uniform(0, 0.3, nv)
    st.abar = np.abs(rng.normal(scale=1e-2, size=(1,) + g.shape))
    eps = rng.normal(scale=5e-3, size=(6,) + g.shape)
    ctx = Context(n, (float(n[0]), float(n[1]), float(n[2])))
    ctx.set_phases(dev(ph), 2)
    ctx.set_material(0, Material.of(synth.MATRIX_J2))
    ctx.set_material(1, Material.of(synth.INCLUSION_EL))
    ctx.set_nonlocal(synth.CONFIG1_ELL, [0])
    ctx.set_control(MASK)
    ctx.set_field(_fgd.FIELD_EPS_P, dev(st.epsp))
    ctx.set_field(_fgd.FIELD_EQPS, dev(st.ep))
    ctx.set_field(_fgd.FIELD_HIST, dev(st.hist))
    ctx.set_field(_fgd.FIELD_NONLOCAL, dev(st.abar[0]))
    ctx.constitutive(dev(eps), None)
    b = apply_projection(g, rng.normal(size=(6,) + g.shape), MASK)
    return g, cell, st, eps, ctx, b


def oracle_tangent(cell, st, eps):
    D = frozen_damage(cell, st, st.abar)
    _, C, _, _, _ = evaluate(cell, eps, st, D)
    return C


@pytest.mark.parametrize("n", [(256, 8, 8), (512, 4, 8), (8, 256, 256)])
def test_compact_cg_vs_oracle(n):
    g, cell, st, eps, ctx, b = damaged_plastic_cell(n, 5)
    C = oracle_tangent(cell, st, eps)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    for k in (1, 2, 6):
        it, _ = ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=k)
        ref, _, _ = cg(g, C, b, MASK, tol=0.0, maxit=k)
        assert it == k
        assert rel(out.cpu().numpy(), ref) <= 1e-10, k
    it, r = ctx.solve_tangent_cg(dev(b), out, tol=1e-8, maxit=4000)
    ref, it_ref, _ = cg(g, C, b, MASK, tol=1e-8, maxit=4000)
    assert abs(it - it_ref) <= 1 and r < 1e-8
    assert rel(out.cpu().numpy(), ref) <= 1e-6
    ctx.close()


def test_compact_cg_256_cube_vs_oracle():
    n = (256, 256, 256)
    g, cell, st, eps, ctx, b = damaged_plastic_cell(n, 6)
    C = oracle_tangent(cell, st, eps)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=2)
    ref, _, _ = cg(g, C, b, MASK, tol=0.0, maxit=2)
    assert rel(out.cpu().numpy(), ref) <= 1e-10
    ctx.close()


def device_cell(n, seed):
    """Same recipe generated on the device (512^3 does not fit the oracle's host arrays)."""
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    f64 = torch.float64
    ctx = Context((n, n, n), (float(n),) * 3)
    ph = (torch.rand((n, n, n), generator=gen, device="cuda", dtype=f64) < 0.2).to(torch.uint8)
    ctx.set_phases(ph, 2)
    ctx.set_material(0, Material.of(synth.MATRIX_J2))
    ctx.set_material(1, Material.of(synth.INCLUSION_EL))
    ctx.set_nonlocal(synth.CONFIG1_ELL, [0])
    ctx.set_control(MASK)
    ctx.set_field(_fgd.FIELD_HIST, torch.rand((n, n, n), generator=gen, device="cuda", dtype=f64) * 0.3)
    ctx.set_field(_fgd.FIELD_NONLOCAL, torch.rand((n, n, n), generator=gen, device="cuda", dtype=f64) * 0.02)
    eps = torch.randn((6, n, n, n), generator=gen, device="cuda", dtype=f64) * 5e-3
    ctx.constitutive(eps, None)
    del eps
    b = torch.empty((6, n, n, n), dtype=f64, device="cuda")
    ctx.mech_residual(np.zeros(6), b)          # a residual: in range(G*) by construction
    return ctx, b


@pytest.mark.parametrize("n", [256, 512])
def test_compact_cg_bitwise_and_vs_packed(n):
    ctx, b = device_cell(n, 11)
    x0 = torch.empty_like(b)
    ctx.solve_tangent_cg(b, x0, tol=0.0, maxit=10)
    x1 = torch.empty_like(b)
    for _ in range(2):
        ctx.solve_tangent_cg(b, x1, tol=0.0, maxit=10)
        assert torch.equal(x0, x1)
    ctx.solve_tangent_cg(b, x0, tol=0.0, maxit=6)
    Cp = torch.empty((21, n, n, n), dtype=torch.float64, device="cuda")
    ctx.get_field(_fgd.FIELD_TANGENT, Cp)          # expanded to the packed 21-component form
    ctx.set_tangent(Cp)                             # now the CG runs the packed instantiation
    del Cp
    torch.cuda.empty_cache()
    ctx.solve_tangent_cg(b, x1, tol=0.0, maxit=6)
    assert float(torch.linalg.vector_norm(x1 - x0) / torch.linalg.vector_norm(x0)) <= 1e-12
    ctx.close()
