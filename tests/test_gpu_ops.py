"""GPU parity: every operator apply of the C ABI against the oracle, element by element.

Bar (BASELINE.json north_star): relative L2 error <= 1e-10 on single operator and
preconditioner applications; Krylov solves are compared on solutions (1e-9) and iteration
counts.  Inputs are seeded (synth/), generated once and handed to both sides.
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

from oracle.helmholtz import apply_helmholtz, apply_precond, ell2_field, solve_helmholtz  # noqa: E402
from oracle.mech import apply_projected_tangent, cg, unpack21  # noqa: E402
from oracle.projection import apply_projection  # noqa: E402
from oracle.spectral import Grid  # noqa: E402
from paper_2103_04770_b200 import Context  # noqa: E402
from synth import bernoulli_phases, gaussian_field, random_spd_tangent  # noqa: E402

TOL_APPLY = 1e-10
GRIDS = [(8, 8, 8), (16, 8, 4), (32, 16, 8), (64, 32, 16), (16, 16, 1), (32, 64, 1), (4, 4, 2), (128, 128, 1),
         (512, 4, 4), (4, 512, 2), (4, 4, 512), (256, 256, 1)]
MASKS = [(1, 1, 0, 1, 1, 1), (0, 1, 0, 0, 0, 1), (0, 0, 0, 0, 0, 0), (1, 1, 1, 1, 1, 1)]


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def dev(x):
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def make_ctx(n, L=(1.0, 0.9, 1.1), scheme=1):
    L = (L[0], L[1], L[2] if n[2] > 1 else L[0] / n[0])
    return Context(n, L, scheme=scheme), Grid(n, L, "willot" if scheme == 1 else "continuous")


@pytest.mark.parametrize("n", GRIDS)
@pytest.mark.parametrize("scheme", [1, 0])
def test_projection(n, scheme):
    ctx, g = make_ctx(n, scheme=scheme)
    mask = MASKS[hash(n) % len(MASKS)]
    ctx.set_control(mask)
    tau = gaussian_field(6, g.shape, 1.0, 2)
    S = np.array([0.1, -0.2, 0.3, 0.05, 0.0, 0.02])
    y = ctx.apply_projection(dev(tau), S).cpu().numpy()
    ref = apply_projection(g, tau, mask, dc_mean_shift=S * np.array(mask))
    assert rel(y, ref) <= TOL_APPLY
    # host-pointer path
    yh = ctx.apply_projection(tau, S)
    assert rel(yh, ref) <= TOL_APPLY


@pytest.mark.parametrize("n", GRIDS)
def test_projected_tangent(n):
    ctx, g = make_ctx(n)
    mask = (1, 1, 0, 1, 1, 1)
    ctx.set_control(mask)
    Cp = random_spd_tangent(g.nvox, 1)
    ctx.set_tangent(dev(Cp))
    x = gaussian_field(6, g.shape, 1e-3, 2)
    y = ctx.apply_projected_tangent(dev(x)).cpu().numpy()
    ref = apply_projected_tangent(g, unpack21(Cp).reshape((6, 6) + g.shape), x, mask)
    assert rel(y, ref) <= TOL_APPLY


def helm_ctx(n, ell=(0.06, 0.12)):
    ctx, g = make_ctx(n)
    ph = bernoulli_phases(g.shape, 0.2, 0)
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(np.array([ell]), [0])
    return ctx, g, ph


@pytest.mark.parametrize("n", GRIDS)
def test_helmholtz_apply_and_precond(n):
    ctx, g, ph = helm_ctx(n)
    e2 = ell2_field(ph, [0.06, 0.12])
    a = gaussian_field(1, g.shape, 1e-3, 4)[0]
    y = ctx.apply_helmholtz(0, dev(a)).cpu().numpy()
    assert rel(y, apply_helmholtz(g, a, e2)) <= TOL_APPLY
    z = ctx.apply_helmholtz_precond(0, dev(a)).cpu().numpy()
    assert rel(z, apply_precond(g, a, e2)) <= TOL_APPLY


@pytest.mark.parametrize("n", [(16, 16, 16), (32, 32, 1), (64, 32, 8)])
def test_helmholtz_pcg(n):
    ctx, g, ph = helm_ctx(n, (0.08, 0.08 / 50))
    e2 = ell2_field(ph, [0.08, 0.08 / 50])
    src = np.random.default_rng(5).random(g.shape)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    it, rr = ctx.solve_helmholtz(0, dev(src), out, tol=1e-12, maxit=2000)
    ref, it_ref, _ = solve_helmholtz(g, src, e2, tol=1e-12, maxit=2000)
    assert abs(it - it_ref) <= 1
    assert rel(out.cpu().numpy(), ref) <= 1e-9
    # fixed-iteration mode: exactly maxit iterations, same iterate as the oracle's
    it5, _ = ctx.solve_helmholtz(0, dev(src), out, tol=0.0, maxit=5)
    ref5, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=5)
    assert it5 == 5
    assert rel(out.cpu().numpy(), ref5) <= 1e-10


@pytest.mark.parametrize("n", [(16, 16, 16), (32, 32, 1), (32, 16, 8)])
def test_mech_cg(n):
    ctx, g = make_ctx(n)
    mask = (1, 1, 0, 1, 1, 1)
    ctx.set_control(mask)
    Cp = random_spd_tangent(g.nvox, 3)
    ctx.set_tangent(dev(Cp))
    C = unpack21(Cp).reshape((6, 6) + g.shape)
    b = apply_projection(g, gaussian_field(6, g.shape, 1.0, 6), mask)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    it, rr = ctx.solve_tangent_cg(dev(b), out, tol=1e-12, maxit=3000)
    ref, it_ref, _ = cg(g, C, b, mask, tol=1e-12, maxit=3000)
    assert abs(it - it_ref) <= 1
    assert rel(out.cpu().numpy(), ref) <= 1e-9
    it7, _ = ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=7)
    ref7, _, _ = cg(g, C, b, mask, tol=0.0, maxit=7)
    assert it7 == 7 and rel(out.cpu().numpy(), ref7) <= 1e-10


def test_errors_and_edge_cases():
    from paper_2103_04770_b200 import FgdError
    with pytest.raises(FgdError):
        Context((12, 8, 8))                      # not a power of two
    ctx, g = make_ctx((8, 8, 8))
    with pytest.raises(FgdError):
        ctx.apply_helmholtz(0, dev(np.zeros(g.shape)))   # before set_phases
    ctx.set_control((0,) * 6)
    z = ctx.apply_projection(dev(np.zeros((6,) + g.shape))).cpu().numpy()
    assert np.all(z == 0)
    # constant field with all strain-controlled components: projection is exactly zero
    y = ctx.apply_projection(dev(np.ones((6,) + g.shape))).cpu().numpy()
    assert np.max(np.abs(y)) < 1e-15
