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
         (512, 4, 4), (4, 512, 2), (4, 4, 512), (256, 256, 1), (4, 4, 256), (8, 4, 128), (4, 8, 64), (16, 256, 4),
         (8, 16, 256), (16, 4, 256)]
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


@pytest.mark.parametrize("n", [(128, 128, 4), (128, 256, 2), (256, 128, 1), (128, 128, 64)])
def test_helmholtz_stencil_tensor_staging(n, monkeypatch):
    """Plane staging of the 27-point stencil by tensor-map TMA boxes (interior CTAs) mixed with the
    per-thread periodic-wrap copies (boundary CTAs), P:704-726 / R-HELM: grids with both kinds of CTA,
    a z extent that is not a multiple of the ring depth and the 2D case.  Against the oracle's Fourier
    form (apply, and PCG iterates), and bit for bit against the cp.async staging (same arithmetic)."""
    ctx, g, ph = helm_ctx(n)
    e2 = ell2_field(ph, [0.06, 0.12])
    a = gaussian_field(1, g.shape, 1e-3, 4)[0]
    src = np.random.default_rng(5).random(g.shape)
    out = {}
    for stage in ("2", "0"):
        monkeypatch.setenv("FGD_ST_STAGE", stage)
        y = ctx.apply_helmholtz(0, dev(a))
        x3 = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        it3, _ = ctx.solve_helmholtz(0, dev(src), x3, tol=0.0, maxit=3)
        assert it3 == 3
        out[stage] = (y, x3)
    assert rel(out["2"][0].cpu().numpy(), apply_helmholtz(g, a, e2)) <= TOL_APPLY
    ref3, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=3)
    assert rel(out["2"][1].cpu().numpy(), ref3) <= 1e-10
    assert torch.equal(out["2"][0], out["0"][0])
    assert torch.equal(out["2"][1], out["0"][1])


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


@pytest.mark.parametrize("n", [(256, 8, 8), (512, 4, 8), (8, 256, 256), (4, 512, 8), (4, 8, 512)])
def test_krylov_iterates_specialised_sizes(n):
    """Fixed-iteration CG and PCG iterates at sizes that select the 256/512-point specialisations:
    bulk-copy tangent/PCG x passes with register FFTs (N1 = 256, 512), register y/z FFTs (N2, N3 =
    256 or 512), the register x-inverse epilogue (N1 = 256), the first-step CG path (no r = b copy)."""
    ctx, g = make_ctx(n)
    mask = (1, 1, 0, 1, 1, 1)
    ctx.set_control(mask)
    Cp = random_spd_tangent(g.nvox, 8)
    ctx.set_tangent(dev(Cp))
    C = unpack21(Cp).reshape((6, 6) + g.shape)
    b = apply_projection(g, gaussian_field(6, g.shape, 1.0, 9), mask)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    for k in (1, 2, 6):
        it, _ = ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=k)
        ref, _, _ = cg(g, C, b, mask, tol=0.0, maxit=k)
        assert it == k and rel(out.cpu().numpy(), ref) <= 1e-10, k
    ph = bernoulli_phases(g.shape, 0.25, 3)
    ctx.set_phases(dev(ph), 2)
    ell = [0.05, 0.001]
    ctx.set_nonlocal(np.array([ell]), [0])
    e2 = ell2_field(ph, ell)
    src = np.random.default_rng(8).random(g.shape)
    o = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    it, _ = ctx.solve_helmholtz(0, dev(src), o, tol=0.0, maxit=4)
    ref4, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=4)
    assert it == 4 and rel(o.cpu().numpy(), ref4) <= 1e-10


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


@pytest.mark.parametrize("n", [128, 256])
def test_full_size_operators_256(n):
    """The config-1 sizes (128^3, and 256^3 of the bench's by_size line) in the launch configuration
    bench.py times.  Projected tangent: at sampled frequencies xi the oracle evaluates, one by one,
    F(y)(xi) = G^*(xi) F(C:x)(xi) (explicit separable DFT sums of the inputs and of the GPU output),
    and then every voxel against the oracle's full apply; Helmholtz apply and preconditioner: every
    voxel against the oracle."""
    import synth
    from oracle.projection import project_spectrum
    from oracle.spectral import cis
    g = Grid((n, n, n), (float(n),) * 3)
    ctx = Context((n, n, n), (float(n),) * 3)
    mask = synth.CONFIG1_MASK
    ctx.set_control(mask)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(7)
    Cd = synth.random_spd_tangent_torch(g.nvox, 1, device="cuda")
    ctx.set_tangent(Cd)
    x = torch.randn((6,) + g.shape, generator=gen, dtype=torch.float64, device="cuda") * 1e-3
    y = ctx.apply_projected_tangent(x)
    # tau = C : x on the device (test infrastructure), then DFT samples on the host
    from oracle.mech import PACKED21
    tau = torch.zeros_like(x)
    for t, (i, j) in enumerate(PACKED21):
        cij = Cd[t].reshape(g.shape)
        tau[i] += cij * x[j]
        if i != j:
            tau[j] += cij * x[i]
    ks = g.symbol(half=True)
    rng = np.random.default_rng(3)
    samples = [(0, 0, 0), (n // 2, 0, 0), (0, n // 2, n // 2), (1, 2, 3)] + \
              [tuple(int(v) for v in rng.integers(0, (n // 2 + 1, n, n))) for _ in range(6)]
    idx = torch.arange(n, device="cuda", dtype=torch.float64)
    for (kx, ky, kz) in samples:
        ex = torch.exp(-2j * np.pi * kx * idx / n)
        ey = torch.exp(-2j * np.pi * ky * idx / n)
        ez = torch.exp(-2j * np.pi * kz * idx / n)
        ft = torch.einsum("czyx,x,y,z->c", tau.to(torch.complex128), ex, ey, ez).cpu().numpy()
        fy = torch.einsum("czyx,x,y,z->c", y.to(torch.complex128), ex, ey, ez).cpu().numpy()
        k = ks[:, kz, ky, kx]
        # batch of two frequencies: a dummy DC slot (index 0) and the sample, unless it is DC
        if (kx, ky, kz) == (0, 0, 0):
            ref = np.asarray(mask) * ft
        else:
            ref = project_spectrum(np.stack([np.zeros(6), ft], 1), np.stack([np.zeros(3), k], 1), mask,
                                   dc_index=(0,))[:, 1]
        scale = max(np.linalg.norm(ft), 1e-300)
        assert np.linalg.norm(fy - ref) <= 1e-10 * scale, (kx, ky, kz)
    del tau
    # and every voxel: the oracle's projected tangent on the whole field (the unpacked 6x6
    # tangent is 4.8 GB of host memory at 256^3)
    Cn = unpack21(Cd.cpu().numpy()).reshape((6, 6) + g.shape)
    del Cd
    ref_full = apply_projected_tangent(g, Cn, x.cpu().numpy(), mask)
    del Cn
    assert rel(y.cpu().numpy(), ref_full) <= TOL_APPLY
    del ref_full
    ph = synth.config1_phases(n, 0)
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(synth.CONFIG1_ELL, [0])
    e2 = ell2_field(ph, synth.CONFIG1_ELL[0])
    a = x[0].cpu().numpy()
    ya = ctx.apply_helmholtz(0, x[0].contiguous()).cpu().numpy()
    assert rel(ya, apply_helmholtz(g, a, e2)) <= TOL_APPLY
    za = ctx.apply_helmholtz_precond(0, x[0].contiguous()).cpu().numpy()
    assert rel(za, apply_precond(g, a, e2)) <= TOL_APPLY


def _dft_sample(f, kx, ky, kz, n):
    """F(f)(xi) of a (C, Nz, Ny, Nx) device field at one frequency (explicit separable DFT sums)."""
    idx = torch.arange(n, device="cuda", dtype=torch.float64)
    ex = torch.exp(-2j * np.pi * kx * idx / n)
    ey = torch.exp(-2j * np.pi * ky * idx / n)
    ez = torch.exp(-2j * np.pi * kz * idx / n)
    out = []
    for c in range(f.shape[0]):
        out.append(torch.einsum("zyx,x,y,z->", f[c].to(torch.complex128), ex, ey, ez).item())
    return np.array(out)


def test_full_size_operators_512():
    """BASELINE's 512^3 metric size, in the launch configuration bench.py --size 512 times (bulk-copy
    tangent pass with 256-thread CTAs, 8x8x8 register y/z FFTs).  At sampled frequencies the oracle's
    per-frequency operators are checked against explicit DFT sums of the GPU input and output:
    projected tangent F(y) = G^*(xi) F(C:x); preconditioner F(z) = F(r) / (1 + <l^2>|k|^2);
    Helmholtz apply with uniform l: F(L a) = (1 + l^2 |k|^2) F(a) (c6 closed form)."""
    import synth
    from oracle.projection import project_spectrum
    from oracle.mech import PACKED21
    n = 512
    g = Grid((n, n, n), (float(n),) * 3)
    ctx = Context((n, n, n), (float(n),) * 3)
    mask = synth.CONFIG1_MASK
    ctx.set_control(mask)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(11)
    Cd = synth.random_spd_tangent_torch(g.nvox, 5, device="cuda")
    ctx.set_tangent(Cd)
    x = torch.randn((6,) + g.shape, generator=gen, dtype=torch.float64, device="cuda") * 1e-3
    y = ctx.apply_projected_tangent(x)
    tau = torch.zeros_like(x)
    for t, (i, j) in enumerate(PACKED21):
        cij = Cd[t].reshape(g.shape)
        tau[i] += cij * x[j]
        if i != j:
            tau[j] += cij * x[i]
    del Cd
    ks = g.symbol(half=True)
    rng = np.random.default_rng(5)
    samples = [(0, 0, 0), (n // 2, 0, 0), (0, n // 2, n // 2), (3, 1, 2)] + \
              [tuple(int(v) for v in rng.integers(0, (n // 2 + 1, n, n))) for _ in range(3)]
    for (kx, ky, kz) in samples:
        ft = _dft_sample(tau, kx, ky, kz, n)
        fy = _dft_sample(y, kx, ky, kz, n)
        if (kx, ky, kz) == (0, 0, 0):
            ref = np.asarray(mask) * ft
        else:
            k = ks[:, kz, ky, kx]
            ref = project_spectrum(np.stack([np.zeros(6), ft], 1), np.stack([np.zeros(3), k], 1), mask,
                                   dc_index=(0,))[:, 1]
        assert np.linalg.norm(fy - ref) <= 1e-10 * max(np.linalg.norm(ft), 1e-300), (kx, ky, kz)
    del tau, y
    # Helmholtz: one phase, l = 3 (uniform) -> diagonal symbols
    ell = 3.0
    ctx.set_phases(torch.zeros(g.shape, dtype=torch.uint8, device="cuda"), 2)
    ctx.set_nonlocal(np.array([[ell, ell]]), [0])
    a = x[0].contiguous()
    ya = ctx.apply_helmholtz(0, a)
    za = ctx.apply_helmholtz_precond(0, a)
    for (kx, ky, kz) in samples:
        fa = _dft_sample(a[None], kx, ky, kz, n)[0]
        k = ks[:, kz, ky, kx]
        sym = 1.0 + ell * ell * float(np.sum(np.abs(k) ** 2))
        assert abs(_dft_sample(ya[None], kx, ky, kz, n)[0] - sym * fa) <= 1e-10 * max(abs(fa) * sym, 1e-300)
        assert abs(_dft_sample(za[None], kx, ky, kz, n)[0] - fa / sym) <= 1e-10 * max(abs(fa), 1e-300)


@pytest.mark.parametrize("n", [(16, 8, 16), (8, 8, 256), (4, 512, 8), (4, 8, 512)])
@pytest.mark.parametrize("P", [2, 4])
def test_emulated_slab_layout(P, n, monkeypatch):
    """Multi-GPU transposition layout (S[r][s] -> R[s][r] block all-to-all, y-slab z pass)
    emulated on one GPU with FGD_EMULATE_SLABS=P: projection, projected tangent, precond,
    CG and PCG must equal the oracle exactly as in the single-slab layout."""
    monkeypatch.setenv("FGD_EMULATE_SLABS", str(P))
    ctx, g = make_ctx(n)
    mask = (1, 1, 0, 1, 1, 1)
    ctx.set_control(mask)
    tau = gaussian_field(6, g.shape, 1.0, 12)
    assert rel(ctx.apply_projection(dev(tau)).cpu().numpy(), apply_projection(g, tau, mask)) <= TOL_APPLY
    Cp = random_spd_tangent(g.nvox, 4)
    ctx.set_tangent(dev(Cp))
    C = unpack21(Cp).reshape((6, 6) + g.shape)
    x = gaussian_field(6, g.shape, 1e-3, 13)
    assert rel(ctx.apply_projected_tangent(dev(x)).cpu().numpy(),
               apply_projected_tangent(g, C, x, mask)) <= TOL_APPLY
    b = apply_projection(g, gaussian_field(6, g.shape, 1.0, 14), mask)
    out = torch.empty((6,) + g.shape, dtype=torch.float64, device="cuda")
    ctx.solve_tangent_cg(dev(b), out, tol=0.0, maxit=6)
    ref, _, _ = cg(g, C, b, mask, tol=0.0, maxit=6)
    assert rel(out.cpu().numpy(), ref) <= 1e-10
    ph = bernoulli_phases(g.shape, 0.3, 2)
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(np.array([[0.1, 0.002]]), [0])
    e2 = ell2_field(ph, [0.1, 0.002])
    a = gaussian_field(1, g.shape, 1.0, 15)[0]
    assert rel(ctx.apply_helmholtz_precond(0, dev(a)).cpu().numpy(), apply_precond(g, a, e2)) <= TOL_APPLY
    o1 = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    ctx.solve_helmholtz(0, dev(np.abs(a)), o1, tol=0.0, maxit=5)
    ref5, _, _ = solve_helmholtz(g, np.abs(a), e2, tol=0.0, maxit=5)
    assert rel(o1.cpu().numpy(), ref5) <= 1e-10


@pytest.mark.parametrize("scheme", [1, 0])
def test_cluster_fused_precond(scheme, monkeypatch):
    """Opt-in cluster/DSMEM kernel (FGD_YZY=1) fusing the y, z (preconditioner) and inverse-y passes
    of the one-component spectrum (N2 = N3 = 256): preconditioner apply and PCG iterates vs oracle."""
    monkeypatch.setenv("FGD_YZY", "1")
    n = (8, 256, 256)
    g = Grid(n, (1.0, 1.0, 1.0))
    ctx = Context(n, (1.0, 1.0, 1.0), scheme=scheme)
    ph = bernoulli_phases(g.shape, 0.3, 4)
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(np.array([[0.03, 0.006]]), [0])
    e2 = ell2_field(ph, [0.03, 0.006])
    gs = Grid(n, (1.0, 1.0, 1.0), scheme="continuous") if scheme == 0 else g
    a = gaussian_field(1, g.shape, 1.0, 21)[0]
    assert rel(ctx.apply_helmholtz_precond(0, dev(a)).cpu().numpy(), apply_precond(gs, a, e2)) <= TOL_APPLY
    if scheme == 1:
        o = torch.empty(g.shape, dtype=torch.float64, device="cuda")
        ctx.solve_helmholtz(0, dev(np.abs(a)), o, tol=0.0, maxit=4)
        ref, _, _ = solve_helmholtz(g, np.abs(a), e2, tol=0.0, maxit=4)
        assert rel(o.cpu().numpy(), ref) <= 1e-10


@pytest.mark.parametrize("n", [(8, 16, 256), (4, 8, 256)])
def test_factorised_z_projection(n, monkeypatch):
    """Opt-in factorised z pass (FGD_ZFAC=1: Willot symbol k_j = A_j m_j(kz), 3 transformed components
    each way): projection with a stress-mask DC and projected tangent against the oracle."""
    monkeypatch.setenv("FGD_ZFAC", "1")
    for mask in [(1, 1, 0, 1, 1, 1), (0, 1, 0, 0, 0, 1)]:
        ctx, g = make_ctx(n)
        ctx.set_control(mask)
        tau = gaussian_field(6, g.shape, 1.0, 31)
        S = np.array([0.3, -0.2, 0.1, 0.05, 0.0, -0.4])
        y = ctx.apply_projection(dev(tau), S).cpu().numpy()
        assert rel(y, apply_projection(g, tau, mask, dc_mean_shift=S)) <= TOL_APPLY
        Cp = random_spd_tangent(g.nvox, 2)
        ctx.set_tangent(dev(Cp))
        x = gaussian_field(6, g.shape, 1e-3, 32)
        yt = ctx.apply_projected_tangent(dev(x)).cpu().numpy()
        assert rel(yt, apply_projected_tangent(g, unpack21(Cp).reshape((6, 6) + g.shape), x, mask)) <= TOL_APPLY


@pytest.mark.parametrize("n", [256, 512])
def test_full_size_run_to_run_bitwise(n):
    """Every kernel on the path reduces in a fixed order, so repeated applies on the same input
    must agree BIT FOR BIT.  A shared-memory race (e.g. a line buffer restaged while another
    plane's warps still exchange through it) shows up here as run-to-run differences long
    before a sampled-frequency parity check happens to hit a corrupted line: at 512^3 the
    y-inverse pass once restaged its line buffers after a per-plane named barrier only and
    corrupted ~2000 z-lines per apply."""
    import synth
    ctx = Context((n, n, n), (float(n),) * 3)
    ctx.set_control(synth.CONFIG1_MASK)
    gen = torch.Generator(device="cuda")
    gen.manual_seed(3)
    ctx.set_tangent(synth.random_spd_tangent_torch(n ** 3, 7, device="cuda"))
    x = torch.randn((6, n, n, n), generator=gen, dtype=torch.float64, device="cuda") * 1e-3
    y0 = ctx.apply_projected_tangent(x)
    for _ in range(4):
        assert torch.equal(ctx.apply_projected_tangent(x), y0)
    p0 = ctx.apply_projection(x)
    for _ in range(3):
        assert torch.equal(ctx.apply_projection(x), p0)
    del y0, p0
    ph = (torch.rand((n, n, n), generator=gen, device="cuda", dtype=torch.float64) < 0.2).to(torch.uint8)
    ctx.set_phases(ph, 2)
    ctx.set_nonlocal(np.array([[2.0, 4.0]]), [0])
    a = x[0].contiguous()
    z0 = ctx.apply_helmholtz_precond(0, a)
    h0 = ctx.apply_helmholtz(0, a)
    for _ in range(4):
        assert torch.equal(ctx.apply_helmholtz_precond(0, a), z0)
        assert torch.equal(ctx.apply_helmholtz(0, a), h0)


@pytest.mark.parametrize("n", [(8, 8, 8), (16, 8, 4), (32, 16, 1), (64, 32, 16), (8, 16, 256), (4, 8, 512)])
def test_helmholtz_continuous_scheme(n):
    """Continuous scheme (k_j = i xi_j, Nyquist zeroed, A-06): the Helmholtz operator in its Fourier
    form (two 3-component FFT round trips, helm_fourier) and the preconditioner against the oracle's
    Fourier form, and PCG iterates (Algorithm 2) after a fixed number of iterations."""
    L = (1.0, 0.9, 1.1 if n[2] > 1 else 1.0 / n[0])
    g = Grid(n, L, "continuous")
    ctx = Context(n, L, scheme=0)
    ph = bernoulli_phases(g.shape, 0.3, 31)
    ell = [0.08, 0.02]
    ctx.set_phases(dev(ph), 2)
    ctx.set_nonlocal(np.array([ell]), [0])
    e2 = ell2_field(ph, ell)
    a = gaussian_field(1, g.shape, 1.0, 32)[0]
    assert rel(ctx.apply_helmholtz(0, dev(a)).cpu().numpy(), apply_helmholtz(g, a, e2)) <= TOL_APPLY
    assert rel(ctx.apply_helmholtz_precond(0, dev(a)).cpu().numpy(), apply_precond(g, a, e2)) <= TOL_APPLY
    src = np.abs(a)
    out = torch.empty(g.shape, dtype=torch.float64, device="cuda")
    ctx.solve_helmholtz(0, dev(src), out, tol=0.0, maxit=4)
    ref, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=4)
    assert rel(out.cpu().numpy(), ref) <= 1e-10
    it, _ = ctx.solve_helmholtz(0, dev(src), out, tol=1e-10, maxit=500)
    ref, it_ref, _ = solve_helmholtz(g, src, e2, tol=1e-10, maxit=500)
    assert abs(it - it_ref) <= 1 and rel(out.cpu().numpy(), ref) <= 1e-8
    ctx.close()
