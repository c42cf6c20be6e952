"""Multi-rank code paths of libfgd (nranks > 1) on ONE GPU through the loopback transport
(fgd_loopback_id, dist.cu): P contexts, one host thread each, every field argument the rank's
z-slab.  Everything that differs from the single-rank library runs here -- the slab layout of the
transposed spectra with the rank's ky offset and local y-slab (Nyl = Ny / P), the zero frequency on
rank 0 only, the block all-to-all transposes, the Helmholtz stencil z-halos (inputs, previous
directions, phase ids), the distributed reductions (local partial -> allreduce -> one-thread
finalise, with the convergence guard), the allreduce-max of the ERR bit patterns and the batched
Krylov loops -- except the NCCL calls themselves, which the loopback replaces by the same block
moves (device-to-device copies ordered by events and host barriers; no kernel waits on another).

Reference: the oracle on the whole cell (the gathered slabs), at the single-apply bar 1e-10,
Krylov iterates 1e-10 after fixed iteration counts, converged solves within their tolerance, and
one staggered increment at the increment bar (<sigma> 1e-6).
"""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

import synth  # noqa: E402
from oracle.helmholtz import apply_helmholtz, apply_precond, ell2_field, solve_helmholtz  # noqa: E402
from oracle.increment import State, Tolerances, make_cell, solve_increment  # noqa: E402
from oracle.mech import apply_projected_tangent, cg, unpack21  # noqa: E402
from oracle.projection import apply_projection  # noqa: E402
from oracle.spectral import Grid  # noqa: E402
from paper_2103_04770_b200 import Context, Material, loopback_id  # noqa: E402
from synth import bernoulli_phases, gaussian_field, random_spd_tangent  # noqa: E402

MASK = (1, 1, 0, 1, 1, 1)


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(np.asarray(b)), 1e-300))


def run_ranks(P, n, L, body):
    """Run body(rank, ctx, z0, nz) on P loopback ranks (one thread and one stream each); returns the
    per-rank results in rank order.  Any exception in a rank is re-raised."""
    lid = loopback_id()
    out = [None] * P
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = Context(n, L, rank=r, nranks=P, nccl_id=lid, stream=s.cuda_stream)
                try:
                    z0, nz = ctx.z0, ctx.nz
                    out[r] = body(r, ctx, z0, nz)
                    s.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:   # noqa: BLE001
            errs.append((r, e))

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    assert not any(t.is_alive() for t in th), "loopback ranks hung"
    if errs:
        raise errs[0][1]
    return out


def slab(a, z0, nz):
    """z-slab [.., z0:z0+nz, :, :] of a numpy field (z is the third-last axis), on the device."""
    return torch.from_numpy(np.ascontiguousarray(a[..., z0:z0 + nz, :, :])).cuda()


def gather(parts):
    return np.concatenate(parts, axis=-3)


GRIDS = [(2, (16, 8, 8)), (4, (16, 8, 8)), (2, (32, 16, 16)), (4, (8, 32, 32)), (2, (256, 8, 8)),
         (2, (16, 256, 256)), (4, (8, 512, 512))]


@pytest.mark.parametrize("overlap", ["1", "4", "3", "peer"])
@pytest.mark.parametrize("P,n", GRIDS)
def test_loopback_operators(P, n, overlap, monkeypatch):
    """Projection (with a stress-controlled macroscopic shift on rank 0's zero frequency), projected
    tangent, Helmholtz apply (z-halos) and preconditioner on P ranks vs the oracle on the cell, with
    the monolithic transposes (FGD_OVERLAP=1) and the kx-chunked round trip overlapped on a second
    stream (4 and 3 chunks)."""
    if overlap == "peer":
        # peer-store transposes (NEXT#4): the y passes write to / read from the peers' z-pass buffers
        monkeypatch.setenv("FGD_PEER", "1")
    else:
        monkeypatch.setenv("FGD_OVERLAP", overlap)
    L = (1.0, 0.9, 1.1)
    g = Grid(n, L)
    tau = gaussian_field(6, g.shape, 1.0, 2)
    S = np.array([0.1, -0.2, 0.3, 0.05, 0.0, 0.02])
    Cp = random_spd_tangent(g.nvox, 4).reshape((21,) + g.shape)
    x = gaussian_field(6, g.shape, 1e-3, 5)
    ph = bernoulli_phases(g.shape, 0.3, 6)
    ell = np.array([[0.1, 0.02]])
    a = gaussian_field(1, g.shape, 1.0, 7)[0]

    def body(r, ctx, z0, nz):
        ctx.set_control(MASK)
        yp = ctx.apply_projection(slab(tau, z0, nz), S).cpu().numpy()
        ctx.set_tangent(slab(Cp, z0, nz))
        yt = ctx.apply_projected_tangent(slab(x, z0, nz)).cpu().numpy()
        ctx.set_phases(slab(ph, z0, nz), 2)
        ctx.set_nonlocal(ell, [0])
        yh = ctx.apply_helmholtz(0, slab(a, z0, nz)).cpu().numpy()
        yz = ctx.apply_helmholtz_precond(0, slab(a, z0, nz)).cpu().numpy()
        return yp, yt, yh, yz

    res = run_ranks(P, n, L, body)
    e2 = ell2_field(ph, ell[0])
    assert rel(gather([r[0] for r in res]), apply_projection(g, tau, MASK, dc_mean_shift=S * np.array(MASK))) <= 1e-10
    C = unpack21(Cp.reshape(21, -1)).reshape((6, 6) + g.shape)
    assert rel(gather([r[1] for r in res]), apply_projected_tangent(g, C, x, MASK)) <= 1e-10
    assert rel(gather([r[2] for r in res]), apply_helmholtz(g, a, e2)) <= 1e-10
    assert rel(gather([r[3] for r in res]), apply_precond(g, a, e2)) <= 1e-10


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("P,n", [(2, (16, 8, 8)), (4, (32, 16, 16)), (2, (256, 8, 8)), (2, (16, 256, 256))])
def test_loopback_krylov(P, n, peer, monkeypatch):
    """Mechanical CG and Helmholtz PCG on P ranks: iterates after a fixed number of iterations
    (distributed finalise) and converged solves (batched loops with the device guard: the
    same iteration count on every rank and +-1 of the oracle's); with the NCCL-style transposes and
    with the peer-store transposes (FGD_PEER=1, NEXT#4)."""
    if peer:
        monkeypatch.setenv("FGD_PEER", "1")
    L = (1.0, 1.0, 1.0)
    g = Grid(n, L)
    Cp = random_spd_tangent(g.nvox, 8).reshape((21,) + g.shape)
    C = unpack21(Cp.reshape(21, -1)).reshape((6, 6) + g.shape)
    b = apply_projection(g, gaussian_field(6, g.shape, 1.0, 9), MASK)
    ph = bernoulli_phases(g.shape, 0.25, 10)
    ell = np.array([[0.08, 0.01]])
    src = np.abs(gaussian_field(1, g.shape, 1.0, 11)[0])

    def body(r, ctx, z0, nz):
        ctx.set_control(MASK)
        ctx.set_tangent(slab(Cp, z0, nz))
        o6 = torch.empty((6, nz) + g.shape[1:], dtype=torch.float64, device="cuda")
        ctx.solve_tangent_cg(slab(b, z0, nz), o6, tol=0.0, maxit=6)
        cg6 = o6.cpu().numpy()
        itc, relc = ctx.solve_tangent_cg(slab(b, z0, nz), o6, tol=1e-9, maxit=3000)
        cgc = o6.cpu().numpy()
        ctx.set_phases(slab(ph, z0, nz), 2)
        ctx.set_nonlocal(ell, [0])
        o1 = torch.empty((nz,) + g.shape[1:], dtype=torch.float64, device="cuda")
        ctx.solve_helmholtz(0, slab(src, z0, nz), o1, tol=0.0, maxit=5)
        h5 = o1.cpu().numpy()
        ith, relh = ctx.solve_helmholtz(0, slab(src, z0, nz), o1, tol=1e-10, maxit=3000)
        hc = o1.cpu().numpy()
        return cg6, (itc, relc), cgc, h5, (ith, relh), hc

    res = run_ranks(P, n, L, body)
    ref6, _, _ = cg(g, C, b, MASK, tol=0.0, maxit=6)
    assert rel(gather([r[0] for r in res]), ref6) <= 1e-10
    refc, itc, _ = cg(g, C, b, MASK, tol=1e-9, maxit=3000)
    its = {r[1][0] for r in res}
    assert len(its) == 1 and abs(its.pop() - itc) <= 1
    assert all(r[1][1] < 1e-9 for r in res)
    assert rel(gather([r[2] for r in res]), refc) <= 1e-7
    e2 = ell2_field(ph, ell[0])
    ref5, _, _ = solve_helmholtz(g, src, e2, tol=0.0, maxit=5)
    assert rel(gather([r[3] for r in res]), ref5) <= 1e-10
    refh, ith, _ = solve_helmholtz(g, src, e2, tol=1e-10, maxit=3000)
    its = {r[4][0] for r in res}
    assert len(its) == 1 and abs(its.pop() - ith) <= 1
    assert rel(gather([r[5] for r in res]), refh) <= 1e-8


@pytest.mark.parametrize("peer", [False, True])
@pytest.mark.parametrize("P", [2, 4])
def test_loopback_increments(P, peer, monkeypatch):
    if peer:
        monkeypatch.setenv("FGD_PEER", "1")
    _loopback_increments(P)


def _loopback_increments(P):
    """Two staggered increments (Algorithm 1) of a 16^3 config-3-type cell (brittle spheres in a
    J2-Lemaitre matrix, two non-local fields) on P ranks: <sigma> and the committed fields against the
    oracle (distributed <sigma>, ERR with the allreduce-max of the strain-change bit patterns)."""
    cfg = synth.config3(n=16, n_spheres=4, phi=0.2, seed=3)
    cfg.dE = 2.0e-3     # plastic from the first increment
    tol = Tolerances(tol_stag=1e-9, tol_newton=1e-10, tol_cg=1e-11, tol_helm=1e-11)
    cell = make_cell(cfg)
    st = State.zero(cell)
    refs = []
    for i in (1, 2):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), tol)
        assert rep.converged
        refs.append(rep.macro_stress.copy())

    def body(r, ctx, z0, nz):
        ctx.set_phases(slab(cfg.phases, z0, nz), len(cfg.materials))
        for q, m in enumerate(cfg.materials):
            ctx.set_material(q, Material.of(m))
        ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
        ctx.set_control(cfg.stress_mask)
        got = []
        for i in (1, 2):
            Et = np.zeros(6)
            Et[cfg.load_comp] = i * cfg.dE
            s, rp = ctx.solve_increment(Et, np.zeros(6), tol.tol_stag, tol.tol_newton, tol.tol_cg, tol.tol_helm,
                                        tol.max_stag, tol.max_newton, tol.max_cg, tol.max_helm)
            assert s == 0, rp
            got.append(rp)
        from paper_2103_04770_b200 import _fgd
        f = torch.empty((nz,) + tuple(cfg.phases.shape[1:]), dtype=torch.float64, device="cuda")
        ctx.get_field(_fgd.FIELD_EQPS, f)
        ep = f.cpu().numpy()
        ctx.get_field(_fgd.FIELD_NONLOCAL + 1, f)
        a1 = f.cpu().numpy()
        return got, ep, a1

    res = run_ranks(P, cfg.n, cfg.L, body)
    for i in range(2):
        for r in range(P):
            assert rel(res[r][0][i]["macro_stress"], refs[i]) <= 1e-6, (i, r)
        assert len({res[r][0][i]["stag"] for r in range(P)}) == 1
    assert st.ep.max() > 0.0
    assert np.abs(gather([r[1] for r in res]).reshape(-1) - st.ep).max() <= 1e-8
    assert rel(gather([r[2] for r in res]), st.abar[1]) <= 1e-6


@pytest.mark.parametrize("P,n", [(2, (16, 8, 8)), (4, (8, 32, 32)), (2, (16, 256, 256))])
def test_loopback_continuous_helmholtz(P, n):
    """The Fourier-form Helmholtz operator (continuous scheme: two 3-component FFT round trips with
    the slab transposes) and its PCG on P ranks vs the oracle's Fourier form."""
    L = (1.0, 0.9, 1.1)
    g = Grid(n, L, "continuous")
    ph = bernoulli_phases(g.shape, 0.3, 41)
    ell = np.array([[0.08, 0.02]])
    a = gaussian_field(1, g.shape, 1.0, 42)[0]

    def body(r, ctx, z0, nz):
        ctx.set_phases(slab(ph, z0, nz), 2)
        ctx.set_nonlocal(ell, [0])
        yh = ctx.apply_helmholtz(0, slab(a, z0, nz)).cpu().numpy()
        o1 = torch.empty((nz,) + g.shape[1:], dtype=torch.float64, device="cuda")
        ctx.solve_helmholtz(0, slab(np.abs(a), z0, nz), o1, tol=0.0, maxit=4)
        return yh, o1.cpu().numpy()

    lid = loopback_id()
    out = [None] * P
    errs = []

    def worker(r):
        try:
            torch.cuda.set_device(0)
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                ctx = Context(n, L, scheme=0, rank=r, nranks=P, nccl_id=lid, stream=s.cuda_stream)
                try:
                    out[r] = body(r, ctx, ctx.z0, ctx.nz)
                    s.synchronize()
                finally:
                    ctx.close()
        except BaseException as e:   # noqa: BLE001
            errs.append(e)

    th = [threading.Thread(target=worker, args=(r,)) for r in range(P)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=900)
    if errs:
        raise errs[0]
    e2 = ell2_field(ph, ell[0])
    assert rel(gather([o[0] for o in out]), apply_helmholtz(g, a, e2)) <= 1e-10
    ref, _, _ = solve_helmholtz(g, np.abs(a), e2, tol=0.0, maxit=4)
    assert rel(gather([o[1] for o in out]), ref) <= 1e-10


def test_loopback_increments_warm_start():
    """Two staggered increments on 2 ranks with warm-started Helmholtz PCG on both sides (R-WARM)."""
    cfg = synth.config3(n=16, n_spheres=4, phi=0.2, seed=3)
    cfg.dE = 2.0e-3
    tol = Tolerances(tol_stag=1e-9, tol_newton=1e-10, tol_cg=1e-11, tol_helm=1e-11, warm_start=True)
    cell = make_cell(cfg)
    st = State.zero(cell)
    refs = []
    for i in (1, 2):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), tol)
        assert rep.converged
        refs.append(rep.macro_stress.copy())

    def body(r, ctx, z0, nz):
        ctx.set_phases(slab(cfg.phases, z0, nz), len(cfg.materials))
        for q, m in enumerate(cfg.materials):
            ctx.set_material(q, Material.of(m))
        ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
        ctx.set_control(cfg.stress_mask)
        got = []
        for i in (1, 2):
            Et = np.zeros(6)
            Et[cfg.load_comp] = i * cfg.dE
            s, rp = ctx.solve_increment(Et, np.zeros(6), tol.tol_stag, tol.tol_newton, tol.tol_cg, tol.tol_helm,
                                        tol.max_stag, tol.max_newton, tol.max_cg, tol.max_helm, warm_start=True)
            assert s == 0, rp
            got.append(rp["macro_stress"])
        return got

    res = run_ranks(2, cfg.n, cfg.L, body)
    for i in range(2):
        for r in range(2):
            assert rel(res[r][i], refs[i]) <= 1e-6, (i, r)
