"""One load increment: mixed-control Newton + Algorithm 1 iterative staggered scheme
(paper Sec. 3.2).

TEST INFRASTRUCTURE (see oracle/__init__.py).

Step by step (readings A-01, A-02, A-07, A-16, A-20-A-22, A-28):
 1. eps^(0) = eps_n + dE, dE applied uniformly on the strain-controlled components
    (dE_c = E_target_c - <eps_n>_c); abar^(0) = abar_n  (A-22).
 2. staggered loop k (iterate UNTIL ERR < TOL_s, A-01):
    a. damage frozen from abar^(k): D = max(D_n, D(abar_m)) (J2 phases), kappa = max(kappa_n,
       abar_p), d = d(kappa) (brittle phases) (A-16, A-18)
    b. Newton r: sigma, C = point update(eps); b = -G*(sigma - Sigma_bar);
       stop if rms(b) < tol_N * max(|<sigma>|, 1e-6 sigma_ref); else CG (mech.cg) and eps += de;
       with Tolerances.line_search (reading R-LS) a step that does not lower rms(b) is halved
       (eps -= lam de, lam = 1/2, 1/4, ..., at most max_backtrack times) before the next CG
    c. alpha_j from the converged point update (A-28): eps_p (J2), eps_eq (brittle), 0 outside
       the source phase
    d. abar_j^(k+1) = Algorithm 2 (helmholtz.solve_helmholtz) for every field j, from
       abar^(0) = 0 as printed, or from abar_j^(k) with Tolerances.warm_start
    e. ERR = max( max_{x,ij}|eps^(k+1) - eps^(k)| / |<eps^(k+1)>|,
                  ||abar_j^(k+1) - abar_j^(k)|| / ||abar_j^(k+1)|| )  (A-02; tensor
       components, Frobenius norm of the mean; denominators < 1e-12 -> absolute term)
 3. commit: eps_n, eps^p_n, eps_p,n <- converged; D_n <- max(D_n, D(abar)); kappa_n <- max(kappa_n,
    abar_p); abar_n <- abar (A-16).
Returns the macroscopic stress <sigma> of the last mechanical solve and <eps>.

Pins (tests/test_oracle_increment.py): homogeneous cell -> uniform fields equal to a 1-voxel
material-point mixed-control Newton; elastic closed forms E*E11 (3D uniaxial stress) and
E/(1-nu^2)*E11 (plane strain); laminate closed form; equilibrium conj(k).sigma^ = 0 and
compatibility at convergence; elastic path independence; re-solving a converged increment is
a fixed point; elastic cell -> ERR = 0 at the 2nd staggered iteration.
Full post-peak load curves: parity unpinned against the paper (no data, A-27).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import gtn as gtn_
from . import material as mat_
from .helmholtz import ell2_field, solve_helmholtz
from .mech import cg
from .projection import apply_projection
from .spectral import Grid

S2 = np.sqrt(2.0)


@dataclass
class Tolerances:
    tol_stag: float = 1e-8
    tol_newton: float = 1e-10
    tol_cg: float = 1e-11
    tol_helm: float = 1e-11
    max_stag: int = 100
    max_newton: int = 50
    max_cg: int = 5000
    max_helm: int = 5000
    warm_start: bool = False    # Helmholtz PCG from abar^(k) instead of 0; Alg. 2 as printed: False
    line_search: bool = True    # Newton with residual backtracking (reading R-LS of DESIGN.md); False: plain N-R
    max_backtrack: int = 5


@dataclass
class Cell:
    grid: Grid
    phases: np.ndarray          # uint8 [z][y][x]
    materials: list
    ell: np.ndarray             # [J][nphases]
    source_phase: list          # [J]
    stress_mask: tuple

    @property
    def J(self):
        return len(self.source_phase)

    def sigma_ref(self):
        sy = [m.sigma_y for m in self.materials if m.sigma_y > 0]
        return max(sy) if sy else max(m.E for m in self.materials) * 1e-3

    def field_of_phase(self, q):
        for j, s in enumerate(self.source_phase):
            if s == q:
                return j
        return None


@dataclass
class State:
    eps: np.ndarray             # (6, Nz, Ny, Nx) committed strain
    epsp: np.ndarray            # (6, n) plastic strain
    ep: np.ndarray              # (n,) equivalent plastic strain
    hist: np.ndarray            # (n,) D_n (J2 phases) / kappa_n (brittle phases)
    abar: np.ndarray            # (J, Nz, Ny, Nx)

    @staticmethod
    def zero(cell: Cell):
        shp = cell.grid.shape
        n = cell.grid.nvox
        return State(np.zeros((6,) + shp), np.zeros((6, n)), np.zeros(n), np.zeros(n),
                     np.zeros((cell.J,) + shp))

    def copy(self):
        return State(self.eps.copy(), self.epsp.copy(), self.ep.copy(), self.hist.copy(), self.abar.copy())


def frozen_damage(cell: Cell, state: State, abar: np.ndarray) -> np.ndarray:
    """Per-voxel damage from the frozen non-local fields (A-16, A-18); returns (n,)."""
    ph = cell.phases.reshape(-1)
    D = np.zeros(ph.shape[0])
    for q, m in enumerate(cell.materials):
        sel = ph == q
        j = cell.field_of_phase(q)
        if m.model == 1 and j is not None:
            D[sel] = mat_.lemaitre_damage(np.maximum(0.0, abar[j].reshape(-1)[sel]), m.eps_c, m.eps_r, m.d_max)
            D[sel] = np.maximum(D[sel], state.hist[sel])
        elif m.model == 2:
            kap = state.hist[sel]
            if j is not None:
                kap = np.maximum(kap, abar[j].reshape(-1)[sel])
            D[sel] = mat_.brittle_damage(kap, m.kappa0, m.kappa_f, m.d_max)
        elif m.model == 3:
            D[sel] = gtn_porosity(cell, q, state, abar)[sel]
    return D


def gtn_porosity(cell: Cell, q: int, state: State, abar: np.ndarray) -> np.ndarray:
    """Frozen porosity f of a GTN phase q (A-30): fields j (ebar0) and j + 1 (trbar) are the
    phase's two non-local fields; f = porosity(f_n, abar^(k), abar_n) per voxel (n,)."""
    j = cell.field_of_phase(q)
    if j is None or j + 1 >= cell.J or cell.source_phase[j + 1] != q:
        raise ValueError("a GTN phase needs two consecutive non-local fields (eps0p, tr eps^p)")
    m = cell.materials[q]
    e0, e0n = abar[j].reshape(-1), state.abar[j].reshape(-1)
    t, tn = abar[j + 1].reshape(-1), state.abar[j + 1].reshape(-1)
    return np.array([gtn_.porosity(state.hist[v], e0[v], e0n[v], t[v], tn[v], m) for v in range(e0.shape[0])])


class ReturnMapFailure(Exception):
    """A GTN return mapping did not converge (the increment is rolled back and cut)."""


def evaluate(cell: Cell, eps: np.ndarray, state: State, D: np.ndarray):
    """Point updates over the cell.  Returns sigma (6,shape), C (6,6,shape), alpha (J,shape),
    epsp (6,n), ep (n,)."""
    shp = cell.grid.shape
    n = cell.grid.nvox
    e = eps.reshape(6, n)
    ph = cell.phases.reshape(-1)
    sigma = np.zeros((6, n))
    C = np.zeros((6, 6, n))
    alpha = np.zeros((cell.J, n))
    epsp = state.epsp.copy()
    ep = state.ep.copy()
    for q, m in enumerate(cell.materials):
        sel = ph == q
        if not np.any(sel):
            continue
        j = cell.field_of_phase(q)
        if m.model == 0:
            s, c = mat_.elastic(e[:, sel], m)
        elif m.model == 1:
            s, c, pp, pe, _, _ = mat_.j2_lemaitre(e[:, sel], state.epsp[:, sel], state.ep[sel], D[sel], m)
            epsp[:, sel] = pp
            ep[sel] = pe
            if j is not None:
                alpha[j, sel] = pe
        elif m.model == 2:
            s, c, eq = mat_.brittle(e[:, sel], D[sel], m)
            if j is not None:
                alpha[j, sel] = eq
        elif m.model == 3:
            s, c, pp, pe, ok = gtn_.gtn(e[:, sel], state.epsp[:, sel], state.ep[sel], D[sel], m)
            if not np.all(ok):
                raise ReturnMapFailure()
            epsp[:, sel] = pp
            ep[sel] = pe
            alpha[j, sel] = pe                         # ebar0 source: eps0p
            alpha[j + 1, sel] = pp[0] + pp[1] + pp[2]  # trbar source: tr eps^p
        else:
            raise ValueError(m.model)
        sigma[:, sel] = s
        C[:, :, sel] = c
    return (sigma.reshape((6,) + shp), C.reshape((6, 6) + shp), alpha.reshape((cell.J,) + shp), epsp, ep)


def _tensor_abs_max(d: np.ndarray) -> float:
    """max over voxels and tensor components of |d_ij| for a Mandel field."""
    w = np.array([1, 1, 1, 1 / S2, 1 / S2, 1 / S2]).reshape((6,) + (1,) * (d.ndim - 1))
    return float(np.max(np.abs(d * w)))


@dataclass
class Report:
    macro_stress: np.ndarray
    macro_strain: np.ndarray
    err: float
    stag_it: int
    newton_it: int
    cg_it: int
    helm_it: int
    converged: bool
    err_hist: list = field(default_factory=list)
    sigma: np.ndarray = None      # stress field of the last mechanical solve


def solve_increment(cell: Cell, state: State, E_target, S_target, tol: Tolerances = Tolerances(),
                    backend="scipy"):
    """Returns (new_state, report).  On non-convergence report.converged is False and the
    input state is returned unchanged (rollback)."""
    g = cell.grid
    mask = np.asarray(cell.stress_mask, dtype=float)
    E_target = np.asarray(E_target, dtype=float)
    S_bar = np.asarray(S_target, dtype=float) * mask
    n = g.nvox
    sref = cell.sigma_ref()
    mean_eps_n = state.eps.reshape(6, n).mean(axis=1)
    dE = (1.0 - mask) * (E_target - mean_eps_n)
    eps = state.eps + dE.reshape((6,) + (1,) * 3)
    abar = state.abar.copy()
    ell2 = [ell2_field(cell.phases, cell.ell[j]) for j in range(cell.J)]
    newton_total = cg_total = helm_total = 0
    err_hist = []
    converged = False
    sigma = None
    for k in range(tol.max_stag):
        D = frozen_damage(cell, state, abar)
        eps_prev = eps.copy()
        newton_ok = False
        rms_prev, lam, nback, de = np.inf, 1.0, 0, None
        for r in range(tol.max_newton + 1):
            try:
                sigma, C, alpha, epsp, ep = evaluate(cell, eps, state, D)
            except ReturnMapFailure:
                return state, Report(np.zeros(6), eps.reshape(6, n).mean(axis=1), np.inf, k + 1, newton_total,
                                     cg_total, helm_total, False, err_hist)
            b = -apply_projection(g, sigma, mask, backend, dc_mean_shift=S_bar)
            smean = sigma.reshape(6, n).mean(axis=1)
            rms = np.sqrt(np.sum(b * b) / n)
            if rms < tol.tol_newton * max(np.linalg.norm(smean), 1e-6 * sref):
                newton_ok = True
                break
            # R-LS: a Newton step that does not lower the residual RMS is halved (at most
            # max_backtrack times), re-evaluating sigma and the residual at eps_r + lam de
            if tol.line_search and de is not None and rms >= rms_prev and nback < tol.max_backtrack:
                lam *= 0.5
                nback += 1
                eps = eps - lam * de
                continue
            if r == tol.max_newton:
                break
            rms_prev, lam, nback = rms, 1.0, 0
            de, it, _ = cg(g, C, b, mask, tol.tol_cg, tol.max_cg, backend)
            cg_total += it
            newton_total += 1
            eps = eps + de
        if not newton_ok:
            return state, Report(smean, eps.reshape(6, n).mean(axis=1), np.inf, k + 1, newton_total,
                                 cg_total, helm_total, False, err_hist)
        abar_new = np.empty_like(abar)
        for j in range(cell.J):
            abar_new[j], it, _ = solve_helmholtz(g, alpha[j], ell2[j], tol.tol_helm, tol.max_helm,
                                                 x0=abar[j] if tol.warm_start else None, backend=backend)
            helm_total += it
        emean = eps.reshape(6, n).mean(axis=1)
        den = np.linalg.norm(emean)
        num = _tensor_abs_max(eps - eps_prev)
        err = num / den if den > 1e-12 else num
        for j in range(cell.J):
            dn = np.linalg.norm(abar_new[j])
            nm = np.linalg.norm(abar_new[j] - abar[j])
            err = max(err, nm / dn if dn > 1e-12 else nm)
        abar = abar_new
        err_hist.append(err)
        if err < tol.tol_stag:
            converged = True
            break
    if not converged:
        return state, Report(smean, eps.reshape(6, n).mean(axis=1), err, k + 1, newton_total,
                             cg_total, helm_total, False, err_hist)
    # commit (A-16)
    new = State(eps, epsp, ep, state.hist.copy(), abar)
    ph = cell.phases.reshape(-1)
    for q, m in enumerate(cell.materials):
        sel = ph == q
        j = cell.field_of_phase(q)
        if j is None:
            continue
        if m.model == 1:
            new.hist[sel] = np.maximum(state.hist[sel], mat_.lemaitre_damage(
                np.maximum(0.0, abar[j].reshape(-1)[sel]), m.eps_c, m.eps_r, m.d_max))
        elif m.model == 2:
            new.hist[sel] = np.maximum(state.hist[sel], abar[j].reshape(-1)[sel])
        elif m.model == 3:
            # f_{n+1} from the converged non-local fields (App. A); eps^p, eps0p are those
            # of the last mechanical solve (f frozen at abar^(k)), A-30
            new.hist[sel] = gtn_porosity(cell, q, state, abar)[sel]
    rep = Report(smean, eps.reshape(6, n).mean(axis=1), err, k + 1, newton_total, cg_total,
                 helm_total, True, err_hist, sigma)
    return new, rep


def make_cell(cfg, scheme="willot") -> Cell:
    """Build an oracle Cell from a synth.CellConfig."""
    g = Grid(cfg.n, cfg.L, scheme)
    return Cell(g, cfg.phases, cfg.materials, np.asarray(cfg.ell, dtype=float), list(cfg.source_phase),
                tuple(cfg.stress_mask))


def run(cfg, n_incr=None, tol: Tolerances = Tolerances(), backend="scipy", max_cutbacks=6, log=None):
    """Fixed-increment driver with deterministic halving on failure (A-21).  Returns a list
    of per-increment dicts at the nominal increments."""
    cell = make_cell(cfg)
    state = State.zero(cell)
    hist = []
    n_incr = cfg.n_incr if n_incr is None else n_incr
    E_prev = 0.0
    for i in range(1, n_incr + 1):
        E_nom = i * cfg.dE
        sub = 1
        while True:
            ok = True
            st = state
            for s in range(1, sub + 1):
                Et = np.zeros(6)
                Et[cfg.load_comp] = E_prev + (E_nom - E_prev) * s / sub
                st2, rep = solve_increment(cell, st, Et, np.zeros(6), tol, backend)
                if not rep.converged:
                    ok = False
                    break
                st = st2
            if ok:
                state = st
                break
            sub *= 2
            if sub > 2 ** max_cutbacks:
                raise RuntimeError(f"increment {i} failed after {max_cutbacks} cutbacks")
        E_prev = E_nom
        rec = dict(incr=i, E=E_nom, stress=rep.macro_stress.tolist(), strain=rep.macro_strain.tolist(),
                   stag=rep.stag_it, newton=rep.newton_it, cg=rep.cg_it, helm=rep.helm_it, sub=sub)
        hist.append(rec)
        if log:
            log(rec)
    return hist, state
