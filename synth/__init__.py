"""Seeded synthetic input generators shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the paper's method (no transforms, projections,
Helmholtz operators, constitutive updates or solvers).  It only draws inputs:
phase maps (disc, RSA spheres, Bernoulli), random SPD tangents, Gaussian fields,
the five BASELINE.json configurations and the non-local GTN cells of the paper's
Sec. 4.1 / 4.2 (config_gtn2d, config_gtn3d) as plain parameter records.

Units: stresses/moduli in MPa, lengths in cell units (L = 1) unless a config says
otherwise.  Array layout: numpy C order [z][y][x] (x fastest) for scalars and
[comp][z][y][x] for fields; Mandel component order (11, 22, 33, 23, 13, 12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

MANDEL = ("11", "22", "33", "23", "13", "12")
# packed upper triangle of a symmetric 6x6 Mandel matrix, row-major: (0,0),(0,1)..(0,5),(1,1)..(5,5)
PACKED21 = tuple((i, j) for i in range(6) for j in range(i, 6))


# ----------------------------------------------------------------------------------------------
# phase maps
# ----------------------------------------------------------------------------------------------
def voxel_centres(n: int, L: float = 1.0) -> np.ndarray:
    """x_i = (1/2 + n_i) L/N."""
    return (0.5 + np.arange(n)) * (L / n)


def disc_phases(n: int, radius: float, L: float = 1.0) -> np.ndarray:
    """2D centred disc (BJ configs 0/2).  Voxel is inclusion (phase 1) iff its centre
    lies inside the disc (A-23).  Returns uint8 array of shape (1, n, n)."""
    x = voxel_centres(n, L)
    X, Y = np.meshgrid(x, x, indexing="xy")  # X varies along axis 1 (x)
    inside = (X - 0.5 * L) ** 2 + (Y - 0.5 * L) ** 2 < radius ** 2
    return inside.astype(np.uint8)[None, :, :]


def rsa_centres(n_spheres: int, phi: float, seed: int, L: float = 1.0, max_tries: int = 2_000_000):
    """Random sequential adsorption with periodic minimum-image distance (A-24).
    r = (phi * 3 / (4 pi n))^(1/3) L.  Returns (centres (n,3) in (x,y,z), r)."""
    r = (phi * 3.0 / (4.0 * math.pi * n_spheres)) ** (1.0 / 3.0) * L
    rng = np.random.default_rng(seed)
    centres = []
    tries = 0
    while len(centres) < n_spheres:
        tries += 1
        if tries > max_tries:
            raise RuntimeError(f"RSA failed: placed {len(centres)}/{n_spheres}")
        c = rng.random(3) * L
        ok = True
        for q in centres:
            d = c - q
            d -= L * np.round(d / L)
            if d @ d < (2.0 * r) ** 2:
                ok = False
                break
        if ok:
            centres.append(c)
    return np.array(centres), r


def sphere_phases(n: int, centres: np.ndarray, r: float, L: float = 1.0) -> np.ndarray:
    """Voxelize periodic spheres (voxel-centre rule, min-image).  uint8 (n, n, n) [z][y][x]."""
    x = voxel_centres(n, L)
    ph = np.zeros((n, n, n), dtype=np.uint8)
    h = L / n
    span = int(math.ceil(r / h)) + 1
    for c in centres:
        idx = [np.arange(int(math.floor(c[a] / h)) - span, int(math.floor(c[a] / h)) + span + 1) for a in range(3)]
        ix, iy, iz = [i % n for i in idx]
        dx = x[ix] - c[0]
        dy = x[iy] - c[1]
        dz = x[iz] - c[2]
        dx -= L * np.round(dx / L)
        dy -= L * np.round(dy / L)
        dz -= L * np.round(dz / L)
        d2 = dz[:, None, None] ** 2 + dy[None, :, None] ** 2 + dx[None, None, :] ** 2
        sub = d2 < r * r
        zz, yy, xx = np.meshgrid(iz, iy, ix, indexing="ij")
        ph[zz[sub], yy[sub], xx[sub]] = 1
    return ph


def bernoulli_phases(shape, p: float, seed: int) -> np.ndarray:
    """Phase 1 with probability p per voxel (BJ config 1): rng(seed).random(N) < p."""
    rng = np.random.default_rng(seed)
    return (rng.random(int(np.prod(shape))) < p).astype(np.uint8).reshape(shape)


# ----------------------------------------------------------------------------------------------
# fields
# ----------------------------------------------------------------------------------------------
def gaussian_field(ncomp: int, shape, std: float, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.normal(0.0, std, size=(ncomp,) + tuple(shape))


def random_spd_tangent(nvox: int, seed: int, lo: float = 1.0e3, hi: float = 1.0e5) -> np.ndarray:
    """Per-voxel random SPD 6x6 Mandel tangent C = Q diag(lam) Q^T (A-29): Q Haar-orthogonal
    (QR of a Gaussian with sign fix), lam ~ U[lo, hi] (MPa; 1..100 GPa).  Returns the
    packed upper triangle, shape (21, nvox)."""
    rng = np.random.default_rng(seed)
    out = np.empty((21, nvox))
    chunk = 1 << 18
    for s in range(0, nvox, chunk):
        m = min(chunk, nvox - s)
        G = rng.normal(size=(m, 6, 6))
        Q, R = np.linalg.qr(G)
        Q = Q * np.sign(np.diagonal(R, axis1=1, axis2=2))[:, None, :]
        lam = rng.uniform(lo, hi, size=(m, 6))
        C = np.einsum("nik,nk,njk->nij", Q, lam, Q)
        for t, (i, j) in enumerate(PACKED21):
            out[t, s:s + m] = C[:, i, j]
    return out


def random_spd_tangent_torch(nvox: int, seed: int, device="cuda", lo: float = 1.0e3, hi: float = 1.0e5):
    """Same recipe as random_spd_tangent, drawn with torch (on the GPU for 256^3/512^3 inputs).
    Returns a (21, nvox) float64 tensor on `device`.  Values differ from the numpy draw; each
    run generates once and hands the SAME tensor to both sides."""
    import torch
    g = torch.Generator(device=device)
    g.manual_seed(seed)
    out = torch.empty((21, nvox), dtype=torch.float64, device=device)
    chunk = 1 << 20
    iu = torch.tensor([i for i, _ in PACKED21], device=device)
    ju = torch.tensor([j for _, j in PACKED21], device=device)
    for s in range(0, nvox, chunk):
        m = min(chunk, nvox - s)
        G = torch.randn((m, 6, 6), generator=g, dtype=torch.float64, device=device)
        # modified Gram-Schmidt on the columns = QR with a positive diagonal of R (Haar Q)
        Q = torch.empty_like(G)
        for i in range(6):
            v = G[:, :, i].clone()
            for j in range(i):
                v -= (Q[:, :, j] * v).sum(dim=1, keepdim=True) * Q[:, :, j]
            Q[:, :, i] = v / v.norm(dim=1, keepdim=True)
        lam = lo + (hi - lo) * torch.rand((m, 6), generator=g, dtype=torch.float64, device=device)
        C = torch.einsum("nik,nk,njk->nij", Q, lam, Q)
        out[:, s:s + m] = C[:, iu, ju].T
    return out


# ----------------------------------------------------------------------------------------------
# configurations (BASELINE.json configs; readings A-12, A-13, A-17, A-18, A-20, A-21, A-24, A-25)
# ----------------------------------------------------------------------------------------------
@dataclass
class Material:
    model: int            # 0 elastic, 1 j2_lemaitre, 2 elastic_brittle, 3 gtn
    E: float
    nu: float
    sigma_y: float = 0.0
    H: float = 0.0
    eps_c: float = 0.0
    eps_r: float = 1.0
    d_max: float = 0.99
    kappa0: float = 0.0
    kappa_f: float = 1.0
    # GTN (model 3, paper Sec. 2.1.1; defaults = the Sec. 4.1 values, cap P:837)
    q1: float = 1.5
    q2: float = 1.0
    q3: float = 2.25
    f_c: float = 0.15
    f_f: float = 0.25
    f_n: float = 0.04
    eps_n: float = 0.3
    s_n: float = 0.1
    n_hard: float = 0.1
    fstar_max: float = 0.6


MATRIX_J2 = Material(model=1, E=70.0e3, nu=0.3, sigma_y=300.0, H=500.0, eps_c=0.005, eps_r=0.025, d_max=0.99)
INCLUSION_EL = Material(model=0, E=400.0e3, nu=0.2)
PARTICLE_BRITTLE = Material(model=2, E=400.0e3, nu=0.2, d_max=0.99, kappa0=0.003, kappa_f=0.006)


@dataclass
class CellConfig:
    name: str
    n: tuple                  # (N1, N2, N3) = (Nx, Ny, Nz); 2D has N3 = 1
    L: tuple
    phases: np.ndarray        # uint8 [z][y][x]
    materials: list           # per phase
    ell: np.ndarray           # [nfields][nphases] in length units
    source_phase: list        # [nfields]
    stress_mask: tuple        # 6 comps, 1 = stress-controlled (A-20)
    load_comp: int            # strain-controlled component that is ramped
    dE: float                 # fixed increment (A-21)
    n_incr: int
    extra: dict = field(default_factory=dict)


def config0(n: int = 32, ell_over_L: float = 2.0 / 32.0) -> CellConfig:
    """BJ config 0 (and config 2 at n=256 with ell = L/16): 2D plane strain, centred disc
    r = 0.2 L, elastic inclusion in J2-Lemaitre matrix; ell_M = 2h at 32^2 (A-13),
    ell_I = ell_M / 50 (A-12); E11 to 2 % in 50 x 4e-4 (A-21); mask (0,1,0,0,0,1) (A-20)."""
    L = 1.0
    ph = disc_phases(n, 0.2 * L, L)
    ellM = ell_over_L * L
    ell = np.array([[ellM, ellM / 50.0]])
    return CellConfig(name=f"config0_{n}", n=(n, n, 1), L=(L, L, L / n), phases=ph,
                      materials=[MATRIX_J2, INCLUSION_EL], ell=ell, source_phase=[0],
                      stress_mask=(0, 1, 0, 0, 0, 1), load_comp=0, dE=4.0e-4, n_incr=50)


def config2(n: int = 256) -> CellConfig:
    c = config0(n, ell_over_L=1.0 / 16.0)
    c.name = f"config2_{n}"
    return c


def config3(n: int = 128, n_spheres: int = 30, phi: float = 0.20, seed: int = 3) -> CellConfig:
    """BJ config 3: RSA spheres (A-24), brittle particles (A-18) in J2-Lemaitre matrix,
    two non-local fields: field 0 = matrix eps_p (ell_m = 5h in matrix, /50 in particles),
    field 1 = particle eps_eq (ell_p = 3h in particles, /50 in matrix); E_zz to 3 % in
    60 x 5e-4, other stresses zero (mask (1,1,0,1,1,1))."""
    L = 1.0
    h = L / n
    centres, r = rsa_centres(n_spheres, phi, seed, L)
    ph = sphere_phases(n, centres, r, L)
    ell = np.array([[5.0 * h, 5.0 * h / 50.0],
                    [3.0 * h / 50.0, 3.0 * h]])
    return CellConfig(name=f"config3_{n}", n=(n, n, n), L=(L, L, L), phases=ph,
                      materials=[MATRIX_J2, PARTICLE_BRITTLE], ell=ell, source_phase=[0, 1],
                      stress_mask=(1, 1, 0, 1, 1, 1), load_comp=2, dE=5.0e-4, n_incr=60,
                      extra={"centres": centres, "radius": r})


def config4(n: int = 512, n_spheres: int = 400, phi: float = 0.25, seed: int = 4) -> CellConfig:
    """BJ config 4: the 512^3 RSA cell, 400 spheres at 25 % volume fraction, same phases,
    materials, two-ell regularisation (ell_m = 5h, ell_p = 3h), mask and loading as config 3."""
    c = config3(n=n, n_spheres=n_spheres, phi=phi, seed=seed)
    c.name = f"config4_{n}"
    return c


# GTN matrices of the paper (model 3): Sec. 4.1 (2D) and Sec. 4.2 (3D)
MATRIX_GTN_2D = Material(model=3, E=300.0e3, nu=0.3, sigma_y=1000.0, q1=1.5, q2=1.0, q3=2.25, f_c=0.15, f_f=0.25,
                         f_n=0.04, eps_n=0.3, s_n=0.1, n_hard=0.1, fstar_max=0.6)
INCLUSION_EL_2D = Material(model=0, E=900.0e3, nu=0.3)
MATRIX_GTN_3D = Material(model=3, E=70.0e3, nu=0.33, sigma_y=200.0, q1=1.5, q2=1.0, q3=2.25, f_c=0.15, f_f=0.25,
                         f_n=0.04, eps_n=0.1, s_n=0.05, n_hard=0.1, fstar_max=0.6)


def config_gtn2d(n: int = 32, ell_over_L: float = 0.05, ell_i_over_L: float = 0.001) -> CellConfig:
    """Non-local GTN in 2D (paper Sec. 4.1): the centred disc r = 0.2 L of config 0,
    GTN matrix (E = 300 GPa, nu = 0.3, sigma_Y = 1 GPa, q1 = 1.5, q2 = 1, q3 = 2.25, f_C = 0.15,
    f_F = 0.25, f_N = 0.04, eps_N = 0.3, s_N = 0.1, Aravas N = 0.1, f* <= 0.6), elastic inclusion
    (E = 900 GPa, nu = 0.3); two non-local fields of the matrix (eps0p, tr eps^p) with
    ell_M = 0.05 L, ell_I = 0.001 L; plane strain E11 ramp (the paper reaches E11 = 0.5;
    fixed increments here, A-21), mask (0,1,0,0,0,1)."""
    L = 1.0
    ph = disc_phases(n, 0.2 * L, L)
    ellM = ell_over_L * L
    row = [ellM, ell_i_over_L * L]     # the local variant of P:843 is ell_M = ell_I = 1e-4 L
    return CellConfig(name=f"gtn2d_{n}", n=(n, n, 1), L=(L, L, L / n), phases=ph,
                      materials=[MATRIX_GTN_2D, INCLUSION_EL_2D], ell=np.array([row, row]), source_phase=[0, 0],
                      stress_mask=(0, 1, 0, 0, 0, 1), load_comp=0, dE=2.5e-3, n_incr=200)


def config_gtn3d(n: int = 32, n_spheres: int = 30, phi: float = 0.20, seed: int = 3) -> CellConfig:
    """Non-local GTN in 3D (paper Sec. 4.2): the RSA sphere cell of config 3 with
    elastic particles (E = 400 GPa, nu = 0.2) in a GTN matrix (E = 70 GPa, nu = 0.33, sigma_Y =
    200 MPa, eps_N = 0.1, s_N = 0.05, other GTN values as in 2D); ell_M = 0.05 L, ell_I = 0.001 L
    for both fields; E_zz ramp, other stresses zero (mask (1,1,0,1,1,1))."""
    L = 1.0
    centres, r = rsa_centres(n_spheres, phi, seed, L)
    ph = sphere_phases(n, centres, r, L)
    row = [0.05 * L, 0.001 * L]
    return CellConfig(name=f"gtn3d_{n}", n=(n, n, n), L=(L, L, L), phases=ph,
                      materials=[MATRIX_GTN_3D, INCLUSION_EL], ell=np.array([row, row]), source_phase=[0, 0],
                      stress_mask=(1, 1, 0, 1, 1, 1), load_comp=2, dE=1.0e-3, n_incr=600,
                      extra={"centres": centres, "radius": r})


def config1_phases(n: int, seed: int = 0) -> np.ndarray:
    """BJ config 1: phases rng(seed).random(N^3) < 0.2."""
    return bernoulli_phases((n, n, n), 0.2, seed)


CONFIG1_ELL = np.array([[2.0, 4.0]])   # L = N (h = 1): ell = 2 (phase 0), 4 (phase 1)
CONFIG1_MASK = (1, 1, 0, 1, 1, 1)
