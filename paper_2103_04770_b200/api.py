"""paper_2103_04770_b200.api -- B200-native (sm_100a, FP64) hot path of the staggered FFT solver for
implicit-gradient ductile damage (Magri et al., arXiv 2103.04770).

The product is libfgd.so (C ABI, include/fgd.h).  This package is its thin Python binding:
`_fgd` mirrors the C functions one to one; `Context` is a convenience object that only
marshals arguments (allocates outputs, converts tensors to pointers, raises on error status).
PyTorch is used for device memory and streams only.
"""
from __future__ import annotations

import ctypes as C

import numpy as np

from . import _fgd
from ._fgd import FgdError, ptr

__all__ = ["Context", "FgdError", "Material", "nccl_id"]


class Material:
    """fgd_material: model 0 elastic, 1 J2-Lemaitre, 2 elastic-brittle, 3 non-local GTN (the GTN
    defaults are the paper's Sec. 4.1 values, with the f* cap 0.6 of P:837)."""

    def __init__(self, model, E, nu, sigma_y=0.0, H=0.0, eps_c=0.0, eps_r=1.0, d_max=0.99, kappa0=0.0,
                 kappa_f=1.0, q1=1.5, q2=1.0, q3=2.25, f_c=0.15, f_f=0.25, f_n=0.04, eps_n=0.3, s_n=0.1,
                 n_hard=0.1, fstar_max=0.6):
        self.model, self.E, self.nu, self.sigma_y, self.H = model, E, nu, sigma_y, H
        self.eps_c, self.eps_r, self.d_max, self.kappa0, self.kappa_f = eps_c, eps_r, d_max, kappa0, kappa_f
        self.q1, self.q2, self.q3, self.f_c, self.f_f = q1, q2, q3, f_c, f_f
        self.f_n, self.eps_n, self.s_n, self.n_hard, self.fstar_max = f_n, eps_n, s_n, n_hard, fstar_max

    @classmethod
    def of(cls, m):
        """From any object carrying the fgd_material attributes (e.g. synth.Material)."""
        return cls(int(m.model), *[float(getattr(m, k)) for k in _fgd.MATERIAL_KEYS])


def _like(x, shape=None):
    if isinstance(x, np.ndarray):
        return np.empty(shape if shape is not None else x.shape, dtype=np.float64)
    import torch
    return torch.empty(shape if shape is not None else x.shape, dtype=torch.float64, device=x.device)


def nccl_id() -> bytes:
    """128-byte NCCL unique id (rank 0); broadcast it to the other ranks and pass to Context."""
    buf = (C.c_ubyte * 128)()
    st = _fgd.fgd_nccl_id(C.cast(buf, C.c_void_p))
    if st != 0:
        raise FgdError(st, "fgd_nccl_id failed")
    return bytes(buf)


def loopback_id() -> bytes:
    """128-byte id of an in-process loopback group (fgd_loopback_id): pass the same id as `nccl_id`
    to `nranks` Contexts of this process, each driven by its own thread, to run the multi-rank
    code paths on one GPU with device-to-device copies instead of NCCL (validation transport)."""
    buf = (C.c_ubyte * 128)()
    st = _fgd.fgd_loopback_id(C.cast(buf, C.c_void_p))
    if st != 0:
        raise FgdError(st, "fgd_loopback_id failed")
    return bytes(buf)


class Context:
    """One libfgd context (one GPU, one stream).  n = (N1, N2, N3); N3 = 1 for 2D.
    Multi-GPU: rank/nranks/nccl_id (from nccl_id() on rank 0); fields are then the rank's
    z-slab (see `local_extent`)."""

    def __init__(self, n, L=None, scheme: int = 1, device: int = 0, stream=None, rank: int = 0, nranks: int = 1,
                 nccl_id: bytes | None = None):
        n = tuple(int(v) for v in n)
        if len(n) == 2:
            n = (n[0], n[1], 1)
        dims = 2 if n[2] == 1 else 3
        if L is None:
            L = (1.0, 1.0, 1.0 if dims == 3 else 1.0 / n[0])
        g = _fgd.fgd_grid(dims, (C.c_int * 3)(*n), (C.c_double * 3)(*[float(v) for v in L]), int(scheme))
        if stream is None:
            try:
                import torch
                if torch.cuda.is_available():
                    stream = torch.cuda.current_stream(device).cuda_stream
            except ImportError:  # pragma: no cover
                stream = None
        self._id = (C.c_ubyte * 128).from_buffer_copy(nccl_id) if nccl_id is not None else None
        d = _fgd.fgd_dist(int(rank), int(nranks), int(device),
                          C.cast(self._id, C.c_void_p) if self._id is not None else None, stream)
        h = C.c_void_p()
        st = _fgd.fgd_create(C.byref(g), C.byref(d), C.byref(h))
        if st != 0:
            raise FgdError(st, "fgd_create failed (see stderr)")
        self.h = h
        self.n = n
        z0, nz = C.c_int(0), C.c_int(0)
        _fgd.fgd_local_extent(h, C.byref(z0), C.byref(nz))
        self.z0, self.nz = z0.value, nz.value
        self.nvox = n[0] * n[1] * self.nz
        self.shape = (self.nz, n[1], n[0])

    # ---- plumbing ---------------------------------------------------------------------------
    def _chk(self, st):
        if st != 0:
            raise FgdError(st, _fgd.fgd_last_error(self.h).decode())
        return st

    def close(self):
        if getattr(self, "h", None):
            _fgd.fgd_destroy(self.h)
            self.h = None

    def __del__(self):  # pragma: no cover
        try:
            self.close()
        except Exception:
            pass

    @property
    def launch_count(self) -> int:
        return int(_fgd.fgd_launch_count(self.h))

    # ---- data ---------------------------------------------------------------------------------
    def set_phases(self, phases, nphases: int):
        self._chk(_fgd.fgd_set_phases(self.h, ptr(phases, np.uint8), int(nphases)))

    def set_material(self, phase: int, m):
        mm = _fgd.fgd_material(int(m.model), *[float(getattr(m, k)) for k in _fgd.MATERIAL_KEYS])
        self._chk(_fgd.fgd_set_material(self.h, int(phase), C.byref(mm)))

    def set_nonlocal(self, ell, source_phase):
        ell = np.ascontiguousarray(np.asarray(ell, dtype=np.float64))
        sp = np.ascontiguousarray(np.asarray(source_phase, dtype=np.int32))
        J = int(sp.shape[0])
        self._chk(_fgd.fgd_set_nonlocal(self.h, J, ell.ctypes.data if J else None, sp.ctypes.data if J else None))

    def set_control(self, stress_mask):
        m = np.ascontiguousarray(np.asarray(stress_mask, dtype=np.int32))
        self._chk(_fgd.fgd_set_control(self.h, m.ctypes.data))

    def set_tangent(self, Cp):
        self._chk(_fgd.fgd_set_tangent(self.h, ptr(Cp)))

    # ---- operators ----------------------------------------------------------------------------
    def apply_projected_tangent(self, x, y=None):
        y = _like(x) if y is None else y
        self._chk(_fgd.fgd_apply_projected_tangent(self.h, ptr(x), ptr(y)))
        return y

    def apply_projection(self, tau, S=None, y=None):
        y = _like(tau) if y is None else y
        Sp = None
        if S is not None:
            S = np.ascontiguousarray(np.asarray(S, dtype=np.float64))
            Sp = S.ctypes.data
        self._chk(_fgd.fgd_apply_projection(self.h, ptr(tau), Sp, ptr(y)))
        return y

    def apply_helmholtz(self, field: int, a, y=None):
        y = _like(a) if y is None else y
        self._chk(_fgd.fgd_apply_helmholtz(self.h, int(field), ptr(a), ptr(y)))
        return y

    def apply_helmholtz_precond(self, field: int, r, z=None):
        z = _like(r) if z is None else z
        self._chk(_fgd.fgd_apply_helmholtz_precond(self.h, int(field), ptr(r), ptr(z)))
        return z

    def solve_helmholtz(self, field: int, src=None, abar=None, tol=1e-10, maxit=1000, check=True):
        it, rel = C.c_int(0), C.c_double(0.0)
        st = _fgd.fgd_solve_helmholtz(self.h, int(field), ptr(src), ptr(abar), float(tol), int(maxit),
                                      C.byref(it), C.byref(rel))
        if check:
            self._chk(st)
        return it.value, rel.value

    def solve_helmholtz_from(self, field: int, src, x0, abar, tol=1e-10, maxit=1000, check=True):
        """Algorithm 2 from the initial guess x0 (None = 0), fgd_solve_helmholtz_from."""
        it, rel = C.c_int(0), C.c_double(0.0)
        st = _fgd.fgd_solve_helmholtz_from(self.h, int(field), ptr(src), ptr(x0), ptr(abar), float(tol), int(maxit),
                                           C.byref(it), C.byref(rel))
        if check:
            self._chk(st)
        return it.value, rel.value

    def solve_helmholtz_all(self, src, x0, abar, nfields: int, tol=1e-10, maxit=1000, check=True):
        """All J fields side by side (fgd_solve_helmholtz_all); src, x0 (None = 0), abar: [J, ...] fields."""
        it = (C.c_int * int(nfields))()
        rel = (C.c_double * int(nfields))()
        st = _fgd.fgd_solve_helmholtz_all(self.h, ptr(src), ptr(x0), ptr(abar), float(tol), int(maxit), it, rel)
        if check:
            self._chk(st)
        return list(it), list(rel)

    def solve_tangent_cg(self, b=None, de=None, tol=1e-10, maxit=1000, check=True):
        it, rel = C.c_int(0), C.c_double(0.0)
        st = _fgd.fgd_solve_tangent_cg(self.h, ptr(b), ptr(de), float(tol), int(maxit), C.byref(it), C.byref(rel))
        if check:
            self._chk(st)
        return it.value, rel.value

    def constitutive(self, eps=None, sigma_out=None):
        m = np.zeros(6)
        self._chk(_fgd.fgd_constitutive(self.h, ptr(eps), ptr(sigma_out), m.ctypes.data))
        return m

    def mech_residual(self, S=None, b_out=None):
        rms = C.c_double(0.0)
        Sp = None
        if S is not None:
            S = np.ascontiguousarray(np.asarray(S, dtype=np.float64))
            Sp = S.ctypes.data
        self._chk(_fgd.fgd_mech_residual(self.h, Sp, ptr(b_out), C.byref(rms)))
        return rms.value

    def solve_increment(self, E_target, S_target=None, tol_stag=1e-8, tol_newton=1e-10, tol_cg=1e-11,
                        tol_helm=1e-11, max_stag=100, max_newton=50, max_cg=5000, max_helm=5000, warm_start=False,
                        line_search=True, stag_stall=0):
        S_target = np.zeros(6) if S_target is None else S_target
        inc = _fgd.fgd_increment((C.c_double * 6)(*map(float, E_target)), (C.c_double * 6)(*map(float, S_target)),
                                 tol_stag, tol_newton, tol_cg, tol_helm, max_stag, max_newton, max_cg, max_helm,
                                 1 if warm_start else 0, 1 if line_search else 0, int(stag_stall))
        rep = _fgd.fgd_report()
        st = _fgd.fgd_solve_increment(self.h, C.byref(inc), C.byref(rep))
        if st not in (0, _fgd.ENOCONV):
            self._chk(st)
        return st, dict(macro_stress=np.array(rep.macro_stress[:]), macro_strain=np.array(rep.macro_strain[:]),
                        err=rep.err, stag=rep.stag_it, newton=rep.newton_it, cg=rep.cg_it, helm=rep.helm_it)

    def get_field(self, which: int, out):
        self._chk(_fgd.fgd_get_field(self.h, int(which), ptr(out)))
        return out

    def set_field(self, which: int, x):
        self._chk(_fgd.fgd_set_field(self.h, int(which), ptr(x)))

    def set_timing(self, enable: bool):
        self._chk(_fgd.fgd_set_timing(self.h, int(bool(enable))))

    def kernel_times(self):
        """{class: (total ms, launches)} since the last set_timing(True)."""
        n = len(_fgd.KCLASS)
        ms = np.zeros(n)
        cnt = np.zeros(n, dtype=np.uint64)
        self._chk(_fgd.fgd_kernel_times(self.h, ms.ctypes.data, cnt.ctypes.data, n))
        return {k: (float(ms[i]), int(cnt[i])) for i, k in enumerate(_fgd.KCLASS)}

    def macro_stress(self):
        m = np.zeros(6)
        self._chk(_fgd.fgd_macro_stress(self.h, m.ctypes.data))
        return m
