"""Thin ctypes binding of libfgd (include/fgd.h).  Argument marshalling only: every step of the
hot path runs in the CUDA kernels of libfgd.so.  There is no CPU fallback -- importing this
module fails loudly if the shared library is missing.

Field arguments may be torch tensors (CUDA or CPU), numpy arrays, or None where the C ABI
accepts NULL.  They must be contiguous float64 (uint8 for phases); layouts are those of fgd.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("FGD_LIB", os.path.join(_HERE, "libfgd.so"))
if not os.path.exists(LIB_PATH):
    raise ImportError(f"libfgd.so not built ({LIB_PATH}); run `python -m paper_2103_04770_b200.build` "
                      "(there is no CPU fallback)")
lib = C.CDLL(LIB_PATH)

OK, EINVAL, ESHAPE, ECUDA, ENCCL, ENOMEM, ENOCONV, ESTATE = 0, -1, -2, -3, -4, -5, -6, -7
STATUS = {0: "FGD_OK", -1: "FGD_EINVAL", -2: "FGD_ESHAPE", -3: "FGD_ECUDA", -4: "FGD_ENCCL",
          -5: "FGD_ENOMEM", -6: "FGD_ENOCONV", -7: "FGD_ESTATE"}
FIELD_STRESS, FIELD_STRAIN, FIELD_EPS_P, FIELD_EQPS, FIELD_HIST, FIELD_TANGENT = 0, 1, 2, 3, 4, 5
FIELD_NONLOCAL, FIELD_SOURCE, FIELD_ITERATE, FIELD_NONLOCAL_ITERATE = 16, 32, 48, 64


class fgd_grid(C.Structure):
    _fields_ = [("dims", C.c_int), ("n", C.c_int * 3), ("L", C.c_double * 3), ("scheme", C.c_int)]


class fgd_dist(C.Structure):
    _fields_ = [("rank", C.c_int), ("nranks", C.c_int), ("device", C.c_int),
                ("nccl_id", C.c_void_p), ("stream", C.c_void_p)]


MATERIAL_KEYS = ("E", "nu", "sigma_y", "H", "eps_c", "eps_r", "d_max", "kappa0", "kappa_f",
                 "q1", "q2", "q3", "f_c", "f_f", "f_n", "eps_n", "s_n", "n_hard", "fstar_max")


class fgd_material(C.Structure):
    _fields_ = [("model", C.c_int)] + [(k, C.c_double) for k in MATERIAL_KEYS]


class fgd_increment(C.Structure):
    _fields_ = [("E_target", C.c_double * 6), ("S_target", C.c_double * 6),
                ("tol_stag", C.c_double), ("tol_newton", C.c_double), ("tol_cg", C.c_double),
                ("tol_helm", C.c_double), ("max_stag", C.c_int), ("max_newton", C.c_int),
                ("max_cg", C.c_int), ("max_helm", C.c_int), ("warm_start", C.c_int),
                ("line_search", C.c_int), ("stag_stall", C.c_int)]


class fgd_report(C.Structure):
    _fields_ = [("macro_stress", C.c_double * 6), ("macro_strain", C.c_double * 6), ("err", C.c_double),
                ("stag_it", C.c_int), ("newton_it", C.c_int), ("cg_it", C.c_int), ("helm_it", C.c_int)]


_P = C.c_void_p
_D = C.c_double
_I = C.c_int
_SIGS = {
    "fgd_create": ([C.POINTER(fgd_grid), C.POINTER(fgd_dist), C.POINTER(C.c_void_p)], _I),
    "fgd_nccl_id": ([_P], _I),
    "fgd_loopback_id": ([_P], _I),
    "fgd_destroy": ([_P], None),
    "fgd_last_error": ([_P], C.c_char_p),
    "fgd_local_extent": ([_P, C.POINTER(_I), C.POINTER(_I)], _I),
    "fgd_launch_count": ([_P], C.c_ulonglong),
    "fgd_set_phases": ([_P, _P, _I], _I),
    "fgd_set_material": ([_P, _I, C.POINTER(fgd_material)], _I),
    "fgd_set_nonlocal": ([_P, _I, _P, _P], _I),
    "fgd_set_control": ([_P, _P], _I),
    "fgd_set_tangent": ([_P, _P], _I),
    "fgd_apply_projected_tangent": ([_P, _P, _P], _I),
    "fgd_apply_projection": ([_P, _P, _P, _P], _I),
    "fgd_apply_helmholtz": ([_P, _I, _P, _P], _I),
    "fgd_apply_helmholtz_precond": ([_P, _I, _P, _P], _I),
    "fgd_solve_helmholtz": ([_P, _I, _P, _P, _D, _I, C.POINTER(_I), C.POINTER(_D)], _I),
    "fgd_solve_helmholtz_from": ([_P, _I, _P, _P, _P, _D, _I, C.POINTER(_I), C.POINTER(_D)], _I),
    "fgd_solve_helmholtz_all": ([_P, _P, _P, _P, _D, _I, C.POINTER(_I), C.POINTER(_D)], _I),
    "fgd_solve_tangent_cg": ([_P, _P, _P, _D, _I, C.POINTER(_I), C.POINTER(_D)], _I),
    "fgd_constitutive": ([_P, _P, _P, _P], _I),
    "fgd_mech_residual": ([_P, _P, _P, C.POINTER(_D)], _I),
    "fgd_solve_increment": ([_P, C.POINTER(fgd_increment), C.POINTER(fgd_report)], _I),
    "fgd_get_field": ([_P, _I, _P], _I),
    "fgd_set_field": ([_P, _I, _P], _I),
    "fgd_macro_stress": ([_P, _P], _I),
    "fgd_set_timing": ([_P, _I], _I),
    "fgd_kernel_times": ([_P, _P, _P, _I], _I),
}
KCLASS = ("xfwd6", "yfwd6", "z6", "yinv6", "xinv6", "xfwd1", "yfwd1", "z1", "yinv1", "xinv1", "stencil",
          "constitutive", "other", "comm", "xfwd6cg")
EXPORTED = tuple(_SIGS)
for _name, (_args, _res) in _SIGS.items():
    _f = getattr(lib, _name)
    _f.argtypes = _args
    _f.restype = _res
    globals()[_name] = _f


class FgdError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def ptr(x, dtype=np.float64):
    """data pointer of a contiguous torch tensor / numpy array (None -> NULL)."""
    if x is None:
        return None
    if isinstance(x, np.ndarray):
        if x.dtype != dtype or not x.flags["C_CONTIGUOUS"]:
            raise ValueError(f"need a C-contiguous {np.dtype(dtype).name} array")
        return x.ctypes.data
    try:
        import torch
    except ImportError:  # pragma: no cover
        torch = None
    if torch is not None and isinstance(x, torch.Tensor):
        want = torch.float64 if dtype == np.float64 else torch.uint8
        if x.dtype != want or not x.is_contiguous():
            raise ValueError(f"need a contiguous {want} tensor")
        return x.data_ptr()
    raise TypeError(f"unsupported field type {type(x)}")
