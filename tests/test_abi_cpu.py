"""CPU-side checks of the C-ABI library: it builds for sm_100a, loads, and exports every symbol
that include/fgd.h declares (no compute calls without a GPU)."""
import ctypes
import os
import re
import shutil

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "fgd.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(fgd_[a-z_]+)\s*\(", src)))


@pytest.fixture(scope="module")
def lib():
    if shutil.which("nvcc") is None and not os.path.exists("/usr/local/cuda/bin/nvcc"):
        pytest.skip("nvcc not available")
    from paper_2103_04770_b200 import build
    path = build.build()
    return ctypes.CDLL(path)


def test_header_declares_boundary():
    syms = declared_symbols()
    for s in ["fgd_create", "fgd_apply_projected_tangent", "fgd_apply_helmholtz", "fgd_apply_helmholtz_precond",
              "fgd_solve_increment", "fgd_get_field", "fgd_macro_stress", "fgd_set_phases", "fgd_set_material"]:
        assert s in syms


def test_library_exports_every_declared_symbol(lib):
    missing = [s for s in declared_symbols() if not hasattr(lib, s)]
    assert not missing, missing


def test_binding_mirrors_header(lib):
    from paper_2103_04770_b200 import _fgd
    assert sorted(_fgd.EXPORTED) == declared_symbols()


def test_library_is_sm100a():
    from paper_2103_04770_b200 import build
    path = build.build()
    out = os.popen(f"/usr/local/cuda/bin/cuobjdump --list-elf {path} 2>&1").read()
    assert "sm_100a" in out


def test_create_without_gpu_fails_cleanly(lib):
    """No GPU here: fgd_create must return an error status, not crash."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    from paper_2103_04770_b200 import Context, FgdError
    with pytest.raises(FgdError):
        Context((8, 8, 8))
