"""Shared-memory race hunting without compute-sanitizer (closed on this pool): the same seeded
computation (every operator apply, packed and compact CG, constitutive update, Newton residual,
Helmholtz apply / preconditioner / PCG) through the production library and through the
race-hunting build libfgd_jitter.so (-DFGD_JITTER: every warp leaving a barrier sleeps a random
0-4 us with probability 1/4, fgd_internal.cuh), on grids that select each family of specialised
kernels.  Every kernel reduces in a fixed order, so the two must agree BIT FOR BIT; an access that
is not ordered by a barrier (the y-inverse 512 restaging race of round 1 was one) reads a
different value under the jittered interleaving."""
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs CUDA", allow_module_level=True)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PKG = os.path.join(ROOT, "paper_2103_04770_b200")
GRIDS = [(16, 16, 16), (32, 32, 1), (256, 8, 8), (512, 4, 8), (8, 256, 256), (4, 512, 512), (256, 256, 256)]


def run(lib, n, path):
    # the same persistent grid in both builds (their occupancies differ), so that the reductions
    # sum the same per-CTA partials in the same order
    env = dict(os.environ, FGD_LIB=lib, FGD_GRID_CAP="96")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "race_case.py"), *map(str, n), path], env=env,
                       capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-3000:]
    return dict(np.load(path))


@pytest.mark.parametrize("n", GRIDS)
def test_jittered_build_is_bitwise_identical(n, tmp_path):
    jit = os.path.join(PKG, "libfgd_jitter.so")
    if not os.path.exists(jit):
        from paper_2103_04770_b200 import build
        build.build(jitter=True)
    a = run(os.path.join(PKG, "libfgd.so"), n, str(tmp_path / "prod.npz"))
    b = run(jit, n, str(tmp_path / "jit.npz"))
    bad = [k for k in a if not np.array_equal(a[k], b[k])]
    assert not bad, {k: float(np.abs(a[k] - b[k]).max()) for k in bad}
