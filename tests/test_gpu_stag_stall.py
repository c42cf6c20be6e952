"""fgd_increment.stag_stall: early exit of a staggered loop whose ERR no longer improves
(the caller's cue to cut the step back, A-34).  Off (0) is Algorithm 1 as printed; a generous
window changes nothing; a stalled loop rolls back like any other failed increment."""
from __future__ import annotations

import os
import sys

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import synth  # noqa: E402
from oracle.increment import State, Tolerances, make_cell, solve_increment  # noqa: E402
from paper_2103_04770_b200 import Context, Material  # noqa: E402
from paper_2103_04770_b200 import _fgd  # noqa: E402

TOL = Tolerances()


def ctx_from_cfg(cfg):
    ctx = Context(cfg.n, cfg.L)
    ctx.set_phases(torch.from_numpy(np.ascontiguousarray(cfg.phases)).cuda(), len(cfg.materials))
    for q, m in enumerate(cfg.materials):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
    ctx.set_control(cfg.stress_mask)
    return ctx


def test_stag_stall_window():
    cfg = synth.config0(16, ell_over_L=2.0 / 16)
    cfg.dE = 8e-4
    cell = make_cell(cfg)
    st = State.zero(cell)
    a, b = ctx_from_cfg(cfg), ctx_from_cfg(cfg)
    args = (TOL.tol_stag, TOL.tol_newton, TOL.tol_cg, TOL.tol_helm, TOL.max_stag, TOL.max_newton, TOL.max_cg,
            TOL.max_helm)
    for i in range(1, 6):
        Et = np.zeros(6)
        Et[cfg.load_comp] = i * cfg.dE
        st, rep = solve_increment(cell, st, Et, np.zeros(6), TOL)
        sa, ra = a.solve_increment(Et, np.zeros(6), *args)
        sb, rb = b.solve_increment(Et, np.zeros(6), *args, stag_stall=1000)
        assert sa == 0 and sb == 0
        # a window that is never reached changes nothing
        assert np.array_equal(ra["macro_stress"], rb["macro_stress"]) and ra["stag"] == rb["stag"]
        assert np.linalg.norm(ra["macro_stress"] - rep.macro_stress) <= 1e-6 * np.linalg.norm(rep.macro_stress)
    # a loop that cannot meet its tolerance (tol_stag = 0) stops improving at the rounding floor:
    # with the window on it gives up long before max_stag, rolls back, and the next increment from
    # the committed state is the one a clean context computes
    Et = np.zeros(6)
    Et[cfg.load_comp] = 6 * cfg.dE
    args0 = (0.0,) + args[1:4] + (60,) + args[5:]
    sb, rb = b.solve_increment(Et, np.zeros(6), *args0, stag_stall=3)
    assert sb == _fgd.ENOCONV and 3 <= rb["stag"] < 60, rb
    sa, ra = a.solve_increment(Et, np.zeros(6), *args)
    sb, rb = b.solve_increment(Et, np.zeros(6), *args, stag_stall=1000)
    assert sa == 0 and sb == 0
    assert np.array_equal(ra["macro_stress"], rb["macro_stress"]) and ra["stag"] == rb["stag"]
    a.close()
    b.close()
