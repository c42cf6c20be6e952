#!/usr/bin/env python
"""Writes the oracle's macroscopic load curves of the BASELINE configurations (golden files for
the config-level GPU parity tests, tests/test_gpu_curves.py).

TEST INFRASTRUCTURE: calls only `oracle/` (and the seeded input recipes of `synth/`, which hold
none of the method's arithmetic).  No value here comes from the CUDA path.

Each case runs Algorithm 1 (oracle.increment.solve_increment) increment by increment
at the parity tolerances of SURVEY 8(c) (TOL_s 1e-8, Newton 1e-10, CG 1e-11, PCG 1e-11) along the
nominal ramp of the configuration (A-21: fixed dE), with deterministic halving on
non-convergence: a failed step is retried at half the size from the last converged state, and
the step grows back (x2) after two consecutive first-try successes, never beyond the nominal dE
(the adaptive rule A-34 with a power-of-two step so that every accepted target is exactly
representable).  The ACCEPTED targets are stored, so the GPU test replays exactly the same
sequence of increments and compares <sigma> at each.

Stored per case: the accepted targets E (load component), the full <sigma> (6 Mandel comps) and
<eps> of every accepted increment, the staggered / Newton / CG / PCG counts, the peak of the
load-component stress, the strain at 50 % post-peak drop (A-26, linear interpolation) and the
run's wall time.  A run stops at the end of the ramp, when the load stress has fallen below
`stop_frac` of the peak (the failure strain is then known), or when the step falls below dE_min
(the record says so: "stalled").

    python tests/golden/make_oracle_curves.py config0_32      # -> tests/golden/curve_config0_32.json
    python tests/golden/make_oracle_curves.py config2_256 --E-max 0.0056   # the pre-peak part only
    python tests/golden/make_oracle_curves.py --list
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle.increment import State, Tolerances, make_cell, solve_increment  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
PARITY_TOL = Tolerances(tol_stag=1e-8, tol_newton=1e-10, tol_cg=1e-11, tol_helm=1e-11, max_stag=100,
                        max_newton=50, max_cg=20000, max_helm=20000)


def cases():
    """name -> (config builder, number of nominal increments or None for the config's ramp)."""
    return {
        # BJ config 0: 32^2 disc, ell_M = 2h = L/16 (also config 2's 32^2 objectivity run, A-13)
        "config0_32": (lambda: synth.config0(32), None),
        # config 2's objectivity runs: ell = L/16 in physical units (A-13)
        "config2_64": (lambda: synth.config2(64), None),
        # BJ config 2 itself (256^2, ell = L/16 = 16h): the oracle run that classifies the GPU's
        # post-peak stall at this size (hours of CPU; not used by the GPU test unless present)
        "config2_256": (lambda: synth.config2(256), None),
        # reduced config 3: 32^3 RSA cell (30 spheres, 20 %), ell_m = 5h, ell_p = 3h, E_zz ramp
        "config3_32": (lambda: synth.config3(n=32), None),
        # BJ config 3 at its own size (128^3, 30 spheres): the first increments only (--incr 2; every
        # oracle CG iteration at this size takes seconds)
        "config3_128": (lambda: synth.config3(n=128), None),
        # small cells for quick checks of the generator itself
        "config0_16": (lambda: synth.config0(16, ell_over_L=1.0 / 8.0), None),
    }


def failure_strain(E, S):
    """First crossing of 50 % of the peak after the peak, linear interpolation (A-26)."""
    ip = int(np.argmax(S))
    for k in range(ip + 1, len(S)):
        if S[k] < 0.5 * S[ip]:
            f = (S[k - 1] - 0.5 * S[ip]) / (S[k - 1] - S[k])
            return float(E[k - 1] + f * (E[k] - E[k - 1]))
    return None


def run_case(name, stop_frac=0.3, de_min_halvings=8, log=None, n_incr=None, E_max=None):
    build, nin = cases()[name]
    cfg = build()
    n_incr = n_incr or nin or cfg.n_incr
    cell = make_cell(cfg)
    state = State.zero(cell)
    E_end = n_incr * cfg.dE
    step_min = cfg.dE / 2 ** de_min_halvings
    E, step, streak = 0.0, cfg.dE, 0
    recs = []
    cut = 0
    stalled = False
    t0 = time.perf_counter()
    while E < E_end - 1e-15:
        dE = min(step, E_end - E)
        Et = np.zeros(6)
        Et[cfg.load_comp] = E + dE
        st2, rep = solve_increment(cell, state, Et, np.zeros(6), PARITY_TOL)
        if rep.converged:
            state = st2
            E = E + dE
            rec = dict(E=E, stress=[float(v) for v in rep.macro_stress], strain=[float(v) for v in rep.macro_strain],
                       stag=rep.stag_it, newton=rep.newton_it, cg=rep.cg_it, helm=rep.helm_it,
                       t=time.perf_counter() - t0)
            recs.append(rec)
            if log:
                log(rec)
            streak += 1
            if streak >= 2 and step < cfg.dE:
                step *= 2.0
                streak = 0
            S = np.array([r["stress"][cfg.load_comp] for r in recs])
            if S.max() > 0 and S[-1] < stop_frac * S.max():
                break
            if E_max is not None and E >= E_max - 1e-15:
                break
        else:
            cut += 1
            streak = 0
            if log:
                log(dict(E_try=E + dE, failed=True, stag=rep.stag_it, newton=rep.newton_it, cg=rep.cg_it,
                         err=float(rep.err), err_hist=[float(v) for v in rep.err_hist[-5:]]))
            step *= 0.5
            if step < step_min:
                stalled = True
                break
    Ev = np.array([0.0] + [r["E"] for r in recs])
    Sv = np.array([0.0] + [r["stress"][cfg.load_comp] for r in recs])
    ip = int(np.argmax(Sv))
    return dict(case=name, config=cfg.name, n=list(cfg.n), load_comp=cfg.load_comp, dE=cfg.dE, n_incr=n_incr,
                tolerances=dict(tol_stag=PARITY_TOL.tol_stag, tol_newton=PARITY_TOL.tol_newton,
                                tol_cg=PARITY_TOL.tol_cg, tol_helm=PARITY_TOL.tol_helm,
                                max_stag=PARITY_TOL.max_stag, max_newton=PARITY_TOL.max_newton,
                                max_cg=PARITY_TOL.max_cg, max_helm=PARITY_TOL.max_helm,
                                warm_start=PARITY_TOL.warm_start, line_search=PARITY_TOL.line_search),
                schedule="halve on failure, x2 after 2 first-try successes, <= dE", cutbacks=cut,
                stalled=stalled, peak_stress=float(Sv[ip]), strain_at_peak=float(Ev[ip]),
                peak_index=ip - 1, strain_at_failure=failure_strain(Ev, Sv),
                wall_s=time.perf_counter() - t0, increments=recs,
                source="oracle/ (NumPy/SciPy FP64) via tests/golden/make_oracle_curves.py")


def main():
    p = argparse.ArgumentParser()
    p.add_argument("case", nargs="?")
    p.add_argument("--list", action="store_true")
    p.add_argument("--out", default=None)
    p.add_argument("--incr", type=int, default=None)
    p.add_argument("--stop-frac", type=float, default=0.3)
    p.add_argument("--E-max", type=float, default=None, help="stop after the increment reaching this strain")
    a = p.parse_args()
    if a.list or not a.case:
        print("\n".join(cases()))
        return
    out = a.out or os.path.join(HERE, f"curve_{a.case}.json")

    def log(r):
        print(json.dumps(r), file=sys.stderr, flush=True)

    res = run_case(a.case, stop_frac=a.stop_frac, log=log, n_incr=a.incr, E_max=a.E_max)
    res["E_max"] = a.E_max
    with open(out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps({k: v for k, v in res.items() if k != "increments"}))


if __name__ == "__main__":
    main()
