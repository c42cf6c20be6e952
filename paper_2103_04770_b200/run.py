"""Full loading runs through the library's increment solver (fgd_solve_increment): the staggered
Alg. 1 per increment, fixed strain increments with deterministic halving on non-convergence
(A-21: up to 6 halvings), the BASELINE configurations 0, 2 and 3 and the non-local GTN cells of the paper's Sec. 4.1 / 4.2
(`synth.config_gtn2d`, `synth.config_gtn3d`) from `synth`.

    python -m paper_2103_04770_b200.run --config 3 [--n 128] [--incr 60] [--tight]
    python -m paper_2103_04770_b200.run --config 4 [--n 512] --incr 4 --log   (first increments of the 512^3 cell)
    python -m paper_2103_04770_b200.run --config gtn2d [--n 64] [--de 2.5e-3] [--incr 200]

prints one JSON line: the macroscopic stress-strain curve (load component), the peak, the strain
at 50 % post-peak drop (A-26), the increment / staggered / Newton / CG / PCG counts and the wall
time.  Default solver tolerances are the performance-run values of SURVEY 8(c) (1e-4 staggered,
1e-6 Newton, 1e-8 CG, 1e-6 PCG); --tight uses the parity-run values.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np


def _context(cfg):
    import torch

    from . import Context, Material
    ctx = Context(cfg.n, cfg.L)
    ctx.set_phases(torch.from_numpy(np.ascontiguousarray(cfg.phases)).cuda(), len(cfg.materials))
    for q, m in enumerate(cfg.materials):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(np.asarray(cfg.ell), cfg.source_phase)
    ctx.set_control(cfg.stress_mask)
    return ctx


def adaptive_schedule(solve, E_end, dE0, dE_max=None, dE_min=1e-5, grow=1.5, grow_after=2, stop=None):
    """Adaptive incrementation (the paper's "variable strain increment",
    P:990, rule A-34 of DESIGN.md): try dE = min(step, E_end - E); on failure halve the step and
    retry from the last converged state; after `grow_after` consecutive first-try successes
    multiply the step by `grow` (at most dE_max = dE0 by default).  Stops with failure when the
    step falls below dE_min.  `solve(E) -> bool` runs one increment to macroscopic strain E (and
    commits it on success); `stop() -> bool` (optional) ends the run early after an accepted
    increment.  Returns (accepted strains, number of cutbacks, reached E_end or stopped)."""
    dE_max = dE0 if dE_max is None else dE_max
    E, step, streak, cuts, accepted = 0.0, dE0, 0, 0, []
    while E < E_end - 1e-15:
        dE = min(step, E_end - E)
        if solve(E + dE):
            E += dE
            accepted.append(E)
            if stop is not None and stop():
                return accepted, cuts, True
            streak += 1
            if streak >= grow_after:
                step = min(step * grow, dE_max)
                streak = 0
        else:
            cuts += 1
            streak = 0
            step *= 0.5
            if step < dE_min:
                return accepted, cuts, False
    return accepted, cuts, True


def run_config(cfg, n_incr=None, tol=(1e-4, 1e-6, 1e-8, 1e-6), max_halvings=6, max_cg=5000, max_helm=5000,
               adaptive=False, de_min=1e-5, log=False, grow=1.5, stop_frac=None, max_stag=100, warm=False,
               max_newton=50, profile=None, stag_stall=0):
    """Load the cell along cfg.load_comp to n_incr * cfg.dE: fixed increments with deterministic
    halving (A-21), or the adaptive schedule (A-34); returns a result dict."""
    import torch

    from . import _fgd
    n_incr = cfg.n_incr if n_incr is None else n_incr
    ctx = _context(cfg)
    tol_stag, tol_newton, tol_cg, tol_helm = tol
    E_done = 0.0
    curve = [(0.0, 0.0)]
    counts = dict(increments=0, substeps=0, stag=0, newton=0, cg=0, helm=0, failed=0)
    torch.cuda.synchronize()
    t0 = time.perf_counter()

    def solve(E_try):
        Et = np.zeros(6)
        Et[cfg.load_comp] = E_try
        st, rep = ctx.solve_increment(Et, np.zeros(6), tol_stag, tol_newton, tol_cg, tol_helm,
                                      max_stag=max_stag, max_newton=max_newton, max_cg=max_cg, max_helm=max_helm,
                                      warm_start=warm, stag_stall=stag_stall)
        for k in ("stag", "newton", "cg", "helm"):
            counts[k] += rep[k]
        if log and st != 0:
            print(json.dumps({"E_try": E_try, "failed": True, "stag": rep["stag"], "newton": rep["newton"],
                              "cg": rep["cg"], "helm": rep["helm"], "err": rep["err"]}), file=sys.stderr, flush=True)
        if st == 0:
            counts["substeps"] += 1
            curve.append((E_try, float(rep["macro_stress"][cfg.load_comp])))
            if log:   # one line per accepted increment: a run cut short still leaves its curve
                print(json.dumps({"E": E_try, "S": curve[-1][1], "t": time.perf_counter() - t0, "stag": rep["stag"],
                                  "newton": rep["newton"], "cg": rep["cg"], "helm": rep["helm"], "err": rep["err"]}),
                      file=sys.stderr, flush=True)
            return True
        if st != _fgd.ENOCONV:
            raise RuntimeError(f"solve_increment failed with status {st}")
        return False

    def stop():
        if stop_frac is None:
            return False
        sv = [c[1] for c in curve]
        return max(sv) > 0 and sv[-1] < stop_frac * max(sv)

    if adaptive:
        acc, cuts, ok = adaptive_schedule(solve, n_incr * cfg.dE, cfg.dE, dE_min=de_min, grow=grow, stop=stop)
        counts.update(increments=len(acc), cutbacks=cuts, failed=int(not ok))
        n_incr = 0
    for i in range(1, n_incr + 1):
        E_goal = i * cfg.dE
        step = cfg.dE
        halvings = 0
        while E_done < E_goal - 1e-15:
            E_try = min(E_done + step, E_goal)
            Et = np.zeros(6)
            Et[cfg.load_comp] = E_try
            st, rep = ctx.solve_increment(Et, np.zeros(6), tol_stag, tol_newton, tol_cg, tol_helm,
                                          max_stag=max_stag, max_newton=max_newton, max_cg=max_cg, max_helm=max_helm,
                                          warm_start=warm, stag_stall=stag_stall)
            counts["stag"] += rep["stag"]
            counts["newton"] += rep["newton"]
            counts["cg"] += rep["cg"]
            counts["helm"] += rep["helm"]
            if st == 0:
                E_done = E_try
                counts["substeps"] += 1
                curve.append((E_try, float(rep["macro_stress"][cfg.load_comp])))
                if log:
                    print(json.dumps({"E": E_try, "S": curve[-1][1], "t": time.perf_counter() - t0,
                                      "cg": counts["cg"], "helm": counts["helm"]}), file=sys.stderr, flush=True)
            elif st == _fgd.ENOCONV and halvings < max_halvings:
                step *= 0.5
                halvings += 1
            else:
                counts["failed"] = 1
                break
        if counts["failed"]:
            break
        counts["increments"] += 1
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    prof = _profiles(ctx, cfg) if profile else None
    ctx.close()
    e = np.array([c[0] for c in curve])
    s = np.array([c[1] for c in curve])
    ip = int(np.argmax(s))
    fail = None
    for k in range(ip + 1, len(s)):          # first crossing of 50 % of the peak, linear (A-26)
        if s[k] < 0.5 * s[ip]:
            f = (s[k - 1] - 0.5 * s[ip]) / (s[k - 1] - s[k])
            fail = float(e[k - 1] + f * (e[k] - e[k - 1]))
            break
    return dict(config=cfg.name, n=list(cfg.n), load_comp=cfg.load_comp, dE=cfg.dE, wall_s=wall,
                peak_stress=float(s[ip]), strain_at_peak=float(e[ip]), strain_at_failure=fail,
                curve=[[float(a), float(b)] for a, b in curve], tolerances=list(tol), max_cg=max_cg,
                max_halvings=max_halvings, adaptive=adaptive, max_stag=max_stag, warm_start=warm, stag_stall=stag_stall,
                ell=np.asarray(cfg.ell).tolist(), **({"profile": prof} if prof else {}), **counts)


def _profiles(ctx, cfg):
    """Committed fields along the row through the cell centre, from the centre to the cell edge
    (the paper's direction r, Fig. impactelli: profiles across the matrix/inclusion
    interface): non-local field 0 (the regularised eps0p / eps_p) and the history variable (GTN:
    porosity f; J2: damage).  Read-back only -- the fields are the library's."""
    import torch

    from . import _fgd
    n1, n2, n3 = cfg.n
    out = torch.empty((n3, n2, n1), dtype=torch.float64, device="cuda")
    row = {}
    for name, fid in (("nonlocal0", _fgd.FIELD_NONLOCAL + 0), ("hist", _fgd.FIELD_HIST), ("eqps", _fgd.FIELD_EQPS)):
        ctx.get_field(fid, out)
        row[name] = out[n3 // 2, n2 // 2, n1 // 2:].cpu().numpy().tolist()
    row["x_over_L"] = [((i + 0.5) / n1 - 0.5) for i in range(n1 // 2, n1)]
    row["phase"] = np.asarray(cfg.phases).reshape(n3, n2, n1)[n3 // 2, n2 // 2, n1 // 2:].astype(int).tolist()
    return row


def main(argv=None):
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import synth
    p = argparse.ArgumentParser()
    p.add_argument("--config", default="0", choices=["0", "2", "3", "4", "gtn2d", "gtn3d"])
    p.add_argument("--de", type=float, default=None, help="override the fixed strain increment")
    p.add_argument("--n", type=int, default=None)
    p.add_argument("--incr", type=int, default=None)
    p.add_argument("--tight", action="store_true")
    p.add_argument("--max-cg", type=int, default=5000)
    p.add_argument("--halvings", type=int, default=6)
    p.add_argument("--adaptive", action="store_true", help="adaptive increments (A-34) instead of fixed + halving")
    p.add_argument("--log", action="store_true", help="one JSON line per accepted increment on stderr")
    p.add_argument("--grow", type=float, default=1.5, help="adaptive: step growth after two first-try successes")
    p.add_argument("--stop-frac", type=float, default=None,
                   help="adaptive: stop once the load stress falls below this fraction of the peak")
    p.add_argument("--max-stag", type=int, default=100)
    p.add_argument("--warm", action="store_true", help="warm-started Helmholtz PCG (S:262)")
    p.add_argument("--stag-stall", type=int, default=0,
                   help="fail an increment once ERR has not improved for this many staggered iterations (0: off)")
    p.add_argument("--max-newton", type=int, default=50)
    p.add_argument("--ell", type=float, default=None,
                   help="gtn2d: matrix ell_M / L (ell_I = min(ell_M, 0.001 L); 1e-4 gives the local variant)")
    p.add_argument("--ell-i", type=float, default=None,
                   help="gtn2d: inclusion ell_I / L (interface-contrast study P:941-952; default min(ell_M, 0.001 L))")
    p.add_argument("--profile", action="store_true",
                   help="add the committed non-local / history fields along the centre row to the result")
    a = p.parse_args(argv)
    if a.config == "0":
        cfg = synth.config0(a.n or 32)
    elif a.config == "2":
        cfg = synth.config2(a.n or 256)
    elif a.config == "3":
        cfg = synth.config3(n=a.n or 128)
    elif a.config == "4":
        cfg = synth.config4(n=a.n or 512)
    elif a.config == "gtn2d":
        ell = a.ell if a.ell else 0.05
        cfg = synth.config_gtn2d(a.n or 64, ell_over_L=ell, ell_i_over_L=a.ell_i if a.ell_i else min(ell, 0.001))
    else:
        cfg = synth.config_gtn3d(a.n or 32)
    if a.de:
        cfg.dE = a.de
    tol = (1e-8, 1e-10, 1e-11, 1e-11) if a.tight else (1e-4, 1e-6, 1e-8, 1e-6)
    print(json.dumps(run_config(cfg, a.incr, tol, a.halvings, a.max_cg, a.max_cg, adaptive=a.adaptive, log=a.log,
                                grow=a.grow, stop_frac=a.stop_frac, max_stag=a.max_stag, warm=a.warm, stag_stall=a.stag_stall,
                                max_newton=a.max_newton, profile=a.profile)), flush=True)


if __name__ == "__main__":
    main()
