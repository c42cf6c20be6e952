#!/usr/bin/env python
"""Benchmark of the FFT-Galerkin / Helmholtz Krylov hot path (BASELINE.json metric:
"FP64 FFT-Galerkin Krylov voxel*iter/s at 256^3/512^3; % of HBM roofline").

One STEP = one staggered Krylov sweep over the whole hot path on
the BASELINE config-1 recipe at the metric size (default 512^3, the cell of the multi-GPU
target, so that the N = 1 line and the scaling lines measure the same cell; --size 256 for 256^3;
on one GPU the other size is measured too and reported under "by_size"):
  a1      constitutive update at the strain field (J2-Lemaitre matrix / elastic inclusion,
          damage frozen from the non-local field) -> sigma, consistent tangent, source alpha
  a3-a5   Newton residual b = -G*(sigma - Sigma_bar)  (5-pass FFT with the projection)
  a2-a6   KCG mechanical CG iterations  (5 fused passes per iteration)
  a7-a9   KH Helmholtz PCG iterations   (27-point stencil + 5-pass preconditioner)
  a10     the device reductions inside the above
value = N_vox * KCG / (step time)  [voxel*iter/s of the mechanical Krylov solver], all ranks.
Inputs are generated on the device (seeded) and stay resident; every field (134 MB/comp at
256^3) and the tangent (2.8 GB) exceed the 126 MB L2, so no explicit flush is needed.
--gpus N without a torchrun environment re-executes itself under torch.distributed.run (N ranks,
one per GPU, 127.0.0.1); the cell is slab-decomposed over the ranks (strong scaling).

--impl reference: the CPU oracle (oracle/, NumPy/SciPy FP64) on a bounded 64^3 sample of the
same recipe, same metric and unit.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "FP64 FFT-Galerkin Krylov voxel·iter/s at 256³/512³; % of HBM roofline"
UNIT = "voxel*iter/s"
CPU_SAMPLE_N = 64          # --impl reference: one sweep per step (keeps the K-step arm within minutes)
CPU_BASELINE_N = 128       # cpu_baseline of our line: the config-1 size (an out-of-cache sample, ~20 s)


def args_():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="ours", choices=["ours", "reference"])
    p.add_argument("--size", dest="n", type=int, default=512, help="cell edge (voxels)")
    p.add_argument("--no-by-size", action="store_true", help="skip the second metric size (256^3 / 512^3)")
    p.add_argument("--kcg", type=int, default=10)
    p.add_argument("--khelm", type=int, default=10)
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--no-cufft", action="store_true", help="skip the cuFFT comparison arm")
    p.add_argument("--no-gtn", action="store_true", help="skip the GTN constitutive measurement")
    return p.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def workload_name(n):
    return (f"config-1 recipe at {n}^3: Bernoulli(0.2) phases (J2-Lemaitre matrix / elastic inclusion), "
            f"strain ~N(0,1e-3), one non-local field l=(2,4) voxels, mask (1,1,0,1,1,1)")


# ---------------------------------------------------------------------------------------------
# reference arm / cpu baseline: the oracle
# ---------------------------------------------------------------------------------------------
def oracle_sweep(n, kcg, khelm):
    import numpy as np

    import synth
    from oracle.helmholtz import ell2_field, solve_helmholtz
    from oracle.increment import Cell, State, evaluate, frozen_damage
    from oracle.mech import cg
    from oracle.projection import apply_projection
    from oracle.spectral import Grid

    g = Grid((n, n, n), (float(n),) * 3)
    ph = synth.config1_phases(n, 0)
    cell = Cell(g, ph, [synth.MATRIX_J2, synth.INCLUSION_EL], synth.CONFIG1_ELL, [0], synth.CONFIG1_MASK)
    st = State.zero(cell)
    eps = synth.gaussian_field(6, g.shape, 1e-3, 2)
    e2 = ell2_field(ph, synth.CONFIG1_ELL[0])

    def step():
        D = frozen_damage(cell, st, st.abar)
        sig, C, alpha, _, _ = evaluate(cell, eps, st, D)
        b = -apply_projection(g, sig, cell.stress_mask)
        cg(g, C, b, cell.stress_mask, tol=0.0, maxit=kcg)
        solve_helmholtz(g, alpha[0], e2, tol=0.0, maxit=khelm)

    return step


def cpu_baseline(kcg, khelm, reps=1):
    step = oracle_sweep(CPU_BASELINE_N, kcg, khelm)
    step()
    ts = []
    for _ in range(reps):
        t = time.perf_counter()
        step()
        ts.append(time.perf_counter() - t)
    t = statistics.median(ts)
    return {"value": CPU_BASELINE_N ** 3 * kcg / t, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
            "sample": f"one sweep of the same recipe at {CPU_BASELINE_N}^3 ({kcg} CG + {khelm} PCG iterations), "
                      f"median of {reps}, scipy.fft workers={os.cpu_count()}; {t:.2f} s per sweep"}


def run_reference(a):
    rank, world, _ = dist_env()
    if rank != 0:
        return
    # sample size: 128^3 (out of cache, ~12 s per sweep on 16 cores: the honest per-voxel rate) while the
    # whole run stays within a few minutes, else the 64^3 sweep (~1.2 s)
    ns = 128
    step = oracle_sweep(ns, a.kcg, a.khelm)
    t = time.perf_counter()
    step()                                        # first sweep: decides the sample, counts as warm-up
    if (a.steps + a.warmup) * (time.perf_counter() - t) > 320.0:
        ns = CPU_SAMPLE_N
        step = oracle_sweep(ns, a.kcg, a.khelm)
        step()
    for _ in range(a.warmup - 1):
        step()
    t = time.perf_counter()
    for _ in range(a.steps):
        step()
    dt = (time.perf_counter() - t) / a.steps
    v = ns ** 3 * a.kcg / dt
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": a.gpus, "steps": a.steps,
            "warmup": a.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_name(a.n), "sample_n": ns, "kcg": a.kcg, "khelm": a.khelm},
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": os.cpu_count(), "kind": "oracle",
                             "sample": f"each step = one sweep at {ns}^3 of the same recipe"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------------------------
# clocks sampler
# ---------------------------------------------------------------------------------------------
class Clocks:
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
    NAMES = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")

    def __init__(self, dev):
        self.dev = dev
        self.p = None
        self.lines = []

    def start(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                                       "-i", str(self.dev), "-lms", "200"], stdout=subprocess.PIPE,
                                      stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.p = None

    def _read(self):
        for ln in self.p.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.p:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.p.terminate()
        try:
            self.p.wait(timeout=2)
        except Exception:
            self.p.kill()
        sm, mx, reasons = [], [], set()
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 6:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for name, v in zip(self.NAMES, f[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------------------------
def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, STREAM-style copy)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


# kernel of each class in the ncu summaries (first candidate present in the newest summary wins)
TRAFFIC_KERNEL = {"xfwd6cg": ["k_xtan_pp<{n}, 2, 1>", "k_xtan<{n}, 2, 1, 2>"], "xinv6": ["k_xipipe<{n}, 1>"],
                  "stencil": ["k_stencil<1, 4, 1, 2>", "k_stencil<1, 2>"],
                  "z6": ["k_zreg512w<6, 0, 0, 1>", "k_zreg512w<6, 0, 0>", "k_zreg256<6, 0, 0>", "k_zreg256<6, 0>"],
                  "yfwd6": ["k_yreg512w", "k_yreg512<0>", "k_yreg256<0>"],
                  "yinv6": ["k_yreg512i", "k_yreg256<1>"]}


def measured_traffic(cls, n):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the class's main
    kernel from the newest committed `ncu --set full` summary (profiles/r*_traffic.json), or None."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_traffic.json")))
    if not files or cls not in TRAFFIC_KERNEL:
        return None, None
    d = json.load(open(files[-1]))
    for k in TRAFFIC_KERNEL[cls]:
        k = k.format(n=n)
        if (str(n) in k or cls == "stencil") and k in d:
            return d[k], os.path.basename(files[-1]) + ":" + k
    return None, None


def class_bytes(n, kcg, khelm, world=1):
    """Algorithmic (compulsory) bytes per STEP and per rank for each kernel class of the fused
    5-pass design.  S = spectral bytes of one component (16 B x Hx*Ny*Nz).
    x forward, 6 comps:
      xfwd6   = residual pass (read sigma 48 B/voxel + write 6S) + the FIRST CG tangent launch,
                which reads r = b (48) and the compact tangent (72) and writes p, x (96) + 6S --
                it reads neither p_old nor x (216 B/voxel + 6S);
      xfwd6cg = every later CG tangent launch (the steady launch): read r, p_old, x (144) +
                compact tangent (72), write p, x (96) + 6S = 312 B/voxel + 6S (~360 B/voxel).
    y/z passes: read + write of the 6-comp spectrum (2 x 6S) per apply.  x inverse: 6S + r
    read/write (96) per CG iteration, 6S + write b (48) for the residual.  1-comp analogues for
    the PCG; stencil 33 B/voxel; constitutive ~300 B/voxel."""
    V = n ** 3 // world
    S = 16 * (n // 2 + 1) * n * n // world
    b = {}
    TB = 72                                                                       # compact J2 tangent (9 doubles)
    b["xfwd6"] = (48 * V + 6 * S) + (1 if kcg > 0 else 0) * ((48 + TB + 96) * V + 6 * S)
    b["xfwd6cg"] = max(0, kcg - 1) * ((144 + TB + 96) * V + 6 * S)
    b["yfwd6"] = b["yinv6"] = b["z6"] = (1 + kcg) * 2 * 6 * S
    b["xinv6"] = (6 * S + 48 * V) + kcg * (6 * S + 96 * V)                      # residual store + CG r update
    b["xfwd1"] = (8 * V + S) + khelm * (32 * V + 16 * V + S)                      # precond init + PCG x/r update
    b["yfwd1"] = b["yinv1"] = b["z1"] = (1 + khelm) * 2 * S
    b["xinv1"] = (1 + khelm) * (S + 16 * V)
    b["stencil"] = khelm * 33 * V
    b["constitutive"] = (48 + 48 + 8 + 8 + 8 + 1 + 48 + TB + 8) * V
    return b


# ---------------------------------------------------------------------------------------------
# measured comparison: the projected-tangent apply through cuFFT (torch.fft) + torch elementwise
# ---------------------------------------------------------------------------------------------
def cufft_comparison(ctx, n, dev, mask, reps=5):
    """y = G*(C:x) built from library pieces -- torch.einsum for C:x, torch.fft.rfftn /
    irfftn (cuFFT) for the transforms, torch elementwise ops for the Galerkin projection with the
    Willot symbol (A-04) -- against the library's fused 5-pass apply on the same x and tangent.
    A comparison arm only (north_star: "a cuFFT-based path is kept only as a measured comparison")."""
    import torch
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    x = torch.randn((6, n, n, n), generator=g, dtype=torch.float64, device=dev) * 1e-3
    Cp = torch.empty((21, n, n, n), dtype=torch.float64, device=dev)
    ctx.get_field(5, Cp)                      # FGD_FIELD_TANGENT (packed upper triangle, Mandel)
    y = torch.empty_like(x)

    def timeit(fn):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps

    t_ours = timeit(lambda: ctx.apply_projected_tangent(x, y))
    pk = {}
    t = 0
    for i in range(6):
        for j in range(i, 6):
            pk[(i, j)] = pk[(j, i)] = t
            t += 1
    idx = torch.tensor([pk[(i, j)] for i in range(6) for j in range(6)], device=dev)
    Cf = Cp.view(21, -1).index_select(0, idx).view(6, 6, -1)
    del Cp
    h = 1.0                                    # L = n, N = n
    def cis(m):
        # e^{2 pi i m / n} with the quarter points exact, so that the rotated-scheme null modes
        # (1 + e^{i pi} = 0) are exactly zero as in the library's tables
        th = 2 * math.pi * m.to(torch.float64) / n
        c, s_ = torch.cos(th), torch.sin(th)
        q = (4 * m) % n == 0
        quarter = (4 * m) // n % 4
        c = torch.where(q, torch.tensor([1.0, 0.0, -1.0, 0.0], dtype=torch.float64, device=dev)[quarter], c)
        s_ = torch.where(q, torch.tensor([0.0, 1.0, 0.0, -1.0], dtype=torch.float64, device=dev)[quarter], s_)
        return torch.complex(c, s_)

    mm = torch.arange(n, device=dev)
    ex = cis(mm[: n // 2 + 1]).view(1, 1, -1)
    ey = cis(mm).view(1, -1, 1)
    ez = cis(mm).view(-1, 1, 1)
    k0 = (ex - 1) * (1 + ey) * (1 + ez) / (4 * h)
    k1 = (1 + ex) * (ey - 1) * (1 + ez) / (4 * h)
    k2 = (1 + ex) * (1 + ey) * (ez - 1) / (4 * h)
    kk = (k0.abs() ** 2 + k1.abs() ** 2 + k2.abs() ** 2)
    inv = torch.where(kk > 0, 1.0 / torch.where(kk > 0, kk, torch.ones_like(kk)), torch.zeros_like(kk))
    r2 = math.sqrt(2.0)
    mk = torch.tensor([float(m) for m in mask], device=dev, dtype=torch.float64)
    yt = torch.empty_like(x)

    def torch_apply():
        tau = torch.einsum("ijv,jv->iv", Cf, x.view(6, -1)).view(6, n, n, n)
        T = torch.fft.rfftn(tau, dim=(1, 2, 3))
        dc = T[:, 0, 0, 0].clone()
        T00, T11, T22, T12, T02, T01 = T[0], T[1], T[2], T[3] / r2, T[4] / r2, T[5] / r2
        c0, c1, c2 = k0.conj(), k1.conj(), k2.conj()
        t0 = T00 * c0 + T01 * c1 + T02 * c2
        t1 = T01 * c0 + T11 * c1 + T12 * c2
        t2 = T02 * c0 + T12 * c1 + T22 * c2
        sv = c0 * t0 + c1 * t1 + c2 * t2
        hs = sv * (0.5 * inv)
        u0, u1, u2 = (t0 - k0 * hs) * (2 * inv), (t1 - k1 * hs) * (2 * inv), (t2 - k2 * hs) * (2 * inv)
        out = torch.stack([u0 * k0, u1 * k1, u2 * k2, (u1 * k2 + k1 * u2) / r2, (u0 * k2 + k0 * u2) / r2,
                           (u0 * k1 + k0 * u1) / r2])
        out[:, 0, 0, 0] = dc * mk
        yt.copy_(torch.fft.irfftn(out, s=(n, n, n), dim=(1, 2, 3)))

    t_torch = timeit(torch_apply)
    rel = float(torch.linalg.vector_norm(yt - y) / torch.linalg.vector_norm(y))
    del Cf
    torch.cuda.empty_cache()
    return {"what": "projected-tangent apply y = G*(C:x) at %d^3: torch.einsum + torch.fft (cuFFT) + torch "
                    "elementwise projection vs the fused 5-pass library apply, same x and tangent" % n,
            "ms_per_apply_cufft_torch": t_torch, "ms_per_apply_ours": t_ours, "speedup": t_torch / t_ours,
            "rel_diff": rel}


GTN_BYTES_PER_VOXEL = (48 + 48 + 8 + 8 + 1 + 16 + 16) + (48 + 72 + 16)   # K1 reads + writes (GTN)


def gtn_measurement(n, dev, peak, reps=5):
    """The non-local GTN constitutive update (material model 3) at the bench
    size: config-1 phases with the Sec. 4.2 GTN matrix, a random committed state that puts most
    matrix voxels on the yield surface across all f* branches, timed by the library's event pair
    around the kernel."""
    import numpy as np
    import torch

    import synth
    from paper_2103_04770_b200 import Context, Material
    from paper_2103_04770_b200 import _fgd
    V = n ** 3
    f64 = torch.float64
    ctx = Context((n, n, n), (1.0, 1.0, 1.0), device=dev.index)
    ctx.set_phases(torch.from_numpy(synth.config1_phases(n, 0)).to(dev), 2)
    mg = synth.MATRIX_GTN_3D
    ctx.set_material(0, Material.of(mg))
    ctx.set_material(1, Material.of(synth.INCLUSION_EL))
    ctx.set_nonlocal(np.array([[0.05, 0.001], [0.05, 0.001]]), [0, 0])
    ctx.set_control(synth.CONFIG1_MASK)
    g = torch.Generator(device=dev)
    g.manual_seed(4321)
    ey = mg.sigma_y / mg.E
    eps = torch.randn((6, n, n, n), generator=g, dtype=f64, device=dev) * (2.5 * ey)
    epsp = torch.randn((6, n, n, n), generator=g, dtype=f64, device=dev) * (0.5 * ey)
    ctx.set_field(_fgd.FIELD_EPS_P, epsp)
    ctx.set_field(_fgd.FIELD_EQPS, torch.randn((n, n, n), generator=g, dtype=f64, device=dev).abs() * (2 * ey))
    ctx.set_field(_fgd.FIELD_HIST, torch.rand((n, n, n), generator=g, dtype=f64, device=dev) * 0.3)
    for j in range(2):
        ab = torch.randn((n, n, n), generator=g, dtype=f64, device=dev).abs() * (2 * ey)
        ctx.set_field(_fgd.FIELD_NONLOCAL + j, ab)
        ctx.set_field(_fgd.FIELD_NONLOCAL_ITERATE + j,
                      ab + torch.randn((n, n, n), generator=g, dtype=f64, device=dev).abs() * (0.5 * ey))
    sig = torch.empty_like(eps)
    ctx.constitutive(eps, sig)
    ctx.set_timing(True)
    for _ in range(reps):
        ctx.constitutive(eps)
    kt = ctx.kernel_times()
    ctx.set_timing(False)
    ms = kt["constitutive"][0] / kt["constitutive"][1]
    # plastic voxels: the stress differs from the elastic trial
    K, mu = mg.E / (3 * (1 - 2 * mg.nu)), mg.E / (2 * (1 + mg.nu))
    ee = eps - epsp
    tr = ee[:3].sum(0)
    trial = 2 * mu * ee
    trial[:3] += (K - 2 * mu / 3) * tr
    matrix = torch.from_numpy(synth.config1_phases(n, 0) == 0).to(dev)
    plastic = ((sig - trial).abs().amax(0) > 1e-8 * trial.abs().amax(0)) & matrix
    gbs = GTN_BYTES_PER_VOXEL * V / (ms * 1e-3) / 1e9
    ctx.close()
    return {"workload": f"config-1 phases at {n}^3, Sec. 4.2 GTN matrix (model 3) + elastic inclusion, random "
                        "committed state (porosity U[0, 0.3], non-local fields and increments ~|N|)",
            "ms_per_update": ms, "voxels_per_s": V / (ms * 1e-3),
            "plastic_fraction": float(plastic.sum().item()) / V,
            "bytes_per_voxel": GTN_BYTES_PER_VOXEL, "GBs": gbs, "frac_hbm": gbs / peak,
            "note": "K1 with the GTN return mapping (3-unknown Newton with cosh/sinh and pow per plastic "
                    "voxel); FP64-ALU bound on plastic voxels, see profiles/ for the ncu pipe utilisation"}


def measure(a, n, rank, world, local, nid, e2e_on, extras):
    """One size: K timed steps (headline), K instrumented steps (kernel classes), optional e2e and,
    with extras (one GPU, n <= 256), the cuFFT comparison arm on the same tangent."""
    import numpy as np
    import torch

    import synth
    from paper_2103_04770_b200 import Context, Material

    V = n ** 3
    dev = torch.device("cuda", local)
    ctx = Context((n, n, n), (float(n),) * 3, device=local, rank=rank, nranks=world, nccl_id=nid)
    nz, z0 = ctx.nz, ctx.z0
    gen = torch.Generator(device=dev)
    gen.manual_seed(1234 + rank)
    ph = torch.from_numpy(synth.config1_phases(n, 0)[z0:z0 + nz].copy()).to(dev)
    eps = torch.randn((6, nz, n, n), generator=gen, dtype=torch.float64, device=dev) * 1e-3
    ctx.set_phases(ph, 2)
    m0, m1 = synth.MATRIX_J2, synth.INCLUSION_EL
    for q, m in enumerate((m0, m1)):
        ctx.set_material(q, Material.of(m))
    ctx.set_nonlocal(synth.CONFIG1_ELL, [0])
    ctx.set_control(synth.CONFIG1_MASK)
    zero6 = np.zeros(6)

    def step(e=eps, de_out=None):
        m = ctx.constitutive(e)
        rms = ctx.mech_residual(zero6)
        _, rel = ctx.solve_tangent_cg(None, de_out, tol=0.0, maxit=a.kcg)
        ctx.solve_helmholtz(0, None, None, tol=0.0, maxit=a.khelm)
        return m, rms, rel

    for _ in range(a.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    clocks = Clocks(local)
    clocks.start()
    time.sleep(0.3)
    stream = torch.cuda.current_stream(dev)
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    # headline: K steps with nothing but the library's own launches on the stream
    l0 = ctx.launch_count
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(a.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    launches = ctx.launch_count - l0
    ms = ev0.elapsed_time(ev1) / a.steps
    # per-kernel-class durations: the same K steps again with a CUDA event pair around every
    # launch (fgd_set_timing) -- the roofline numbers come from this instrumented pass
    if world > 1:
        torch.distributed.barrier()
    ctx.set_timing(True)
    torch.cuda.synchronize()
    ev0.record(stream)
    for _ in range(a.steps):
        step()
    ev1.record(stream)
    torch.cuda.synchronize()
    kt = ctx.kernel_times()
    ctx.set_timing(False)
    ms_instr = ev0.elapsed_time(ev1) / a.steps
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = V * a.kcg / (ms * 1e-3)          # strong scaling: the global n^3 cell, all ranks

    # roofline of the dominant kernel class (its launches inside the timed region)
    peak, peak_src = peaks()
    cb = class_bytes(n, a.kcg, a.khelm, world)
    per_class = {}
    step_ms_sum = sum(v[0] for v in kt.values())
    for k, (tms, cnt) in kt.items():
        if cnt == 0:
            continue
        entry = {"ms_per_step": tms / a.steps, "launches_per_step": cnt / a.steps,
                 "share": tms / step_ms_sum if step_ms_sum else None}
        if k in cb:
            entry["GBs"] = cb[k] * a.steps / (tms * 1e-3) / 1e9
            entry["frac"] = entry["GBs"] / peak
        per_class[k] = entry
    dom = max((k for k in per_class if k in cb), key=lambda k: per_class[k]["ms_per_step"])
    d = per_class[dom]
    traffic, traffic_src = measured_traffic(dom, n)
    alg = cb[dom] / d["launches_per_step"]
    roof = {"bound": "hbm", "kernel": dom, "achieved": d["GBs"], "peak": peak, "unit": "GB/s", "frac": d["frac"],
            "traffic": traffic, "traffic_source": traffic_src, "peak_source": peak_src,
            "algorithmic_bytes_per_launch": alg,
            "traffic_vs_algorithmic": (traffic / alg) if traffic else None}
    # whole-step efficiency against the fused-design byte model
    step_bytes = sum(cb.values())
    step_eff = {"bytes_per_step": step_bytes, "GBs": step_bytes / (ms * 1e-3) / 1e9,
                "frac": step_bytes / (ms * 1e-3) / 1e9 / peak,
                "ms_per_step_instrumented": ms_instr,
                "note": "kernel-class times from a second K-step pass with an event pair per launch"}

    e2e = None
    if e2e_on:
        host = torch.empty((6, nz, n, n), dtype=torch.float64, pin_memory=True)
        host.copy_(eps.cpu())
        host_de = torch.empty((6, nz, n, n), dtype=torch.float64, pin_memory=True)
        step(host, host_de)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        t = time.perf_counter()
        for _ in range(a.steps):
            # H2D of the strain inside fgd_constitutive; D2H of the Krylov solution field (the Newton
            # correction) into pinned host memory, plus <sigma>, rms and relres
            m, rms, rel = step(host, host_de)
        torch.cuda.synchronize()
        te = (time.perf_counter() - t) / a.steps
        if world > 1:
            tt = torch.tensor([te], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(tt, op=torch.distributed.ReduceOp.MAX)
            te = float(tt.item())
        e2e = {"value": V * a.kcg / te, "unit": UNIT, "h2d_bytes_per_step": 48 * V,
               "d2h_bytes_per_step": 48 * V + world * (48 + 8 + 8 + 8), "ms_per_step": te * 1e3,
               "what": "the same step through the C ABI with host buffers: the strain field staged from pinned "
                       "host memory into fgd_constitutive, the CG solution field read back into pinned host "
                       "memory by fgd_solve_tangent_cg"}

    cmp_cufft = None
    if extras and world == 1 and not a.no_cufft:
        cmp_cufft = cufft_comparison(ctx, n, dev, synth.CONFIG1_MASK)

    # multi-GPU: share and achieved bandwidth of the slab transposes; every operator
    # apply moves (P-1)/P of the rank's spectrum twice (before and after the z pass)
    comm = None
    if world > 1 and "comm" in per_class:
        S_loc = 16 * (n // 2 + 1) * n * n // world
        a2a_bytes = 2 * (world - 1) / world * S_loc * (6 * (a.kcg + 1) + (a.khelm + 1))
        cms = per_class["comm"]["ms_per_step"]
        comm = {"ms_per_step": cms, "share": cms / ms, "alltoall_bytes_sent_per_gpu_per_step": a2a_bytes,
                "alltoall_GBs_per_gpu": a2a_bytes / (cms * 1e-3) / 1e9 if cms else None,
                "nvlink_GBs_per_direction": 900.0, "nvlink_measured_peer_GBs": 770.0,
                "note": "comm = NCCL all-to-all transposes + stencil z-halos + Krylov allreduces (event-timed)"}
    # per-solver rates inside the step (kernel-class times, this rank): one mechanical apply = the
    # five 6-comp passes (the residual projection costs the same passes as a CG iteration), one PCG
    # iteration = the stencil + the five 1-comp passes
    t_mech = sum(per_class[k]["ms_per_step"] for k in ("xfwd6", "xfwd6cg", "yfwd6", "z6", "yinv6", "xinv6")
                 if k in per_class)
    t_helm = sum(per_class[k]["ms_per_step"] for k in ("xfwd1", "yfwd1", "z1", "yinv1", "xinv1", "stencil")
                 if k in per_class)
    b_mech = sum(cb[k] for k in ("xfwd6", "xfwd6cg", "yfwd6", "z6", "yinv6", "xinv6") if k in per_class)
    b_helm = sum(cb[k] for k in ("xfwd1", "yfwd1", "z1", "yinv1", "xinv1", "stencil") if k in per_class)
    op_roof = {"what": "operator-level roofline: algorithmic bytes of the kernel classes of the mechanical Krylov "
                       "solve (projected-tangent applies incl. the fused CG updates) and of the Helmholtz PCG "
                       "(stencil + preconditioner passes incl. the fused updates) over their event-timed duration",
               "mech_GBs": b_mech / (t_mech * 1e-3) / 1e9 if t_mech else None,
               "mech_frac": b_mech / (t_mech * 1e-3) / 1e9 / peak if t_mech else None,
               "helm_GBs": b_helm / (t_helm * 1e-3) / 1e9 if t_helm else None,
               "helm_frac": b_helm / (t_helm * 1e-3) / 1e9 / peak if t_helm else None}
    mech_apply_ms = t_mech / (a.kcg + 1) if t_mech else None
    helm_iter_ms = t_helm / (a.khelm + 1) if t_helm else None
    rates = {"mech_cg_iter_per_s": 1e3 / mech_apply_ms if mech_apply_ms else None,
             "mech_apply_ms": mech_apply_ms,
             "mech_cg_voxel_iter_per_s": V / (mech_apply_ms * 1e-3) if mech_apply_ms else None,
             "helm_pcg_iter_per_s": 1e3 / helm_iter_ms if helm_iter_ms else None,
             "helm_pcg_iter_ms": helm_iter_ms,
             "helm_pcg_voxel_iter_per_s": V / (helm_iter_ms * 1e-3) if helm_iter_ms else None,
             "operator_roofline": op_roof,
             "note": "Krylov iteration rates from the event-timed kernel classes of one rank (the step's "
                     "constitutive update and reductions excluded); value/ms_per_step is the whole step"}
    ctx.close()
    del eps
    torch.cuda.empty_cache()
    return dict(value=value, ms=ms, launches=launches, clocks=clk, roofline=roof, step_roofline=step_eff, e2e=e2e,
                kernels=per_class, rates=rates, comm=comm, cufft=cmp_cufft, peak=peak)


def run_ours(a):
    import torch

    rank, world, local = dist_env()
    if world != a.gpus:
        print(f"bench.py: --gpus {a.gpus} but WORLD_SIZE = {world}", file=sys.stderr)
        sys.exit(2)
    torch.cuda.set_device(local)
    from paper_2103_04770_b200 import nccl_id

    nid = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        t = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            t.copy_(torch.frombuffer(bytearray(nccl_id()), dtype=torch.uint8))
        dist.broadcast(t, 0)
        nid = bytes(t.cpu().numpy().tobytes())
    n = a.n
    dev = torch.device("cuda", local)
    main = measure(a, n, rank, world, local, nid, e2e_on=not a.no_e2e, extras=n <= 256)
    # the other metric size (BASELINE metric "at 256^3/512^3"), one GPU only
    by_size = {}
    cmp_cufft = main["cufft"]
    if world == 1 and not a.no_by_size:
        for m in (256, 512):
            if m == n:
                continue
            o = measure(a, m, rank, world, local, nid, e2e_on=False, extras=m <= 256)
            cmp_cufft = cmp_cufft or o["cufft"]
            by_size[str(m)] = {"value": o["value"], "unit": UNIT, "ms_per_step": o["ms"], "roofline": o["roofline"],
                               "step_roofline": o["step_roofline"], "rates": o["rates"], "gpu_launches": o["launches"],
                               "clocks": o["clocks"], "workload": workload_name(m)}
    cpu = None
    if rank == 0 and world == 1 and not a.no_cpu:
        cpu = cpu_baseline(a.kcg, a.khelm)
    gtn = None
    if world == 1 and not a.no_gtn:
        gtn = gtn_measurement(256, dev, main["peak"])   # a second context: keep it at 256^3
        k = main["kernels"] if n == 256 else by_size.get("256", {}).get("kernels")
        if k and "constitutive" in k:
            gtn["j2_ms_per_update"] = k["constitutive"]["ms_per_step"]
    if rank == 0:
        line = {"metric": METRIC, "value": main["value"], "unit": UNIT, "n_gpus": world, "steps": a.steps,
                "warmup": a.warmup, "ms_per_step": main["ms"], "higher_is_better": True,
                "scaling": "strong",
                "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": {"workload": workload_name(n), "n": n, "kcg": a.kcg, "khelm": a.khelm,
                           "parallelism": "single GPU" if world == 1 else
                           f"z-slab decomposition over {world} GPUs (NCCL all-to-all transposes, allreduce)",
                           "l2": "no flush: every input field (>=134 MB) and the tangent (>=2.8 GB) exceed the "
                                 "126 MB L2"},
                "roofline": main["roofline"], "step_roofline": main["step_roofline"], "cpu_baseline": cpu,
                "e2e": main["e2e"], "gpu_launches": main["launches"], "clocks": main["clocks"],
                "kernels": main["kernels"], "rates": main["rates"], "by_size": by_size or None,
                "cufft_comparison": cmp_cufft, "gtn_constitutive": gtn, "comm": main["comm"]}
        print(json.dumps(line), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


def relaunch_under_torchrun(a):
    """`bench.py --gpus N` without a torchrun environment: re-exec this command as N ranks of one
    node (one process per GPU, rendezvous on 127.0.0.1), as the driver does for its scaling runs."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={a.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    os.execv(sys.executable, cmd)


def main():
    a = args_()
    if a.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(a)
    if a.impl == "reference":
        run_reference(a)
    else:
        run_ours(a)


if __name__ == "__main__":
    main()
