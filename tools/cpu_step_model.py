"""Modelled CPU time of one BASELINE cfg5 TR-BDF2 step (96^3 Q2/Q1) for the reference
("cfg5 (20 steps ~ 100 h on CPU): reported as modelled (CPU per-apply times x
the oracle-vs-GPU iteration counts), labelled as such").

Per-apply times of the unmodified reference (oracle/_ref, 1 core) are measured on one
96 x 96 x 4 z-slab of the cfg5 mesh (identical cells, tools of bench.py) -- median of 3
after a warm-up -- and scaled by the slab count (24).  The step model counts what the
restated driver (oracle/trbdf2_cpu.hpp) does per stage: one momentum RHS (~1 apply), one
momentum diagonal (~0.6 apply), GMRES(50) with one apply + (k+1) dot/axpy pairs per
iteration, the mass solves, the pressure RHS, Helmholtz diagonal and CG with one pressure
apply + 5 vector passes per iteration.  Iteration counts: the device's for the cfg5 steps
(identical to the reference's at every size compared).  Prints one JSON line.
usage: python tools/cpu_step_model.py [its json: [[gm1, gm2, cg1, cg2, m0..m3], ...]]"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import reforacle as ref

g = 2.0 - 2.0 ** 0.5


def med(fn, reps=3):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return float(np.median(ts))


def model(cfg, its):
    """Per-apply times on one z-slab (x slab count) and the per-stage call count of the
    restated driver -> modelled seconds per step for each iteration-count set."""
    n, nz, ku, kp, Re, seed = {"cfg5": (96, 4, 2, 1, 1600.0, 4), "cfg2": (32, 4, 2, 1, 100.0, 1)}[cfg]
    nslab = n // nz
    R = ref.RefCtx.slab(n, n // 2 - nz // 2, nz, ku, kp)
    f = ref.SynthField(3, seed)
    w = f.interpolate(R)
    x = ref.seeded_uniform(1000 + seed, R.n_u)
    xp = ref.seeded_uniform(2000 + seed, R.n_p)
    dt = 0.5 * (3.0 ** 0.5 / n) / ku if cfg == "cfg5" else 1e-3
    coefs = (1.0 / (g * dt), 1.0 / (2 * Re), 0.5, 0.0)
    pmc = 1.0 / (1e6 * g * g * dt * dt)
    t_mom = med(lambda: R.momentum(coefs, w, x)) * nslab
    t_prs = med(lambda: R.pressure(pmc, xp)) * nslab
    t_mass = med(lambda: R.mass(0, x)) * nslab
    t_diag = med(lambda: R.momentum_diag(coefs, w), 1) * nslab
    N_u, N_p = 3 * 27 * n ** 3, 8 * n ** 3
    v = ref.seeded_uniform(1, N_u // nslab)
    t0 = time.perf_counter()
    for _ in range(5):
        ref.kern("axpy", 0.3, v, v)
    t_pass = (time.perf_counter() - t0) / 5 * nslab  # one axpy over N_u
    steps = []
    for it in its:
        gm, cg, ms = it[0:2], it[2:4], it[4:8]
        t = 0.0
        for s in range(2):
            t += 2.0 * t_mom + t_diag                               # RHS (fields + data) + diagonal
            k = gm[s]
            t += k * (t_mom + (min(k, 50) / 2.0 + 2) * 2 * t_pass)  # GMRES: apply + MGS dot/axpy pairs
            t += sum(ms[2 * s:2 * s + 2]) * (t_mass + 4 * t_pass)  # mass CG solves
            t += 0.9 * t_mom + t_prs                                # gradient / divergence, pressure RHS
            t += cg[s] * (t_prs + 5 * t_pass * (N_p / N_u))         # pressure CG
        steps.append(t)
    return steps, {"momentum": t_mom, "pressure": t_prs, "mass_u": t_mass, "momentum_diag": t_diag,
                   "axpy_N_u": t_pass}


def measured_cfg2_step():
    R = ref.RefCtx(3, 32, 2, 1)
    f = ref.SynthField(3, 1)
    u0 = f.interpolate(R, os.cpu_count() or 1)
    for bid in range(6):
        R.set_bc(bid, 0, f.fn_ptr, f.user_ptr)
    t0 = time.perf_counter()
    _, _, its = R.step([1e-3, 100.0, 1e3, 0.0, 50, 1e-10, 1e-10, 1e-12, 10000, 1.0], u0, u0, np.zeros(R.n_p))
    return time.perf_counter() - t0, its[:8]


if __name__ == "__main__":
    its5 = json.loads(sys.argv[1]) if len(sys.argv) > 1 else [[28, 27, 1586, 1487, 0, 1, 1, 1],
                                                               [44, 46, 1463, 1409, 1, 1, 1, 1]]
    t2, its2 = measured_cfg2_step()
    m2, _ = model("cfg2", [its2])
    cal = t2 / m2[0]
    m5, per = model("cfg5", its5)
    print(json.dumps({
        "config": "cfg5 96^3 Q2/Q1, Re 1600, CFL 0.5: MODELLED reference CPU TR-BDF2 step time, 1 core",
        "modelled_s_per_step": [cal * t for t in m5], "iterations_used": its5,
        "calibration": {"cfg2_measured_step_s": t2, "cfg2_its": its2, "cfg2_modelled_s": m2[0], "factor": cal},
        "per_apply_s_cfg5": per,
        "method": "per-apply times of the unmodified reference on one 96x96x4 z-slab of the cfg5 mesh x 24 "
                  "(median of 3 after 1 warm-up) x the driver's call counts per stage with the device's cfg5 "
                  "iteration counts (first / last of the 20-step run), scaled by measured / modelled for a real "
                  f"cfg2 step on the same host; backend {ref.lib().ref_backend().decode()}"}))
