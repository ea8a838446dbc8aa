#!/usr/bin/env python3
"""Benchmark of the B200 DG hot path (one JSON line on rank 0).

Workload (BASELINE.json configs[2], the north-star config): 3D unit cube,
64^3 affine hex mesh, velocity DG Q3 (3 comps, 50,331,648 DoF), pressure Q2
(7,077,888 DoF), fp64.  A "step" is one pass of the hot path over one batch
of synthetic input: ONE momentum-operator apply (stage-1 TR-BDF2 operator,
mass 1/(gamma dt) + visc 1/(2Re) + LF advection 1/2 with w = u^0, the seeded
curl-of-vector-potential field, seed 2) followed by ONE pressure-Helmholtz
apply (mass_coef 1/(c^2 gamma^2 dt^2)), on U[-1,1] seeded vectors (seeds
1002 / 2002).  value = (N_u + N_p) / step time [GDoF/s], whole job over N GPUs
(replicas: the path is single-GPU; each rank runs its own copy, weak scaling).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]

--impl reference times the unmodified reference CPU implementation
(oracle/_ref/libdgref.so: /root/reference/proj/src compiled as-is) on the same
cfg3 workload with all host threads: the 64^3 mesh as z-slabs, one reference
context per slab (the reference is single-threaded), inputs from the oracle-side
generator (no product library in that process).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

GAMMA = 2.0 - math.sqrt(2.0)
CFG = dict(workload="cfg3: 3D 64^3 unit cube affine, Q3/Q2 velocity/pressure, fp64 "
                    "(1 momentum apply + 1 pressure apply per step)",
           dim=3, n_el=64, ku=3, kp=2, seed=2, Re=1000.0, dt=1e-3, c=1e3)
# algorithmic fp64 flop / DoF and bytes / DoF at cfg3
FLOP_PER_DOF = {"momentum": 545.9, "pressure": 406.2}
BYTES_PER_DOF = {"momentum": 24.0, "pressure": 16.0}
METRIC = "fp64 DG op-apply throughput (momentum + pressure), GDoF/s"
DATA = "synthetic (seeded; BASELINE cfg3 vector-potential field, U[-1,1] vectors)"


def bench_config(ws: int) -> dict:
    """The config dict both arms print (identical, so the driver can pair them)."""
    n, ku, kp = CFG["n_el"], CFG["ku"], CFG["kp"]
    return {"workload": CFG["workload"], "mesh": f"{n}^3", "degrees": f"Q{ku}/Q{kp}",
            "n_u": 3 * n ** 3 * (ku + 1) ** 3, "n_p": n ** 3 * (kp + 1) ** 3,
            "Re": CFG["Re"], "dt": CFG["dt"], "c": CFG["c"], "parallelism": f"replicas x{ws}",
            "l2": "inputs larger than L2 (x, w 403 MB each); the momentum apply streams 1.2 GB between "
                  "pressure applies"}


def coefficients():
    dt, Re, c = CFG["dt"], CFG["Re"], CFG["c"]
    mom = (1.0 / (GAMMA * dt), 1.0 / (2.0 * Re), 0.5, 0.0)
    pmc = 1.0 / (c * c * GAMMA * GAMMA * dt * dt)
    return mom, pmc


def profile_json(name):
    """A committed evidence file under profiles/ (None if absent)."""
    try:
        with open(os.path.join(ROOT, "profiles", name)) as f:
            return json.load(f)
    except Exception:
        return None


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f)
    except Exception:
        return {"hbm_gbs": 6650.0, "_fallback": True}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self.proc = None
        self.thread = None

    def start(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.thread = threading.Thread(target=self._read, daemon=True)
        self.thread.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_info():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_max(x: float) -> float:
    """Max over ranks (device timing rule: the job takes as long as its slowest rank).
    NCCL on GPU ranks, gloo on CPU (tests/test_multirank.py)."""
    import torch
    import torch.distributed as tdist
    if not (tdist.is_available() and tdist.is_initialized()) or tdist.get_world_size() == 1:
        return x
    dev = torch.device("cuda", torch.cuda.current_device()) if tdist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(ws: int, units_per_rank: int, ms_max: float) -> float:
    """Replicas (weak scaling): every rank processes its own copy of the workload;
    value = all units processed / the slowest rank's time."""
    return ws * units_per_rank / (ms_max * 1e-3)


# ---------------------------------------------------------------------------
# reference CPU leg (TEST INFRASTRUCTURE: the unmodified reference, oracle/_ref)
# ---------------------------------------------------------------------------
def reference_slabs(nslabs: int, z_list=None, nthreads: int = 1):
    """The cfg3 workload for the unmodified reference, cut into z-slabs.

    The 64^3 mesh is split into `nslabs` slabs of 64 x 64 x (64 / nslabs) cells; each
    slab is its own reference Mesh / GeometryCache / FunctionSpace pair (oracle
    ref_create_slab: cells bit-identical to the full mesh's, the slab's own z-ends are
    boundary faces) holding the cfg3 inputs of its cells: w = the seeded
    vector-potential field interpolated by FunctionSpace::interpolate, x / xp = its
    contiguous cell range of the full U[-1,1] vectors (seeds 1002 / 2002).  Inputs come
    from the oracle-side generator only (reforacle; no product library is loaded).
    Returns the RefCtx list (each ready for pair_rounds) and the DoFs it covers."""
    import reforacle as ref
    n, ku, kp = CFG["n_el"], CFG["ku"], CFG["kp"]
    nz = n // nslabs
    nbu, nbp = 3 * (ku + 1) ** 3, (kp + 1) ** 3
    mom, pmc = coefficients()
    f = ref.SynthField(3, CFG["seed"])
    x = ref.seeded_uniform(CFG["seed"] + 1000, n ** 3 * nbu)
    xp = ref.seeded_uniform(CFG["seed"] + 2000, n ** 3 * nbp)
    ctxs, dofs = [], 0
    for s in (range(nslabs) if z_list is None else z_list):
        R = ref.RefCtx.slab(n, s * nz, nz, ku, kp)
        c0, c1 = s * nz * n * n, (s + 1) * nz * n * n
        R.pair_setup(mom, f.interpolate(R, nthreads), x[c0 * nbu:c1 * nbu], pmc, xp[c0 * nbp:c1 * nbp])
        ctxs.append(R)
        dofs += R.n_u + R.n_p
    return ctxs, dofs


def reference_nslabs(ncores: int) -> int:
    """Smallest power of two >= the host threads (one slab per thread), within 16..64."""
    k = 16
    while k < min(ncores, 64):
        k *= 2
    return k


def cpu_baseline_1core():
    """SURVEY 8(d) CPU baseline: the reference on ONE host core, median of 3 applies
    after one warm-up apply (the warm-up also pays the lazy GeometryCache build), on a
    bounded sample of the cfg3 workload: one 64 x 64 x 4 z-slab (1/16 of the cells)."""
    import reforacle as ref
    ctxs, dofs = reference_slabs(16, z_list=[8])
    ref.pair_rounds(ctxs, 1, 1)
    t = float(np.median(ref.pair_rounds(ctxs, 1, 3)))
    return {"value": dofs / t / 1e9, "unit": "GDoF/s", "cores": 1, "kind": "reference",
            "sample": "cfg3 workload, one 64x64x4 z-slab of the 64^3 mesh (16,384 of 262,144 cells, cfg3 inputs of "
                      "those cells): median of 3 momentum+pressure apply pairs after 1 warm-up, 1 core, reference "
                      f"backend {ref.lib().ref_backend().decode()}",
            "detail": {"s_per_apply_pair": t, "dofs": dofs,
                       "modelled_full_cfg3_s_per_apply_pair": t * 16}}


def run_reference(args):
    ws, rank, _ = dist_info()
    if rank != 0:
        return
    import reforacle as ref
    ncores = max(1, os.cpu_count() or 1)
    nslabs = reference_nslabs(ncores)
    t0 = time.time()
    ctxs, dofs = reference_slabs(nslabs, nthreads=ncores)
    ref.pair_rounds(ctxs, ncores, max(1, args.warmup))  # the first round builds the lazy geometry
    setup_s = time.time() - t0
    times = ref.pair_rounds(ctxs, ncores, max(1, args.steps))
    secs = float(times.sum())
    val = dofs * len(times) / secs / 1e9
    desc = (f"the whole cfg3 64^3 Q3/Q2 workload every step, as {nslabs} z-slabs of 64x64x{CFG['n_el'] // nslabs} "
            f"cells (one reference context each; slab ends are boundary faces) spread over {ncores} host threads; "
            f"reference backend {ref.lib().ref_backend().decode()}")
    line = {"metric": METRIC, "value": val, "unit": "GDoF/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": max(1, args.warmup), "ms_per_step": secs / len(times) * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": DATA, "config": bench_config(ws),
            "impl": "reference",
            "cpu_baseline": {"value": val, "unit": "GDoF/s", "cores": ncores, "kind": "reference", "sample": desc},
            "e2e": {"value": val, "unit": "GDoF/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "detail": {"dofs_per_step": dofs, "setup_and_warmup_s": setup_s,
                       "step_s": [float(t) for t in times]}}
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# device leg
# ---------------------------------------------------------------------------
def trbdf2_step_time(D, dg, torch, stream, precond="jacobi"):
    """Second of two consecutive first-order-start TR-BDF2 steps from u^0 (the first
    warms the solver workspaces), timed with CUDA events on the context stream.
    precond: the pressure CG preconditioner ("jacobi" = the reference's, iteration-count
    parity; "mg" = the hybrid multigrid of mg.cu)."""
    f = dg.SynthField(CFG["dim"], CFG["seed"])
    for bid in range(2 * CFG["dim"]):
        D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros()
    dg.interpolate_synth_device(D, f, u0)
    p0 = D.zeros(dg.SPACE_P)
    u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
    sp = dg.StepParams(dt=CFG["dt"], Re=CFG["Re"], c=CFG["c"], restart=30, first_step=True, pressure_precond=precond)
    dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    l0 = D.launch_count()
    e0.record(stream)
    its = dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
    e1.record(stream)
    torch.cuda.synchronize()
    return {"s_per_step": e0.elapsed_time(e1) * 1e-3, "krylov_its": [int(i) for i in its],
            "its_legend": "[gmres s1, gmres s2, cg s1, cg s2, mass-cg s1 (pre), s1 (post), s2 (pre), s2 (post)]",
            "gpu_launches": int(D.launch_count() - l0),
            "config": "cfg3 stage pair from u^0 (seed 2), Dirichlet = u^0 trace, p^0 = 0, dt 1e-3, Re 1000, "
                      "c 1e3, GMRES restart 30 / CG, rel tol 1e-10 (mass 1e-12); pressure CG preconditioner: " + precond}


def cfg4_run(dg, torch, stream, hbm_peak):
    """BASELINE configs[3] (cfg4): 48^3 deformed Q4/Q3 (interior vertices displaced by
    U[-0.1h, 0.1h], seed 3; per-quadrature-point geometry).  Momentum / pressure apply
    times (CUDA events, 10 applies after 3) against the HBM roofline with SURVEY 8(d)'s
    per-DoF bytes, then one TR-BDF2 step (second of two from u^0) with the reference's
    Jacobi CG and with the multigrid pressure CG.  Outside the timed op-apply region."""
    import time as _t
    n_el, ku, kp, seed, Re = 48, 4, 3, 3, 100.0
    t0 = _t.time()
    D = dg.DGContext(3, n_el, ku, kp, 0.1 / n_el, seed)
    setup = _t.time() - t0
    f = dg.SynthField(3, seed)
    for bid in range(6):
        D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros()
    dg.interpolate_synth_device(D, f, u0)
    x = torch.from_numpy(dg.seeded_uniform(seed + 1000, D.n_u)).cuda()
    xp = torch.from_numpy(dg.seeded_uniform(seed + 2000, D.n_p)).cuda()
    y, yp = D.zeros(), D.zeros(dg.SPACE_P)
    g = 2.0 - 2.0 ** 0.5
    ctx = dg.MomentumCtx(1.0 / (g * 1e-3), 1.0 / (2.0 * Re), 0.5, 0.0, advecting=u0)
    pmc = 1.0 / (1e6 * g * g * 1e-6)
    out = {"config": "cfg4: 3D 48^3 unit cube, interior vertices displaced U[-0.1h, 0.1h] (seed 3), Q4/Q3, "
                     "per-quadrature-point geometry, Re 100, dt 1e-3, GMRES restart 50 / CG tol 1e-10",
           "setup_s": setup, "fast_path": "deformed" if D.fast_path_active else "generic",
           "n_u": D.n_u, "n_p": D.n_p}
    for name, fn, n, bpd in (("momentum", lambda: dg.apply_momentum(D, ctx, x, y), D.n_u, 182.6),
                             ("pressure", lambda: dg.apply_pressure_helmholtz(D, pmc, xp, yp), D.n_p, 378.5)):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(10):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        gbs = bpd * n / ms / 1e6
        out[name] = {"ms": ms, "gdofs": n / ms / 1e6, "hbm_gbs_alg": gbs, "bytes_per_dof_alg": bpd,
                     "hbm_frac": gbs / hbm_peak if hbm_peak else None}
    del x, xp, y, yp
    p0 = D.zeros(dg.SPACE_P)
    u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
    for precond in ("jacobi", "mg"):
        sp = dg.StepParams(dt=1e-3, Re=Re, c=1e3, restart=50, first_step=True, pressure_precond=precond)
        dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        its = dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
        e1.record(stream)
        torch.cuda.synchronize()
        out["step_" + precond] = {"s_per_step": e0.elapsed_time(e1) * 1e-3, "krylov_its": [int(i) for i in its]}
    del D, u0, p0, u1, p1
    torch.cuda.empty_cache()
    return out


def cfg5_steps(dg, torch, stream, precond="jacobi", nsteps=20):
    """BASELINE configs[4]: 20 consecutive TR-BDF2 steps at 96^3 Q2/Q1, Re 1600, initial
    field (seed 4) scaled to max nodal |u| = 1, dt for CFL 0.5, GMRES(50) /
    CG at 1e-10, after one discarded warm-up step (first-use allocations).  Same protocol
    as tools/cfg5_steps.py; CUDA events on the context stream."""
    import math
    n_el, ku, kp, seed, Re = 96, 2, 1, 4, 1600.0
    D = dg.DGContext(3, n_el, ku, kp)
    f1 = dg.SynthField(3, seed)
    u = D.zeros()
    dg.interpolate_synth_device(D, f1, u)
    umax = float(u.view(D.ncells, 3, -1).pow(2).sum(1).sqrt().max())
    f = dg.SynthField(3, seed, 1.0 / umax)
    for bid in range(6):
        D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros()
    dg.interpolate_synth_device(D, f, u0)
    dt = 0.5 * (math.sqrt(3.0) / n_el) / ku
    p0 = D.zeros(dg.SPACE_P)
    wu, wp = D.zeros(), D.zeros(dg.SPACE_P)
    dg.trbdf2_step(D, dg.StepParams(dt=dt, Re=Re, c=1e3, restart=50, first_step=True, pressure_precond=precond),
                   u0, u0, p0, wu, wp)
    del wu, wp
    bufs = [(u0, p0), (D.zeros(), D.zeros(dg.SPACE_P)), (D.zeros(), D.zeros(dg.SPACE_P))]
    u_nm1, (u_n, p_n) = u0, bufs[0]
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its_all = []
    e0.record(stream)
    for n in range(nsteps):
        u_np1, p_np1 = bufs[(n + 1) % 3]
        if u_np1.data_ptr() == u_nm1.data_ptr():
            u_np1, p_np1 = bufs[(n + 2) % 3]
        sp = dg.StepParams(dt=dt, Re=Re, c=1e3, time=n * dt, restart=50, first_step=(n == 0),
                           pressure_precond=precond)
        its_all.append([int(i) for i in dg.trbdf2_step(D, sp, u_nm1, u_n, p_n, u_np1, p_np1)])
        u_nm1, u_n, p_n = u_n, u_np1, p_np1
    e1.record(stream)
    torch.cuda.synchronize()
    total = e0.elapsed_time(e1) * 1e-3
    del D, bufs, u, u0
    torch.cuda.empty_cache()
    return {"s_per_step": total / nsteps, "total_s": total, "steps": nsteps, "dt": dt,
            "krylov_its_first_last": [its_all[0], its_all[-1]], "pressure_precond": precond}


def run_device(args):
    import torch
    import paper_2107_07776_b200 as dg

    ws, rank, local = dist_info()
    if ws > 1:
        import torch.distributed as tdist
        tdist.init_process_group("nccl", init_method="env://")
    torch.cuda.set_device(local)
    dev = torch.device(f"cuda:{local}")
    mom, pmc = coefficients()
    t0 = time.time()
    D = dg.DGContext(CFG["dim"], CFG["n_el"], CFG["ku"], CFG["kp"], device=local)
    stream = D.stream
    f = dg.SynthField(CFG["dim"], CFG["seed"])
    w = D.zeros()
    dg.interpolate_synth_device(D, f, w)
    x_h = torch.from_numpy(dg.seeded_uniform(CFG["seed"] + 1000, D.n_u))
    xp_h = torch.from_numpy(dg.seeded_uniform(CFG["seed"] + 2000, D.n_p))
    x = x_h.to(dev)
    xp = xp_h.to(dev)
    y = D.zeros()
    yp = D.zeros(dg.SPACE_P)
    ctx = dg.MomentumCtx(*mom, advecting=w)
    setup_s = time.time() - t0
    peak_dfma = dg.fp64_peak_tflops(D)
    peak_dmma = dg.fp64_peak_dmma_tflops(D)
    peak_fp64 = max(peak_dfma, peak_dmma)  # both measured, the higher is the denominator

    def step():
        dg.apply_momentum(D, ctx, x, y)
        dg.apply_pressure_helmholtz(D, pmc, xp, yp)

    # warm-up: at least W steps, and the GPU kept busy while the clock sampler (an
    # nvidia-smi child, ~0.3 s to start) comes up, so the timed region does not begin
    # from an idle, down-clocked GPU
    sampler = ClockSampler(local)
    sampler.start()
    t_warm = time.time()
    nwarm = 0
    while nwarm < max(3, args.warmup) or (time.time() - t_warm < 0.4 and nwarm < 400):
        step()
        nwarm += 1
        if nwarm % 16 == 0:
            torch.cuda.synchronize()
    torch.cuda.synchronize()
    if ws > 1:
        tdist.barrier()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * args.steps + 2)]
    launches0 = D.launch_count()
    ev[0].record(stream)
    for k in range(args.steps):
        dg.apply_momentum(D, ctx, x, y)
        ev[1 + 2 * k].record(stream)
        dg.apply_pressure_helmholtz(D, pmc, xp, yp)
        ev[2 + 2 * k].record(stream)
    torch.cuda.synchronize()
    launches = D.launch_count() - launches0
    clocks = sampler.stop()
    total_ms = ev[0].elapsed_time(ev[2 * args.steps])
    t_mom = [ev[2 * k].elapsed_time(ev[1 + 2 * k]) if k else ev[0].elapsed_time(ev[1]) for k in range(args.steps)]
    t_prs = [ev[1 + 2 * k].elapsed_time(ev[2 + 2 * k]) for k in range(args.steps)]
    ms_step = reduce_max(total_ms / args.steps)
    dofs_step = D.n_u + D.n_p
    value = whole_job_rate(ws, dofs_step, ms_step) / 1e9

    # ---- end-to-end through the public API with HOST buffers (pinned): the host-buffer
    #      applies copy x, w / xp in and y / yp out every step (inside the timed region),
    #      pipelined against the kernels over z-slabs
    xh = x_h.pin_memory()
    wh = w.cpu().pin_memory()
    xph = xp_h.pin_memory()
    yh = torch.empty(D.n_u, dtype=torch.float64).pin_memory()
    yph = torch.empty(D.n_p, dtype=torch.float64).pin_memory()

    def e2e_step():
        dg.apply_momentum_host(D, mom, wh, xh, yh)
        dg.apply_pressure_helmholtz_host(D, pmc, xph, yph)

    for _ in range(2):
        e2e_step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne2e = max(1, min(args.steps, 5))
    e0.record(stream)
    for _ in range(ne2e):
        e2e_step()
    e1.record(stream)
    torch.cuda.synchronize()
    e2e_ms = reduce_max(e0.elapsed_time(e1) / ne2e)
    e2e_val = whole_job_rate(ws, dofs_step, e2e_ms) / 1e9

    # ---- one full TR-BDF2 step on device (cfg3 construction, GMRES restart 30, tol 1e-10):
    #      the "s / TR-BDF2 step" half of the metric; outside the timed op-apply region
    trbdf2 = None
    if not args.no_step:
        trbdf2 = trbdf2_step_time(D, dg, torch, stream)
        trbdf2["s_per_step"] = reduce_max(trbdf2["s_per_step"])
        mg = trbdf2_step_time(D, dg, torch, stream, "mg")
        ref3 = profile_json("cfg3_full_step_parity_r02.json")
        if ref3:  # the same step through the restated reference driver, 1 host core (tools/full_step_parity.py)
            trbdf2["reference_cpu"] = {"s_per_step": ref3.get("reference_s_1core"), "cores": 1,
                                       "krylov_its": ref3.get("its_reference"),
                                       "parity": {k: ref3.get(k) for k in ("max_its_diff", "rel_l2_u",
                                                                           "rel_l2_p_mean_free")},
                                       "source": "profiles/cfg3_full_step_parity_r02.json (measured once, "
                                                 "not in this run)"}
        trbdf2["mg"] = {"s_per_step": reduce_max(mg["s_per_step"]), "krylov_its": mg["krylov_its"],
                        "gpu_launches": mg["gpu_launches"],
                        "note": "same step with the multigrid-preconditioned pressure CG (opt-in; not the reference's "
                                "Jacobi, so CG iteration counts differ by design; fields agree to the solve tolerance)"}

    # ---- BASELINE configs[3] (cfg4, deformed): applies vs the HBM roofline + one step each solver
    cfg4 = None
    if not args.no_step and not args.no_cfg4:
        cfg4 = cfg4_run(dg, torch, stream, measured_peaks().get("hbm_gbs"))
        for k in ("step_jacobi", "step_mg"):
            cfg4[k]["s_per_step"] = reduce_max(cfg4[k]["s_per_step"])

    # ---- BASELINE configs[4] (cfg5): 20 consecutive steps, the parity (Jacobi) solver and
    #      the multigrid pressure CG; outside the timed op-apply region
    cfg5 = None
    if not args.no_step and not args.no_cfg5:
        cfg5 = {"config": "cfg5: 3D 96^3 affine Q2/Q1, Re 1600, max|u| = 1, CFL 0.5, GMRES(50) / CG tol 1e-10, "
                          "20 consecutive steps after one discarded warm-up step"}
        j = cfg5_steps(dg, torch, stream, "jacobi")
        m = cfg5_steps(dg, torch, stream, "mg")
        m5 = profile_json("cfg5_cpu_model_r02.json")
        if m5:
            cfg5["reference_cpu_modelled"] = {"s_per_step": m5.get("modelled_s_per_step"), "cores": 1,
                                              "method": m5.get("method"),
                                              "source": "profiles/cfg5_cpu_model_r02.json (MODELLED, "
                                                        "tools/cpu_step_model.py)"}
        cfg5.update({"s_per_step": reduce_max(j["s_per_step"]), "dt": j["dt"],
                     "krylov_its_first_last": j["krylov_its_first_last"],
                     "mg": {"s_per_step": reduce_max(m["s_per_step"]),
                            "krylov_its_first_last": m["krylov_its_first_last"]}})

    if rank != 0:
        if ws > 1:
            tdist.barrier()
            tdist.destroy_process_group()
        return
    # ---- roofline of the dominant kernel (momentum apply, fp64-bound at cfg3)
    tm = float(np.mean(t_mom)) * 1e-3
    tp = float(np.mean(t_prs)) * 1e-3
    mom_tflops = FLOP_PER_DOF["momentum"] * D.n_u / tm / 1e12
    prs_tflops = FLOP_PER_DOF["pressure"] * D.n_p / tp / 1e12
    peaks = measured_peaks()
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "momentum_traffic.json")) as fh:
            traffic = json.load(fh).get("dram_bytes_per_launch")
    except Exception:
        pass
    roofline = {"bound": "fp64", "achieved": mom_tflops, "peak": peak_fp64, "unit": "TFLOP/s",
                "frac": mom_tflops / peak_fp64, "traffic": traffic,
                "kernel": "k_momentum (dgb_momentum_apply)",
                "algorithmic": f"{FLOP_PER_DOF['momentum']} flop/DoF x {D.n_u} DoF per launch (SURVEY 8d)",
                "peak_source": "FP64 pipe peak measured live: the higher of the DMMA (mma.sync m8n8k4.f64, "
                               "dgb_fp64_peak_dmma) and DFMA (dgb_fp64_peak) microbenchmarks; MEASURED_PEAKS.json "
                               "has no fp64.  The kernels issue DFMA only (DMMA shares the pipe and lost on the line "
                               "contractions, profiles/experiments_r02.md)",
                "peak_dfma": peak_dfma, "peak_dmma": peak_dmma, "frac_vs_dfma": mom_tflops / peak_dfma}
    roofline_hbm = {"achieved": BYTES_PER_DOF["momentum"] * D.n_u / tm / 1e9, "peak": peaks.get("hbm_gbs"),
                    "unit": "GB/s",
                    "frac": BYTES_PER_DOF["momentum"] * D.n_u / tm / 1e9 / peaks.get("hbm_gbs", 6535.7)}
    # ---- CPU baseline: reference on one host core, bounded sample
    cpu = None
    if ws == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_1core()
        except Exception as e:  # oracle not built on this box
            cpu = {"value": None, "unit": "GDoF/s", "cores": 1, "kind": "reference", "sample": f"unavailable: {e}"}
    line = {
        "metric": METRIC,
        "value": value, "unit": "GDoF/s", "n_gpus": ws, "steps": args.steps, "warmup": max(3, args.warmup),
        "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": DATA, "config": bench_config(ws), "warmup_steps_run": nwarm,
        "ops": {"momentum": {"ms": tm * 1e3, "gdofs": D.n_u / tm / 1e9, "tflops_alg": mom_tflops},
                "pressure": {"ms": tp * 1e3, "gdofs": D.n_p / tp / 1e9, "tflops_alg": prs_tflops,
                             "fp64_frac_alg": prs_tflops / peak_fp64,
                             "hbm_frac_alg": BYTES_PER_DOF["pressure"] * D.n_p / tp / 1e9 / peaks.get("hbm_gbs", 6535.7),
                             "note": "algorithmic = the reference's dense-table flop count (SURVEY 8d, 406.2 flop/DoF); "
                                     "the exact line split of k_sip_cell executes ~130 flop/DoF"}},
        "roofline": roofline, "roofline_hbm": roofline_hbm, "cpu_baseline": cpu,
        "e2e": {"value": e2e_val, "unit": "GDoF/s", "h2d_bytes_per_step": 8 * (2 * D.n_u + D.n_p),
                "d2h_bytes_per_step": 8 * (D.n_u + D.n_p)},
        "gpu_launches": int(launches), "clocks": clocks, "setup_s": setup_s,
        "trbdf2": trbdf2,
        "cfg4": cfg4,
        "cfg5_steps": cfg5,
    }
    print(json.dumps(line), flush=True)
    if ws > 1:
        tdist.barrier()
        tdist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="dgb", choices=["dgb", "reference"])
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline sample")
    ap.add_argument("--no-step", action="store_true", help="skip the full TR-BDF2 step timing")
    ap.add_argument("--no-cfg5", action="store_true", help="skip the cfg5 20-step runs")
    ap.add_argument("--no-cfg4", action="store_true", help="skip the cfg4 (deformed) applies and steps")
    args = ap.parse_args()
    if args.impl == "reference":
        run_reference(args)
    else:
        run_device(args)


if __name__ == "__main__":
    main()
