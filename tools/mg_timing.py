"""Pressure solve and TR-BDF2 step: Jacobi-CG (the reference's) vs multigrid-CG, cfg2/3/5."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
cfgs = {"cfg2": (32, 2, 1, 1, 100.0, 1e-3, 50), "cfg3": (64, 3, 2, 2, 1000.0, 1e-3, 30),
        "cfg5": (96, 2, 1, 4, 1600.0, 4.510549e-3, 50)}
for name in (sys.argv[1:] or list(cfgs)):
    n, ku, kp, seed, Re, dt, restart = cfgs[name]
    D = dg.DGContext(3, n, ku, kp)
    g = 2 - 2 ** 0.5
    mc = 1 / (1e6 * (g * dt) ** 2)
    b = torch.from_numpy(dg.seeded_uniform(seed + 2000, D.n_p)).cuda()
    s = dg.SolverSettings(rel_tol=1e-10, max_iter=20000)
    d = D.zeros(dg.SPACE_P); dg.helmholtz_diagonal(D, mc, d)
    M = dg.JacobiPreconditioner(D, d)
    for pc in ("jacobi", "mg"):
        for rep in range(2):
            x = D.zeros(dg.SPACE_P)
            torch.cuda.synchronize(); t0 = time.time()
            r = dg.cg_solve(D, dg.LinearOperator.pressure_helmholtz(mc), b, s, M, x) if pc == "jacobi" else \
                dg.pressure_cg_mg(D, mc, b, s, x)
            torch.cuda.synchronize()
        print(f"{name} pressure solve {pc}: {time.time()-t0:.4f} s, {r.iterations} its", flush=True)
    f = dg.SynthField(3, seed)
    for bid in range(6):
        D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros(); dg.interpolate_synth_device(D, f, u0)
    p0 = D.zeros(dg.SPACE_P)
    for pc in ("jacobi", "mg"):
        u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
        for rep in range(2):
            sp = dg.StepParams(dt=dt, Re=Re, c=1e3, restart=restart, first_step=True, pressure_precond=pc)
            torch.cuda.synchronize(); t0 = time.time()
            its = dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
            torch.cuda.synchronize()
        print(f"{name} step {pc}: {time.time()-t0:.3f} s, its {its}", flush=True)
    del D
    torch.cuda.empty_cache()
