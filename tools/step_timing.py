"""Time one device TR-BDF2 step (BASELINE configs) and report Krylov iteration counts."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
cfg = os.environ.get("CFG", "3")
P = {"1": (2, 32, 2, 1, 0, 100.0, 1e-3, 50), "2": (3, 32, 2, 1, 1, 100.0, 1e-3, 50),
     "3": (3, 64, 3, 2, 2, 1000.0, 1e-3, 30), "4": (3, 48, 4, 3, 3, 100.0, 1e-3, 50)}[cfg]
dim, n_el, ku, kp, seed, Re, dt, restart = P
# cfg4: interior vertices displaced by U[-0.1h, 0.1h] (seed 3), per-qp geometry
D = dg.DGContext(dim, n_el, ku, kp, 0.1 / n_el, 3) if cfg == "4" else dg.DGContext(dim, n_el, ku, kp)
f = dg.SynthField(dim, seed)
t0 = time.time()
for bid in range(2 * dim):
    D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
print("dirichlet table", time.time() - t0, "s")
u0 = D.zeros(); dg.interpolate_synth_device(D, f, u0)
p0 = D.zeros(dg.SPACE_P)
u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
sp = dg.StepParams(dt=dt, Re=Re, c=1e3, restart=restart, first_step=True,
                   pressure_precond=os.environ.get("PRECOND", "jacobi"))
torch.cuda.synchronize()
for rep in range(2):
    t0 = time.time(); l0 = D.launch_count()
    its = dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
    torch.cuda.synchronize()
    print(f"cfg{cfg} step {rep}: {time.time()-t0:.3f} s, its {its}, launches {D.launch_count()-l0}")
