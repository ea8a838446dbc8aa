"""One-off parity evidence at a full BASELINE size: one TR-BDF2 step of cfg2 (3D 32^3,
Q2/Q1, Re 100, dt 1e-3, seed 1; minutes on one CPU core for the reference) through the
restated reference driver (oracle/_ref, CPU) and through the device, from the same
synthetic u^0 (Dirichlet data = its trace, p^0 = 0).  Prints a JSON line with the
Krylov iteration counts of both sides and the relative L2 field differences.
CFG_N / KU override the mesh and degree."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2107_07776_b200 as dg
import reforacle as ref

n_el, ku = int(os.environ.get("CFG_N", "32")), int(os.environ.get("KU", "2"))
kp, seed, Re, dt = ku - 1, 1, 100.0, 1e-3
R = ref.RefCtx(3, n_el, ku, kp, 0.0, 7)
D = dg.DGContext(3, n_el, ku, kp)
f = dg.SynthField(3, seed)
for bid in range(6):
    R.set_bc(bid, 0, f.fn_ptr, f.user_ptr)
    D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
u0 = f.interpolate(D)
p0 = np.zeros(R.n_p)
t0 = time.time()
u1, p1, its_ref = R.step([dt, Re, 1e3, 0.0, 50, 1e-10, 1e-10, 1e-12, 10000, 1.0], u0, u0, p0)
t_ref = time.time() - t0
du0 = torch.from_numpy(u0).cuda()
dp0 = torch.from_numpy(p0).cuda()
du1, dp1 = D.zeros(), D.zeros(dg.SPACE_P)
torch.cuda.synchronize()
t0 = time.time()
its = dg.trbdf2_step(D, dg.StepParams(dt=dt, Re=Re, c=1e3, restart=50, first_step=True), du0, du0, dp0, du1, dp1)
torch.cuda.synchronize()
t_dev = time.time() - t0
hu, hp = du1.cpu().numpy(), dp1.cpu().numpy()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(json.dumps({"config": f"3D {n_el}^3 Q{ku}/Q{kp}, Re {Re}, dt {dt}, seed {seed}, one TR-BDF2 step from u^0",
                  "n_u": D.n_u, "n_p": D.n_p, "its_device": its[:8], "its_reference": its_ref[:8],
                  "max_its_diff": max(abs(a - b) for a, b in zip(its[:8], its_ref[:8])),
                  "rel_l2_u": rel(hu, u1), "rel_l2_p_mean_free": rel(hp - hp.mean(), p1 - p1.mean()),
                  "reference_s": t_ref, "device_s": t_dev}))
