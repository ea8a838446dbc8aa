"""One-off parity evidence at full BASELINE sizes: one momentum apply (stage-1
coefficients, w = the synthetic field) and one pressure Helmholtz apply on the seeded
U[-1,1] vectors through the unmodified reference (oracle/_ref, CPU; its lazy geometry
build alone takes minutes and ~10+ GB) and through the device fast kernels.
Usage: python tools/full_apply_parity.py cfg2|cfg3|cfg4|cfg5 ; prints a JSON line."""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2107_07776_b200 as dg
import reforacle as ref

name = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
n_el, ku, amp, seed, Re = {"cfg2": (32, 2, 0.0, 1, 100.0), "cfg3": (64, 3, 0.0, 2, 1000.0),
                            "cfg4": (48, 4, 0.1 / 48, 3, 100.0), "cfg5": (96, 2, 0.0, 4, 1600.0)}[name]
kp = ku - 1
g = 2 - 2 ** 0.5
coefs = (1 / (g * 1e-3), 1 / (2 * Re), 0.5, 0.0)
pmc = 1 / (1e6 * g * g * 1e-6)
t0 = time.time()
R = ref.RefCtx(3, n_el, ku, kp, amp, 3 if amp else 0)
D = dg.DGContext(3, n_el, ku, kp, amp, 3) if amp else dg.DGContext(3, n_el, ku, kp)
f = dg.SynthField(3, seed)
w = f.interpolate(D)
x = dg.seeded_uniform(seed + 1000, D.n_u)
xp = dg.seeded_uniform(seed + 2000, D.n_p)
t_setup = time.time() - t0
t0 = time.time()
want_u = R.momentum(coefs, w, x)
t_ref_u = time.time() - t0
t0 = time.time()
want_p = R.pressure(pmc, xp)
t_ref_p = time.time() - t0
y, yp = D.zeros(), D.zeros(dg.SPACE_P)
dg.apply_momentum(D, dg.MomentumCtx(*coefs, advecting=torch.from_numpy(w).cuda()), torch.from_numpy(x).cuda(), y)
dg.apply_pressure_helmholtz(D, pmc, torch.from_numpy(xp).cuda(), yp)
torch.cuda.synchronize()
rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
print(json.dumps({"config": name, "mesh": f"{n_el}^3", "degrees": f"Q{ku}/Q{kp}", "deformed": bool(amp),
                  "kernels": ["generic", "fast axis-aligned", "fast deformed"][dg.lib().dgb_fast_path_active(D.handle)],
                  "n_u": D.n_u, "n_p": D.n_p, "rel_l2_momentum": rel(y.cpu().numpy(), want_u),
                  "rel_l2_pressure": rel(yp.cpu().numpy(), want_p), "reference_momentum_s_incl_lazy_geometry": t_ref_u,
                  "reference_pressure_s": t_ref_p, "setup_s": t_setup}))
