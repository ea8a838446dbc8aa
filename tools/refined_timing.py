"""Momentum / pressure applies on an axis-aligned REFINED mesh (1-irregular, hanging faces):
the line-split fast kernels + hang.cu against the generic kernels + hang.cu.

The mesh comes from the reference's own refinement (oracle/_ref: generate_cartesian +
Mesh::refine_and_coarsen of the cells inside a ball), handed to the device through
dgb_ctx_create_mesh_hanging as a reference-side binding would.
  python tools/refined_timing.py [n_el=24] [ku=3] [radius=0.3]
"""
import json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import torch
import paper_2107_07776_b200 as dg
import reforacle as ref

n_el = int(sys.argv[1]) if len(sys.argv) > 1 else 24
ku = int(sys.argv[2]) if len(sys.argv) > 2 else 3
rad = float(sys.argv[3]) if len(sys.argv) > 3 else 0.3
kp = ku - 1
i = np.arange(n_el ** 3)
cx = ((i % n_el) + 0.5) / n_el - 0.5
cy = (((i // n_el) % n_el) + 0.5) / n_el - 0.5
cz = ((i // (n_el * n_el)) + 0.5) / n_el - 0.5
refine = np.nonzero(cx * cx + cy * cy + cz * cz < rad * rad)[0]
t0 = time.time()
R = ref.RefCtx.refined(3, n_el, ku, kp, refine)
xv, cv, bid, it, emb = R.mesh_arrays()
hang = it[:, 4] == 1
D = dg.DGContext(3, 0, ku, kp, mesh_arrays=(xv, cv, bid, it[hang, :4], emb[hang]))
setup = time.time() - t0
g = 2 - 2 ** 0.5
w = torch.from_numpy(dg.seeded_uniform(1, D.n_u)).cuda()
x = torch.from_numpy(dg.seeded_uniform(2, D.n_u)).cuda()
xp = torch.from_numpy(dg.seeded_uniform(3, D.n_p)).cuda()
y, yp = D.zeros(), D.zeros(dg.SPACE_P)
ctx = dg.MomentumCtx(1 / (g * 1e-3), 1 / 2000.0, 0.5, 0.0, advecting=w)
pmc = 1 / (1e6 * g * g * 1e-6)
out = {"mesh": f"{n_el}^3 base, cells within {rad} of the centre refined once", "ncells": D.ncells,
       "n_hanging": D.n_hanging, "degrees": f"Q{ku}/Q{kp}", "n_u": D.n_u, "n_p": D.n_p, "setup_s": setup}
res = {}
for fast in (True, False):
    D.set_fast_path(fast)
    for op in ("momentum", "pressure"):
        fn = (lambda: dg.apply_momentum(D, ctx, x, y)) if op == "momentum" else (
            lambda: dg.apply_pressure_helmholtz(D, pmc, xp, yp))
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[(fast, op)] = (e0.elapsed_time(e1) / 10, (y if op == "momentum" else yp).cpu().numpy().copy())
for op, n in (("momentum", D.n_u), ("pressure", D.n_p)):
    tf, yf = res[(True, op)]
    tg, yg = res[(False, op)]
    out[op] = {"fast_ms": tf, "generic_ms": tg, "speedup": tg / tf, "fast_gdofs": n / tf / 1e6,
               "rel_l2_fast_vs_generic": float(np.linalg.norm(yf - yg) / np.linalg.norm(yg))}
# one TR-BDF2 step (Dirichlet data = the synthetic field's trace, Re 1000, dt 1e-3, GMRES(30) / Jacobi-CG)
if os.environ.get("STEP", "1") != "0":
    f = dg.SynthField(3, 2)
    for b in range(6):
        D.set_dirichlet_fn(b, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros(); dg.interpolate_synth_device(D, f, u0)
    p0 = D.zeros(dg.SPACE_P)
    sp = dg.StepParams(dt=1e-3, Re=1000.0, c=1e3, restart=30, first_step=True)
    out["trbdf2_step"] = {}
    fields = {}
    for fast in (True, False):
        D.set_fast_path(fast)
        u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
        for rep in range(2):
            torch.cuda.synchronize(); t0 = time.time()
            its = dg.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
            torch.cuda.synchronize(); t = time.time() - t0
        out["trbdf2_step"]["fast" if fast else "generic"] = {"s": t, "its": [int(i) for i in its]}
        fields[fast] = (u1.cpu().numpy(), p1.cpu().numpy())
    out["trbdf2_step"]["rel_l2_u_fast_vs_generic"] = float(
        np.linalg.norm(fields[True][0] - fields[False][0]) / np.linalg.norm(fields[False][0]))
    D.set_fast_path(True)
print(json.dumps(out))
