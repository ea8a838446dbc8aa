"""Smallest cases of the hot kernels, for compute-sanitizer (racecheck / synccheck /
memcheck): one momentum + one pressure apply on the fast axis-aligned kernels
(k_momentum_axis<3>, k_sip_axis<2>; 4^3 Q3/Q2 -- several CTAs, CTA-internal and
external neighbours), the same on the deformed kernels (k_momentum_qp<4>, k_sip_qp<3>;
distorted 3^3 Q4/Q3), K = 2 / K = 1 variants (2^3 ... 5^3), and a few Jacobi-CG /
GMRES iterations (cg_* / gs_* kernels), plus the RHS / diagonal kernels of one stage.
Usage: compute-sanitizer --tool racecheck python tools/sanitize_cases.py"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

import paper_2107_07776_b200 as dg


def case(n_el, ku, amp=0.0, steps=False):
    D = dg.DGContext(3, n_el, ku, ku - 1, amp, 3) if amp else dg.DGContext(3, n_el, ku, ku - 1)
    w = torch.from_numpy(dg.seeded_uniform(1, D.n_u)).cuda()
    x = torch.from_numpy(dg.seeded_uniform(2, D.n_u)).cuda()
    xp = torch.from_numpy(dg.seeded_uniform(3, D.n_p)).cuda()
    y, yp = D.zeros(), D.zeros(dg.SPACE_P)
    ctx = dg.MomentumCtx(3.7, 0.01, 0.5, 0.0, advecting=w)
    dg.apply_momentum(D, ctx, x, y)
    dg.apply_pressure_helmholtz(D, 2.3, xp, yp)
    s = dg.SolverSettings(rel_tol=1e-10, max_iter=12, restart=5)
    for solve, op, b, n in ((dg.cg_solve, dg.LinearOperator.pressure_helmholtz(2.3), xp, D.n_p),
                            (dg.gmres_solve, dg.LinearOperator.momentum(ctx), x, D.n_u)):
        z = torch.zeros(n, dtype=torch.float64, device="cuda")
        try:
            solve(D, op, b, s, None, z)
        except dg.SolverError:
            pass  # 12 iterations: not converged, by design
    if steps:
        f = dg.SynthField(3, 1)
        for bid in range(6):
            D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
        u0 = D.zeros()
        dg.interpolate_synth_device(D, f, u0)
        u1, p1 = D.zeros(), D.zeros(dg.SPACE_P)
        dg.trbdf2_step(D, dg.StepParams(dt=1e-3, Re=100.0, c=1e3, restart=20, first_step=True),
                       u0, u0, D.zeros(dg.SPACE_P), u1, p1)
    torch.cuda.synchronize()
    print(f"ok {n_el}^3 Q{ku} amp {amp}", flush=True)


if __name__ == "__main__":
    case(4, 3, steps=True)
    case(3, 4, 0.03, steps=True)
    case(3, 2)
    case(2, 4)
