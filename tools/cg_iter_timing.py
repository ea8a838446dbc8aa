"""Time per Jacobi-CG iteration of the cfg3 / cfg5 pressure solve (400 iterations, CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
n, ku = (96, 2) if os.environ.get("CFG", "3") == "5" else (64, 3)
D = dg.DGContext(3, n, ku, ku - 1)
g = 2 - 2 ** 0.5
mc = 1 / (1e6 * (g * 1e-3) ** 2)
b = torch.from_numpy(dg.seeded_uniform(7, D.n_p)).cuda()
d = D.zeros(dg.SPACE_P); dg.helmholtz_diagonal(D, mc, d)
M = dg.JacobiPreconditioner(D, d)
for rep in range(3):
    x = D.zeros(dg.SPACE_P)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    try:
        dg.cg_solve(D, dg.LinearOperator.pressure_helmholtz(mc), b, dg.SolverSettings(rel_tol=1e-30, max_iter=400), M, x)
    except dg.SolverError:
        pass
    e1.record(); torch.cuda.synchronize()
    print(f"cfg{os.environ.get('CFG', '3')} {e0.elapsed_time(e1) / 400 * 1e3:.1f} us per CG iteration")
