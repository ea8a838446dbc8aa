"""ncu driver: a few Jacobi-CG iterations of the cfg5 (96^3 Q1) / cfg3 pressure solve."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
n, ku = (96, 2) if os.environ.get("CFG", "5") == "5" else (64, 3)
D = dg.DGContext(3, n, ku, ku - 1)
g = 2 - 2 ** 0.5
mc = 1 / (1e6 * (g * 1e-3) ** 2)
b = torch.from_numpy(dg.seeded_uniform(7, D.n_p)).cuda()
d = D.zeros(dg.SPACE_P); dg.helmholtz_diagonal(D, mc, d)
M = dg.JacobiPreconditioner(D, d)
x = D.zeros(dg.SPACE_P)
try:
    dg.cg_solve(D, dg.LinearOperator.pressure_helmholtz(mc), b, dg.SolverSettings(rel_tol=1e-10, max_iter=40), M, x)
except dg.SolverError:
    pass
torch.cuda.synchronize()
print("ok")
