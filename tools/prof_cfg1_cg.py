import os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2107_07776_b200 as dg
D = dg.DGContext(2, 32, 2, 1)
mc = 2.9
b = torch.from_numpy(dg.seeded_uniform(7, D.n_p)).cuda()
d = D.zeros(dg.SPACE_P); dg.helmholtz_diagonal(D, mc, d)
M = dg.JacobiPreconditioner(D, d)
x = D.zeros(dg.SPACE_P)
try:
    dg.cg_solve(D, dg.LinearOperator.pressure_helmholtz(mc), b, dg.SolverSettings(rel_tol=1e-10, max_iter=40), M, x)
except dg.SolverError:
    pass
torch.cuda.synchronize()
