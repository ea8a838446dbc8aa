import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_07776_b200 as dg, reforacle as ref
coefs = (1.0 / (0.2929 * 1e-3), 0.005, 0.5, 0.0)
for order in ("diag_first", "apply_first"):
    D = dg.DGContext(3, 3, 2, 1); R = ref.RefCtx(3, 3, 2, 1)
    w = dg.seeded_uniform(21, R.n_u); x = dg.seeded_uniform(22, R.n_u)
    wd = torch.from_numpy(w).cuda(); ctx = dg.MomentumCtx(*coefs, advecting=wd)
    def diag():
        d = D.zeros(); dg.momentum_diagonal(D, ctx, d); torch.cuda.synchronize(); return d.cpu().numpy()
    def apply():
        y = D.zeros(); dg.apply_momentum(D, ctx, torch.from_numpy(x).cuda(), y); torch.cuda.synchronize(); return y.cpu().numpy()
    if order == "diag_first":
        d = diag(); y = apply()
    else:
        y = apply(); d = diag()
    wd_ = R.momentum_diag(coefs, w)
    print(order, "diag nan", np.isnan(d).sum(), "rel", np.linalg.norm(d-wd_)/np.linalg.norm(wd_), "apply rel", np.linalg.norm(y-R.momentum(coefs,w,x))/np.linalg.norm(R.momentum(coefs,w,x)))
    print("  w on device still intact:", np.abs(wd.cpu().numpy()-w).max())
