import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_07776_b200 as dg, reforacle as ref
for (dim, n, k, kp) in [(2, 4, 2, 1), (2,1,2,1), (3, 2, 2, 1)]:
    D = dg.DGContext(dim, n, k, kp); R = ref.RefCtx(dim, n, k, kp)
    w = dg.seeded_uniform(21, R.n_u); x = dg.seeded_uniform(22, R.n_u)
    for coefs in [(1,0,0,0),(0,1,0,0),(0,0,1,0),(0,0,0,1)]:
        want = R.momentum(coefs, w, x)
        y = D.zeros()
        dg.apply_momentum(D, dg.MomentumCtx(*coefs, advecting=torch.from_numpy(w).cuda()), torch.from_numpy(x).cuda(), y)
        torch.cuda.synchronize(); h = y.cpu().numpy()
        err = np.abs(h - want); i = int(err.argmax())
        print(dim, n, k, coefs, "rel", np.linalg.norm(h-want)/np.linalg.norm(want), "worst dof", i, h[i], want[i])
