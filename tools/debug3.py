import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_07776_b200 as dg, reforacle as ref
for (n, k, coefs) in [(3, 2, (1,0,0,0)), (3,2,(0,1,0,0)), (3,2,(0,0,1,0)), (2,2,(0,1,0,0)), (3,3,(0,1,0,0)), (3,1,(0,1,0,0)),(1,2,(0,1,0,0))]:
    D = dg.DGContext(3, n, k, k-1 if k>1 else 1); R = ref.RefCtx(3, n, k, k-1 if k>1 else 1)
    w = dg.seeded_uniform(21, R.n_u); x = dg.seeded_uniform(22, R.n_u)
    want = R.momentum(coefs, w, x)
    outs = []
    for fast in (True, False):
        D.set_fast_path(fast)
        y = D.zeros()
        dg.apply_momentum(D, dg.MomentumCtx(*coefs, advecting=torch.from_numpy(w).cuda()), torch.from_numpy(x).cuda(), y)
        torch.cuda.synchronize(); outs.append(y.cpu().numpy())
    h = outs[0]; err = np.abs(h - want); i = int(err.argmax())
    nb = (k+1)**3
    print(n, k, coefs, D.fast_path_active, "fast rel", np.linalg.norm(h-want)/np.linalg.norm(want), "generic rel", np.linalg.norm(outs[1]-want)/np.linalg.norm(want),
          "worst", i, "cell", i//(3*nb), "comp", (i%(3*nb))//nb, "node", i%nb, h[i], want[i])
