import os, sys, time
sys.path.insert(0, os.getcwd())
import torch, paper_2107_07776_b200 as dg
D = dg.DGContext(3, 48, 4, 3, 0.1 / 48, 3)
f = dg.SynthField(3, 3)
for bid in range(6): D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
u = D.zeros(); dg.interpolate_synth_device(D, f, u)
p = torch.from_numpy(dg.seeded_uniform(5, D.n_p)).cuda()
y = D.zeros()
specs = {"full": dg.MomentumRhs(mass=[(1.0, u)], visc=[(0.005, u)], adv=[(0.5, u, u)], pres=[(1.0, p)], dir_visc_coef=0.005, dir_adv_coef=0.5, dir_w=u),
         "ops only": dg.MomentumRhs(mass=[(1.0, u)], visc=[(0.005, u)], adv=[(0.5, u, u)]),
         "pres only": dg.MomentumRhs(pres=[(1.0, p)]),
         "data only": dg.MomentumRhs(dir_visc_coef=0.005, dir_adv_coef=0.5, dir_w=u)}
for k, s in specs.items():
    for _ in range(2): dg.momentum_rhs(D, s, y)
    torch.cuda.synchronize(); t0 = time.time()
    for _ in range(5): dg.momentum_rhs(D, s, y)
    torch.cuda.synchronize(); print(k, (time.time() - t0) / 5 * 1e3, "ms")
