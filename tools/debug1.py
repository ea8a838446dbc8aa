import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import paper_2107_07776_b200 as dg, reforacle as ref
D = dg.DGContext(2, 4, 2, 1)
R = ref.RefCtx(2, 4, 2, 1)
x = dg.seeded_uniform(11, R.n_p)
xd = torch.from_numpy(x).cuda()
y = D.zeros(dg.SPACE_P)
rc = dg.lib().dgb_pressure_apply(D.handle, 2.3, xd.data_ptr(), y.data_ptr())
print("rc", rc, dg.lib().dgb_last_error())
D.sync(); torch.cuda.synchronize()
print(y[:8].cpu().numpy()); print(R.pressure(2.3, x)[:8])
m = D.zeros(dg.SPACE_P); dg.apply_mass(D, 1, xd, m); D.sync(); print("mass", m[:4].cpu().numpy(), R.mass(1, x)[:4])
print("launches", D.launch_count())
