import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
D = dg.DGContext(3, 64, 3, 2)
w = D.zeros()
x = torch.from_numpy(dg.seeded_uniform(1002, D.n_u)).cuda()
y = D.zeros()
f = dg.SynthField(3, 2); dg.interpolate_synth_device(D, f, w); ctx = dg.MomentumCtx(0.0, 0.0, 0.5, 0.0, advecting=w)
for _ in range(3):
    dg.apply_momentum(D, ctx, x, y)
torch.cuda.synchronize()
print("ok")
