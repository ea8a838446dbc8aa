"""Minimal driver for ncu: cfg5 (96^3 affine Q2/Q1) momentum + pressure applies (2 each)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
D = dg.DGContext(3, 96, 2, 1)
f = dg.SynthField(3, 4)
w = D.zeros(); dg.interpolate_synth_device(D, f, w)
x = torch.from_numpy(dg.seeded_uniform(1003, D.n_u)).cuda()
xp = torch.from_numpy(dg.seeded_uniform(2003, D.n_p)).cuda()
y, yp = D.zeros(), D.zeros(dg.SPACE_P)
g = 2 - 2 ** 0.5
ctx = dg.MomentumCtx(1 / (g * 1e-3), 1 / 3200.0, 0.5, 0.0, advecting=w)
for _ in range(2):
    dg.apply_momentum(D, ctx, x, y)
    dg.apply_pressure_helmholtz(D, 1 / (1e6 * g * g * 1e-6), xp, yp)
torch.cuda.synchronize()
print("ok", float(y.norm()), float(yp.norm()))
