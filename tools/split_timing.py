"""Time the momentum apply with only pass A / only pass B / both (cfg3)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
D = dg.DGContext(3, 64, 3, 2)
f = dg.SynthField(3, 2)
w = D.zeros(); dg.interpolate_synth_device(D, f, w)
x = torch.from_numpy(dg.seeded_uniform(1002, D.n_u)).cuda()
y = D.zeros()
g = 2 - 2 ** 0.5
for name, co in [("full", (1 / (g * 1e-3), 1 / 2000.0, 0.5, 0.0)), ("passA", (1 / (g * 1e-3), 1 / 2000.0, 0.0, 0.0)),
                 ("passB", (0.0, 0.0, 0.5, 0.0)), ("mass", (1.0, 0.0, 0.0, 0.0))]:
    ctx = dg.MomentumCtx(*co, advecting=w)
    for _ in range(3):
        dg.apply_momentum(D, ctx, x, y)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dg.apply_momentum(D, ctx, x, y)
    e1.record(); torch.cuda.synchronize()
    print(f"{name:6s} {e0.elapsed_time(e1) / 10:.3f} ms")
