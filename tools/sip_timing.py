"""Time the pressure Helmholtz apply (cfg3 / cfg2 sizes)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
for n_el, ku in ((64, 3), (32, 2), (96, 2)):
    D = dg.DGContext(3, n_el, ku, ku - 1)
    xp = torch.from_numpy(dg.seeded_uniform(2002, D.n_p)).cuda()
    yp = D.zeros(dg.SPACE_P)
    g = 2 - 2 ** 0.5
    for _ in range(3):
        dg.apply_pressure_helmholtz(D, 1 / (1e6 * g * g * 1e-6), xp, yp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        dg.apply_pressure_helmholtz(D, 1 / (1e6 * g * g * 1e-6), xp, yp)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print(f"n_el {n_el} kp {ku-1}: {ms:.4f} ms  {D.n_p / ms / 1e6:.1f} GDoF/s")
    del D
