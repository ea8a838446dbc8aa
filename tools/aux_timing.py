"""Time the once-per-stage auxiliary operators at cfg3 (divergence, gradient, mass, diagonals)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
D = dg.DGContext(3, 64, 3, 2)
f = dg.SynthField(3, 2)
u = D.zeros(); dg.interpolate_synth_device(D, f, u)
p = torch.from_numpy(dg.seeded_uniform(5, D.n_p)).cuda()
yu, yp = D.zeros(), D.zeros(dg.SPACE_P)
ops = {
    "divergence": lambda: dg.divergence_functional(D, u, yp),
    "gradient": lambda: dg.pressure_gradient_rhs(D, p, yu),
    "mass_u": lambda: dg.apply_mass(D, dg.SPACE_U, u, yu),
    "mass_p": lambda: dg.apply_mass(D, dg.SPACE_P, p, yp),
    "helmholtz_diag": lambda: dg.helmholtz_diagonal(D, 2.3, yp),
    "mass_diag_u": lambda: dg.mass_diagonal(D, dg.SPACE_U, yu),
}
for name, fn in ops.items():
    for _ in range(2):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        fn()
    e1.record(); torch.cuda.synchronize()
    print(f"{name:16s} {e0.elapsed_time(e1) / 5:8.3f} ms")
