"""Per-call times of the non-Krylov operators of a step (mass, gradient, divergence,
pressure diagonal) on cfg3 / cfg4, fast and generic paths (CUDA events)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
CFGS = {"cfg3": (64, 3, 0.0), "cfg4": (48, 4, 0.1 / 48)}
for name in sys.argv[1:] or list(CFGS):
    n_el, ku, amp = CFGS[name]
    D = dg.DGContext(3, n_el, ku, ku - 1, amp, 3 if amp else 0)
    x = torch.from_numpy(dg.seeded_uniform(5, D.n_u)).cuda()
    xp = torch.from_numpy(dg.seeded_uniform(6, D.n_p)).cuda()
    y, yp = D.zeros(), D.zeros(dg.SPACE_P)
    ops = {"mass_u": lambda: dg.apply_mass(D, dg.SPACE_U, x, y),
           "mass_p": lambda: dg.apply_mass(D, dg.SPACE_P, xp, yp),
           "gradient": lambda: dg.pressure_gradient_rhs(D, xp, y),
           "divergence": lambda: dg.divergence_functional(D, x, yp),
           "p_diag": lambda: dg.helmholtz_diagonal(D, 2.0, yp),
           "mass_diag_u": lambda: dg.mass_diagonal(D, dg.SPACE_U, y)}
    for fast in (True, False):
        D.set_fast_path(fast)
        out = []
        for k, fn in ops.items():
            for _ in range(2):
                fn()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                fn()
            e1.record(); torch.cuda.synchronize()
            out.append(f"{k} {e0.elapsed_time(e1) / 5:.3f}")
        print(f"{name} fast={fast}: " + ", ".join(out) + " ms", flush=True)
    del D
    torch.cuda.empty_cache()
