"""Momentum / pressure apply throughput on the BASELINE 3D configs (2-5)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2107_07776_b200 as dg
g = 2 - 2 ** 0.5
# cfg: (n_el, ku, amp, seed, Re, flop/DoF mom, prs, bytes/DoF mom, prs)
CFGS = {"cfg2": (32, 2, 0.0, 1, 100.0, 530.6, 470.2, 24, 16), "cfg3": (64, 3, 0.0, 2, 1000.0, 545.9, 406.2, 24, 16),
        "cfg4": (48, 4, 0.1 / 48, 3, 100.0, 631.7, 450.9, 182.6, 378.5),
        "cfg5": (96, 2, 0.0, 4, 1600.0, 530.6, 470.2, 24, 16)}
sel = sys.argv[1:] or list(CFGS)
for name in sel:
    n_el, ku, amp, seed, Re, fm, fp, bm, bp = CFGS[name]
    t0 = time.time()
    D = dg.DGContext(3, n_el, ku, ku - 1, amp, 3 if amp else 0)
    f = dg.SynthField(3, seed)
    w = D.zeros(); dg.interpolate_synth_device(D, f, w)
    x = torch.from_numpy(dg.seeded_uniform(seed + 1000, D.n_u)).cuda()
    xp = torch.from_numpy(dg.seeded_uniform(seed + 2000, D.n_p)).cuda()
    y = D.zeros(); yp = D.zeros(dg.SPACE_P)
    ctx = dg.MomentumCtx(1 / (g * 1e-3), 1 / (2 * Re), 0.5, 0.0, advecting=w)
    pmc = 1 / (1e6 * g * g * 1e-6)
    setup = time.time() - t0
    res = {}
    for op in ("mom", "prs"):
        fn = (lambda: dg.apply_momentum(D, ctx, x, y)) if op == "mom" else (lambda: dg.apply_pressure_helmholtz(D, pmc, xp, yp))
        for _ in range(3):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fn()
        e1.record(); torch.cuda.synchronize()
        res[op] = e0.elapsed_time(e1) / 10
    nu, np_ = D.n_u, D.n_p
    print(f"{name}: setup {setup:.1f}s fast={D.fast_path_active} | mom {res['mom']:.3f} ms {nu/res['mom']/1e6:.1f} GDoF/s "
          f"{fm*nu/res['mom']/1e9:.1f} TF/s {bm*nu/res['mom']/1e6:.0f} GB/s | prs {res['prs']:.4f} ms "
          f"{np_/res['prs']/1e6:.1f} GDoF/s {fp*np_/res['prs']/1e9:.1f} TF/s {bp*np_/res['prs']/1e6:.0f} GB/s", flush=True)
    del D, w, x, xp, y, yp
    torch.cuda.empty_cache()
