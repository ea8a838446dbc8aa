"""A/B timing of libdgb variants (tools/ab_build.sh) on the cfg3 momentum / pressure applies:
each variant in its own process (DGB_LIB), rounds interleaved; prints the median per variant.
usage: python tools/ab_time.py rounds name [name ...]"""
import json, os, statistics, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CHILD = r'''
import os, sys, json
sys.path.insert(0, os.environ["ROOT"])
import torch
import paper_2107_07776_b200 as dg
cfg = os.environ.get("CFG", "cfg3")
n_el, ku, seed, Re, amp = {"cfg2": (32, 2, 1, 100.0, 0.0), "cfg3": (64, 3, 2, 1000.0, 0.0),
                            "cfg4": (48, 4, 3, 100.0, 0.1 / 48), "cfg5": (96, 2, 4, 1600.0, 0.0)}[cfg]
D = dg.DGContext(3, n_el, ku, ku - 1, amp, 3) if amp else dg.DGContext(3, n_el, ku, ku - 1)
f = dg.SynthField(3, seed)
w = D.zeros(); dg.interpolate_synth_device(D, f, w)
x = torch.from_numpy(dg.seeded_uniform(seed + 1000, D.n_u)).cuda()
xp = torch.from_numpy(dg.seeded_uniform(seed + 2000, D.n_p)).cuda()
y = D.zeros(); yp = D.zeros(dg.SPACE_P)
g = 2 - 2 ** 0.5
ctx = dg.MomentumCtx(1 / (g * 1e-3), 1 / (2 * Re), 0.5, 0.0, advecting=w)
out = {}
for op, fn in (("mom", lambda: dg.apply_momentum(D, ctx, x, y)),
               ("prs", lambda: dg.apply_pressure_helmholtz(D, 1 / (1e6 * g * g * 1e-6), xp, yp))):
    for _ in range(5): fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): fn()
    e1.record(); torch.cuda.synchronize()
    out[op] = e0.elapsed_time(e1) / 20
out["norm"] = float(y.norm())
print(json.dumps(out))
'''
rounds, names = int(sys.argv[1]), sys.argv[2:]
res = {n: [] for n in names}
for r in range(rounds):
    for n in names:
        lib = os.path.join(ROOT, "paper_2107_07776_b200", "libdgb.so") if n == "main" else os.path.join(ROOT, "tune", f"libdgb_{n}.so")
        env = dict(os.environ, DGB_LIB=lib, ROOT=ROOT)
        o = subprocess.run([sys.executable, "-c", CHILD], env=env, capture_output=True, text=True)
        if o.returncode:
            print(n, "FAILED", o.stderr[-500:]); continue
        res[n].append(json.loads(o.stdout.strip().splitlines()[-1]))
for n in names:
    if res[n]:
        print(f"{n:14s} mom {statistics.median(v['mom'] for v in res[n]):.4f} ms  prs {statistics.median(v['prs'] for v in res[n]):.4f} ms"
              f"  (n={len(res[n])}, |y| {res[n][0]['norm']:.10e})", flush=True)
