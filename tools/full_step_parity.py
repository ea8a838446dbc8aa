"""Full-size TR-BDF2 step parity (VERDICT r01 "next round" item 1).

One TR-BDF2 step of a BASELINE config from the synthetic u^0 (Dirichlet data = its
trace on every boundary, p^0 = 0) through the restated reference driver
(oracle/trbdf2_cpu.hpp over the unmodified reference, oracle/_ref) and through the
device (dgb_trbdf2_step).  The two halves run on different machines, because the
cfg3 CPU step takes hours and ~26 GB:

  python tools/full_step_parity.py cpu cfg3      # here (no GPU): writes parity_data/cfg3_step_ref.*
  python tools/full_step_parity.py gpu cfg3      # on the GPU box: device step, compares, prints JSON

A gpurun snapshot is limited to 512 MiB, so the cfg3 velocity (403 MB) is compared in parts:
  python tools/full_step_parity.py split cfg3 3          # here: u -> 3 chunk files
  python tools/full_step_parity.py gpu cfg3 0/3          # one gpurun call per part (the other
                                                         # chunks listed in .gpurunignore):
                                                         # device step, sums over that chunk
  python tools/full_step_parity.py merge cfg3 3 dir      # here: the parts' JSON -> one report

Inputs come from the oracle-side generator (reforacle.SynthField, bit-identical to the
product's, tests/test_oracle_inputs.py) on both sides, and the GPU half checks the
SHA-256 of u^0 against the one the CPU half recorded.  parity_data/ is git-ignored
but travels to the GPU box with the gpurun snapshot.
"""
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np

import reforacle as ref

# name: (n_el, ku, seed, Re, dt, restart)  -- BASELINE.json configs, SURVEY Appendix C3/C12
CFGS = {"cfg2": (32, 2, 1, 100.0, 1e-3, 50), "cfg3": (64, 3, 2, 1000.0, 1e-3, 30)}
DATA = os.path.join(ROOT, "parity_data")


def inputs(name, nthreads):
    n_el, ku, seed, Re, dt, restart = CFGS[name]
    R = ref.RefCtx(3, n_el, ku, ku - 1, 0.0, 0)
    f = ref.SynthField(3, seed)
    u0 = f.interpolate(R, nthreads)
    return R, f, u0, hashlib.sha256(u0.tobytes()).hexdigest()


def cpu(name):
    n_el, ku, seed, Re, dt, restart = CFGS[name]
    os.makedirs(DATA, exist_ok=True)
    R, f, u0, sha = inputs(name, os.cpu_count() or 1)
    for bid in range(6):
        R.set_bc(bid, 0, f.fn_ptr, f.user_ptr)
    p0 = np.zeros(R.n_p)
    t0 = time.time()
    u1, p1, its = R.step([dt, Re, 1e3, 0.0, restart, 1e-10, 1e-10, 1e-12, 10000, 1.0], u0, u0, p0)
    t = time.time() - t0
    np.save(os.path.join(DATA, f"{name}_step_ref_u.npy"), u1)
    np.save(os.path.join(DATA, f"{name}_step_ref_p.npy"), p1)
    meta = {"config": name, "n_u": R.n_u, "n_p": R.n_p, "u0_sha256": sha, "its_reference": its[:8],
            "reference_s": t, "backend": ref.lib().ref_backend().decode()}
    json.dump(meta, open(os.path.join(DATA, f"{name}_step_ref.json"), "w"))
    print(json.dumps(meta))


def split(name, k):
    u = np.load(os.path.join(DATA, f"{name}_step_ref_u.npy"))
    for i, c in enumerate(np.array_split(u, k)):
        np.save(os.path.join(DATA, f"{name}_step_ref_u.{i}of{k}.npy"), c)
    os.remove(os.path.join(DATA, f"{name}_step_ref_u.npy"))


def merge(name, k, d):
    parts = [json.load(open(os.path.join(d, f"{name}_step_part{i}of{k}.json"))) for i in range(k)]
    out = dict(parts[0])
    du2, u2 = sum(p["du2"] for p in parts), sum(p["u2"] for p in parts)
    for key in ("du2", "u2", "part"):
        out.pop(key, None)
    out["rel_l2_u"] = float(np.sqrt(du2 / u2))
    out["device_runs"] = [{"its_device": p["its_device"], "device_s_incl_first_use_alloc": p["device_s_incl_first_use_alloc"]}
                          for p in parts]
    out["max_its_diff"] = max(p["max_its_diff"] for p in parts)
    out["note"] = (f"velocity compared in {k} parts (one device step per gpurun call, snapshot size limit); "
                   "every part's device step has the same iteration counts")
    out["pass"] = bool(out["max_its_diff"] <= 1 and out["rel_l2_u"] <= 1e-9 and out["rel_l2_p_mean_free"] <= 1e-9)
    print(json.dumps(out))


def gpu(name, part=None):
    import torch

    import paper_2107_07776_b200 as dg
    n_el, ku, seed, Re, dt, restart = CFGS[name]
    meta = json.load(open(os.path.join(DATA, f"{name}_step_ref.json")))
    R, f, u0, sha = inputs(name, os.cpu_count() or 1)
    assert sha == meta["u0_sha256"], "u^0 differs from the CPU half's"
    D = dg.DGContext(3, n_el, ku, ku - 1)
    g = dg.SynthField(3, seed)  # product generator: the device's Dirichlet callback (same values)
    assert (g.user == f.user).all()
    for bid in range(6):
        D.set_dirichlet_fn(bid, g.fn_ptr, g.user_ptr, 0.0)
    du0 = torch.from_numpy(u0).cuda()
    dp0 = torch.zeros(D.n_p, dtype=torch.float64, device="cuda")
    du1, dp1 = D.zeros(), D.zeros(dg.SPACE_P)
    torch.cuda.synchronize()
    t0 = time.time()
    its = dg.trbdf2_step(D, dg.StepParams(dt=dt, Re=Re, c=1e3, restart=restart, first_step=True),
                         du0, du0, dp0, du1, dp1)
    torch.cuda.synchronize()
    t_dev = time.time() - t0
    p1 = np.load(os.path.join(DATA, f"{name}_step_ref_p.npy"))
    hu, hp = du1.cpu().numpy(), dp1.cpu().numpy()
    if part is not None:  # one chunk of the velocity: partial sums only
        i, k = part
        u1c = np.load(os.path.join(DATA, f"{name}_step_ref_u.{i}of{k}.npy"))
        hc = np.array_split(hu, k)[i]
        assert hc.shape == u1c.shape
        u1 = None
    else:
        u1 = np.load(os.path.join(DATA, f"{name}_step_ref_u.npy"))
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    out = {"config": f"{name}: 3D {n_el}^3 Q{ku}/Q{ku - 1}, Re {Re}, dt {dt}, seed {seed}, GMRES({restart}) + "
                     f"Jacobi, CG + Jacobi, rel tol 1e-10 (mass 1e-12); one TR-BDF2 step from u^0",
           "n_u": D.n_u, "n_p": D.n_p, "u0_sha256": sha,
           "its_legend": "[gmres s1, gmres s2, cg s1, cg s2, mass-cg s1 pre, s1 post, s2 pre, s2 post]",
           "its_device": its[:8], "its_reference": meta["its_reference"],
           "max_its_diff": max(abs(a - b) for a, b in zip(its[:8], meta["its_reference"])),
           "rel_l2_u": rel(hu, u1) if u1 is not None else None,
           "rel_l2_p_mean_free": rel(hp - hp.mean(), p1 - p1.mean()),
           "reference_s_1core": meta["reference_s"], "reference_backend": meta["backend"],
           "device_s_incl_first_use_alloc": t_dev}
    if part is not None:
        out["part"] = f"{part[0]}/{part[1]}"
        out["du2"] = float(np.sum((hc - u1c) ** 2))
        out["u2"] = float(np.sum(u1c ** 2))
        os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
        json.dump(out, open(os.path.join(ROOT, "gpurun_out", f"{name}_step_part{part[0]}of{part[1]}.json"), "w"))
    else:
        out["pass"] = bool(out["max_its_diff"] <= 1 and out["rel_l2_u"] <= 1e-9 and out["rel_l2_p_mean_free"] <= 1e-9)
    print(json.dumps(out))


if __name__ == "__main__":
    cmd, name = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "cfg3"
    if cmd == "cpu":
        cpu(name)
    elif cmd == "split":
        split(name, int(sys.argv[3]))
    elif cmd == "merge":
        merge(name, int(sys.argv[3]), sys.argv[4])
    else:
        part = tuple(int(v) for v in sys.argv[3].split("/")) if len(sys.argv) > 3 else None
        gpu(name, part)
