"""Generate golden vectors from the COMPILED REFERENCE (oracle/_ref/libdgref.so,
built from /root/reference/proj/src by oracle/Makefile).

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
Writes tests/golden/<case>.npz with the mesh (vertex coordinates, cell vertex
ids, boundary ids), the seeded inputs and the reference outputs.  These pin the
numpy restatement (oracle/dg_numpy.py) without needing the reference at test
time.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import reforacle  # noqa: E402


def uniform(seed, n):
    rng = np.random.default_rng(seed)
    return rng.uniform(-1.0, 1.0, n)


CASES = {
    # name: dim, n_el, ku, kp, distort amplitude, seed, outlet id
    "d2_k2_distorted": (2, 2, 2, 1, 0.05, 7, None),
    "d2_k3_outlet": (2, 3, 3, 2, 0.0, 0, 1),
    "d3_k2_distorted": (3, 2, 2, 1, 0.03, 7, None),
}

COEFS = (3.7, 1.3, 0.9, -0.45)
COEFS_STAGE = (1.0 / ((2 - 2 ** 0.5) * 0.2), 0.005, 0.5, 0.0)
MC = 2.3


def mesh_arrays(R):
    xv = R.cell_vertices()  # [nc][2^d][d]
    flat = xv.reshape(-1, R.dim)
    uniq, inv = np.unique(np.round(flat, 15), axis=0, return_inverse=True)
    # keep the exact coordinates of the first occurrence
    verts = np.zeros_like(uniq)
    verts[inv] = flat
    cells = inv.reshape(R.ncells, 1 << R.dim)
    it, im, bd, bm = R.faces()
    bids = -np.ones((R.ncells, 2 * R.dim), dtype=np.int64)
    for c, f, b in bd:
        bids[c, f] = b
    return verts, cells, bids, it, bd


def main():
    for name, (dim, n_el, ku, kp, amp, seed, outlet) in CASES.items():
        R = reforacle.RefCtx(dim, n_el, ku, kp, amp, seed)
        if outlet is not None:
            R.set_bc(outlet, 1)
        verts, cells, bids, it, bd = mesh_arrays(R)
        w = uniform(11, R.n_u)
        x = uniform(12, R.n_u)
        xp = uniform(13, R.n_p)
        out = dict(dim=dim, ku=ku, kp=kp, outlet=-1 if outlet is None else outlet, verts=verts, cells=cells,
                   bids=bids, interior=it, boundary=bd, w=w, x=x, xp=xp, coefs=np.array(COEFS),
                   coefs_stage=np.array(COEFS_STAGE), mc=MC)
        out["momentum"] = R.momentum(COEFS, w, x)
        out["momentum_stage"] = R.momentum(COEFS_STAGE, w, x)
        out["momentum_diag"] = R.momentum_diag(COEFS, w)
        out["pressure"] = R.pressure(MC, xp)
        out["helmholtz_diag"] = R.helmholtz_diag(MC)
        out["laplace_dir"] = R.laplace(True, xp)
        out["mass_u"] = R.mass(0, x)
        out["mass_p"] = R.mass(1, xp)
        out["mass_diag_u"] = R.mass_diag(0)
        out["divergence"] = R.divergence(x)
        out["gradient"] = R.gradient(xp)
        out["pressure_rhs"] = R.pressure_rhs(1.7, x, 7.3, xp)
        out["kinetic"] = R.kinetic_energy(x)
        xs, its, res = R.solve(1, 0, (MC, 0, 0, 0), None, xp, np.zeros(R.n_p))
        out["cg_x"], out["cg_its"] = xs, its
        xg, itg, _ = R.solve(0, 1, COEFS_STAGE, w, x, np.zeros(R.n_u), restart=5)
        out["gmres_x"], out["gmres_its"] = xg, itg
        np.savez_compressed(os.path.join(HERE, name + ".npz"), **out)
        print(name, R.n_u, R.n_p, "cg its", its, "gmres its", itg)


if __name__ == "__main__":
    main()
