"""CPU restatement of the reference DG operators and Krylov solvers in numpy.

TEST INFRASTRUCTURE ONLY (the parity oracle): never imported by the product
package.  It restates, owner-based and with dense tables exactly like the
reference, the algorithms of /root/reference/proj/src:

  quadrature.cpp:11-69   gauss_legendre / gauss_lobatto (Newton)
  lagrange.cpp:10-90     barycentric Lagrange values / derivatives, tensor tables
  mesh.cpp:250-378       conforming face lists (owner = lower index), embeddings
  space.cpp:60-162       GeometryCache (Jinv, detJ*w, Nanson normals, w_ds)
  space.cpp:205-237      cell_table / trace_table
  forms.cpp:16-109       Eval / TestAcc (evaluate / integrate with dense tables)
  forms.cpp:148-243      scalar_sip_apply          forms.cpp:246-329 scalar_sip_diagonal
  forms.cpp:337-383      apply_mass / mass_diagonal
  forms.cpp:389-604      apply_momentum            forms.cpp:606-810 momentum_diagonal
  forms.cpp:816-1084     momentum_rhs
  forms.cpp:1118-1233    divergence_functional / pressure_rhs / pressure_gradient_rhs
  forms.cpp:1239-1260    kinetic_energy
  krylov.cpp:27-207      JacobiPreconditioner, cg_solve, gmres_solve

Pinned against golden vectors produced by the compiled reference
(tests/golden/make_golden.py -> tests/golden/*.npz).  Small meshes only.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Optional, Tuple

import numpy as np


# ----------------------------------------------------------------------------- 1D rules
def _legendre(n: int, t: float) -> Tuple[float, float]:  # quadrature.cpp:13-23
    if n == 0:
        return 1.0, 0.0
    p0, p1 = 1.0, t
    for k in range(2, n + 1):
        pk = ((2.0 * k - 1.0) * t * p1 - (k - 1.0) * p0) / k
        p0, p1 = p1, pk
    return p1, n * (t * p1 - p0) / (t * t - 1.0)


def gauss_legendre(n: int) -> Tuple[np.ndarray, np.ndarray]:  # quadrature.cpp:25-46
    x = np.zeros(n)
    w = np.zeros(n)
    for i in range(n):
        t = math.cos(math.pi * (i + 0.75) / (n + 0.5))
        for _ in range(100):
            p, dp = _legendre(n, t)
            step = p / dp
            t -= step
            if abs(step) < 1e-16:
                break
        p, dp = _legendre(n, t)
        x[n - 1 - i] = 0.5 * (t + 1.0)
        w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp)
    return x, w


def gauss_lobatto(n: int) -> np.ndarray:  # quadrature.cpp:48-69
    x = np.zeros(n)
    x[-1] = 1.0
    m = n - 1
    for i in range(1, m):
        t = math.cos(math.pi * (m - i) / m)
        for _ in range(100):
            p, dp = _legendre(m, t)
            d2p = (2.0 * t * dp - m * (m + 1.0) * p) / (1.0 - t * t)
            step = dp / d2p
            t -= step
            if abs(step) < 1e-16:
                break
        x[i] = 0.5 * (t + 1.0)
    return x


class Lagrange1D:  # lagrange.cpp:10-50
    def __init__(self, nodes: np.ndarray):
        self.nodes = np.asarray(nodes, dtype=float)
        m = len(nodes)
        self.bary = np.ones(m)
        for i in range(m):
            for j in range(m):
                if j != i:
                    self.bary[i] /= (nodes[i] - nodes[j])

    def values(self, t: float) -> np.ndarray:
        m = len(self.nodes)
        for i in range(m):
            if t == self.nodes[i]:
                out = np.zeros(m)
                out[i] = 1.0
                return out
        l = np.prod(t - self.nodes)
        return l * self.bary / (t - self.nodes)

    def derivatives(self, t: float) -> np.ndarray:
        m = len(self.nodes)
        out = np.zeros(m)
        for i in range(m):
            s = 0.0
            for k in range(m):
                if k == i:
                    continue
                p = 1.0
                for j in range(m):
                    if j != i and j != k:
                        p *= (t - self.nodes[j])
                s += p
            out[i] = self.bary[i] * s
        return out


def tensor_points(dim: int, n1d: int) -> Tuple[np.ndarray, np.ndarray]:  # quadrature.cpp:71-92
    x1, w1 = gauss_legendre(n1d)
    n = n1d ** dim
    X = np.zeros((n, max(dim, 1)))
    W = np.ones(n)
    for i in range(n):
        rem = i
        for d in range(dim):
            idx = rem % n1d
            rem //= n1d
            X[i, d] = x1[idx]
            W[i] *= w1[idx]
    return X, W


def tabulate(basis: Lagrange1D, pts: np.ndarray, dim: int):  # lagrange.cpp:52-90
    m = len(basis.nodes)
    nb = m ** dim
    nq = len(pts)
    val = np.zeros((nb, nq))
    der = np.zeros((dim, nb, nq))
    for q in range(nq):
        v = [basis.values(pts[q, d]) for d in range(dim)]
        g = [basis.derivatives(pts[q, d]) for d in range(dim)]
        for i in range(nb):
            rem = i
            ids = []
            for d in range(dim):
                ids.append(rem % m)
                rem //= m
            val[i, q] = np.prod([v[d][ids[d]] for d in range(dim)])
            for a in range(dim):
                der[a, i, q] = np.prod([(g[d][ids[d]] if d == a else v[d][ids[d]]) for d in range(dim)])
    return val, der


# ----------------------------------------------------------------------------- mesh
def face_corner_vertex(dim: int, face: int, corner: int) -> int:  # mesh.cpp:27-38
    a, s = face // 2, face % 2
    v = s << a
    t = 0
    for d in range(dim):
        if d == a:
            continue
        v |= ((corner >> t) & 1) << d
        t += 1
    return v


def vertex_ref(dim: int, v: int) -> np.ndarray:
    return np.array([(v >> d) & 1 for d in range(dim)], dtype=float)


@dataclass
class Face:
    cell_in: int
    face_in: int
    cell_out: int = -1
    face_out: int = -1
    boundary_id: int = -1
    emb_in: Tuple[np.ndarray, np.ndarray] = None   # origin, tangents [dim-1][dim]
    emb_out: Tuple[np.ndarray, np.ndarray] = None
    measure: float = 0.0


class Mesh:
    """Conforming mesh from arrays (vertices [nv][dim], cells [nc][2^dim], boundary ids [nc][2dim])."""

    def __init__(self, vertices, cells, boundary_ids):
        self.X = np.asarray(vertices, dtype=float)
        self.cells = np.asarray(cells, dtype=int)
        self.bids = np.asarray(boundary_ids, dtype=int)
        self.dim = self.X.shape[1]
        self.nc = self.cells.shape[0]
        self._build_faces()
        self.measure = np.array([self.cell_measure(c) for c in range(self.nc)])

    def map_point(self, c, ref):  # mesh.cpp:44-53
        x = np.zeros(self.dim)
        for v in range(1 << self.dim):
            s = 1.0
            for d in range(self.dim):
                s *= ref[d] if (v >> d) & 1 else (1.0 - ref[d])
            x += s * self.X[self.cells[c, v]]
        return x

    def jacobian(self, c, ref):  # mesh.cpp:55-72 (J[d][a] = dx_d / dxi_a)
        dim = self.dim
        J = np.zeros((dim, dim))
        for v in range(1 << dim):
            for a in range(dim):
                s = 1.0
                for d in range(dim):
                    if d == a:
                        s *= 1.0 if (v >> d) & 1 else -1.0
                    else:
                        s *= ref[d] if (v >> d) & 1 else (1.0 - ref[d])
                J[:, a] += s * self.X[self.cells[c, v]]
        return J

    def cell_measure(self, c):  # mesh.cpp:101-109
        X, W = tensor_points(self.dim, 2)
        return sum(np.linalg.det(self.jacobian(c, X[i])) * W[i] for i in range(len(W)))

    def _face_measure(self, c, f):  # mesh.cpp:271-292
        dim = self.dim
        pts = [self.X[self.cells[c, face_corner_vertex(dim, f, j)]] for j in range(1 << (dim - 1))]
        if dim == 2:
            return float(np.linalg.norm(pts[1] - pts[0]))

        def tri(a, b, p):
            return 0.5 * np.linalg.norm(np.cross(b - a, p - a))
        return tri(pts[0], pts[1], pts[3]) + tri(pts[0], pts[3], pts[2])

    def _canonical(self, f):  # mesh.cpp:239-248
        dim = self.dim
        o = vertex_ref(dim, face_corner_vertex(dim, f, 0))
        T = np.array([vertex_ref(dim, face_corner_vertex(dim, f, 1 << t)) - o for t in range(dim - 1)])
        return o, T

    def _conforming(self, c, f, n, fn):  # mesh.cpp:296-314
        dim = self.dim
        perm = []
        for j in range(1 << (dim - 1)):
            vid = self.cells[c, face_corner_vertex(dim, f, j)]
            perm.append([j2 for j2 in range(1 << (dim - 1))
                         if self.cells[n, face_corner_vertex(dim, fn, j2)] == vid][0])
        r0 = vertex_ref(dim, face_corner_vertex(dim, fn, perm[0]))
        T = np.array([vertex_ref(dim, face_corner_vertex(dim, fn, perm[1 << t])) - r0 for t in range(dim - 1)])
        return r0, T

    def _build_faces(self):  # mesh.cpp:316-377 (conforming part)
        dim = self.dim
        key = {}
        for c in range(self.nc):
            for f in range(2 * dim):
                if self.bids[c, f] >= 0:
                    continue
                k = tuple(sorted(self.cells[c, face_corner_vertex(dim, f, j)] for j in range(1 << (dim - 1))))
                key.setdefault(k, []).append((c, f))
        nbr = {}
        for k, lst in key.items():
            assert len(lst) == 2, "only conforming meshes"
            (c1, f1), (c2, f2) = lst
            nbr[(c1, f1)] = (c2, f2)
            nbr[(c2, f2)] = (c1, f1)
        self.interior: List[Face] = []
        self.boundary: List[Face] = []
        for c in range(self.nc):
            for f in range(2 * dim):
                if self.bids[c, f] >= 0:
                    self.boundary.append(Face(c, f, boundary_id=int(self.bids[c, f]), emb_in=self._canonical(f),
                                              measure=self._face_measure(c, f)))
                    continue
                n, fn = nbr[(c, f)]
                if c > n:
                    continue
                self.interior.append(Face(c, f, n, fn, emb_in=self._canonical(f),
                                          emb_out=self._conforming(c, f, n, fn), measure=self._face_measure(c, f)))


# ----------------------------------------------------------------------------- geometry + tables
@dataclass
class CellGeo:
    detJw: np.ndarray
    Jinv: np.ndarray  # [nq][dim][dim], Jinv[q][a][j] = dxi_a / dx_j
    xq: np.ndarray


@dataclass
class FaceGeo:
    w_ds: np.ndarray
    n: np.ndarray
    xq: np.ndarray
    Jinv_in: np.ndarray
    Jinv_out: Optional[np.ndarray]


class Geometry:  # space.cpp:60-162
    def __init__(self, mesh: Mesh):
        self.mesh = mesh
        self._cache = {}

    def bundle(self, n1d):
        if n1d in self._cache:
            return self._cache[n1d]
        m = self.mesh
        dim = m.dim
        X, W = tensor_points(dim, n1d)
        cells = []
        for c in range(m.nc):
            Ji = np.zeros((len(W), dim, dim))
            dw = np.zeros(len(W))
            xq = np.zeros((len(W), dim))
            for q in range(len(W)):
                J = m.jacobian(c, X[q])
                Ji[q] = np.linalg.inv(J)
                dw[q] = np.linalg.det(J) * W[q]
                xq[q] = m.map_point(c, X[q])
            cells.append(CellGeo(dw, Ji, xq))
        XF, WF = tensor_points(dim - 1, n1d)

        def face(fi: Face, interior: bool):
            axis, sgn = fi.face_in // 2, (1.0 if fi.face_in % 2 == 1 else -1.0)
            nq = len(WF)
            g = FaceGeo(np.zeros(nq), np.zeros((nq, dim)), np.zeros((nq, dim)), np.zeros((nq, dim, dim)),
                        np.zeros((nq, dim, dim)) if interior else None)
            o, T = fi.emb_in
            for q in range(nq):
                r = o + XF[q, :dim - 1] @ T
                J = m.jacobian(fi.cell_in, r)
                g.Jinv_in[q] = np.linalg.inv(J)
                g.xq[q] = m.map_point(fi.cell_in, r)
                tau = np.array([J @ T[t] for t in range(dim - 1)])
                ds = math.hypot(tau[0][0], tau[0][1]) if dim == 2 else float(np.linalg.norm(np.cross(tau[0], tau[1])))
                g.w_ds[q] = ds * WF[q]
                nn = sgn * g.Jinv_in[q][axis, :]
                g.n[q] = nn / np.linalg.norm(nn)
                if interior:
                    o2, T2 = fi.emb_out
                    g.Jinv_out[q] = np.linalg.inv(m.jacobian(fi.cell_out, o2 + XF[q, :dim - 1] @ T2))
            return g

        b = (cells, [face(f, True) for f in m.interior], [face(f, False) for f in m.boundary])
        self._cache[n1d] = b
        return b


class Space:  # space.cpp:188-237
    def __init__(self, mesh: Mesh, degree: int, ncomp: int):
        self.mesh, self.degree, self.nc = mesh, degree, ncomp
        self.basis = Lagrange1D(gauss_lobatto(degree + 1))
        self.nb = (degree + 1) ** mesh.dim
        self.ndofs = mesh.nc * ncomp * self.nb
        self._ct, self._tt = {}, {}

    def off(self, c):
        return c * self.nc * self.nb

    def cell_table(self, n1d):
        if n1d not in self._ct:
            X, _ = tensor_points(self.mesh.dim, n1d)
            self._ct[n1d] = tabulate(self.basis, X, self.mesh.dim)
        return self._ct[n1d]

    def trace_table(self, n1d, emb):
        o, T = emb
        k = (n1d, tuple(np.round(o * 4).astype(int)), tuple(np.round(T.ravel() * 4).astype(int)))
        if k not in self._tt:
            XF, _ = tensor_points(self.mesh.dim - 1, n1d)
            pts = np.array([o + XF[q, :self.mesh.dim - 1] @ T for q in range(len(XF))])
            self._tt[k] = tabulate(self.basis, pts, self.mesh.dim)
        return self._tt[k]


def sip_sigma(deg, fm, cm):  # forms.hpp:175-177
    return (deg + 1) ** 2 * fm / cm


# evaluate values [nc][nq] and physical gradients [nc][dim][nq] (forms.cpp:39-60)
def _eval(tab, coeff, nc, Jinv=None):
    val, der = tab
    nb = val.shape[0]
    C = coeff.reshape(nc, nb)
    v = C @ val
    if Jinv is None:
        return v, None
    dr = np.einsum("cb,abq->caq", C, der)
    g = np.einsum("qad,caq->cdq", Jinv, dr)
    return v, g


# integrate (forms.cpp:90-108): out[c][b] += sum_q val[b,q] sv[c,q] + sum_a der[a,b,q] (sum_d Ji[q,a,d] sg[c,d,q])
def _flush(tab, Jinv, sv, sg, nc):
    val, der = tab
    out = sv @ val.T
    if sg is not None:
        r = np.einsum("qad,cdq->caq", Jinv, sg)
        out += np.einsum("abq,caq->cb", der, r)
    return out.reshape(-1)


# ----------------------------------------------------------------------------- operators
class Forms:
    def __init__(self, mesh: Mesh, ku: int, kp: int):
        self.mesh, self.geom = mesh, Geometry(mesh)
        self.Vu, self.Vp = Space(mesh, ku, mesh.dim), Space(mesh, kp, 1)
        self.bc_type: Dict[int, str] = {}
        self.bc_value: Dict[int, Callable] = {}

    def outlet(self, bid):
        return self.bc_type.get(bid, "dirichlet") == "outlet"

    def _penalty(self, V, fi, boundary=False):  # forms.cpp:111-129
        m = self.mesh
        s_in = sip_sigma(V.degree, fi.measure, m.measure[fi.cell_in])
        if boundary:
            return s_in
        return 0.5 * (s_in + sip_sigma(V.degree, fi.measure, m.measure[fi.cell_out]))

    # forms.cpp:148-243
    def scalar_sip(self, V: Space, mass_coef, dirichlet, x):
        m, dim = self.mesh, self.mesh.dim
        rule = V.degree + 2
        cells, ifg, bfg = self.geom.bundle(rule)
        tab = V.cell_table(rule)
        out = np.zeros(V.ndofs)
        for c in range(m.nc):
            cg = cells[c]
            v, g = _eval(tab, x[V.off(c):V.off(c) + V.nb], 1, cg.Jinv)
            out[V.off(c):V.off(c) + V.nb] += _flush(tab, cg.Jinv, mass_coef * v * cg.detJw, g * cg.detJw, 1)
        for fi, fg in zip(m.interior, ifg):
            tin, tout = V.trace_table(rule, fi.emb_in), V.trace_table(rule, fi.emb_out)
            a, o = V.off(fi.cell_in), V.off(fi.cell_out)
            vi, gi = _eval(tin, x[a:a + V.nb], 1, fg.Jinv_in)
            vo, go = _eval(tout, x[o:o + V.nb], 1, fg.Jinv_out)
            Cp = self._penalty(V, fi)
            dni = np.einsum("cdq,qd->cq", gi, fg.n)
            dno = np.einsum("cdq,qd->cq", go, fg.n)
            ju = vi - vo
            flux = (-0.5 * (dni + dno) + Cp * ju) * fg.w_ds
            ssym = (-0.5 * ju * fg.w_ds)[:, None, :] * fg.n.T[None]
            out[a:a + V.nb] += _flush(tin, fg.Jinv_in, flux, ssym, 1)
            out[o:o + V.nb] += _flush(tout, fg.Jinv_out, -flux, ssym, 1)
        if dirichlet:
            for fi, fg in zip(m.boundary, bfg):
                tin = V.trace_table(rule, fi.emb_in)
                a = V.off(fi.cell_in)
                vi, gi = _eval(tin, x[a:a + V.nb], 1, fg.Jinv_in)
                sK = self._penalty(V, fi, True)
                dn = np.einsum("cdq,qd->cq", gi, fg.n)
                fl = (-dn + 2.0 * sK * vi) * fg.w_ds
                ssym = (-vi * fg.w_ds)[:, None, :] * fg.n.T[None]
                out[a:a + V.nb] += _flush(tin, fg.Jinv_in, fl, ssym, 1)
        return out

    def apply_pressure_helmholtz(self, mass_coef, x):  # forms.cpp:1090-1095
        return self.scalar_sip(self.Vp, mass_coef, False, x)

    # forms.cpp:337-360
    def apply_mass(self, V: Space, x):
        m = self.mesh
        rule = V.degree + (2 if V.nc == 1 else 1)
        cells, _, _ = self.geom.bundle(rule)
        tab = V.cell_table(rule)
        out = np.zeros(V.ndofs)
        for c in range(m.nc):
            s = slice(V.off(c), V.off(c) + V.nc * V.nb)
            v, _ = _eval(tab, x[s], V.nc)
            out[s] += _flush(tab, cells[c].Jinv, v * cells[c].detJw, None, V.nc)
        return out

    # forms.cpp:389-604
    def apply_momentum(self, coefs, w, x):
        mass, visc, adv, skew = coefs
        m, dim, V = self.mesh, self.mesh.dim, self.Vu
        nc, nb = V.nc, V.nb
        out = np.zeros(V.ndofs)
        if mass != 0.0 or visc != 0.0:
            rule = V.degree + 1
            cells, ifg, bfg = self.geom.bundle(rule)
            tab = V.cell_table(rule)
            for c in range(m.nc):
                cg = cells[c]
                s = slice(V.off(c), V.off(c) + nc * nb)
                v, g = _eval(tab, x[s], nc, cg.Jinv)
                out[s] += _flush(tab, cg.Jinv, mass * v * cg.detJw, visc * g * cg.detJw, nc)
            if visc != 0.0:
                for fi, fg in zip(m.interior, ifg):
                    tin, tout = V.trace_table(rule, fi.emb_in), V.trace_table(rule, fi.emb_out)
                    a, o = slice(V.off(fi.cell_in), V.off(fi.cell_in) + nc * nb), slice(V.off(fi.cell_out), V.off(fi.cell_out) + nc * nb)
                    vi, gi = _eval(tin, x[a], nc, fg.Jinv_in)
                    vo, go = _eval(tout, x[o], nc, fg.Jinv_out)
                    Cu = self._penalty(V, fi)
                    dni = np.einsum("cdq,qd->cq", gi, fg.n)
                    dno = np.einsum("cdq,qd->cq", go, fg.n)
                    ju = vi - vo
                    flux = visc * (-0.5 * (dni + dno) + Cu * ju) * fg.w_ds
                    ssym = (-visc * 0.5 * ju * fg.w_ds)[:, None, :] * fg.n.T[None]
                    out[a] += _flush(tin, fg.Jinv_in, flux, ssym, nc)
                    out[o] += _flush(tout, fg.Jinv_out, -flux, ssym, nc)
                for fi, fg in zip(m.boundary, bfg):
                    if self.outlet(fi.boundary_id):
                        continue
                    tin = V.trace_table(rule, fi.emb_in)
                    a = slice(V.off(fi.cell_in), V.off(fi.cell_in) + nc * nb)
                    vi, gi = _eval(tin, x[a], nc, fg.Jinv_in)
                    sK = self._penalty(V, fi, True)
                    dn = np.einsum("cdq,qd->cq", gi, fg.n)
                    fl = visc * (-dn + 2.0 * sK * vi) * fg.w_ds
                    ssym = (-visc * vi * fg.w_ds)[:, None, :] * fg.n.T[None]
                    out[a] += _flush(tin, fg.Jinv_in, fl, ssym, nc)
        if adv != 0.0 or skew != 0.0:
            rule = V.degree + 2
            cells, ifg, bfg = self.geom.bundle(rule)
            tab = V.cell_table(rule)
            for c in range(m.nc):
                cg = cells[c]
                s = slice(V.off(c), V.off(c) + nc * nb)
                u, _ = _eval(tab, x[s], nc)
                wv, wg = _eval(tab, w[s], nc, cg.Jinv)
                divw = np.einsum("ddq->q", wg) if skew != 0.0 else 0.0
                sg = -adv * u[:, None, :] * wv[None, :, :] * cg.detJw
                sv = skew * divw * u * cg.detJw
                out[s] += _flush(tab, cg.Jinv, sv, sg, nc)
            if adv != 0.0:
                for fi, fg in zip(m.interior, ifg):
                    tin, tout = V.trace_table(rule, fi.emb_in), V.trace_table(rule, fi.emb_out)
                    a, o = slice(V.off(fi.cell_in), V.off(fi.cell_in) + nc * nb), slice(V.off(fi.cell_out), V.off(fi.cell_out) + nc * nb)
                    ui, _ = _eval(tin, x[a], nc)
                    uo, _ = _eval(tout, x[o], nc)
                    wi, _ = _eval(tin, w[a], nc)
                    wo, _ = _eval(tout, w[o], nc)
                    wni = np.einsum("dq,qd->q", wi, fg.n)
                    wno = np.einsum("dq,qd->q", wo, fg.n)
                    lam = np.maximum(np.abs(wni), np.abs(wno))
                    flux = adv * (0.5 * (ui * wni + uo * wno) + 0.5 * lam * (ui - uo)) * fg.w_ds
                    out[a] += _flush(tin, fg.Jinv_in, flux, None, nc)
                    out[o] += _flush(tout, fg.Jinv_out, -flux, None, nc)
                for fi, fg in zip(m.boundary, bfg):
                    tin = V.trace_table(rule, fi.emb_in)
                    a = slice(V.off(fi.cell_in), V.off(fi.cell_in) + nc * nb)
                    ui, _ = _eval(tin, x[a], nc)
                    wi, _ = _eval(tin, w[a], nc)
                    wn = np.einsum("dq,qd->q", wi, fg.n)
                    coef = wn if self.outlet(fi.boundary_id) else np.abs(wn)
                    out[a] += _flush(tin, fg.Jinv_in, adv * coef * ui * fg.w_ds, None, nc)
        return out

    # forms.cpp:1118-1197
    def divergence(self, u):
        m, Vu, Vp = self.mesh, self.Vu, self.Vp
        rule = Vu.degree + 1
        cells, ifg, bfg = self.geom.bundle(rule)
        tab, ptab = Vu.cell_table(rule), Vp.cell_table(rule)
        nc, nb = Vu.nc, Vu.nb
        out = np.zeros(Vp.ndofs)
        for c in range(m.nc):
            ue, _ = _eval(tab, u[Vu.off(c):Vu.off(c) + nc * nb], nc)
            out[Vp.off(c):Vp.off(c) + Vp.nb] += _flush(ptab, cells[c].Jinv, np.zeros((1, len(cells[c].detJw))),
                                                       (ue * cells[c].detJw)[None], 1)
        for fi, fg in zip(m.interior, ifg):
            ui, _ = _eval(Vu.trace_table(rule, fi.emb_in), u[Vu.off(fi.cell_in):Vu.off(fi.cell_in) + nc * nb], nc)
            uo, _ = _eval(Vu.trace_table(rule, fi.emb_out), u[Vu.off(fi.cell_out):Vu.off(fi.cell_out) + nc * nb], nc)
            un = np.einsum("dq,qd->q", 0.5 * (ui + uo), fg.n)
            out[Vp.off(fi.cell_in):Vp.off(fi.cell_in) + Vp.nb] += _flush(Vp.trace_table(rule, fi.emb_in), None, (-un * fg.w_ds)[None], None, 1)
            out[Vp.off(fi.cell_out):Vp.off(fi.cell_out) + Vp.nb] += _flush(Vp.trace_table(rule, fi.emb_out), None, (un * fg.w_ds)[None], None, 1)
        for fi, fg in zip(m.boundary, bfg):
            if self.outlet(fi.boundary_id):
                continue
            ui, _ = _eval(Vu.trace_table(rule, fi.emb_in), u[Vu.off(fi.cell_in):Vu.off(fi.cell_in) + nc * nb], nc)
            un = np.einsum("dq,qd->q", ui, fg.n)
            out[Vp.off(fi.cell_in):Vp.off(fi.cell_in) + Vp.nb] += _flush(Vp.trace_table(rule, fi.emb_in), None, (-un * fg.w_ds)[None], None, 1)
        return out

    def pressure_rhs(self, inv_adt, u, mass_coef, p_old):  # forms.cpp:1199-1210
        out = self.divergence(u)
        if inv_adt != 1.0:
            out = out * inv_adt
        if p_old is not None and mass_coef != 0.0:
            out = out + mass_coef * self.apply_mass(self.Vp, p_old)
        return out

    def pressure_gradient(self, p):  # forms.cpp:1212-1233
        m, Vu, Vp = self.mesh, self.Vu, self.Vp
        rule = Vu.degree + 1
        cells, _, _ = self.geom.bundle(rule)
        tab, ptab = Vu.cell_table(rule), Vp.cell_table(rule)
        out = np.zeros(Vu.ndofs)
        for c in range(m.nc):
            _, g = _eval(ptab, p[Vp.off(c):Vp.off(c) + Vp.nb], 1, cells[c].Jinv)
            out[Vu.off(c):Vu.off(c) + Vu.nc * Vu.nb] += _flush(tab, cells[c].Jinv, g[0] * cells[c].detJw, None, Vu.nc)
        return out

    def kinetic_energy(self, u):  # forms.cpp:1239-1260
        m, V = self.mesh, self.Vu
        rule = V.degree + 2
        cells, _, _ = self.geom.bundle(rule)
        tab = V.cell_table(rule)
        ke = 0.0
        for c in range(m.nc):
            ue, _ = _eval(tab, u[V.off(c):V.off(c) + V.nc * V.nb], V.nc)
            ke += float(np.sum(0.5 * np.sum(ue * ue, axis=0) * cells[c].detJw))
        return ke

    # exact diagonals by materialising unit vectors (small meshes only)
    def diagonal(self, apply, n):
        d = np.zeros(n)
        e = np.zeros(n)
        for i in range(n):
            e[:] = 0.0
            e[i] = 1.0
            d[i] = apply(e)[i]
        return d


# ----------------------------------------------------------------------------- Krylov (krylov.cpp)
class SolverError(RuntimeError):
    def __init__(self, msg, history):
        super().__init__(msg)
        self.history = history


def jacobi(diag):  # krylov.cpp:27-36
    for i, v in enumerate(diag):
        if v == 0.0:
            raise SolverError(f"jacobi preconditioner: zero diagonal at dof {i}", [])
    return 1.0 / np.asarray(diag)


def cg_solve(A, b, x, rel_tol=1e-10, abs_tol=0.0, max_iter=10000, inv=None):  # krylov.cpp:43-101
    bnorm = math.sqrt(float(b @ b))
    if bnorm == 0.0:
        x[:] = 0.0
        return 0, 0.0
    tol = max(rel_tol * bnorm, abs_tol)
    it, hist = 0, []
    while True:
        r = b - A(x)
        rnorm = math.sqrt(float(r @ r))
        if rnorm <= tol:
            return it, rnorm
        if it >= max_iter:
            raise SolverError("cg: no convergence", hist)
        first, rho_old = True, 0.0
        while it < max_iter:
            z = r * inv if inv is not None else r.copy()
            rho = float(r @ z)
            if rho == 0.0:
                raise SolverError("cg: breakdown, <r,z> = 0", hist)
            p = z.copy() if first else z + (rho / rho_old) * p
            first, rho_old = False, rho
            q = A(p)
            pq = float(p @ q)
            if pq <= 0.0:
                raise SolverError("cg: operator not positive definite, <p,Ap> <= 0", hist)
            alpha = rho / pq
            x += alpha * p
            r -= alpha * q
            it += 1
            rnorm = math.sqrt(float(r @ r))
            hist.append(rnorm)
            if rnorm <= tol:
                break


def gmres_solve(A, b, x, rel_tol=1e-10, abs_tol=0.0, max_iter=10000, restart=50, inv=None):  # krylov.cpp:103-207
    bnorm = math.sqrt(float(b @ b))
    if bnorm == 0.0:
        x[:] = 0.0
        return 0, 0.0
    tol = max(rel_tol * bnorm, abs_tol)
    m = max(1, restart)
    it, hist = 0, []
    M = (lambda v: v * inv) if inv is not None else (lambda v: v.copy())
    while True:
        r = b - A(x)
        beta = math.sqrt(float(r @ r))
        if beta <= tol:
            return it, beta
        if it >= max_iter:
            raise SolverError("gmres: no convergence", hist)
        V = [r / beta]
        H = np.zeros((m + 1, m))
        cs, sn, g = np.zeros(m), np.zeros(m), np.zeros(m + 1)
        g[0] = beta
        k = 0
        while k < m and it < max_iter:
            w = A(M(V[k]))
            it += 1
            for i in range(k + 1):
                h = float(w @ V[i])
                H[i, k] = h
                w = w - h * V[i]
            hk1 = math.sqrt(float(w @ w))
            H[k + 1, k] = hk1
            for i in range(k):
                t = cs[i] * H[i, k] + sn[i] * H[i + 1, k]
                H[i + 1, k] = -sn[i] * H[i, k] + cs[i] * H[i + 1, k]
                H[i, k] = t
            denom = math.hypot(H[k, k], H[k + 1, k])
            cs[k], sn[k] = (1.0, 0.0) if denom == 0.0 else (H[k, k] / denom, H[k + 1, k] / denom)
            H[k, k], H[k + 1, k] = denom, 0.0
            g[k + 1] = -sn[k] * g[k]
            g[k] = cs[k] * g[k]
            res = abs(g[k + 1])
            hist.append(res)
            k += 1
            if res <= tol or hk1 == 0.0:
                break
            if k < m:
                V.append(w / hk1)
        y = np.zeros(k)
        for i in range(k - 1, -1, -1):
            y[i] = (g[i] - H[i, i + 1:k] @ y[i + 1:k]) / H[i, i]
        wsum = sum(y[j] * V[j] for j in range(k))
        x += M(wsum)
