"""ctypes wrapper of oracle/_ref/libdgref.so — TEST INFRASTRUCTURE ONLY.

Drives the unmodified reference library (proj/src, compiled by oracle/Makefile)
through oracle/ref_capi.cpp on numpy arrays.  Used only as the checker by the
tests, __graft_entry__.smoke() and bench.py's CPU-baseline legs.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF_SO = os.path.join(ROOT, "oracle", "_ref", "libdgref.so")

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
BC_FN = C.CFUNCTYPE(None, _dp, C.c_double, _dp, C.c_void_p)

_lib = None


def available() -> bool:
    return os.path.exists(REF_SO)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(REF_SO)
        L.ref_last_error.restype = C.c_char_p
        L.ref_backend.restype = C.c_char_p
        L.ref_create_cartesian.restype = C.c_void_p
        L.ref_create_cartesian.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, C.c_int, C.c_int, C.c_int]
        L.ref_create_refined.restype = C.c_void_p
        L.ref_create_refined.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, C.c_int, C.c_int, C.c_int, _ip]
        L.ref_mesh_arrays.argtypes = [C.c_void_p, _dp, _ip, _ip, _dp]
        L.ref_create_from_text.restype = C.c_void_p
        L.ref_create_from_text.argtypes = [C.c_char_p, C.c_int, C.c_int]
        L.ref_create_from_arrays.restype = C.c_void_p
        L.ref_create_from_arrays.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, C.c_int, C.c_int]
        L.ref_create_cylinder.restype = C.c_void_p
        L.ref_create_cylinder.argtypes = [C.c_int, C.c_int, C.c_int]
        L.ref_destroy.argtypes = [C.c_void_p]
        L.ref_info.argtypes = [C.c_void_p, C.POINTER(C.c_longlong)]
        L.ref_set_bc.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p]
        L.ref_apply_momentum.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp]
        L.ref_momentum_diagonal.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_apply_pressure.argtypes = [C.c_void_p, C.c_double, _dp, _dp]
        L.ref_helmholtz_diagonal.argtypes = [C.c_void_p, C.c_double, _dp]
        L.ref_apply_laplace.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.ref_laplace_diagonal.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_apply_mass.argtypes = [C.c_void_p, C.c_int, _dp, _dp]
        L.ref_mass_diagonal.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_momentum_rhs.argtypes = [C.c_void_p, C.c_int, _dp, C.POINTER(_dp), C.c_int, _dp, C.POINTER(_dp),
                                       C.c_int, _dp, C.POINTER(_dp), C.POINTER(_dp), C.c_int, _dp,
                                       C.POINTER(_dp), C.c_double, C.c_double, _dp, C.c_double, _dp]
        L.ref_divergence.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_pressure_rhs.argtypes = [C.c_void_p, C.c_double, _dp, C.c_double, _dp, _dp]
        L.ref_pressure_gradient.argtypes = [C.c_void_p, _dp, _dp]
        L.ref_kinetic_energy.argtypes = [C.c_void_p, _dp]
        L.ref_kinetic_energy.restype = C.c_double
        L.ref_solve.argtypes = [C.c_void_p, C.c_int, C.c_int, _dp, _dp, _dp, C.c_double, C.c_double, C.c_int,
                                C.c_int, C.c_int, _dp, _ip, _dp, _dp, C.c_int, _ip]
        L.ref_trbdf2_step.argtypes = [C.c_void_p, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
        L.ref_scheme_step.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, _dp, _dp, _dp, _ip]
        L.ref_faces.argtypes = [C.c_void_p, _ip, _dp, _ip, _dp]
        L.ref_cell_vertices.argtypes = [C.c_void_p, _dp]
        L.ref_bface_points.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_node_points.argtypes = [C.c_void_p, C.c_int, _dp]
        L.ref_bench.argtypes = [C.c_void_p, C.c_int, _dp, _dp, _dp, C.c_int, C.c_int]
        L.ref_bench.restype = C.c_double
        L.ref_dense_momentum.argtypes = [C.c_void_p, _dp, _dp, _dp]
        L.ref_dense_scalar_sip.argtypes = [C.c_void_p, C.c_double, C.c_int, C.c_int, _dp]
        L.ref_seeded_uniform.argtypes = [C.c_ulonglong, C.c_size_t, C.c_double, C.c_double, _dp]
        L.ref_synth_init.argtypes = [C.c_int, C.c_ulonglong, C.c_double, _dp]
        L.ref_synth_eval.argtypes = [_dp, C.c_double, _dp, C.c_void_p]
        L.ref_interpolate_fn.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, _dp, C.c_int]
        L.ref_create_slab.restype = C.c_void_p
        L.ref_create_slab.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, C.c_int]
        L.ref_kern.argtypes = [C.c_int, C.c_size_t, C.c_double, C.c_double, _dp, _dp]
        L.ref_kern.restype = C.c_double
        L.ref_pair_setup.argtypes = [C.c_void_p, _dp, _dp, _dp, C.c_double, _dp]
        L.ref_pair_rounds.argtypes = [C.POINTER(C.c_void_p), C.c_int, C.c_int, C.c_int, _dp]
        _lib = L
    return _lib


def kern(op: str, a: float, x, y, b: float = 0.0):
    """The reference's kern:: BLAS-1 (active backend).  axpy / axpby / scal return the
    updated copy of y (scal: of x); dot / max_abs_diff return the scalar."""
    code = {"axpy": 0, "axpby": 1, "scal": 2, "dot": 3, "max_abs_diff": 4}[op]
    yy = np.array(x if op == "scal" else y, dtype=np.float64, copy=True)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    r = lib().ref_kern(code, len(yy), a, b, P(xx), P(yy))
    return yy if code <= 2 else r


def pair_rounds(ctxs, nthreads: int, rounds: int):
    """Wall seconds of `rounds` rounds of one momentum + one pressure apply on every
    context in ctxs (after RefCtx.pair_setup), spread over nthreads host threads."""
    hs = (C.c_void_p * len(ctxs))(*[c.h for c in ctxs])
    t = np.zeros(rounds)
    lib().ref_pair_rounds(hs, len(ctxs), int(nthreads), int(rounds), P(t))
    return t


def seeded_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0):
    """U[lo,hi) from mt19937_64(seed) (same values as the product's dgb_seeded_uniform)."""
    out = np.empty(n)
    lib().ref_seeded_uniform(seed, n, lo, hi, P(out))
    return out


class SynthField:
    """BASELINE initial field (curl of a seeded stream function / vector potential),
    oracle-side restatement: its fn_ptr is a plain C function inside libdgref.so."""

    def __init__(self, dim: int, seed: int, scale: float = 1.0):
        self.dim = dim
        self.user = np.zeros(512)
        lib().ref_synth_init(dim, seed, scale, P(self.user))

    @property
    def user_ptr(self):
        return self.user.ctypes.data_as(C.c_void_p)

    @property
    def fn_ptr(self):
        return C.cast(lib().ref_synth_eval, C.c_void_p)

    def eval(self, x):
        out = np.zeros(self.dim)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        lib().ref_synth_eval(P(xx), 0.0, P(out), self.user_ptr)
        return out

    def interpolate(self, R: "RefCtx", nthreads: int = 1):
        """FunctionSpace::interpolate (space.cpp:239-253) of the field on R's velocity space."""
        out = np.zeros(R.n_u)
        lib().ref_interpolate_fn(R.h, self.fn_ptr, self.user_ptr, P(out), int(nthreads))
        return out


def P(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


class RefSolverError(RuntimeError):
    def __init__(self, msg, history):
        super().__init__(msg)
        self.history = history


class RefCtx:
    """Reference Mesh + GeometryCache + FunctionSpace(ku, dim) + FunctionSpace(kp, 1)."""

    def __init__(self, dim=2, n_el=2, ku=2, kp=1, amp=0.0, seed=0, refine_first=False, handle=None):
        L = lib()
        h = handle if handle is not None else L.ref_create_cartesian(dim, n_el, amp, seed, ku, kp, int(refine_first))
        if not h:
            raise RuntimeError(L.ref_last_error().decode())
        self.h = h
        info = (C.c_longlong * 10)()
        L.ref_info(h, info)
        (self.ncells, self.n_u, self.n_p, self.n_interior, self.n_boundary, self.ku, self.kp, self.dim,
         self.nverts, self.n_hanging) = [int(v) for v in info]
        self._keep = []

    @classmethod
    def refined(cls, dim: int, n_el: int, ku: int, kp: int, refine, amp: float = 0.0, seed: int = 0):
        """generate_cartesian (+ distort) then Mesh::refine_and_coarsen(refine, {}): hanging faces."""
        r = np.ascontiguousarray(refine, dtype=np.int32)
        h = lib().ref_create_refined(dim, n_el, amp, seed, ku, kp, len(r), r.ctypes.data_as(_ip))
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        return cls(handle=h)

    def mesh_arrays(self):
        """(vertices [nv][dim], active cell vertices [n][2^dim], boundary ids [n][2dim],
        interior faces [ni][5] (cell_in, face_in, cell_out, face_out, hanging), emb_out [ni][dim*dim])."""
        xv = np.zeros((self.nverts, self.dim))
        cv = np.zeros((self.ncells, 1 << self.dim), dtype=np.int32)
        bid = np.zeros((self.ncells, 2 * self.dim), dtype=np.int32)
        emb = np.zeros((self.n_interior, self.dim * self.dim))
        lib().ref_mesh_arrays(self.h, P(xv), cv.ctypes.data_as(_ip), bid.ctypes.data_as(_ip), P(emb))
        it, _, _, _ = self.faces()
        return xv, cv, bid, it, emb

    @classmethod
    def slab(cls, n_el: int, z0: int, nz: int, ku: int, kp: int):
        """z-slab [z0, z0+nz) of the 3D n_el^3 Cartesian mesh (identical cells; slab ends are boundary faces)."""
        h = lib().ref_create_slab(n_el, z0, nz, ku, kp)
        if not h:
            raise RuntimeError(lib().ref_last_error().decode())
        return cls(handle=h)

    def __del__(self):
        try:
            lib().ref_destroy(self.h)
        except Exception:
            pass

    def set_bc(self, bid, bc_type, fn_ptr=None, user=None):
        self._keep.append(user)
        lib().ref_set_bc(self.h, bid, bc_type, fn_ptr, user)

    def momentum(self, coefs, w, x):
        y = np.zeros(self.n_u)
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        if lib().ref_apply_momentum(self.h, P(c), P(w), P(x), P(y)):
            raise RuntimeError(lib().ref_last_error().decode())
        return y

    def momentum_diag(self, coefs, w):
        y = np.zeros(self.n_u)
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        if lib().ref_momentum_diagonal(self.h, P(c), P(w), P(y)):
            raise RuntimeError(lib().ref_last_error().decode())
        return y

    def pressure(self, mc, x):
        y = np.zeros(self.n_p)
        lib().ref_apply_pressure(self.h, mc, P(x), P(y))
        return y

    def helmholtz_diag(self, mc):
        y = np.zeros(self.n_p)
        lib().ref_helmholtz_diagonal(self.h, mc, P(y))
        return y

    def laplace(self, dirichlet, x):
        y = np.zeros(self.n_p)
        lib().ref_apply_laplace(self.h, int(dirichlet), P(x), P(y))
        return y

    def laplace_diag(self, dirichlet):
        y = np.zeros(self.n_p)
        lib().ref_laplace_diagonal(self.h, int(dirichlet), P(y))
        return y

    def mass(self, space, x):
        y = np.zeros(self.n_u if space == 0 else self.n_p)
        lib().ref_apply_mass(self.h, space, P(x), P(y))
        return y

    def mass_diag(self, space):
        y = np.zeros(self.n_u if space == 0 else self.n_p)
        lib().ref_mass_diagonal(self.h, space, P(y))
        return y

    def momentum_rhs(self, mass=(), visc=(), adv=(), pres=(), dir_visc=0.0, dir_adv=0.0, dir_w=None, time=0.0):
        def arr(lst, idx):
            return (_dp * max(1, len(lst)))(*[P(t[idx]) for t in lst])

        def coefs(lst):
            return np.ascontiguousarray([t[0] for t in lst] + [0.0], dtype=np.float64)

        cm, cv, ca, cp = coefs(mass), coefs(visc), coefs(adv), coefs(pres)
        y = np.zeros(self.n_u)
        rc = lib().ref_momentum_rhs(self.h, len(mass), P(cm), arr(mass, 1), len(visc), P(cv), arr(visc, 1),
                                    len(adv), P(ca), arr(adv, 1), arr(adv, 2), len(pres), P(cp), arr(pres, 1),
                                    dir_visc, dir_adv, P(dir_w), time, P(y))
        if rc:
            raise RuntimeError(lib().ref_last_error().decode())
        return y

    def divergence(self, u):
        y = np.zeros(self.n_p)
        lib().ref_divergence(self.h, P(u), P(y))
        return y

    def pressure_rhs(self, inv_adt, u, mc, p_old):
        y = np.zeros(self.n_p)
        lib().ref_pressure_rhs(self.h, inv_adt, P(u), mc, P(p_old), P(y))
        return y

    def gradient(self, p):
        y = np.zeros(self.n_u)
        lib().ref_pressure_gradient(self.h, P(p), P(y))
        return y

    def kinetic_energy(self, u):
        return lib().ref_kinetic_energy(self.h, P(u))

    def solve(self, op, solver, coefs, w, b, x0, rel_tol=1e-10, abs_tol=0.0, max_iter=10000, restart=50,
              precond=True):
        x = np.array(x0, dtype=np.float64, copy=True)
        it = C.c_int()
        res = C.c_double()
        hist = np.zeros(100000)
        hl = C.c_int()
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        rc = lib().ref_solve(self.h, op, solver, P(c), P(w), P(b), rel_tol, abs_tol, max_iter, restart,
                             int(precond), P(x), C.byref(it), C.byref(res), P(hist), 100000, C.byref(hl))
        if rc == 2:
            raise RefSolverError(lib().ref_last_error().decode(), hist[: hl.value].tolist())
        if rc:
            raise RuntimeError(lib().ref_last_error().decode())
        return x, it.value, res.value

    def step(self, params, u_nm1, u_n, p_n):
        prm = np.ascontiguousarray(params, dtype=np.float64)
        u1 = np.zeros(self.n_u)
        p1 = np.zeros(self.n_p)
        if len(prm) < 13:  # no fixed point
            prm = np.concatenate([prm, [0.0, 1e-8, 100.0][len(prm) - 10:]])
        its = (C.c_int * 10)()
        if lib().ref_trbdf2_step(self.h, P(prm), P(u_nm1), P(u_n), P(p_n), P(u1), P(p1), its):
            raise RuntimeError(lib().ref_last_error().decode())
        return u1, p1, list(its)

    def scheme_step(self, scheme, params, u_nm1, u_n, p_n):
        """scheme 1 = BCG, 2 = GQ-BDF2 (oracle/trbdf2_cpu.hpp); params as step()."""
        prm = np.ascontiguousarray(params, dtype=np.float64)
        if len(prm) < 13:
            prm = np.concatenate([prm, [0.0, 1e-8, 100.0][len(prm) - 10:]])
        u1 = np.zeros(self.n_u)
        p1 = np.zeros(self.n_p)
        its = (C.c_int * 10)()
        if lib().ref_scheme_step(self.h, scheme, P(prm), P(u_nm1), P(u_n), P(p_n), P(u1), P(p1), its):
            raise RuntimeError(lib().ref_last_error().decode())
        return u1, p1, list(its)

    def faces(self):
        it = np.zeros((self.n_interior, 5), dtype=np.int32)
        im = np.zeros(self.n_interior)
        bd = np.zeros((self.n_boundary, 3), dtype=np.int32)
        bm = np.zeros(self.n_boundary)
        lib().ref_faces(self.h, it.ctypes.data_as(_ip), P(im), bd.ctypes.data_as(_ip), P(bm))
        return it, im, bd, bm

    def cell_vertices(self):
        xv = np.zeros((self.ncells, 1 << self.dim, self.dim))
        lib().ref_cell_vertices(self.h, P(xv))
        return xv

    def bface_points(self, rule):
        xq = np.zeros((self.n_boundary, rule ** (self.dim - 1), self.dim))
        lib().ref_bface_points(self.h, rule, P(xq))
        return xq

    def bench(self, op, coefs, w, x, nthreads, napplies):
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        return lib().ref_bench(self.h, op, P(c), P(w), P(x), nthreads, napplies)

    def pair_setup(self, coefs, w, x, mass_coef, xp):
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        lib().ref_pair_setup(self.h, P(c), P(w), P(x), mass_coef, P(xp))

    def dense_momentum(self, coefs, w):
        A = np.zeros((self.n_u, self.n_u))
        c = np.ascontiguousarray(coefs, dtype=np.float64)
        lib().ref_dense_momentum(self.h, P(c), P(w), P(A))
        return A

    def dense_scalar_sip(self, mc, dirichlet, rule):
        A = np.zeros((self.n_p, self.n_p))
        lib().ref_dense_scalar_sip(self.h, mc, int(dirichlet), rule, P(A))
        return A
