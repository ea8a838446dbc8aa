"""B200-native DG / TR-BDF2 hot path: Python mirror of the reference interface.

The reference (``/root/reference/proj/src``) exposes free C++ functions over
``FunctionSpace`` / ``GeometryCache`` / ``Field`` (forms.hpp:105-170) and the
Krylov solvers (krylov.hpp:22-66).  This module mirrors those names, argument
meanings and error behaviour on top of the C-ABI ``libdgb.so`` (include/dgb.h);
fields are CUDA ``torch.float64`` tensors in the reference DoF layout
(space.hpp:5-8).  There is no CPU fallback: without the built extension or a
GPU every call raises.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass, field
from typing import List, Optional, Sequence, Tuple

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("DGB_LIB") or os.path.join(_HERE, "libdgb.so")  # DGB_LIB: tuning builds only

# status codes (include/dgb.h)
OK, E_ARG, E_NO_CONVERGENCE, E_BREAKDOWN, E_NOT_SPD, E_ZERO_DIAG, E_CUDA, E_UNSUPPORTED, E_MISSING_FIELD = range(9)
BC_DIRICHLET, BC_OUTLET = 0, 1
SPACE_U, SPACE_P = 0, 1
OP_MOMENTUM, OP_PRESSURE, OP_MASS_U, OP_MASS_P, OP_LAPLACE = range(5)

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int)
_llp = C.POINTER(C.c_longlong)


class SolverError(RuntimeError):
    """krylov.hpp:31-36: raised on non-convergence / breakdown, carries the residual history."""

    def __init__(self, msg: str, history: Sequence[float] = ()):
        super().__init__(msg)
        self.history = list(history)


class DGBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[dgb status {code}] {msg}")
        self.code = code


class _RhsDesc(C.Structure):
    _fields_ = [
        ("n_mass", C.c_int), ("n_visc", C.c_int), ("n_adv", C.c_int), ("n_pres", C.c_int),
        ("mass_coef", C.c_double * 4), ("visc_coef", C.c_double * 4),
        ("adv_coef", C.c_double * 4), ("pres_coef", C.c_double * 4),
        ("mass_f", C.c_void_p * 4), ("visc_f", C.c_void_p * 4), ("adv_f", C.c_void_p * 4),
        ("adv_w", C.c_void_p * 4), ("pres_f", C.c_void_p * 4),
        ("dir_visc_coef", C.c_double), ("dir_adv_coef", C.c_double), ("dir_w", C.c_void_p),
    ]


class _Settings(C.Structure):
    _fields_ = [("rel_tol", C.c_double), ("abs_tol", C.c_double), ("max_iter", C.c_int), ("restart", C.c_int)]


class _Result(C.Structure):
    _fields_ = [("iterations", C.c_int), ("residual", C.c_double)]


class _Operator(C.Structure):
    _fields_ = [("op", C.c_int), ("coefs", C.c_double * 4), ("d_w", C.c_void_p), ("dirichlet_bdry", C.c_int)]


class _StepParams(C.Structure):
    _fields_ = [("dt", C.c_double), ("Re", C.c_double), ("c", C.c_double), ("time", C.c_double),
                ("restart", C.c_int), ("tol_mom", C.c_double), ("tol_p", C.c_double),
                ("tol_mass", C.c_double), ("max_iter", C.c_int), ("first_step", C.c_int),
                ("pressure_precond", C.c_int), ("fixed_point", C.c_int), ("fp_tol", C.c_double),
                ("fp_max_iter", C.c_int)]


BC_FN = C.CFUNCTYPE(None, _dp, C.c_double, _dp, C.c_void_p)

_lib = None


def lib() -> C.CDLL:
    """Load libdgb.so (fails loudly if the extension has not been built)."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} missing: build it with `make -C paper_2107_07776_b200` "
                          "(or __graft_entry__.build()); there is no CPU fallback")
    L = C.CDLL(LIB_PATH)
    L.dgb_last_error.restype = C.c_char_p
    L.dgb_version.restype = C.c_char_p
    L.dgb_ctx_create_cartesian.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, C.c_int, C.c_int, C.c_int,
                                           C.POINTER(C.c_void_p)]
    L.dgb_ctx_create_mesh.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, C.c_int, C.c_int, C.c_int,
                                      C.POINTER(C.c_void_p)]
    L.dgb_ctx_create_mesh_hanging.argtypes = [C.c_int, C.c_int, _dp, C.c_int, _ip, _ip, C.c_int, _ip, _dp,
                                              C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
    L.dgb_ctx_destroy.argtypes = [C.c_void_p]
    L.dgb_ctx_destroy.restype = None
    L.dgb_ctx_info.argtypes = [C.c_void_p, _llp]
    L.dgb_set_stream.argtypes = [C.c_void_p, C.c_void_p]
    L.dgb_sync.argtypes = [C.c_void_p]
    L.dgb_set_boundary_type.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.dgb_set_dirichlet_table.argtypes = [C.c_void_p, _dp]
    L.dgb_set_dirichlet_fn.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_double]
    L.dgb_set_dirichlet_time_dependent.argtypes = [C.c_void_p, C.c_int]
    L.dgb_set_cell_range.argtypes = [C.c_void_p, C.c_int, C.c_int]
    L.dgb_set_debug.argtypes = [C.c_void_p, C.c_int]
    L.dgb_boundary_points.argtypes = [C.c_void_p, C.c_int, _dp]
    L.dgb_node_points.argtypes = [C.c_void_p, C.c_int, _dp]
    L.dgb_face_lists.argtypes = [C.c_void_p, _ip, _ip]
    for name in ("dgb_copy_h2d", "dgb_copy_d2h", "dgb_copy_d2d"):
        getattr(L, name).argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_size_t]
    L.dgb_fill.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.c_size_t]
    L.dgb_momentum_apply.argtypes = [C.c_void_p, _dp, C.c_void_p, C.c_void_p, C.c_void_p]
    L.dgb_momentum_diag.argtypes = [C.c_void_p, _dp, C.c_void_p, C.c_void_p]
    L.dgb_pressure_apply.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    L.dgb_momentum_apply_host.argtypes = [C.c_void_p, _dp, C.c_void_p, C.c_void_p, C.c_void_p]
    L.dgb_pressure_apply_host.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    L.dgb_helmholtz_diag.argtypes = [C.c_void_p, C.c_double, C.c_void_p]
    L.dgb_laplace_apply.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.dgb_laplace_diag.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.dgb_mass_apply.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]
    L.dgb_mass_diag.argtypes = [C.c_void_p, C.c_int, C.c_void_p]
    L.dgb_momentum_rhs.argtypes = [C.c_void_p, C.POINTER(_RhsDesc), C.c_void_p]
    L.dgb_divergence.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.dgb_pressure_rhs.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    L.dgb_pressure_gradient.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
    L.dgb_kinetic_energy.argtypes = [C.c_void_p, C.c_void_p, _dp]
    L.dgb_axpy.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_void_p, C.c_void_p]
    L.dgb_axpby.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_void_p, C.c_double, C.c_void_p]
    L.dgb_scal.argtypes = [C.c_void_p, C.c_size_t, C.c_double, C.c_void_p]
    L.dgb_dot.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, _dp]
    L.dgb_max_abs_diff.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p, _dp]
    L.dgb_norm.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, _dp]
    L.dgb_jacobi_inverse.argtypes = [C.c_void_p, C.c_size_t, C.c_void_p, C.c_void_p]
    for name in ("dgb_cg", "dgb_gmres"):
        getattr(L, name).argtypes = [C.c_void_p, C.POINTER(_Operator), C.POINTER(_Settings), C.c_void_p,
                                     C.c_void_p, C.c_void_p, C.POINTER(_Result), _dp, C.c_int, _ip]
    L.dgb_trbdf2_step.argtypes = [C.c_void_p, C.POINTER(_StepParams), C.c_void_p, C.c_void_p, C.c_void_p,
                                  C.c_void_p, C.c_void_p, _ip]
    L.dgb_pressure_cg_mg.argtypes = [C.c_void_p, C.c_double, C.POINTER(_Settings), C.c_void_p, C.c_void_p,
                                     C.POINTER(_Result)]
    L.dgb_pressure_mg_vcycle.argtypes = [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p]
    L.dgb_projection_step.argtypes = [C.c_void_p, C.c_int, C.POINTER(_StepParams), C.c_void_p, C.c_void_p,
                                      C.c_void_p, C.c_void_p, C.c_void_p, _ip]
    L.dgb_l2_norm.argtypes = [C.c_void_p, C.c_int, C.c_void_p, _dp]
    L.dgb_check_steady.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_double, _ip, _dp]
    L.dgb_stability_params.argtypes = [C.c_void_p, C.c_double, C.c_double, C.c_double, _dp, _dp]
    L.dgb_seeded_uniform.argtypes = [C.c_ulonglong, C.c_size_t, C.c_double, C.c_double, _dp]
    L.dgb_synth_init.argtypes = [C.c_int, C.c_ulonglong, C.c_double, _dp]
    L.dgb_synth_eval.argtypes = [_dp, C.c_double, _dp, C.c_void_p]
    L.dgb_synth_eval.restype = None
    L.dgb_interpolate_synth.argtypes = [C.c_void_p, _dp, _dp]
    L.dgb_interpolate_synth_device.argtypes = [C.c_void_p, _dp, C.c_void_p]
    L.dgb_timer_start.argtypes = [C.c_void_p]
    L.dgb_timer_stop.argtypes = [C.c_void_p, C.POINTER(C.c_float)]
    L.dgb_fp64_peak.argtypes = [C.c_void_p, _dp]
    L.dgb_fp64_peak_dmma.argtypes = [C.c_void_p, _dp]
    L.dgb_launch_count.argtypes = [C.c_void_p]
    L.dgb_launch_count.restype = C.c_longlong
    L.dgb_host_mesh_cartesian.argtypes = [C.c_int, C.c_int, C.c_double, C.c_uint, _llp, _ip, _ip, _dp, _dp, _dp]
    L.dgb_host_tables.argtypes = [C.c_int, C.c_int, _dp, _dp, _dp, _dp]
    L.dgb_set_fast_path.argtypes = [C.c_void_p, C.c_int]
    L.dgb_fast_path_active.argtypes = [C.c_void_p]
    L.dgb_hanging_mode.argtypes = [C.c_void_p]
    _lib = L
    return L


def _ptr(t) -> Optional[int]:
    if t is None:
        return None
    import torch
    if not (t.is_cuda and t.dtype == torch.float64 and t.is_contiguous()):
        raise ValueError("fields must be contiguous CUDA float64 tensors")
    return t.data_ptr()


def _host_ptr(t) -> Optional[int]:
    """Host field: contiguous CPU float64 torch tensor (pinned for copy/compute overlap)
    or numpy array."""
    if t is None:
        return None
    import numpy as np
    if isinstance(t, np.ndarray):
        if not (t.dtype == np.float64 and t.flags.c_contiguous):
            raise ValueError("host fields must be contiguous float64 arrays")
        return t.ctypes.data
    import torch
    if t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError("host fields must be contiguous CPU float64 tensors")
    return t.data_ptr()


def _np_ptr(a):
    return a.ctypes.data_as(_dp)


def _check(code: int) -> None:
    if code != OK:
        msg = lib().dgb_last_error().decode()
        if code == E_MISSING_FIELD:
            raise RuntimeError(msg)
        if code == E_ZERO_DIAG:
            raise SolverError(msg, [])
        raise DGBError(code, msg)


# ---------------------------------------------------------------------------
# Context = (Mesh, GeometryCache, FunctionSpace Vu, FunctionSpace Vp) on one GPU
# ---------------------------------------------------------------------------
@dataclass
class BoundaryTable:
    """forms.hpp:29-51: per boundary id a type and optional data callback g(x, t)."""
    types: dict = field(default_factory=dict)


class DGContext:
    """Device-resident mesh + geometry + the velocity (degree ku, dim comps) and
    pressure (degree kp, scalar) spaces.  Mirrors what the reference builds from
    ``generate_cartesian`` / ``distort`` / ``GeometryCache`` / ``FunctionSpace``."""

    def __init__(self, dim: int, n_el: int, ku: int, kp: int, distort_amp: float = 0.0, distort_seed: int = 0,
                 device: int = 0, *, mesh_arrays=None):
        import torch
        L = lib()
        h = C.c_void_p()
        if mesh_arrays is None:
            _check(L.dgb_ctx_create_cartesian(dim, n_el, float(distort_amp), distort_seed, ku, kp, device,
                                              C.byref(h)))
        else:
            import numpy as np
            verts, cells, bids = mesh_arrays[:3]
            verts = np.ascontiguousarray(verts, dtype=np.float64)
            cells = np.ascontiguousarray(cells, dtype=np.int32)
            bids = np.ascontiguousarray(bids, dtype=np.int32)
            if len(mesh_arrays) > 3:  # hanging subfaces: (fine, f, coarse, fN) records + emb_out
                hf = np.ascontiguousarray(mesh_arrays[3], dtype=np.int32).reshape(-1, 4)
                he = np.ascontiguousarray(mesh_arrays[4], dtype=np.float64).reshape(len(hf), dim * dim)
                _check(L.dgb_ctx_create_mesh_hanging(dim, verts.shape[0], _np_ptr(verts), cells.shape[0],
                                                     cells.ctypes.data_as(_ip), bids.ctypes.data_as(_ip), len(hf),
                                                     hf.ctypes.data_as(_ip), _np_ptr(he), ku, kp, device,
                                                     C.byref(h)))
            else:
                _check(L.dgb_ctx_create_mesh(dim, verts.shape[0], _np_ptr(verts), cells.shape[0],
                                             cells.ctypes.data_as(_ip), bids.ctypes.data_as(_ip), ku, kp, device,
                                             C.byref(h)))
        self._h = h
        self.device = device
        info = (C.c_longlong * 16)()
        _check(L.dgb_ctx_info(h, info))
        (self.ncells, self.n_u, self.n_p, self.n_interior, self.n_boundary, self.ku, self.kp, self.dim,
         affine, self.nqf_bdry) = [int(v) for v in info[:10]]
        self.n_hanging = int(info[11])
        self.affine = bool(affine)
        # run on torch's current stream so torch ops and our kernels are ordered
        with torch.cuda.device(device):
            self.stream = torch.cuda.current_stream()
        _check(L.dgb_set_stream(h, C.c_void_p(self.stream.cuda_stream)))
        self._keep = []

    @property
    def handle(self):
        return self._h

    def close(self):
        if getattr(self, "_h", None):
            lib().dgb_ctx_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- fields -----------------------------------------------------------
    def zeros(self, space: int = SPACE_U):
        import torch
        n = self.n_u if space == SPACE_U else self.n_p
        return torch.zeros(n, dtype=torch.float64, device=f"cuda:{self.device}")

    def sync(self):
        _check(lib().dgb_sync(self._h))

    # -- boundary table ---------------------------------------------------
    def set_boundary_type(self, boundary_id: int, bc_type: int):
        _check(lib().dgb_set_boundary_type(self._h, boundary_id, bc_type))

    def set_dirichlet_table(self, g):
        import numpy as np
        g = None if g is None else np.ascontiguousarray(g, dtype=np.float64)
        _check(lib().dgb_set_dirichlet_table(self._h, None if g is None else _np_ptr(g)))

    def set_dirichlet_fn(self, boundary_id: int, fn_ptr, user, t: float = 0.0):
        """fn_ptr: a C function pointer (e.g. lib().dgb_synth_eval) with its user data."""
        _check(lib().dgb_set_dirichlet_fn(self._h, boundary_id, C.cast(fn_ptr, C.c_void_p), user, t))

    def set_dirichlet_time_dependent(self, enable: bool):
        """Re-evaluate the registered Dirichlet callbacks at every stage time of a step
        (MomentumRhs::time semantics, forms.cpp:1061-1062)."""
        _check(lib().dgb_set_dirichlet_time_dependent(self._h, int(bool(enable))))

    def boundary_points(self, q1d: int):
        import numpy as np
        nq = q1d ** (self.dim - 1)
        out = np.zeros((self.n_boundary, nq, self.dim))
        _check(lib().dgb_boundary_points(self._h, q1d, _np_ptr(out)))
        return out

    def face_lists(self):
        import numpy as np
        it = np.zeros((self.n_interior, 4), dtype=np.int32)
        bd = np.zeros((self.n_boundary, 3), dtype=np.int32)
        _check(lib().dgb_face_lists(self._h, it.ctypes.data_as(_ip), bd.ctypes.data_as(_ip)))
        return it, bd

    def set_fast_path(self, enable: bool):
        """Fast axis-aligned 3D kernels (default) or the generic kernels."""
        _check(lib().dgb_set_fast_path(self._h, int(bool(enable))))

    @property
    def fast_path_active(self) -> bool:
        return bool(lib().dgb_fast_path_active(self._h))

    @property
    def hanging_mode(self) -> int:
        """0: conforming mesh, 1: dense-table subface kernels, 2: sum-factorised (axis-aligned 3D)."""
        return int(lib().dgb_hanging_mode(self._h))

    def launch_count(self) -> int:
        return int(lib().dgb_launch_count(self._h))


# ---------------------------------------------------------------------------
# forms.hpp mirror
# ---------------------------------------------------------------------------
@dataclass
class MomentumCtx:
    """forms.hpp:56-64"""
    mass_coef: float = 0.0
    visc_coef: float = 0.0
    adv_coef: float = 0.0
    skew_coef: float = 0.0
    advecting: object = None  # CUDA tensor (w)

    def coefs(self):
        return (C.c_double * 4)(self.mass_coef, self.visc_coef, self.adv_coef, self.skew_coef)


@dataclass
class MomentumRhs:
    """forms.hpp:89-100 (lists of (coef, field) / (coef, field, w))."""
    mass: List[Tuple[float, object]] = field(default_factory=list)
    visc: List[Tuple[float, object]] = field(default_factory=list)
    adv: List[Tuple[float, object, object]] = field(default_factory=list)
    pres: List[Tuple[float, object]] = field(default_factory=list)
    dir_visc_coef: float = 0.0
    dir_adv_coef: float = 0.0
    dir_w: object = None


def apply_momentum(V: DGContext, ctx: MomentumCtx, x, out):
    _check(lib().dgb_momentum_apply(V.handle, ctx.coefs(), _ptr(ctx.advecting), _ptr(x), _ptr(out)))


def apply_momentum_host(V: DGContext, coefs, w_host, x_host, out_host):
    """apply_momentum on HOST fields (blocking): copies in, applies and copies back with
    the copies pipelined against the apply over z-slabs on uniform 3D meshes."""
    c = (C.c_double * 4)(*[float(v) for v in coefs])
    _check(lib().dgb_momentum_apply_host(V.handle, c, _host_ptr(w_host), _host_ptr(x_host), _host_ptr(out_host)))


def apply_pressure_helmholtz_host(V: DGContext, mass_coef: float, x_host, out_host):
    _check(lib().dgb_pressure_apply_host(V.handle, float(mass_coef), _host_ptr(x_host), _host_ptr(out_host)))


def momentum_diagonal(V: DGContext, ctx: MomentumCtx, diag):
    _check(lib().dgb_momentum_diag(V.handle, ctx.coefs(), _ptr(ctx.advecting), _ptr(diag)))


def apply_pressure_helmholtz(V: DGContext, mass_coef: float, x, out):
    _check(lib().dgb_pressure_apply(V.handle, float(mass_coef), _ptr(x), _ptr(out)))


def helmholtz_diagonal(V: DGContext, mass_coef: float, diag):
    _check(lib().dgb_helmholtz_diag(V.handle, float(mass_coef), _ptr(diag)))


def apply_scalar_laplace(V: DGContext, dirichlet_bdry: bool, x, out):
    _check(lib().dgb_laplace_apply(V.handle, int(bool(dirichlet_bdry)), _ptr(x), _ptr(out)))


def scalar_laplace_diagonal(V: DGContext, dirichlet_bdry: bool, diag):
    _check(lib().dgb_laplace_diag(V.handle, int(bool(dirichlet_bdry)), _ptr(diag)))


def apply_mass(V: DGContext, space: int, x, out):
    _check(lib().dgb_mass_apply(V.handle, space, _ptr(x), _ptr(out)))


def mass_diagonal(V: DGContext, space: int, diag):
    _check(lib().dgb_mass_diag(V.handle, space, _ptr(diag)))


def momentum_rhs(V: DGContext, spec: MomentumRhs, out):
    d = _RhsDesc()
    for name in ("mass", "visc", "pres"):
        terms = getattr(spec, name)
        if len(terms) > 4:
            raise ValueError("at most 4 terms per list")
        setattr(d, "n_" + name, len(terms))
        for i, (c, f) in enumerate(terms):
            getattr(d, name + "_coef")[i] = c
            getattr(d, name + "_f")[i] = _ptr(f)
    d.n_adv = len(spec.adv)
    for i, (c, f, w) in enumerate(spec.adv):
        d.adv_coef[i] = c
        d.adv_f[i] = _ptr(f)
        d.adv_w[i] = _ptr(w)
    d.dir_visc_coef = spec.dir_visc_coef
    d.dir_adv_coef = spec.dir_adv_coef
    d.dir_w = _ptr(spec.dir_w)
    _check(lib().dgb_momentum_rhs(V.handle, C.byref(d), _ptr(out)))


def divergence_functional(V: DGContext, u, out):
    _check(lib().dgb_divergence(V.handle, _ptr(u), _ptr(out)))


def pressure_rhs(V: DGContext, inv_adt: float, u, mass_coef: float, p_old, out):
    _check(lib().dgb_pressure_rhs(V.handle, float(inv_adt), _ptr(u), float(mass_coef), _ptr(p_old), _ptr(out)))


def pressure_gradient_rhs(V: DGContext, p, out):
    _check(lib().dgb_pressure_gradient(V.handle, _ptr(p), _ptr(out)))


def kinetic_energy(V: DGContext, u) -> float:
    r = C.c_double()
    _check(lib().dgb_kinetic_energy(V.handle, _ptr(u), C.byref(r)))
    return r.value


# ---------------------------------------------------------------------------
# BLAS-1 (kern::axpy/axpby/scal/dot/max_abs_diff, kernels.hpp:34-43) on device vectors
# ---------------------------------------------------------------------------
def _n(x) -> int:
    return int(x.numel())


def axpy(V: DGContext, a: float, x, y) -> None:
    """y += a x  (kern::axpy)"""
    _check(lib().dgb_axpy(V.handle, _n(y), float(a), _ptr(x), _ptr(y)))


def axpby(V: DGContext, a: float, x, b: float, y) -> None:
    """y = a x + b y  (kern::axpby)"""
    _check(lib().dgb_axpby(V.handle, _n(y), float(a), _ptr(x), float(b), _ptr(y)))


def scal(V: DGContext, a: float, x) -> None:
    """x *= a  (kern::scal)"""
    _check(lib().dgb_scal(V.handle, _n(x), float(a), _ptr(x)))


def dot(V: DGContext, x, y) -> float:
    """<x, y>  (kern::dot)"""
    r = C.c_double()
    _check(lib().dgb_dot(V.handle, _n(x), _ptr(x), _ptr(y), C.byref(r)))
    return r.value


def norm(V: DGContext, x) -> float:
    """sqrt(<x, x>)  (the solvers' 2-norm, krylov.cpp:54-56)"""
    r = C.c_double()
    _check(lib().dgb_norm(V.handle, _n(x), _ptr(x), C.byref(r)))
    return r.value


def max_abs_diff(V: DGContext, x, y) -> float:
    """max_i |x_i - y_i|  (kern::max_abs_diff)"""
    r = C.c_double()
    _check(lib().dgb_max_abs_diff(V.handle, _n(x), _ptr(x), _ptr(y), C.byref(r)))
    return r.value


def l2_norm(V: DGContext, x, space: int = SPACE_U) -> float:
    """sqrt(x^T M x) on the device (diagnostics)."""
    r = C.c_double()
    _check(lib().dgb_l2_norm(V.handle, space, _ptr(x), C.byref(r)))
    return r.value


def check_steady(V: DGContext, u_new, u_old, tol: float):
    """(max |u_new - u_old| < tol, that max), computed on the device."""
    st, d = C.c_int(), C.c_double()
    _check(lib().dgb_check_steady(V.handle, _ptr(u_new), _ptr(u_old), tol, C.byref(st), C.byref(d)))
    return bool(st.value), d.value


def stability_params(V: DGContext, dt: float, Re: float, U: float):
    """(C, mu) = (k U dt / H, k^2 dt / (Re H^2)), H = min cell diameter."""
    c, mu = C.c_double(), C.c_double()
    _check(lib().dgb_stability_params(V.handle, dt, Re, U, C.byref(c), C.byref(mu)))
    return c.value, mu.value


# ---------------------------------------------------------------------------
# krylov.hpp mirror
# ---------------------------------------------------------------------------
@dataclass
class SolverSettings:
    """krylov.hpp:24-29"""
    rel_tol: float = 1e-10
    abs_tol: float = 0.0
    max_iter: int = 10000
    restart: int = 50


@dataclass
class SolveResult:
    iterations: int
    residual: float


class JacobiPreconditioner:
    """krylov.hpp:40-48: holds 1/diag; raises SolverError naming the first zero-diagonal dof."""

    def __init__(self, V: DGContext, diag):
        self.inv = diag.new_empty(diag.shape)
        _check(lib().dgb_jacobi_inverse(V.handle, diag.numel(), _ptr(diag), _ptr(self.inv)))


@dataclass
class LinearOperator:
    """The LinearOp closure of krylov.hpp:22, restricted to the device operators."""
    op: int
    coefs: Tuple[float, float, float, float] = (0.0, 0.0, 0.0, 0.0)
    w: object = None
    dirichlet_bdry: bool = False

    @staticmethod
    def momentum(ctx: MomentumCtx):
        return LinearOperator(OP_MOMENTUM, (ctx.mass_coef, ctx.visc_coef, ctx.adv_coef, ctx.skew_coef), ctx.advecting)

    @staticmethod
    def pressure_helmholtz(mass_coef: float):
        return LinearOperator(OP_PRESSURE, (mass_coef, 0.0, 0.0, 0.0))

    def _c(self):
        o = _Operator()
        o.op = self.op
        for i in range(4):
            o.coefs[i] = self.coefs[i]
        o.d_w = _ptr(self.w)
        o.dirichlet_bdry = int(self.dirichlet_bdry)
        return o


def _solve(fn, V, A: LinearOperator, b, s: SolverSettings, M: Optional[JacobiPreconditioner], x):
    res = _Result()
    cap = 100000
    import numpy as np
    hist = np.zeros(cap)
    hl = C.c_int()
    st = _Settings(s.rel_tol, s.abs_tol, s.max_iter, s.restart)
    op = A._c()
    code = fn(V.handle, C.byref(op), C.byref(st), _ptr(M.inv) if M is not None else None, _ptr(b), _ptr(x),
              C.byref(res), _np_ptr(hist), cap, C.byref(hl))
    if code in (E_NO_CONVERGENCE, E_BREAKDOWN, E_NOT_SPD):
        raise SolverError(lib().dgb_last_error().decode(), hist[: min(hl.value, cap)].tolist())
    _check(code)
    return SolveResult(res.iterations, res.residual)


def cg_solve(V: DGContext, A: LinearOperator, b, s: SolverSettings, M: Optional[JacobiPreconditioner], x):
    """krylov.hpp:58-60: x is initial guess and solution."""
    return _solve(lib().dgb_cg, V, A, b, s, M, x)


def gmres_solve(V: DGContext, A: LinearOperator, b, s: SolverSettings, M: Optional[JacobiPreconditioner], x):
    """krylov.hpp:64-66"""
    return _solve(lib().dgb_gmres, V, A, b, s, M, x)


def pressure_cg_mg(V: DGContext, mass_coef: float, b, s: SolverSettings, x) -> SolveResult:
    """(mass_coef M + K_SIP) x = b by CG with the hybrid multigrid V-cycle (not in the
    reference, which uses Jacobi: SURVEY 8(f) item 1).  x: initial guess and solution."""
    res = _Result()
    st = _Settings(s.rel_tol, s.abs_tol, s.max_iter, s.restart)
    code = lib().dgb_pressure_cg_mg(V.handle, mass_coef, C.byref(st), _ptr(b), _ptr(x), C.byref(res))
    if code in (E_NO_CONVERGENCE, E_BREAKDOWN, E_NOT_SPD):
        raise SolverError(lib().dgb_last_error().decode())
    _check(code)
    return SolveResult(res.iterations, res.residual)


def pressure_mg_vcycle(V: DGContext, mass_coef: float, r, z) -> None:
    """z = B r, one V-cycle of the pressure multigrid preconditioner."""
    _check(lib().dgb_pressure_mg_vcycle(V.handle, mass_coef, _ptr(r), _ptr(z)))


# ---------------------------------------------------------------------------
# TR-BDF2 step
# ---------------------------------------------------------------------------
@dataclass
class StepParams:
    dt: float = 1e-3
    Re: float = 100.0
    c: float = 1e3
    time: float = 0.0
    restart: int = 50
    tol_mom: float = 1e-10
    tol_p: float = 1e-10
    tol_mass: float = 1e-12
    max_iter: int = 10000
    first_step: bool = True
    pressure_precond: str = "jacobi"  # "jacobi" (the reference's) or "mg" (pressure_cg_mg)
    fixed_point: bool = False         # trbdf2_step_fixedpoint
    fp_tol: float = 1e-8
    fp_max_iter: int = 100

    def _c(self):
        pc = {"jacobi": 0, "mg": 1}[self.pressure_precond]
        return _StepParams(self.dt, self.Re, self.c, self.time, self.restart, self.tol_mom, self.tol_p,
                           self.tol_mass, self.max_iter, int(self.first_step), pc, int(self.fixed_point),
                           self.fp_tol, self.fp_max_iter)


SCHEME_TRBDF2, SCHEME_BCG, SCHEME_GQ_BDF2 = 0, 1, 2


def projection_step(V: DGContext, scheme: int, P: StepParams, u_nm1, u_n, p_n, u_np1, p_np1) -> List[int]:
    """One step of SCHEME_TRBDF2 / SCHEME_BCG / SCHEME_GQ_BDF2; for the two
    baseline schemes returns [gmres, 0, cg, 0, mass-cg pre, mass-cg post, 0, 0, fixed-point re-solves, 0]."""
    its = (C.c_int * 10)()
    code = lib().dgb_projection_step(V.handle, scheme, C.byref(P._c()), _ptr(u_nm1), _ptr(u_n), _ptr(p_n),
                                     _ptr(u_np1), _ptr(p_np1), its)
    if code in (E_NO_CONVERGENCE, E_BREAKDOWN, E_NOT_SPD):
        raise SolverError(lib().dgb_last_error().decode())
    _check(code)
    return list(its)[: 10 if (P.fixed_point or scheme != SCHEME_TRBDF2) else 8]


def trbdf2_step(V: DGContext, P: StepParams, u_nm1, u_n, p_n, u_np1, p_np1) -> List[int]:
    """Returns [gmres s1, gmres s2, cg s1, cg s2, mass-cg x4] (+ [fixed-point re-solves s1, s2]
    when P.fixed_point)."""
    its = (C.c_int * 10)()
    code = lib().dgb_trbdf2_step(V.handle, C.byref(P._c()), _ptr(u_nm1), _ptr(u_n), _ptr(p_n), _ptr(u_np1),
                                 _ptr(p_np1), its)
    if code in (E_NO_CONVERGENCE, E_BREAKDOWN, E_NOT_SPD):
        raise SolverError(lib().dgb_last_error().decode())
    _check(code)
    return list(its)[: 10 if P.fixed_point else 8]


# ---------------------------------------------------------------------------
# synthetic inputs (BASELINE.json configs)
# ---------------------------------------------------------------------------
def seeded_uniform(seed: int, n: int, lo: float = -1.0, hi: float = 1.0):
    import numpy as np
    out = np.empty(n)
    _check(lib().dgb_seeded_uniform(seed, n, lo, hi, _np_ptr(out)))
    return out


class SynthField:
    """Curl of a random stream function (2D) / vector potential (3D)."""

    def __init__(self, dim: int, seed: int, scale: float = 1.0):
        import numpy as np
        self.user = np.zeros(512)
        _check(lib().dgb_synth_init(dim, seed, scale, _np_ptr(self.user)))
        self.dim = dim

    @property
    def user_ptr(self):
        return self.user.ctypes.data_as(C.c_void_p)

    @property
    def fn_ptr(self):
        return C.cast(lib().dgb_synth_eval, C.c_void_p)

    def eval(self, x):
        import numpy as np
        out = np.zeros(self.dim)
        xx = np.ascontiguousarray(x, dtype=np.float64)
        lib().dgb_synth_eval(_np_ptr(xx), 0.0, _np_ptr(out), self.user_ptr)
        return out

    def interpolate(self, V: DGContext):
        import numpy as np
        out = np.zeros(V.n_u)
        _check(lib().dgb_interpolate_synth(V.handle, _np_ptr(self.user), _np_ptr(out)))
        return out


def interpolate_synth_device(V: DGContext, f: "SynthField", out):
    _check(lib().dgb_interpolate_synth_device(V.handle, _np_ptr(f.user), _ptr(out)))


def fp64_peak_tflops(V: DGContext) -> float:
    r = C.c_double()
    _check(lib().dgb_fp64_peak(V.handle, C.byref(r)))
    return r.value


def fp64_peak_dmma_tflops(V: DGContext) -> float:
    """FP64 peak through the tensor-core instruction (DMMA m8n8k4): the pipe's upper peak."""
    r = C.c_double()
    _check(lib().dgb_fp64_peak_dmma(V.handle, C.byref(r)))
    return r.value


__all__ = [n for n in dir() if not n.startswith("_")]
