"""Hanging faces (1-irregular refinement) on the device vs the unmodified reference.

The reference refines with Mesh::refine_and_coarsen (mesh.hpp:125-128) and records one
interior face per hanging subface with its embedding into the coarse cell
(mesh.cpp:344-375); its operators integrate such faces like any interior face
(test_forms.cpp:145-179 checks them against dense assembly).  Here the reference's own
refined mesh is handed to the device through dgb_ctx_create_mesh_hanging (the arrays a
reference-side binding passes) and every face-carrying operator,
diagonal, right-hand side, Krylov solve and TR-BDF2 step is compared on the same seeded
inputs.  Gates as everywhere: per-apply relative L2 <= 1e-12, iteration counts +-1,
fields <= 1e-9.
"""
import numpy as np
import pytest

from test_gpu_parity import TOL_APPLY, TOL_FIELD, dev, host, rel

pytestmark = pytest.mark.gpu


def hpair(ref, gpu, dim, n_el, ku, kp, refine, amp=0.0, seed=7, dirichlet_seed=None, outlet=None):
    R = ref.RefCtx.refined(dim, n_el, ku, kp, refine, amp, seed)
    xv, cv, bid, it, emb = R.mesh_arrays()
    hang = it[:, 4] == 1
    assert hang.sum() == R.n_hanging > 0
    D = gpu.DGContext(dim, 0, ku, kp, mesh_arrays=(xv, cv, bid, it[hang, :4], emb[hang]))
    assert (R.n_u, R.n_p, R.ncells, R.n_interior, R.n_boundary) == (D.n_u, D.n_p, D.ncells, D.n_interior,
                                                                     D.n_boundary)
    assert D.n_hanging == R.n_hanging
    # 3D refined meshes whose cells are all axis-aligned boxes run the line-split fast kernels
    # (hanging slots = zero-weight face type) + the subface supplement; everything else the
    # generic kernels + the supplement
    assert D.fast_path_active == (1 if dim == 3 and amp == 0.0 else 0)
    assert D.hanging_mode == (2 if dim == 3 and amp == 0.0 else 1)
    if outlet is not None:
        R.set_bc(outlet, 1)
        D.set_boundary_type(outlet, gpu.BC_OUTLET)
    if dirichlet_seed is not None:
        f = gpu.SynthField(dim, dirichlet_seed)
        for b in range(2 * dim):
            if b == outlet:
                continue
            R.set_bc(b, 0, f.fn_ptr, f.user_ptr)
            D.set_dirichlet_fn(b, f.fn_ptr, f.user_ptr, 0.0)
        R._keep.append(f)
        D._keep.append(f)
    return R, D


CASES = [
    # dim, n_el, ku, kp, refine (active indices), amp
    (2, 2, 2, 1, [0], 0.0),        # the reference's own hanging-face test mesh (test_forms.cpp:145-149)
    (2, 4, 3, 2, [5, 6, 9], 0.0),
    (2, 3, 2, 1, [4], 0.06),       # distorted before refinement: per-qp geometry on both sides
    (2, 3, 4, 3, [0, 8], 0.0),
    (3, 2, 2, 1, [0], 0.0),
    (3, 3, 3, 2, [13], 0.0),       # centre cell: six coarse faces with four subfaces each
    (3, 3, 2, 1, [0, 26], 0.04),
    (3, 4, 3, 2, [0, 21, 22, 42, 63], 0.0),  # fine cells next to each other, at corners and inside
    (3, 2, 4, 3, [7], 0.0),        # degree 4 / 3: the N = 5 subface kernels
]
IDS = [f"d{c[0]}n{c[1]}k{c[2]}{c[3]}r{len(c[4])}a{c[5]}" for c in CASES]


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,amp", CASES, ids=IDS)
def test_face_lists_match_reference(ref, gpu, dim, n_el, ku, kp, refine, amp):
    """Interior faces incl. one record per hanging subface from the fine side, in the
    reference order (mesh.cpp:316-377); boundary faces likewise."""
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, amp)
    it, _, bd, _ = R.faces()
    di, db = D.face_lists()
    np.testing.assert_array_equal(di, it[:, :4])
    np.testing.assert_array_equal(db, bd)


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,amp", CASES, ids=IDS)
@pytest.mark.parametrize("coefs", [(1.9, 1.1, 0.7, 0.0), (1.0 / (0.2929 * 1e-3), 0.005, 0.5, -0.4)])
def test_momentum_apply_and_diag(ref, gpu, dim, n_el, ku, kp, refine, amp, coefs):
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, amp)
    w = gpu.seeded_uniform(31, R.n_u)
    x = gpu.seeded_uniform(32, R.n_u)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    y = D.zeros()
    gpu.apply_momentum(D, ctx, dev(x), y)
    assert rel(host(y), R.momentum(coefs, w, x)) <= TOL_APPLY
    d = D.zeros()
    gpu.momentum_diagonal(D, ctx, d)
    assert rel(host(d), R.momentum_diag(coefs, w)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,amp", CASES, ids=IDS)
def test_pressure_laplace_mass(ref, gpu, dim, n_el, ku, kp, refine, amp):
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, amp)
    x = gpu.seeded_uniform(33, R.n_p)
    for mc in (2.3, 0.0):
        y = D.zeros(gpu.SPACE_P)
        gpu.apply_pressure_helmholtz(D, mc, dev(x), y)
        assert rel(host(y), R.pressure(mc, x)) <= TOL_APPLY
        d = D.zeros(gpu.SPACE_P)
        gpu.helmholtz_diagonal(D, mc, d)
        assert rel(host(d), R.helmholtz_diag(mc)) <= TOL_APPLY
    for dirichlet in (False, True):
        y = D.zeros(gpu.SPACE_P)
        gpu.apply_scalar_laplace(D, dirichlet, dev(x), y)
        assert rel(host(y), R.laplace(dirichlet, x)) <= TOL_APPLY
        d = D.zeros(gpu.SPACE_P)
        gpu.scalar_laplace_diagonal(D, dirichlet, d)
        assert rel(host(d), R.laplace_diag(dirichlet)) <= TOL_APPLY
    xu = gpu.seeded_uniform(34, R.n_u)
    y = D.zeros()
    gpu.apply_mass(D, gpu.SPACE_U, dev(xu), y)
    assert rel(host(y), R.mass(0, xu)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,amp", CASES, ids=IDS)
def test_divergence_gradient_pressure_rhs(ref, gpu, dim, n_el, ku, kp, refine, amp):
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, amp)
    u = gpu.seeded_uniform(35, R.n_u)
    p = gpu.seeded_uniform(36, R.n_p)
    y = D.zeros(gpu.SPACE_P)
    gpu.divergence_functional(D, dev(u), y)
    assert rel(host(y), R.divergence(u)) <= TOL_APPLY
    y = D.zeros()
    gpu.pressure_gradient_rhs(D, dev(p), y)
    assert rel(host(y), R.gradient(p)) <= TOL_APPLY
    y = D.zeros(gpu.SPACE_P)
    gpu.pressure_rhs(D, 1.7, dev(u), 7.3, dev(p), y)
    assert rel(host(y), R.pressure_rhs(1.7, u, 7.3, p)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,amp", CASES, ids=IDS)
def test_momentum_rhs_full(ref, gpu, dim, n_el, ku, kp, refine, amp):
    """test_forms.cpp:255-310 terms (2 viscous, 2 advective, pressure, Dirichlet data) on a
    refined mesh: the explicit interior-face fluxes cross every hanging subface."""
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, amp, dirichlet_seed=5)
    un, ug, wx = (gpu.seeded_uniform(s, R.n_u) for s in (41, 42, 43))
    pp = gpu.seeded_uniform(44, R.n_p)
    want = R.momentum_rhs(mass=[(2.9, un)], visc=[(0.65, un), (0.3, ug)], adv=[(0.5, un, wx), (0.25, ug, ug)],
                          pres=[(1.0, pp)], dir_visc=0.65, dir_adv=0.5, dir_w=wx, time=0.0)
    dun, dug, dwx, dpp = dev(un), dev(ug), dev(wx), dev(pp)
    spec = gpu.MomentumRhs(mass=[(2.9, dun)], visc=[(0.65, dun), (0.3, dug)],
                           adv=[(0.5, dun, dwx), (0.25, dug, dug)], pres=[(1.0, dpp)], dir_visc_coef=0.65,
                           dir_adv_coef=0.5, dir_w=dwx)
    y = D.zeros()
    gpu.momentum_rhs(D, spec, y)
    assert rel(host(y), want) <= TOL_APPLY


def test_outlet_boundary_with_hanging_faces(ref, gpu):
    R, D = hpair(ref, gpu, 2, 4, 2, 1, [5, 10], outlet=1)
    coefs = (3.7, 1.3, 0.9, 0.0)
    w, x = gpu.seeded_uniform(51, R.n_u), gpu.seeded_uniform(52, R.n_u)
    y = D.zeros()
    gpu.apply_momentum(D, gpu.MomentumCtx(*coefs, advecting=dev(w)), dev(x), y)
    assert rel(host(y), R.momentum(coefs, w, x)) <= TOL_APPLY


def test_operators_are_linear_and_pressure_symmetric(ref, gpu):
    """Size-independent properties: the SIP operator stays symmetric across hanging
    subfaces (both sides' consistency / symmetry terms), the momentum operator linear."""
    R, D = hpair(ref, gpu, 3, 3, 2, 1, [13])
    a, b = gpu.seeded_uniform(81, R.n_p), gpu.seeded_uniform(82, R.n_p)
    ya, yb = D.zeros(gpu.SPACE_P), D.zeros(gpu.SPACE_P)
    gpu.apply_pressure_helmholtz(D, 0.3, dev(a), ya)
    gpu.apply_pressure_helmholtz(D, 0.3, dev(b), yb)
    ha, hb = host(ya), host(yb)
    assert abs(b @ ha - a @ hb) <= 1e-12 * abs(b @ ha)
    coefs = (2.0, 0.7, 0.6, 0.0)
    w = gpu.seeded_uniform(83, R.n_u)
    xa, xb = gpu.seeded_uniform(84, R.n_u), gpu.seeded_uniform(85, R.n_u)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    outs = []
    for x in (xa, xb, 2.0 * xa - 3.0 * xb):
        y = D.zeros()
        gpu.apply_momentum(D, ctx, dev(x), y)
        outs.append(host(y))
    assert rel(outs[2], 2.0 * outs[0] - 3.0 * outs[1]) <= 1e-13
    # determinism: the subface scatter adds in a fixed order
    y2 = D.zeros()
    gpu.apply_momentum(D, ctx, dev(xa), y2)
    assert np.array_equal(host(y2), outs[0])


@pytest.mark.parametrize("dim,n_el,ku,kp,refine", [(2, 4, 2, 1, [5, 6]), (3, 3, 2, 1, [13]), (3, 2, 3, 2, [0])])
def test_krylov_iteration_parity(ref, gpu, dim, n_el, ku, kp, refine):
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine)
    mc = 1.0 / (1e6 * 0.2929 ** 2 * 1e-6)
    b = gpu.seeded_uniform(61, R.n_p)
    x_ref, it_ref, _ = R.solve(1, 0, (mc, 0, 0, 0), None, b, np.zeros(R.n_p))
    diag = D.zeros(gpu.SPACE_P)
    gpu.helmholtz_diagonal(D, mc, diag)
    x = D.zeros(gpu.SPACE_P)
    res = gpu.cg_solve(D, gpu.LinearOperator.pressure_helmholtz(mc), dev(b), gpu.SolverSettings(),
                       gpu.JacobiPreconditioner(D, diag), x)
    assert abs(res.iterations - it_ref) <= 1
    assert rel(host(x), x_ref) <= 1e-8
    coefs = (1.0 / (0.2929 * 1e-2), 0.005, 0.5, 0.0)
    w, bu = gpu.seeded_uniform(62, R.n_u), gpu.seeded_uniform(63, R.n_u)
    xu_ref, itu_ref, _ = R.solve(0, 1, coefs, w, bu, np.zeros(R.n_u), restart=10)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    diag = D.zeros()
    gpu.momentum_diagonal(D, ctx, diag)
    xu = D.zeros()
    res = gpu.gmres_solve(D, gpu.LinearOperator.momentum(ctx), dev(bu), gpu.SolverSettings(restart=10),
                          gpu.JacobiPreconditioner(D, diag), xu)
    assert abs(res.iterations - itu_ref) <= 1
    assert rel(host(xu), xu_ref) <= 1e-8


@pytest.mark.parametrize("dim,n_el,ku,kp,refine,steps", [(2, 6, 2, 1, [14, 15, 20, 21], 2),
                                                         (3, 3, 2, 1, [13], 1), (3, 2, 3, 2, [0], 1)])
def test_trbdf2_steps_on_refined_mesh(ref, gpu, dim, n_el, ku, kp, refine, steps):
    """Full TR-BDF2 steps (restated driver) on a refined mesh: every
    solve's iteration count +-1, fields <= 1e-9."""
    R, D = hpair(ref, gpu, dim, n_el, ku, kp, refine, dirichlet_seed=3)
    f = gpu.SynthField(dim, 3)
    u0 = f.interpolate(D)
    p0 = np.zeros(R.n_p)
    u_prev, u, p = u0.copy(), u0.copy(), p0.copy()
    du_prev, du, dp = dev(u0), dev(u0), dev(p0)
    dt, Re = 1e-3, 100.0
    for n in range(steps):
        params = [dt, Re, 1e3, n * dt, 50, 1e-10, 1e-10, 1e-12, 10000, 1.0 if n == 0 else 0.0, 0.0, 1e-8, 100]
        u1, p1, its_ref = R.step(params, u_prev, u, p)
        P = gpu.StepParams(dt=dt, Re=Re, c=1e3, time=n * dt, restart=50, first_step=(n == 0))
        du1, dp1 = D.zeros(), D.zeros(gpu.SPACE_P)
        its = gpu.trbdf2_step(D, P, du_prev, du, dp, du1, dp1)
        for a, b in zip(its, its_ref):
            assert abs(a - b) <= 1, (its, its_ref)
        u_prev, u, p = u, u1, p1
        du_prev, du, dp = du, du1, dp1
    hu, hp = host(du), host(dp)
    assert rel(hu, u) <= TOL_FIELD
    assert rel(hp - hp.mean(), p - p.mean()) <= TOL_FIELD


def test_cell_range_rejected_on_refined_mesh(ref, gpu):
    """The subface kernels always cover every hanging face: owned-cell ranges (z-slabs) are only
    defined on conforming meshes."""
    R, D = hpair(ref, gpu, 3, 2, 2, 1, [0])
    assert gpu.lib().dgb_set_cell_range(D.handle, 0, 4) != 0
    assert gpu.lib().dgb_set_cell_range(D.handle, 0, -1) == 0


def test_bad_hanging_records_rejected(ref, gpu):
    R = ref.RefCtx.refined(2, 2, 2, 1, [0])
    xv, cv, bid, it, emb = R.mesh_arrays()
    hang = it[:, 4] == 1
    rec = it[hang, :4].copy()
    rec[0, 1] = 2  # fine face on the domain boundary (boundary id 2)
    with pytest.raises(gpu.DGBError):
        gpu.DGContext(2, 0, 2, 1, mesh_arrays=(xv, cv, bid, rec, emb[hang]))
    with pytest.raises(gpu.DGBError):  # subfaces left out: unmatched interior faces
        gpu.DGContext(2, 0, 2, 1, mesh_arrays=(xv, cv, bid))


@pytest.mark.parametrize("n_el,ku,kp,refine", [(3, 2, 1, [0, 13]), (4, 3, 2, [0, 21, 22, 42, 63])])
def test_fast_kernels_match_generic_on_refined_mesh(ref, gpu, n_el, ku, kp, refine):
    """Axis-aligned refined meshes: the line-split fast kernels (hanging slots as the
    zero-weight face type 3) + hang.cu against the generic kernels + hang.cu, every
    face-carrying operator, with an outlet and Dirichlet data."""
    R, D = hpair(ref, gpu, 3, n_el, ku, kp, refine, 0.0, dirichlet_seed=5, outlet=1)
    w, x, un = (gpu.seeded_uniform(s, R.n_u) for s in (51, 52, 53))
    p = gpu.seeded_uniform(54, R.n_p)
    dw, dx, dun, dp = dev(w), dev(x), dev(un), dev(p)
    ctx = gpu.MomentumCtx(1.0 / (0.2929 * 1e-3), 0.005, 0.5, 0.0, advecting=dw)
    spec = gpu.MomentumRhs(mass=[(2.9, dun)], visc=[(0.65, dun)], adv=[(0.5, dun, dw)], pres=[(1.0, dp)],
                           dir_visc_coef=0.65, dir_adv_coef=0.5, dir_w=dw)
    out = {}
    for fast in (True, False):
        D.set_fast_path(fast)
        assert D.fast_path_active == (1 if fast else 0)
        r = []
        y = D.zeros(); gpu.apply_momentum(D, ctx, dx, y); r.append(host(y))
        y = D.zeros(); gpu.momentum_diagonal(D, ctx, y); r.append(host(y))
        y = D.zeros(gpu.SPACE_P); gpu.apply_pressure_helmholtz(D, 2.3, dp, y); r.append(host(y))
        y = D.zeros(gpu.SPACE_P); gpu.helmholtz_diagonal(D, 2.3, y); r.append(host(y))
        y = D.zeros(gpu.SPACE_P); gpu.apply_scalar_laplace(D, True, dp, y); r.append(host(y))
        y = D.zeros(gpu.SPACE_P); gpu.scalar_laplace_diagonal(D, True, y); r.append(host(y))
        y = D.zeros(gpu.SPACE_P); gpu.divergence_functional(D, dx, y); r.append(host(y))
        y = D.zeros(); gpu.momentum_rhs(D, spec, y); r.append(host(y))
        out[fast] = r
    D.set_fast_path(True)
    for a, b in zip(out[True], out[False]):
        assert rel(a, b) <= TOL_APPLY
