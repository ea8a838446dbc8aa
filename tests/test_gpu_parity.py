"""Device path vs the reference CPU implementation on identical seeded inputs.

Gate (BASELINE.json north_star): per-apply relative L2 <= 1e-12 in fp64,
Krylov iteration counts within +-1, end-of-run fields within relative L2 1e-9.
Every device call goes through the C-ABI (libdgb.so); the checker is the
unmodified reference library (oracle/_ref/libdgref.so).
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

TOL_APPLY = 1e-12   # per-apply relative L2 (north_star)
TOL_FIELD = 1e-9    # end-of-run fields (north_star)


def rel(a, b):
    nb = np.linalg.norm(b)
    return np.linalg.norm(a - b) / (nb if nb > 0 else 1.0)


def dev(t):
    import torch
    return torch.from_numpy(np.ascontiguousarray(t, dtype=np.float64)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


def pair(ref, gpu, dim, n_el, ku, kp, amp=0.0, seed=7, outlet=None, dirichlet_seed=None):
    R = ref.RefCtx(dim, n_el, ku, kp, amp, seed)
    D = gpu.DGContext(dim, n_el, ku, kp, amp, seed)
    assert (R.n_u, R.n_p, R.ncells) == (D.n_u, D.n_p, D.ncells)
    assert (R.n_interior, R.n_boundary) == (D.n_interior, D.n_boundary)
    if outlet is not None:
        R.set_bc(outlet, 1)
        D.set_boundary_type(outlet, gpu.BC_OUTLET)
    if dirichlet_seed is not None:
        f = gpu.SynthField(dim, dirichlet_seed)
        for bid in range(2 * dim):
            if bid == outlet:
                continue
            R.set_bc(bid, 0, f.fn_ptr, f.user_ptr)
            D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
        R._keep.append(f)
        D._keep.append(f)
    return R, D


CASES = [
    # dim, n_el, ku, kp, amp
    (2, 4, 2, 1, 0.0),
    (2, 3, 3, 2, 0.05),
    (2, 3, 4, 3, 0.0),
    (3, 2, 2, 1, 0.03),
    (3, 3, 2, 1, 0.0),
    (3, 2, 3, 2, 0.0),
    (3, 2, 3, 2, 0.03),
    (3, 2, 4, 3, 0.02),
]


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", CASES)
def test_pressure_helmholtz_apply_and_diag(ref, gpu, dim, n_el, ku, kp, amp):
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp)
    x = gpu.seeded_uniform(11, R.n_p)
    for mc in (2.3, 0.0):
        want = R.pressure(mc, x)
        y = D.zeros(gpu.SPACE_P)
        gpu.apply_pressure_helmholtz(D, mc, dev(x), y)
        assert rel(host(y), want) <= TOL_APPLY
        d = D.zeros(gpu.SPACE_P)
        gpu.helmholtz_diagonal(D, mc, d)
        assert rel(host(d), R.helmholtz_diag(mc)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", [(2, 3, 3, 2, 0.05), (3, 2, 3, 2, 0.03)])
def test_scalar_laplace_dirichlet(ref, gpu, dim, n_el, ku, kp, amp):
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp)
    x = gpu.seeded_uniform(12, R.n_p)
    for dirichlet in (True, False):
        y = D.zeros(gpu.SPACE_P)
        gpu.apply_scalar_laplace(D, dirichlet, dev(x), y)
        assert rel(host(y), R.laplace(dirichlet, x)) <= TOL_APPLY
        d = D.zeros(gpu.SPACE_P)
        gpu.scalar_laplace_diagonal(D, dirichlet, d)
        assert rel(host(d), R.laplace_diag(dirichlet)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", CASES)
@pytest.mark.parametrize("coefs", [(3.7, 1.3, 0.9, -0.45), (1.0 / (0.2929 * 1e-3), 0.005, 0.5, 0.0)])
def test_momentum_apply_and_diag(ref, gpu, dim, n_el, ku, kp, amp, coefs):
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp)
    w = gpu.seeded_uniform(21, R.n_u)
    x = gpu.seeded_uniform(22, R.n_u)
    want = R.momentum(coefs, w, x)
    y = D.zeros()
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    gpu.apply_momentum(D, ctx, dev(x), y)
    assert rel(host(y), want) <= TOL_APPLY
    d = D.zeros()
    gpu.momentum_diagonal(D, ctx, d)
    assert rel(host(d), R.momentum_diag(coefs, w)) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", [(2, 3, 2, 1, 0.05), (3, 2, 2, 1, 0.0)])
def test_momentum_outlet_switch(ref, gpu, dim, n_el, ku, kp, amp):
    """test_forms.cpp:312-363: outlet faces drop viscous terms and use w.n advection."""
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp, outlet=1)
    w = gpu.seeded_uniform(31, R.n_u)
    x = gpu.seeded_uniform(32, R.n_u)
    coefs = (1.0, 0.9, 0.8, 0.0)
    y = D.zeros()
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    gpu.apply_momentum(D, ctx, dev(x), y)
    assert rel(host(y), R.momentum(coefs, w, x)) <= TOL_APPLY
    d = D.zeros()
    gpu.momentum_diagonal(D, ctx, d)
    assert rel(host(d), R.momentum_diag(coefs, w)) <= TOL_APPLY
    u = gpu.seeded_uniform(33, R.n_u)
    b = D.zeros(gpu.SPACE_P)
    gpu.divergence_functional(D, dev(u), b)
    assert rel(host(b), R.divergence(u)) <= TOL_APPLY


@pytest.mark.parametrize("n_el,ku,kp", [(3, 1, 1), (3, 2, 1), (4, 3, 2), (2, 3, 3), (5, 2, 1)])
@pytest.mark.parametrize("outlet", [None, 1])
def test_fast_axis_path_matches_reference(ref, gpu, n_el, ku, kp, outlet):
    """The axis-aligned 3D fast kernels (fast_axis.cuh) against the reference, and
    against the generic device kernels on the same inputs."""
    R, D = pair(ref, gpu, 3, n_el, ku, kp, 0.0, outlet=outlet)
    assert D.fast_path_active
    w = gpu.seeded_uniform(81, R.n_u)
    x = gpu.seeded_uniform(82, R.n_u)
    xp = gpu.seeded_uniform(83, R.n_p)
    coefs = (1.0 / (0.2929 * 1e-3), 1.0 / 2000.0, 0.5, 0.0)
    want = R.momentum(coefs, w, x)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    outs = []
    for fast in (True, False):
        D.set_fast_path(fast)
        y = D.zeros()
        gpu.apply_momentum(D, ctx, dev(x), y)
        outs.append(host(y))
        assert rel(outs[-1], want) <= TOL_APPLY, fast
    want_d = R.momentum_diag(coefs, w)
    for fast in (True, False):
        D.set_fast_path(fast)
        d = D.zeros()
        gpu.momentum_diagonal(D, ctx, d)
        assert rel(host(d), want_d) <= TOL_APPLY, ("diag", fast)
    D.set_fast_path(True)
    # a viscous-dominated operator exercises the face terms harder
    coefs2 = (0.3, 2.0, 1.5, 0.0)
    want2 = R.momentum(coefs2, w, x)
    D.set_fast_path(True)
    y = D.zeros()
    gpu.apply_momentum(D, gpu.MomentumCtx(*coefs2, advecting=dev(w)), dev(x), y)
    assert rel(host(y), want2) <= TOL_APPLY
    for mc in (1.0 / (1e6 * 0.2929 ** 2 * 1e-6), 0.0):
        yp = D.zeros(gpu.SPACE_P)
        gpu.apply_pressure_helmholtz(D, mc, dev(xp), yp)
        assert rel(host(yp), R.pressure(mc, xp)) <= TOL_APPLY
    for dirichlet in (True, False):
        yl = D.zeros(gpu.SPACE_P)
        gpu.apply_scalar_laplace(D, dirichlet, dev(xp), yl)
        assert rel(host(yl), R.laplace(dirichlet, xp)) <= TOL_APPLY


def test_missing_advecting_field_raises(gpu):
    D = gpu.DGContext(2, 2, 2, 1)
    with pytest.raises(RuntimeError, match="advecting field missing"):
        gpu.apply_momentum(D, gpu.MomentumCtx(1.0, 1.0, 1.0, 0.0), D.zeros(), D.zeros())


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", CASES)
def test_mass_divergence_gradient_kinetic(ref, gpu, dim, n_el, ku, kp, amp):
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp)
    u = gpu.seeded_uniform(41, R.n_u)
    p = gpu.seeded_uniform(42, R.n_p)
    for space, v in ((0, u), (1, p)):
        y = D.zeros(space)
        gpu.apply_mass(D, space, dev(v), y)
        assert rel(host(y), R.mass(space, v)) <= TOL_APPLY
        d = D.zeros(space)
        gpu.mass_diagonal(D, space, d)
        assert rel(host(d), R.mass_diag(space)) <= TOL_APPLY
    if kp == ku - 1:
        b = D.zeros(gpu.SPACE_P)
        gpu.divergence_functional(D, dev(u), b)
        assert rel(host(b), R.divergence(u)) <= TOL_APPLY
        g = D.zeros()
        gpu.pressure_gradient_rhs(D, dev(p), g)
        assert rel(host(g), R.gradient(p)) <= TOL_APPLY
        pr = D.zeros(gpu.SPACE_P)
        gpu.pressure_rhs(D, 1.7, dev(u), 7.3, dev(p), pr)
        assert rel(host(pr), R.pressure_rhs(1.7, u, 7.3, p)) <= TOL_APPLY
    ke = gpu.kinetic_energy(D, dev(u))
    assert abs(ke - R.kinetic_energy(u)) <= 1e-12 * abs(R.kinetic_energy(u))


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", [(2, 2, 2, 1, 0.05), (2, 3, 3, 2, 0.0), (3, 2, 2, 1, 0.03),
                                                (3, 2, 3, 2, 0.0)])
def test_momentum_rhs_full(ref, gpu, dim, n_el, ku, kp, amp):
    """test_forms.cpp:255-310: 2 viscous, 2 advective, pressure and Dirichlet data terms."""
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp, dirichlet_seed=5)
    un = gpu.seeded_uniform(41, R.n_u)
    ug = gpu.seeded_uniform(42, R.n_u)
    wx = gpu.seeded_uniform(43, R.n_u)
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


def test_rhs_outlet_drops_pressure_boundary_flux(ref, gpu):
    R, D = pair(ref, gpu, 2, 2, 2, 1, 0.0, outlet=1)
    pp = gpu.seeded_uniform(52, R.n_p)
    want = R.momentum_rhs(pres=[(1.0, pp)])
    y = D.zeros()
    gpu.momentum_rhs(D, gpu.MomentumRhs(pres=[(1.0, dev(pp))]), y)
    assert rel(host(y), want) <= TOL_APPLY


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", [(2, 4, 2, 1, 0.05), (3, 3, 2, 1, 0.0), (3, 2, 3, 2, 0.03)])
def test_krylov_iteration_parity(ref, gpu, dim, n_el, ku, kp, amp):
    """Jacobi-CG on the pressure Helmholtz operator and Jacobi-GMRES on the momentum
    operator (test_krylov.cpp:215-274): iteration counts within +-1, solutions agree."""
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp)
    mc = 1.0 / (1e6 * 0.2929 ** 2 * 1e-6)
    b = gpu.seeded_uniform(61, R.n_p)
    x_ref, it_ref, _ = R.solve(1, 0, (mc, 0, 0, 0), None, b, np.zeros(R.n_p))
    diag = D.zeros(gpu.SPACE_P)
    gpu.helmholtz_diagonal(D, mc, diag)
    M = gpu.JacobiPreconditioner(D, diag)
    x = D.zeros(gpu.SPACE_P)
    res = gpu.cg_solve(D, gpu.LinearOperator.pressure_helmholtz(mc), dev(b), gpu.SolverSettings(), M, x)
    assert abs(res.iterations - it_ref) <= 1
    assert rel(host(x), x_ref) <= 1e-8

    coefs = (1.0 / (0.2929 * 1e-2), 0.005, 0.5, 0.0)
    w = gpu.seeded_uniform(62, R.n_u)
    bu = gpu.seeded_uniform(63, R.n_u)
    xu_ref, itu_ref, _ = R.solve(0, 1, coefs, w, bu, np.zeros(R.n_u), restart=10)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    diag = D.zeros()
    gpu.momentum_diagonal(D, ctx, diag)
    M = gpu.JacobiPreconditioner(D, diag)
    xu = D.zeros()
    res = gpu.gmres_solve(D, gpu.LinearOperator.momentum(ctx), dev(bu), gpu.SolverSettings(restart=10), M, xu)
    assert abs(res.iterations - itu_ref) <= 1
    assert rel(host(xu), xu_ref) <= 1e-8


def test_gmres_long_restart_multi_chunk(ref, gpu):
    """GMRES(80) with 147 reference iterations on a 3^3 Q3/Q2 advection-dominated momentum
    system: Arnoldi steps with up to 80 basis vectors exercise every Gram-Schmidt chunking
    path (32-vector dot passes, 16-vector update passes); iterations +-1, solution 1e-8."""
    R, D = pair(ref, gpu, 3, 3, 3, 2)
    coefs = (10.0, 1e-3, 1.0, 0.0)
    w = gpu.seeded_uniform(62, R.n_u)
    bu = gpu.seeded_uniform(63, R.n_u)
    xu_ref, itu_ref, _ = R.solve(0, 1, coefs, w, bu, np.zeros(R.n_u), restart=80)
    assert itu_ref > 80
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    diag = D.zeros()
    gpu.momentum_diagonal(D, ctx, diag)
    M = gpu.JacobiPreconditioner(D, diag)
    xu = D.zeros()
    res = gpu.gmres_solve(D, gpu.LinearOperator.momentum(ctx), dev(bu), gpu.SolverSettings(restart=80), M, xu)
    assert abs(res.iterations - itu_ref) <= 1
    assert rel(host(xu), xu_ref) <= 1e-8


def test_solver_budget_exhaustion_raises_with_history(ref, gpu):
    """test_krylov.cpp:317-341: SolverError carries a history of length max_iter."""
    R, D = pair(ref, gpu, 2, 4, 2, 1)
    b = gpu.seeded_uniform(71, R.n_p)
    with pytest.raises(gpu.SolverError) as ei:
        gpu.cg_solve(D, gpu.LinearOperator.pressure_helmholtz(0.0), dev(b),
                     gpu.SolverSettings(max_iter=3), None, D.zeros(gpu.SPACE_P))
    assert len(ei.value.history) == 3
    with pytest.raises(ref.RefSolverError) as er:
        R.solve(1, 0, (0.0, 0, 0, 0), None, b, np.zeros(R.n_p), max_iter=3, precond=False)
    assert len(er.value.history) == 3


def test_jacobi_zero_diagonal_names_dof(gpu):
    D = gpu.DGContext(2, 2, 2, 1)
    d = D.zeros(gpu.SPACE_P) + 1.0
    d[2] = 0.0
    with pytest.raises(gpu.SolverError, match="dof 2"):
        gpu.JacobiPreconditioner(D, d)


def test_zero_rhs_zero_iterations(gpu):
    D = gpu.DGContext(2, 2, 2, 1)
    x = D.zeros(gpu.SPACE_P) + 3.0
    r = gpu.cg_solve(D, gpu.LinearOperator.pressure_helmholtz(1.0), D.zeros(gpu.SPACE_P),
                     gpu.SolverSettings(), None, x)
    assert r.iterations == 0 and float(x.abs().max()) == 0.0


def _step_case(ref, gpu, dim, n_el, ku, kp, Re, dt, seed, steps, restart=50, fixed_point=False, amp=0.0,
               outlet=None):
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp, outlet=outlet, dirichlet_seed=seed)
    f = gpu.SynthField(dim, seed)
    u0 = f.interpolate(D)
    p0 = np.zeros(R.n_p)
    u_prev, u, p = u0.copy(), u0.copy(), p0.copy()
    du_prev, du, dp = dev(u0), dev(u0), dev(p0)
    for n in range(steps):
        params = [dt, Re, 1e3, n * dt, restart, 1e-10, 1e-10, 1e-12, 10000, 1.0 if n == 0 else 0.0,
                  1.0 if fixed_point else 0.0, 1e-8, 100]
        u1, p1, its_ref = R.step(params, u_prev, u, p)
        P = gpu.StepParams(dt=dt, Re=Re, c=1e3, time=n * dt, restart=restart, first_step=(n == 0),
                           fixed_point=fixed_point)
        du1, dp1 = D.zeros(), D.zeros(gpu.SPACE_P)
        its = gpu.trbdf2_step(D, P, du_prev, du, dp, du1, dp1)
        for i, (a, b) in enumerate(zip(its, its_ref)):
            # with fixed point, its[0:2] sum 1 + its[8:10] GMRES solves, each within +-1
            slack = 1 + (its_ref[8 + i] if fixed_point and i < 2 else 0)
            assert abs(a - b) <= slack, (its, its_ref)
        u_prev, u, p = u, u1, p1
        du_prev, du, dp = du, du1, dp1
    hu, hp = host(du), host(dp)
    assert rel(hu, u) <= TOL_FIELD
    # pressure compared after removing its mean
    assert rel(hp - hp.mean(), p - p.mean()) <= TOL_FIELD or rel(hp, p) <= TOL_FIELD
    return its_ref


def test_trbdf2_step_2d_small(ref, gpu):
    _step_case(ref, gpu, 2, 8, 2, 1, Re=100.0, dt=1e-3, seed=0, steps=2)


def test_trbdf2_step_cfg1(ref, gpu):
    """BASELINE configs[0]: 2D 32x32, Q2/Q1, nu = 1/100, dt = 1e-3, seed 0 (one full step)."""
    _step_case(ref, gpu, 2, 32, 2, 1, Re=100.0, dt=1e-3, seed=0, steps=1)


def test_trbdf2_cfg1_ten_steps(ref, gpu):
    """BASELINE configs[0] over 10 consecutive steps (second-order extrapolation from step 1
    on): per-solve iteration counts within +-1 and end-of-run fields <= 1e-9 (no drift)."""
    _step_case(ref, gpu, 2, 32, 2, 1, Re=100.0, dt=1e-3, seed=0, steps=10)


def test_trbdf2_q3q2_3d_two_steps(ref, gpu):
    """cfg3's degrees (Q3/Q2), Re 1000, GMRES restart 30, on a 4^3 mesh: the axis-aligned
    fast kernels inside two full device steps vs the restated reference driver."""
    _step_case(ref, gpu, 3, 4, 3, 2, Re=1000.0, dt=1e-3, seed=2, steps=2, restart=30)


def test_trbdf2_deformed_q4q3_step(ref, gpu):
    """cfg4's degrees (Q4/Q3) on a distorted 3^3 mesh: the deformed fast kernels
    (k_momentum_qp / k_sip_qp) inside two full device steps vs the restated driver."""
    _step_case(ref, gpu, 3, 3, 4, 3, Re=100.0, dt=1e-3, seed=3, steps=2, amp=0.03)


@pytest.mark.parametrize("dim,n_el,ku,kp,amp", [(2, 8, 2, 1, 0.0), (3, 3, 3, 2, 0.0), (3, 3, 2, 1, 0.04)])
def test_trbdf2_steps_with_outlet(ref, gpu, dim, n_el, ku, kp, amp):
    """Two steps with an outlet on boundary id 1 (no Dirichlet data there: natural
    viscous terms, w.n advective flux, pressure boundary flux dropped) vs the restated
    driver; fast axis-aligned, deformed and 2D paths."""
    _step_case(ref, gpu, dim, n_el, ku, kp, Re=100.0, dt=1e-3, seed=1, steps=2, amp=amp, outlet=1)


def test_trbdf2_step_3d_small(ref, gpu):
    _step_case(ref, gpu, 3, 3, 2, 1, Re=100.0, dt=1e-3, seed=1, steps=1)


@pytest.mark.parametrize("dim,n_el,ku,kp,amp,steps", [(2, 8, 2, 1, 0.0, 2), (3, 3, 2, 1, 0.0, 1),
                                                      (3, 3, 3, 2, 0.03, 1)])
def test_trbdf2_fixed_point_step(ref, gpu, dim, n_el, ku, kp, amp, steps):
    """trbdf2_step_fixedpoint (decision FP1): device vs the restated
    oracle, fixed-point re-solve counts within +-1, fields <= 1e-9."""
    its = _step_case(ref, gpu, dim, n_el, ku, kp, Re=100.0, dt=1e-3, seed=1, steps=steps, fixed_point=True,
                     amp=amp)
    assert its[8] >= 1 and its[9] >= 1


# ---------------------------------------------------------------- graded axis-aligned meshes
def graded_box(n):
    """3D box with graded (non-uniform) tensor-product spacing: axis-aligned cells of
    different sizes, so the fast kernels take their mesh-table path (no uniform grid).
    Returns the reference mesh text (mesh.cpp:793-817 format) and the C-ABI arrays."""
    t = np.linspace(0.0, 1.0, n + 1)
    axes = [t ** 1.4, 0.5 * (t + t ** 2), np.sin(0.5 * np.pi * t)]
    nv1 = n + 1
    verts = np.array([[axes[0][i], axes[1][j], axes[2][k]] for k in range(nv1) for j in range(nv1)
                      for i in range(nv1)])
    cells, bids = [], []
    for k in range(n):
        for j in range(n):
            for i in range(n):
                cells.append([(i + dx) + nv1 * (j + dy) + nv1 * nv1 * (k + dz)
                              for dz in (0, 1) for dy in (0, 1) for dx in (0, 1)])
                co = (i, j, k)
                bids.append([2 * a + s if co[a] == (0 if s == 0 else n - 1) else -1
                             for a in range(3) for s in (0, 1)])
    lines = [f"3 {len(verts)} {len(cells)}"]
    lines += [" ".join(repr(float(v)) for v in p) for p in verts]
    lines += [" ".join(str(v) for v in c) for c in cells]
    lines += [f"{c} {f} {b}" for c, row in enumerate(bids) for f, b in enumerate(row) if b >= 0]
    return "\n".join(lines) + "\n", (verts, np.array(cells, dtype=np.int32), np.array(bids, dtype=np.int32))


def graded_pair(ref, gpu, n, ku, kp, outlet=None, dirichlet_seed=None):
    _, arrays = graded_box(n)
    verts, cells, bids = arrays
    verts = np.ascontiguousarray(verts, dtype=np.float64)
    h = ref.lib().ref_create_from_arrays(3, len(verts), ref.P(verts), len(cells), cells.ctypes.data_as(ref._ip),
                                         bids.ctypes.data_as(ref._ip), ku, kp)
    assert h, ref.lib().ref_last_error().decode()
    R = ref.RefCtx(handle=h)
    D = gpu.DGContext(3, n, ku, kp, mesh_arrays=arrays)
    assert (R.n_u, R.n_p, R.ncells) == (D.n_u, D.n_p, D.ncells)
    if outlet is not None:
        R.set_bc(outlet, 1)
        D.set_boundary_type(outlet, gpu.BC_OUTLET)
    if dirichlet_seed is not None:
        f = gpu.SynthField(3, dirichlet_seed)
        for bid in range(6):
            if bid == outlet:
                continue
            R.set_bc(bid, 0, f.fn_ptr, f.user_ptr)
            D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
        R._keep.append(f)
        D._keep.append(f)
    return R, D


@pytest.mark.parametrize("n,ku,kp", [(3, 2, 1), (3, 3, 2), (2, 4, 3)])
@pytest.mark.parametrize("outlet", [None, 1])
def test_graded_axis_mesh_operators(ref, gpu, n, ku, kp, outlet):
    """Non-uniform axis-aligned cells: fast kernels with mesh tables (no uniform-grid
    shortcut) against the reference on the same imported mesh."""
    R, D = graded_pair(ref, gpu, n, ku, kp, outlet=outlet, dirichlet_seed=9)
    assert D.fast_path_active
    w = gpu.seeded_uniform(91, R.n_u)
    x = gpu.seeded_uniform(92, R.n_u)
    xp = gpu.seeded_uniform(93, R.n_p)
    for coefs in ((1.0 / (0.2929 * 1e-3), 1.0 / 2000.0, 0.5, 0.0), (0.3, 2.0, 1.5, 0.0)):
        y = D.zeros()
        gpu.apply_momentum(D, gpu.MomentumCtx(*coefs, advecting=dev(w)), dev(x), y)
        assert rel(host(y), R.momentum(coefs, w, x)) <= TOL_APPLY
        dg_ = D.zeros()
        gpu.momentum_diagonal(D, gpu.MomentumCtx(*coefs, advecting=dev(w)), dg_)
        assert rel(host(dg_), R.momentum_diag(coefs, w)) <= TOL_APPLY
    for mc in (2.3, 0.0):
        yp = D.zeros(gpu.SPACE_P)
        gpu.apply_pressure_helmholtz(D, mc, dev(xp), yp)
        assert rel(host(yp), R.pressure(mc, xp)) <= TOL_APPLY
        dp = D.zeros(gpu.SPACE_P)
        gpu.helmholtz_diagonal(D, mc, dp)
        assert rel(host(dp), R.helmholtz_diag(mc)) <= TOL_APPLY
    b = D.zeros(gpu.SPACE_P)
    gpu.divergence_functional(D, dev(x), b)
    assert rel(host(b), R.divergence(x)) <= TOL_APPLY
    ug = gpu.seeded_uniform(94, R.n_u)
    want = R.momentum_rhs(mass=[(2.9, x)], visc=[(0.65, x), (0.3, ug)], adv=[(0.5, x, w), (0.25, ug, ug)],
                          pres=[(1.0, xp), (-0.4, xp)], dir_visc=0.65, dir_adv=0.5, dir_w=w, time=0.0)
    spec = gpu.MomentumRhs(mass=[(2.9, dev(x))], visc=[(0.65, dev(x)), (0.3, dev(ug))],
                           adv=[(0.5, dev(x), dev(w)), (0.25, dev(ug), dev(ug))],
                           pres=[(1.0, dev(xp)), (-0.4, dev(xp))], dir_visc_coef=0.65, dir_adv_coef=0.5,
                           dir_w=dev(w))
    y = D.zeros()
    gpu.momentum_rhs(D, spec, y)
    assert rel(host(y), want) <= TOL_APPLY


@pytest.mark.parametrize("n_el,ku,kp", [(3, 2, 1), (2, 3, 2), (2, 4, 3)])
@pytest.mark.parametrize("outlet", [None, 1])
def test_fast_rhs_matches_reference_and_generic(ref, gpu, n_el, ku, kp, outlet):
    """Stage right-hand side through the fast launches (uniform grid) vs the reference
    and the generic device kernel; also single-term lists (pressure only, mass only)."""
    R, D = pair(ref, gpu, 3, n_el, ku, kp, 0.0, outlet=outlet, dirichlet_seed=4)
    assert D.fast_path_active
    un = gpu.seeded_uniform(61, R.n_u)
    ug = gpu.seeded_uniform(62, R.n_u)
    wv = gpu.seeded_uniform(63, R.n_u)
    pp = gpu.seeded_uniform(64, R.n_p)
    cases = [
        (dict(mass=[(2.9, un)], visc=[(0.3, ug), (0.65, un)], adv=[(0.25, ug, ug), (0.5, un, un)],
              pres=[(1.0, pp)], dir_visc=0.65, dir_adv=0.5, dir_w=wv), True),
        (dict(pres=[(1.3, pp)]), False),
        (dict(mass=[(0.7, ug)]), False),
        (dict(adv=[(0.5, un, wv)], dir_adv=0.5, dir_w=wv), True),
    ]
    for kw, has_dir in cases:
        want = R.momentum_rhs(time=0.0, **kw)
        tr = lambda lst: [tuple(dev(v) if isinstance(v, np.ndarray) else v for v in t) for t in lst]
        spec = gpu.MomentumRhs(mass=tr(kw.get("mass", [])), visc=tr(kw.get("visc", [])),
                               adv=tr(kw.get("adv", [])), pres=tr(kw.get("pres", [])),
                               dir_visc_coef=kw.get("dir_visc", 0.0), dir_adv_coef=kw.get("dir_adv", 0.0),
                               dir_w=dev(kw["dir_w"]) if "dir_w" in kw else None)
        outs = []
        for fast in (True, False):
            D.set_fast_path(fast)
            y = D.zeros()
            gpu.momentum_rhs(D, spec, y)
            outs.append(host(y))
            assert rel(outs[-1], want) <= TOL_APPLY, (kw.keys(), fast)
        D.set_fast_path(True)


@pytest.mark.parametrize("n_el,ku,kp,graded", [(5, 3, 2, False), (7, 2, 1, False), (3, 3, 2, True)])
def test_host_buffer_applies_match_device_applies(ref, gpu, n_el, ku, kp, graded):
    """dgb_*_apply_host (z-slab pipelined copies on uniform grids, copy/apply/copy
    otherwise) give bit-identical results to the device-buffer applies and match the
    reference."""
    import torch
    if graded:
        R, D = graded_pair(ref, gpu, n_el, ku, kp)
    else:
        R, D = pair(ref, gpu, 3, n_el, ku, kp, 0.0)
    w = gpu.seeded_uniform(71, R.n_u)
    x = gpu.seeded_uniform(72, R.n_u)
    xp = gpu.seeded_uniform(73, R.n_p)
    coefs = (1.0 / (0.2929 * 1e-3), 1.0 / 2000.0, 0.5, 0.0)
    y_dev = D.zeros()
    gpu.apply_momentum(D, gpu.MomentumCtx(*coefs, advecting=dev(w)), dev(x), y_dev)
    wh, xh = torch.from_numpy(w).pin_memory(), torch.from_numpy(x).pin_memory()
    yh = torch.zeros(R.n_u, dtype=torch.float64).pin_memory()
    gpu.apply_momentum_host(D, coefs, wh, xh, yh)
    assert np.array_equal(yh.numpy(), host(y_dev))
    assert rel(yh.numpy(), R.momentum(coefs, w, x)) <= TOL_APPLY
    yp_dev = D.zeros(gpu.SPACE_P)
    gpu.apply_pressure_helmholtz(D, 2.3, dev(xp), yp_dev)
    yph = np.zeros(R.n_p)
    gpu.apply_pressure_helmholtz_host(D, 2.3, np.ascontiguousarray(xp), yph)  # pageable numpy buffers
    assert np.array_equal(yph, host(yp_dev))
    assert rel(yph, R.pressure(2.3, xp)) <= TOL_APPLY


@pytest.mark.parametrize("n_el,ku,kp,amp", [(3, 1, 1, 0.05), (3, 2, 1, 0.05), (2, 3, 2, 0.04), (2, 4, 3, 0.03)])
def test_deformed_mass_kernel_matches_reference_and_generic(ref, gpu, n_el, ku, kp, amp):
    """fast_deformed.cuh k_mass_qp (sum-factorised B^T detJw B from the compact per-qp
    records) vs the reference apply_mass and the generic device kernel, velocity (rule
    ku+1, 3 components) and pressure (rule kp+2) spaces on distorted 3D meshes."""
    R, D = pair(ref, gpu, 3, n_el, ku, kp, amp)
    assert not D.affine
    for space, n in ((gpu.SPACE_U, R.n_u), (gpu.SPACE_P, R.n_p)):
        x = gpu.seeded_uniform(77 + space, n)
        want = R.mass(space, x)
        outs = []
        for fast in (True, False):
            D.set_fast_path(fast)
            y = D.zeros(space)
            gpu.apply_mass(D, space, dev(x), y)
            outs.append(host(y))
            assert rel(outs[-1], want) <= TOL_APPLY, (space, fast)
        assert rel(outs[0], outs[1]) <= 1e-14
    for fast in (True, False):  # velocity mass diagonal: k_momentum_diag_qp with mass only
        D.set_fast_path(fast)
        d = D.zeros()
        gpu.mass_diagonal(D, gpu.SPACE_U, d)
        assert rel(host(d), R.mass_diag(gpu.SPACE_U)) <= TOL_APPLY, ("mass diag", fast)
    D.set_fast_path(True)


@pytest.mark.parametrize("n_el,kp,amp", [(3, 1, 0.05), (2, 2, 0.04), (2, 3, 0.03)])
def test_deformed_sip_kernel_matches_reference_and_generic(ref, gpu, n_el, kp, amp):
    """fast_deformed.cuh k_sip_qp (per-qp geometry streamed) vs the reference and the
    generic device kernel on distorted 3D meshes: pressure Helmholtz and the Dirichlet /
    natural scalar Laplacian."""
    R, D = pair(ref, gpu, 3, n_el, kp + 1, kp, amp)
    assert not D.affine
    xp = gpu.seeded_uniform(95, R.n_p)
    for mc in (2.3, 0.0):
        want = R.pressure(mc, xp)
        for fast in (True, False):
            D.set_fast_path(fast)
            yp = D.zeros(gpu.SPACE_P)
            gpu.apply_pressure_helmholtz(D, mc, dev(xp), yp)
            assert rel(host(yp), want) <= TOL_APPLY, (mc, fast)
    for dirichlet in (True, False):
        want = R.laplace(dirichlet, xp)
        for fast in (True, False):
            D.set_fast_path(fast)
            yl = D.zeros(gpu.SPACE_P)
            gpu.apply_scalar_laplace(D, dirichlet, dev(xp), yl)
            assert rel(host(yl), want) <= TOL_APPLY, (dirichlet, fast)
    # diagonals: k_momentum_diag_qp<kp, SCALAR> vs reference and generic
    for fast in (True, False):
        D.set_fast_path(fast)
        d = D.zeros(gpu.SPACE_P)
        gpu.helmholtz_diagonal(D, 2.3, d)
        assert rel(host(d), R.helmholtz_diag(2.3)) <= TOL_APPLY, ("helmholtz diag", fast)
        for dirichlet in (True, False):
            gpu.scalar_laplace_diagonal(D, dirichlet, d)
            assert rel(host(d), R.laplace_diag(dirichlet)) <= TOL_APPLY, ("laplace diag", dirichlet, fast)
    D.set_fast_path(True)


@pytest.mark.parametrize("n_el,ku,amp,outlet", [(3, 2, 0.05, None), (2, 3, 0.04, 1), (2, 4, 0.03, None),
                                               (2, 4, 0.03, 4), (3, 1, 0.05, None)])
@pytest.mark.parametrize("coefs", [(1.0 / (0.2929 * 1e-3), 0.005, 0.5, 0.0), (3.7, 1.3, 0.9, 0.0),
                                   (2.1, 0.0, 0.7, 0.0), (0.0, 0.0, 1.1, 0.0), (1.9, 0.6, 0.0, 0.0)])
def test_deformed_momentum_kernel_matches_reference_and_generic(ref, gpu, n_el, ku, amp, outlet, coefs):
    """fast_deformed.cuh k_momentum_qp (pass A through the per-field SIP body at rule k+1,
    Lax-Friedrichs advection at rule k+2 with per-qp geometry) and k_momentum_diag_qp vs
    the reference and the generic device kernels on distorted 3D meshes, with walls / an
    outlet and every combination of mass / viscous / advective coefficients."""
    R, D = pair(ref, gpu, 3, n_el, ku, ku - 1 if ku > 1 else 1, amp, outlet=outlet)
    assert not D.affine
    w = gpu.seeded_uniform(41, R.n_u)
    x = gpu.seeded_uniform(42, R.n_u)
    want = R.momentum(coefs, w, x)
    want_d = R.momentum_diag(coefs, w)
    ctx = gpu.MomentumCtx(*coefs, advecting=dev(w))
    for fast in (True, False):
        D.set_fast_path(fast)
        y = D.zeros()
        gpu.apply_momentum(D, ctx, dev(x), y)
        assert rel(host(y), want) <= TOL_APPLY, fast
        d = D.zeros()
        gpu.momentum_diagonal(D, ctx, d)  # k_momentum_diag_qp (fast) / k_momentum_diag
        assert rel(host(d), want_d) <= TOL_APPLY, ("diag", fast)
    D.set_fast_path(True)


@pytest.mark.parametrize("scheme_name", ["BCG", "GQ_BDF2"])
@pytest.mark.parametrize("dim,n_el,ku,kp,amp,steps", [(2, 8, 2, 1, 0.0, 3), (3, 3, 2, 1, 0.0, 2),
                                                      (3, 2, 3, 2, 0.03, 2)])
def test_baseline_schemes_match_oracle(ref, gpu, scheme_name, dim, n_el, ku, kp, amp, steps):
    """The paper's comparison schemes (decisions in DESIGN.md): device
    dgb_projection_step vs the restated oracle (oracle/trbdf2_cpu.hpp bcg_step /
    gq_bdf2_step) over several steps (GQ-BDF2 starts with a BCG step)."""
    scheme = getattr(gpu, "SCHEME_" + scheme_name)
    R, D = pair(ref, gpu, dim, n_el, ku, kp, amp, dirichlet_seed=1)
    f = gpu.SynthField(dim, 1)
    u0 = f.interpolate(D)
    p0 = np.zeros(R.n_p)
    u_prev, u, p = u0.copy(), u0.copy(), p0.copy()
    du_prev, du, dp = dev(u0), dev(u0), dev(p0)
    dt, Re = 1e-3, 100.0
    for n in range(steps):
        params = [dt, Re, 1e3, n * dt, 50, 1e-10, 1e-10, 1e-12, 10000, 1.0 if n == 0 else 0.0, 0.0, 1e-8, 100]
        u1, p1, its_ref = R.scheme_step(scheme, params, u_prev, u, p)
        P = gpu.StepParams(dt=dt, Re=Re, c=1e3, time=n * dt, restart=50, first_step=(n == 0))
        du1, dp1 = D.zeros(), D.zeros(gpu.SPACE_P)
        its = gpu.projection_step(D, scheme, P, du_prev, du, dp, du1, dp1)
        for i, (a, b) in enumerate(zip(its, its_ref)):
            slack = 1 + (its_ref[8] if i == 0 else 0)
            assert abs(a - b) <= slack, (n, its, its_ref)
        u_prev, u, p = u, u1, p1
        du_prev, du, dp = du, du1, dp1
    hu, hp = host(du), host(dp)
    assert rel(hu, u) <= TOL_FIELD
    assert rel(hp - hp.mean(), p - p.mean()) <= TOL_FIELD or rel(hp, p) <= TOL_FIELD


def test_diagnostics(ref, gpu):
    """On-device diagnostics: L2 norms against the reference's kinetic
    energy (forms.cpp:1239-1260) and its mass apply, check_steady, stability parameters
    (cfg5's dt gives C = 0.5 by construction)."""
    R, D = pair(ref, gpu, 3, 3, 2, 1, 0.0)  # Cartesian: the mass and kinetic-energy rules are both exact
    u = gpu.seeded_uniform(61, R.n_u)
    p = gpu.seeded_uniform(62, R.n_p)
    nu = gpu.l2_norm(D, dev(u))
    assert abs(nu * nu - 2.0 * R.kinetic_energy(u)) <= 1e-12 * nu * nu
    mp = R.mass(gpu.SPACE_P, p)
    npn = gpu.l2_norm(D, dev(p), gpu.SPACE_P)
    assert abs(npn * npn - float(p @ mp)) <= 1e-12 * npn * npn
    du, du2 = dev(u), dev(u)
    du2[5] += 1e-6
    assert gpu.check_steady(D, du, du, 1e-7) == (True, 0.0)
    steady, d = gpu.check_steady(D, du2, du, 1e-7)
    assert not steady and abs(d - 1e-6) < 1e-12
    D5 = gpu.DGContext(3, 8, 2, 1)
    c, mu = gpu.stability_params(D5, 0.5 * (3 ** 0.5 / 8) / 2.0, 1600.0, 1.0)
    assert abs(c - 0.5) < 1e-12
    H = 3 ** 0.5 / 8
    assert abs(mu - 4 * (0.5 * H / 2.0) / (1600.0 * H * H)) < 1e-12


@pytest.mark.parametrize("n_el,kp", [(4, 1), (3, 2), (3, 3), (32, 1)])
def test_2d_axis_sip_kernel_matches_reference_and_generic(ref, gpu, n_el, kp):
    """fast_axis.cuh k_sip_axis2 (2D line split, one thread per cell) vs the reference and
    the generic device kernel: pressure Helmholtz and the Dirichlet / natural Laplacian."""
    R, D = pair(ref, gpu, 2, n_el, kp + 1, kp, 0.0)
    xp = gpu.seeded_uniform(97, R.n_p)
    for mc in (2.3, 0.0):
        want = R.pressure(mc, xp)
        for fast in (True, False):
            D.set_fast_path(fast)
            yp = D.zeros(gpu.SPACE_P)
            gpu.apply_pressure_helmholtz(D, mc, dev(xp), yp)
            assert rel(host(yp), want) <= TOL_APPLY, (mc, fast)
    for dirichlet in (True, False):
        want = R.laplace(dirichlet, xp)
        for fast in (True, False):
            D.set_fast_path(fast)
            yl = D.zeros(gpu.SPACE_P)
            gpu.apply_scalar_laplace(D, dirichlet, dev(xp), yl)
            assert rel(host(yl), want) <= TOL_APPLY, (dirichlet, fast)
    D.set_fast_path(True)


@pytest.mark.parametrize("n_el,ku,amp,outlet", [(2, 2, 0.03, None), (2, 3, 0.03, 1), (2, 4, 0.02, None),
                                               (3, 2, 0.05, 4)])
def test_deformed_rhs_matches_reference_and_generic(ref, gpu, n_el, ku, amp, outlet):
    """Stage RHS on distorted 3D meshes through RHS-mode k_momentum_qp launches (mass,
    consistency-only viscous, central advective terms), k_pgrad_qp (weak pressure gradient)
    and the generic boundary-data terms, vs the reference and the all-generic path; walls,
    an outlet, Dirichlet data."""
    R, D = pair(ref, gpu, 3, n_el, ku, ku - 1, amp, outlet=outlet, dirichlet_seed=5)
    un = gpu.seeded_uniform(61, R.n_u)
    ug = gpu.seeded_uniform(62, R.n_u)
    wx = gpu.seeded_uniform(63, R.n_u)
    pp = gpu.seeded_uniform(64, R.n_p)
    want = R.momentum_rhs(mass=[(2.9, un), (-0.7, ug)], visc=[(0.65, un), (0.3, ug)],
                          adv=[(0.5, un, wx), (0.25, ug, ug)], pres=[(1.0, pp)], dir_visc=0.65, dir_adv=0.5,
                          dir_w=wx, time=0.0)
    dun, dug, dwx, dpp = dev(un), dev(ug), dev(wx), dev(pp)
    spec = gpu.MomentumRhs(mass=[(2.9, dun), (-0.7, dug)], visc=[(0.65, dun), (0.3, dug)],
                           adv=[(0.5, dun, dwx), (0.25, dug, dug)], pres=[(1.0, dpp)], dir_visc_coef=0.65,
                           dir_adv_coef=0.5, dir_w=dwx)
    for fast in (True, False):
        D.set_fast_path(fast)
        y = D.zeros()
        gpu.momentum_rhs(D, spec, y)
        assert rel(host(y), want) <= TOL_APPLY, fast
    D.set_fast_path(True)


@pytest.mark.parametrize("n_el,ku,amp,outlet", [(2, 2, 0.03, None), (3, 2, 0.05, 4), (2, 3, 0.03, 1),
                                               (3, 3, 0.04, None), (2, 4, 0.02, 0), (3, 4, 0.03, None)])
def test_deformed_mixed_forms_match_reference_and_generic(ref, gpu, n_el, ku, amp, outlet):
    """The mixed velocity-pressure forms on distorted 3D meshes (k_div_qp, k_pgrad_qp):
    divergence_functional (forms.cpp:1118-1197), pressure_rhs (:1199-1210) and the pressure
    terms of momentum_rhs alone (:850-855, :895-912, :940-948; two pressure fields with
    different coefficients), vs the reference and the generic kernels; walls and an outlet."""
    R, D = pair(ref, gpu, 3, n_el, ku, ku - 1, amp, outlet=outlet)
    assert D.fast_path_active
    u = gpu.seeded_uniform(71, R.n_u)
    p1 = gpu.seeded_uniform(72, R.n_p)
    p2 = gpu.seeded_uniform(73, R.n_p)
    want_div = R.divergence(u)
    want_prhs = R.pressure_rhs(1.7, u, 7.3, p1)
    want_grad = R.momentum_rhs(pres=[(1.0, p1), (-0.35, p2)], time=0.0)
    du, dp1, dp2 = dev(u), dev(p1), dev(p2)
    for fast in (True, False):
        D.set_fast_path(fast)
        b = D.zeros(gpu.SPACE_P)
        gpu.divergence_functional(D, du, b)
        assert rel(host(b), want_div) <= TOL_APPLY, fast
        pr = D.zeros(gpu.SPACE_P)
        gpu.pressure_rhs(D, 1.7, du, 7.3, dp1, pr)
        assert rel(host(pr), want_prhs) <= TOL_APPLY, fast
        y = D.zeros()
        gpu.momentum_rhs(D, gpu.MomentumRhs(pres=[(1.0, dp1), (-0.35, dp2)]), y)
        assert rel(host(y), want_grad) <= TOL_APPLY, fast
    D.set_fast_path(True)
