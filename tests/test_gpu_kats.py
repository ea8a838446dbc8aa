"""The reference's own known-answer tests, run against the device path.

* BLAS-1 (test_kernels.cpp:31-84 "scalar kernels match naive loops exactly"): the
  device kernels against the reference's kern:: kernels (AVX2 backend) on the same
  odd-sized vectors -- axpy / axpby / scal / max_abs_diff bit-exact, dot / norm within
  the reassociation bound of a sum of n products.
* Free stream (test_forms.cpp:365-433): a uniform velocity is annihilated by the
  stage-1 operator minus the stage-1 RHS (<= 1e-12 on a Cartesian mesh, <= 1e-9 on a
  distorted one), and its projection right-hand side vanishes.  Same meshes, same
  coefficients, extended to the 3D fast kernels.
* The multigrid-preconditioned pressure CG against the reference's cg_solve
  (krylov.cpp:43-101, Jacobi) on the same system.
"""
import ctypes as C

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def host(t):
    import torch
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("n", [257, 4096 + 3, (1 << 22) + 1])
def test_blas1_match_reference_kernels(ref, gpu, n):
    D = gpu.DGContext(3, 1, 1, 1)
    x, y = ref.seeded_uniform(1, n), ref.seeded_uniform(2, n)
    dx, dy = dev(x), dev(y)
    gpu.axpy(D, 0.37, dx, dy)
    assert np.array_equal(host(dy), ref.kern("axpy", 0.37, x, y))
    dy = dev(y)
    gpu.axpby(D, 0.37, dx, -1.25, dy)
    assert np.array_equal(host(dy), ref.kern("axpby", 0.37, x, y, -1.25))
    dx2 = dev(x)
    gpu.scal(D, -3.5, dx2)
    assert np.array_equal(host(dx2), ref.kern("scal", -3.5, x, None))
    assert gpu.max_abs_diff(D, dx, dev(y)) == ref.kern("max_abs_diff", 0.0, x, y)
    # dot: any summation order is within n * eps * sum |x_i y_i| of the exact sum
    import math
    exact = math.fsum((x * y).tolist())
    bound = n * np.finfo(float).eps * float(np.abs(x * y).sum())
    assert abs(gpu.dot(D, dx, dev(y)) - exact) <= bound
    assert abs(ref.kern("dot", 0.0, x, y) - exact) <= bound
    nrm = math.sqrt(math.fsum((x * x).tolist()))
    assert abs(gpu.norm(D, dx) - nrm) <= n * np.finfo(float).eps * nrm


# ---------------------------------------------------------------------------- free stream
U0 = {2: (1.7, -0.6), 3: (1.7, -0.6, 0.45)}
_BC = C.CFUNCTYPE(None, C.POINTER(C.c_double), C.c_double, C.POINTER(C.c_double), C.c_void_p)


def _const_fn(dim):
    u0 = U0[dim]

    def f(x, t, out, user):
        for d in range(dim):
            out[d] = u0[d]
    return _BC(f)


def _box_arrays(dim, n, hi):
    """generate_cartesian<dim>(n, 0, hi) (mesh.cpp:572-615) as C-ABI arrays."""
    nv1 = n + 1
    idx = np.indices((nv1,) * dim).reshape(dim, -1)[::-1].T  # x fastest
    verts = np.array([[hi[d] * i[d] / n for d in range(dim)] for i in idx], dtype=np.float64)
    cells, bids = [], []
    for c in np.indices((n,) * dim).reshape(dim, -1)[::-1].T:
        cells.append([sum((c[d] + ((b >> d) & 1)) * nv1 ** d for d in range(dim)) for b in range(1 << dim)])
        bids.append([2 * a + s if c[a] == (0 if s == 0 else n - 1) else -1 for a in range(dim) for s in (0, 1)])
    return verts, np.array(cells, dtype=np.int32), np.array(bids, dtype=np.int32)


def _free_stream_residuals(gpu, D):
    """test_forms.cpp:369-422 on the device: lhs = stage-1 operator applied to the
    uniform field, rhs = stage-1 RHS of the same field; returns (max|lhs - rhs|,
    max|pressure_rhs|)."""
    gamma, dt, nu = 2.0 - 2.0 ** 0.5, 0.2, 0.01
    dim = D.dim
    fn = _const_fn(dim)
    D._keep.append(fn)
    for bid in range(2 * dim):
        D.set_dirichlet_fn(bid, C.cast(fn, C.c_void_p), None, 0.0)
    nb = (D.ku + 1) ** dim
    uc = dev(np.tile(np.repeat(np.array(U0[dim]), nb), D.ncells))
    pz = D.zeros(gpu.SPACE_P)
    lhs, rhs = D.zeros(), D.zeros()
    gpu.apply_momentum(D, gpu.MomentumCtx(1.0 / (gamma * dt), 0.5 * nu, 0.5, 0.0, advecting=uc), uc, lhs)
    spec = gpu.MomentumRhs(mass=[(1.0 / (gamma * dt), uc)], visc=[(0.5 * nu, uc)], adv=[(0.5, uc, uc)],
                           pres=[(1.0, pz)], dir_visc_coef=0.5 * nu, dir_adv_coef=0.5, dir_w=uc)
    gpu.momentum_rhs(D, spec, rhs)
    prhs = D.zeros(gpu.SPACE_P)
    gpu.pressure_rhs(D, 1.0 / (gamma * dt), uc, 7.3, pz, prhs)
    return float(np.abs(host(lhs) - host(rhs)).max()), float(np.abs(host(prhs)).max())


@pytest.mark.parametrize("dim,n,ku,hi", [(2, 2, 2, (1.2, 0.8)), (3, 2, 2, (1.2, 0.8, 1.0)),
                                         (3, 3, 3, (1.0, 1.0, 1.0)), (3, 2, 4, (0.7, 1.1, 0.9))])
def test_free_stream_cartesian(gpu, dim, n, ku, hi):
    """test_forms.cpp:426-428: Cartesian mesh, exact cancellation (<= 1e-12); the 3D
    cases run the fast axis-aligned kernels."""
    D = gpu.DGContext(dim, n, ku, ku - 1, mesh_arrays=_box_arrays(dim, n, hi))
    r_mom, r_prs = _free_stream_residuals(gpu, D)
    assert r_mom <= 1e-12 and r_prs <= 1e-12, (r_mom, r_prs)


@pytest.mark.parametrize("dim,amp,ku", [(2, 0.05, 2), (3, 0.03, 2), (3, 0.03, 4)])
def test_free_stream_distorted(gpu, dim, amp, ku):
    """test_forms.cpp:429-432: small_distorted_mesh (generate_cartesian(2) + distort(amp,
    7)), quadrature-limited cancellation (<= 1e-9); 3D runs the deformed fast kernels."""
    D = gpu.DGContext(dim, 2, ku, ku - 1, amp, 7)
    r_mom, r_prs = _free_stream_residuals(gpu, D)
    assert r_mom <= 1e-9 and r_prs <= 1e-9, (r_mom, r_prs)


# ------------------------------------------------------------- multigrid CG vs reference CG
@pytest.mark.parametrize("n_el,kp,amp", [(8, 1, 0.0), (6, 2, 0.0), (6, 2, 0.02)])
def test_multigrid_cg_matches_reference_cg(ref, gpu, n_el, kp, amp):
    """the multigrid-preconditioned pressure CG solves the same system as
    the reference's Jacobi cg_solve (krylov.cpp:43-101) to the solver tolerance."""
    R = ref.RefCtx(3, n_el, kp + 1, kp, amp, 3)
    D = gpu.DGContext(3, n_el, kp + 1, kp, amp, 3)
    G = 2.0 - 2.0 ** 0.5
    mc = 1.0 / (1e6 * G * G * 1e-6)
    b = ref.seeded_uniform(77, R.n_p)
    x_ref, it_ref, _ = R.solve(1, 0, (mc, 0, 0, 0), None, b, np.zeros(R.n_p), rel_tol=1e-10)
    x = D.zeros(gpu.SPACE_P)
    res = gpu.pressure_cg_mg(D, mc, dev(b), gpu.SolverSettings(rel_tol=1e-10, max_iter=10000), x)
    e = np.linalg.norm(host(x) - x_ref) / np.linalg.norm(x_ref)
    assert e <= 1e-7, (e, res, it_ref)
    assert res.iterations < it_ref


# ------------------------------------------------------------- time-dependent Dirichlet data
@pytest.mark.parametrize("dim,n_el,ku,amp", [(2, 4, 2, 0.0), (3, 2, 2, 0.03), (3, 3, 3, 0.0)])
def test_trbdf2_step_time_dependent_dirichlet(ref, gpu, dim, n_el, ku, amp):
    """Dirichlet data g(x, t) that changes in time: the reference evaluates it at each
    stage time t* (MomentumRhs::time, forms.cpp:1061-1062; Appendix A stage 1 t^n + gamma
    dt, stage 2 t^n + dt).  With set_dirichlet_time_dependent the device step does the
    same: iteration counts +-1, fields <= 1e-9 against the restated reference driver."""
    import math

    def g(x, t, out, user):
        for d in range(dim):
            out[d] = math.sin(1.3 * x[(d + 1) % dim] + 0.7 * d + 40.0 * t) * math.cos(0.9 * x[d])
    cb = _BC(g)
    R = ref.RefCtx(dim, n_el, ku, ku - 1, amp, 7)
    D = gpu.DGContext(dim, n_el, ku, ku - 1, amp, 7)
    D._keep.append(cb)
    R._keep.append(cb)
    for bid in range(2 * dim):
        R.set_bc(bid, 0, C.cast(cb, C.c_void_p), None)
        D.set_dirichlet_fn(bid, C.cast(cb, C.c_void_p), None, 0.0)
    D.set_dirichlet_time_dependent(True)
    u0 = ref.seeded_uniform(5, R.n_u)
    p0 = np.zeros(R.n_p)
    t0, dt = 0.1, 2e-3
    u1, p1, its_ref = R.step([dt, 100.0, 1e3, t0, 50, 1e-10, 1e-10, 1e-12, 10000, 0.0], u0, u0, p0)
    du1, dp1 = D.zeros(), D.zeros(gpu.SPACE_P)
    its = gpu.trbdf2_step(D, gpu.StepParams(dt=dt, Re=100.0, c=1e3, time=t0, restart=50, first_step=False),
                          dev(u0), dev(u0), dev(p0), du1, dp1)
    assert all(abs(a - b) <= 1 for a, b in zip(its[:8], its_ref[:8])), (its, its_ref)
    hu, hp = host(du1), host(dp1)
    assert np.linalg.norm(hu - u1) / np.linalg.norm(u1) <= 1e-9
    hp, p1 = hp - hp.mean(), p1 - p1.mean()
    assert np.linalg.norm(hp - p1) / np.linalg.norm(p1) <= 1e-9


# ------------------------------------------------------------- caller alignment
def test_gmres_accepts_a_misaligned_jacobi_inverse(gpu):
    """dgb_gmres reads the Jacobi inverse as double2 in its Gram-Schmidt update pass; a
    caller's view at an odd element offset is copied to an aligned slot first (dgb.h),
    so the solve is the same as with the aligned vector (no misaligned-address fault)."""
    import torch
    D = gpu.DGContext(3, 3, 2, 1)
    w = torch.from_numpy(gpu.seeded_uniform(1, D.n_u)).cuda()
    b = torch.from_numpy(gpu.seeded_uniform(2, D.n_u)).cuda()
    ctx = gpu.MomentumCtx(3.7, 0.01, 0.5, 0.0, advecting=w)
    d = D.zeros()
    gpu.momentum_diagonal(D, ctx, d)
    M = gpu.JacobiPreconditioner(D, d)
    s = gpu.SolverSettings(rel_tol=1e-10, restart=20)
    x1 = D.zeros()
    r1 = gpu.gmres_solve(D, gpu.LinearOperator.momentum(ctx), b, s, M, x1)
    buf = torch.zeros(D.n_u + 1, dtype=torch.float64, device="cuda")
    buf[1:] = M.inv
    M.inv = buf[1:]  # data_ptr 8 bytes past a 16-byte boundary
    assert M.inv.data_ptr() % 16 == 8
    x2 = D.zeros()
    r2 = gpu.gmres_solve(D, gpu.LinearOperator.momentum(ctx), b, s, M, x2)
    assert r1.iterations == r2.iterations and torch.equal(x1, x2)
