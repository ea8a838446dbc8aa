"""Pressure multigrid preconditioner (mg.cu, not in the reference):
the MG-preconditioned CG solves the same pressure system as the reference's Jacobi-CG
(whose iteration counts are pinned in test_gpu_parity.py) to the solver tolerance, in far
fewer iterations; the V-cycle is symmetric positive definite; a TR-BDF2 step with it
matches the Jacobi step to the solve tolerances."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()


def _rel(a, b):
    return float((a - b).norm() / b.norm())


@pytest.mark.parametrize("n_el,kp", [(8, 1), (8, 2), (6, 3), (12, 2), (6, 1)])
def test_mg_cg_matches_jacobi_cg(gpu, n_el, kp):
    D = gpu.DGContext(3, n_el, kp + 1, kp)
    mc = 2.9
    b = _dev(gpu.seeded_uniform(300 + n_el, D.n_p))
    s = gpu.SolverSettings(rel_tol=1e-11, max_iter=20000)
    A = gpu.LinearOperator.pressure_helmholtz(mc)
    d = D.zeros(gpu.SPACE_P)
    gpu.helmholtz_diagonal(D, mc, d)
    xj = D.zeros(gpu.SPACE_P)
    rj = gpu.cg_solve(D, A, b, s, gpu.JacobiPreconditioner(D, d), xj)
    xm = D.zeros(gpu.SPACE_P)
    rm = gpu.pressure_cg_mg(D, mc, b, s, xm)
    assert _rel(xm, xj) <= 1e-8, (rm, rj)
    assert rm.iterations * 3 <= rj.iterations, (rm.iterations, rj.iterations)
    # the residual it reports is the true one
    y = D.zeros(gpu.SPACE_P)
    gpu.apply_pressure_helmholtz(D, mc, xm, y)
    assert float((y - b).norm() / b.norm()) <= 1e-11


def test_mg_vcycle_is_spd(gpu):
    D = gpu.DGContext(3, 8, 3, 2)
    mc = 0.7
    x = _dev(gpu.seeded_uniform(1, D.n_p))
    y = _dev(gpu.seeded_uniform(2, D.n_p))
    bx, by = D.zeros(gpu.SPACE_P), D.zeros(gpu.SPACE_P)
    gpu.pressure_mg_vcycle(D, mc, x, bx)
    gpu.pressure_mg_vcycle(D, mc, y, by)
    a, c = float((by * x).sum()), float((bx * y).sum())
    assert abs(a - c) <= 1e-11 * abs(a)
    assert float((bx * x).sum()) > 0.0 and float((by * y).sum()) > 0.0
    # linear: B(2x + y) = 2 Bx + By
    bz = D.zeros(gpu.SPACE_P)
    gpu.pressure_mg_vcycle(D, mc, 2 * x + y, bz)
    assert _rel(bz, 2 * bx + by) <= 1e-12


@pytest.mark.parametrize("n_el,kp,amp", [(8, 1, 0.1 / 8), (6, 2, 0.1 / 6), (8, 3, 0.1 / 8)])
def test_mg_cg_on_deformed_mesh(gpu, n_el, kp, amp):
    """cfg4-type meshes (interior vertices moved by up to 0.1 h): the Q1 levels approximate
    the deformed operator by the undeformed grid's; still the same solution, far fewer
    iterations."""
    D = gpu.DGContext(3, n_el, kp + 1, kp, amp, 3)
    assert not D.affine
    mc = 2.9
    b = _dev(gpu.seeded_uniform(400 + n_el, D.n_p))
    s = gpu.SolverSettings(rel_tol=1e-11, max_iter=20000)
    d = D.zeros(gpu.SPACE_P)
    gpu.helmholtz_diagonal(D, mc, d)
    xj = D.zeros(gpu.SPACE_P)
    rj = gpu.cg_solve(D, gpu.LinearOperator.pressure_helmholtz(mc), b, s, gpu.JacobiPreconditioner(D, d), xj)
    xm = D.zeros(gpu.SPACE_P)
    rm = gpu.pressure_cg_mg(D, mc, b, s, xm)
    assert _rel(xm, xj) <= 1e-8, (rm, rj)
    assert rm.iterations * 3 <= rj.iterations, (rm.iterations, rj.iterations)


def test_mg_unsupported_mesh_fails_loudly(gpu):
    D = gpu.DGContext(2, 8, 2, 1)  # 2D: no hierarchy
    b = _dev(gpu.seeded_uniform(3, D.n_p))
    with pytest.raises(Exception):
        gpu.pressure_cg_mg(D, 1.0, b, gpu.SolverSettings(), D.zeros(gpu.SPACE_P))


def test_trbdf2_step_with_mg_matches_jacobi(gpu):
    D = gpu.DGContext(3, 8, 2, 1)
    f = gpu.SynthField(3, 1)
    for bid in range(6):
        D.set_dirichlet_fn(bid, f.fn_ptr, f.user_ptr, 0.0)
    u0 = D.zeros()
    gpu.interpolate_synth_device(D, f, u0)
    p0 = D.zeros(gpu.SPACE_P)
    out = {}
    for pc in ("jacobi", "mg"):
        u1, p1 = D.zeros(), D.zeros(gpu.SPACE_P)
        sp = gpu.StepParams(dt=1e-3, Re=100.0, c=1e3, first_step=True, pressure_precond=pc)
        its = gpu.trbdf2_step(D, sp, u0, u0, p0, u1, p1)
        out[pc] = (u1, p1 - p1.mean(), its)
    uj, pj, ij = out["jacobi"]
    um, pm, im = out["mg"]
    assert _rel(um, uj) <= 1e-9
    assert _rel(pm, pj) <= 1e-7
    assert im[2] * 3 <= ij[2] and im[3] * 3 <= ij[3], (im, ij)
    assert abs(im[0] - ij[0]) <= 1 and abs(im[1] - ij[1]) <= 1
