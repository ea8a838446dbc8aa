"""The numpy restatement (oracle/dg_numpy.py) against golden vectors produced by
the compiled reference (tests/golden/make_golden.py).  CPU only."""
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(os.path.dirname(HERE), "oracle"))
import dg_numpy as O  # noqa: E402

CASES = sorted(f[:-4] for f in os.listdir(os.path.join(HERE, "golden")) if f.endswith(".npz"))


@pytest.fixture(scope="module", params=CASES)
def case(request):
    g = dict(np.load(os.path.join(HERE, "golden", request.param + ".npz")))
    mesh = O.Mesh(g["verts"], g["cells"], g["bids"])
    F = O.Forms(mesh, int(g["ku"]), int(g["kp"]))
    if int(g["outlet"]) >= 0:
        F.bc_type[int(g["outlet"])] = "outlet"
    return g, F


def rel(a, b):
    return np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300)


def test_face_lists_match_reference(case):
    g, F = case
    it = np.array([[f.cell_in, f.face_in, f.cell_out, f.face_out] for f in F.mesh.interior])
    bd = np.array([[f.cell_in, f.face_in, f.boundary_id] for f in F.mesh.boundary])
    assert np.array_equal(it, g["interior"][:, :4])
    assert np.array_equal(bd, g["boundary"])


def test_operators_match_reference(case):
    g, F = case
    assert rel(F.apply_momentum(tuple(g["coefs"]), g["w"], g["x"]), g["momentum"]) <= 1e-12
    assert rel(F.apply_momentum(tuple(g["coefs_stage"]), g["w"], g["x"]), g["momentum_stage"]) <= 1e-12
    assert rel(F.apply_pressure_helmholtz(float(g["mc"]), g["xp"]), g["pressure"]) <= 1e-12
    assert rel(F.scalar_sip(F.Vp, 0.0, True, g["xp"]), g["laplace_dir"]) <= 1e-12
    assert rel(F.apply_mass(F.Vu, g["x"]), g["mass_u"]) <= 1e-12
    assert rel(F.apply_mass(F.Vp, g["xp"]), g["mass_p"]) <= 1e-12
    assert rel(F.divergence(g["x"]), g["divergence"]) <= 1e-12
    assert rel(F.pressure_gradient(g["xp"]), g["gradient"]) <= 1e-12
    assert rel(F.pressure_rhs(1.7, g["x"], 7.3, g["xp"]), g["pressure_rhs"]) <= 1e-12
    assert abs(F.kinetic_energy(g["x"]) - float(g["kinetic"])) <= 1e-12 * abs(float(g["kinetic"]))


def test_diagonals_match_reference(case):
    g, F = case
    cf = tuple(g["coefs"])
    d = F.diagonal(lambda e: F.apply_momentum(cf, g["w"], e), F.Vu.ndofs)
    assert rel(d, g["momentum_diag"]) <= 1e-12
    dh = F.diagonal(lambda e: F.apply_pressure_helmholtz(float(g["mc"]), e), F.Vp.ndofs)
    assert rel(dh, g["helmholtz_diag"]) <= 1e-12


def test_krylov_restatement_matches_reference(case):
    g, F = case
    mc = float(g["mc"])
    dh = F.diagonal(lambda e: F.apply_pressure_helmholtz(mc, e), F.Vp.ndofs)
    x = np.zeros(F.Vp.ndofs)
    its, _ = O.cg_solve(lambda v: F.apply_pressure_helmholtz(mc, v), g["xp"], x, inv=O.jacobi(dh))
    assert abs(its - int(g["cg_its"])) <= 1
    assert rel(x, g["cg_x"]) <= 1e-8
    cs = tuple(g["coefs_stage"])
    dm = F.diagonal(lambda e: F.apply_momentum(cs, g["w"], e), F.Vu.ndofs)
    xu = np.zeros(F.Vu.ndofs)
    its, _ = O.gmres_solve(lambda v: F.apply_momentum(cs, g["w"], v), g["x"], xu, restart=5, inv=O.jacobi(dm))
    assert abs(its - int(g["gmres_its"])) <= 1
    assert rel(xu, g["gmres_x"]) <= 1e-8


def test_jacobi_zero_diagonal_names_dof():
    with pytest.raises(O.SolverError, match="dof 2"):
        O.jacobi(np.array([1.0, 2.0, 0.0, 4.0]))


def test_gauss_rules_exactness():
    """quadrature.cpp contract: n-point rule exact to degree 2n-1, weights sum to 1."""
    for n in range(1, 8):
        x, w = O.gauss_legendre(n)
        assert abs(w.sum() - 1.0) < 1e-14
        for p in range(2 * n):
            assert abs((w * x ** p).sum() - 1.0 / (p + 1)) < 1e-13
    for n in range(2, 7):
        xl = O.gauss_lobatto(n)
        assert xl[0] == 0.0 and xl[-1] == 1.0 and np.all(np.diff(xl) > 0)
