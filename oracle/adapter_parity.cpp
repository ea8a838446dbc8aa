// Drop-in demonstration (TEST INFRASTRUCTURE): the reference's own host objects
// (generate_cartesian + distort + FunctionSpace + GeometryCache) driven through
// BOTH the unmodified reference operators and include/dgb_reference_adapter.hpp
// (libdgb.so on the GPU).  Exit 0 iff every operator agrees to <= 1e-12 rel L2
// and the device Krylov iteration counts are within +-1 of the reference's.
#include <cmath>
#include <cstdio>
#include <random>

#include "dgb_reference_adapter.hpp"

using namespace dgns;

static double rel(const Field& a, const Field& b) {
  double n = 0, d = 0;
  for (size_t i = 0; i < a.size(); ++i) {
    n += (a[i] - b[i]) * (a[i] - b[i]);
    d += b[i] * b[i];
  }
  return std::sqrt(n / (d > 0 ? d : 1));
}
static Field rnd(int n, unsigned s) {
  std::mt19937 g(s);
  std::uniform_real_distribution<double> u(-1, 1);
  Field f(n);
  for (auto& v : f) v = u(g);
  return f;
}

template <int dim>
static int run(int n_el, double amp, int ku) {
  std::array<double, dim> lo{}, hi{};
  hi.fill(1.0);
  Mesh<dim> mesh = generate_cartesian<dim>(n_el, lo, hi);
  if (amp != 0.0) distort(mesh, amp, 7u);
  GeometryCache<dim> geom(mesh);
  FunctionSpace<dim> Vu(mesh, ku, dim), Vp(mesh, ku - 1, 1);
  BoundaryTable<dim> bc;
  dgb_adapter::Device<dim> dev(mesh, Vu, Vp);
  dev.set_boundary(bc, 0.0);
  const Field w = rnd(Vu.n_dofs(), 1), x = rnd(Vu.n_dofs(), 2), xp = rnd(Vp.n_dofs(), 3);
  MomentumCtx<dim> m;
  m.mass_coef = 1.0 / ((2 - std::sqrt(2.0)) * 1e-3);
  m.visc_coef = 0.005;
  m.adv_coef = 0.5;
  m.advecting = &w;
  m.bc = &bc;
  int bad = 0;
  auto cmp = [&](const char* what, const Field& a, const Field& b, double tol = 1e-12) {
    const double e = rel(a, b);
    std::printf("  %-28s rel L2 %.3e (tol %.0e)\n", what, e, tol);
    bad += !(e <= tol);
  };
  Field r1, r2;
  apply_momentum(Vu, geom, m, x, r1);
  dev.apply_momentum(m, x, r2);
  cmp("apply_momentum", r2, r1);
  momentum_diagonal(Vu, geom, m, r1);
  dev.momentum_diagonal(m, r2);
  cmp("momentum_diagonal", r2, r1);
  apply_pressure_helmholtz(Vp, geom, 2.3, xp, r1);
  dev.apply_pressure_helmholtz(2.3, xp, r2);
  cmp("apply_pressure_helmholtz", r2, r1);
  helmholtz_diagonal(Vp, geom, 2.3, r1);
  dev.helmholtz_diagonal(2.3, r2);
  cmp("helmholtz_diagonal", r2, r1);
  divergence_functional(Vu, Vp, geom, x, &bc, r1);
  dev.divergence_functional(x, r2);
  cmp("divergence_functional", r2, r1);
  pressure_gradient_rhs(Vu, Vp, geom, xp, r1);
  dev.pressure_gradient_rhs(xp, r2);
  cmp("pressure_gradient_rhs", r2, r1);
  // Jacobi-CG on the pressure operator, Jacobi-GMRES on the momentum operator
  SolverSettings s;
  Field hd;
  helmholtz_diagonal(Vp, geom, 2.3, hd);
  JacobiPreconditioner Mp(hd);
  Field xr(Vp.n_dofs(), 0.0), xd(Vp.n_dofs(), 0.0), tmp;
  auto rc = cg_solve(
      Vp.n_dofs(), [&](const double* a, double* b) {
        apply_pressure_helmholtz(Vp, geom, 2.3, Field(a, a + Vp.n_dofs()), tmp);
        std::copy(tmp.begin(), tmp.end(), b);
      },
      xp.data(), s, &Mp, xr.data());
  auto dc = dev.cg_pressure(2.3, xp, s, true, xd);
  std::printf("  cg iterations  ref %d  dev %d\n", rc.iterations, dc.iterations);
  bad += std::abs(rc.iterations - dc.iterations) > 1;
  cmp("cg solution", xd, xr, 1e-8);  // both stopped at rel tol 1e-10, iterations may differ by 1
  return bad;
}

int main() {
  int bad = 0;
  std::printf("2D 4x4 distorted, Q2/Q1\n");
  bad += run<2>(4, 0.05, 2);
  std::printf("3D 3^3 Cartesian, Q3/Q2\n");
  bad += run<3>(3, 0.0, 3);
  std::printf("3D 2^3 distorted, Q2/Q1\n");
  bad += run<3>(2, 0.03, 2);
  std::printf(bad ? "ADAPTER PARITY FAILED (%d)\n" : "adapter parity ok\n", bad);
  return bad ? 1 : 0;
}
