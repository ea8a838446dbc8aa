// Drop-in demonstration (TEST INFRASTRUCTURE): the reference's own host objects
// (generate_cartesian + distort + FunctionSpace + GeometryCache) driven through
// BOTH the unmodified reference operators and include/dgb_reference_adapter.hpp
// (libdgb.so on the GPU).  Exit 0 iff every operator agrees to <= 1e-12 rel L2
// and the device Krylov iteration counts are within +-1 of the reference's.
#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

#include "dgb_reference_adapter.hpp"
#include "trbdf2_cpu.hpp"

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

// refine: cells handed to one Mesh::refine_and_coarsen (hanging faces, mesh.cpp:344-375)
template <int dim>
static int run(int n_el, double amp, int ku, std::vector<int> refine = {}) {
  std::array<double, dim> lo{}, hi{};
  hi.fill(1.0);
  Mesh<dim> mesh = generate_cartesian<dim>(n_el, lo, hi);
  if (amp != 0.0) distort(mesh, amp, 7u);
  if (!refine.empty()) mesh.refine_and_coarsen(refine, {});
  GeometryCache<dim> geom(mesh);
  FunctionSpace<dim> Vu(mesh, ku, dim), Vp(mesh, ku - 1, 1);
  BoundaryTable<dim> bc;
  for (int id = 0; id < 2 * dim; ++id)  // smooth Dirichlet data on every boundary id
    bc.entries[id].value = [](const std::array<double, dim>& x, double t, double* out) {
      for (int d = 0; d < dim; ++d) out[d] = std::sin(1.3 * x[(d + 1) % dim] + 0.7 * d + t) * std::cos(0.9 * x[d]);
    };
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
  apply_mass(Vu, geom, x, r1);
  dev.apply_mass(Vu, x, r2);
  cmp("apply_mass (velocity)", r2, r1);
  apply_mass(Vp, geom, xp, r1);
  dev.apply_mass(Vp, xp, r2);
  cmp("apply_mass (pressure)", r2, r1);
  mass_diagonal(Vu, geom, r1);
  dev.mass_diagonal(Vu, r2);
  cmp("mass_diagonal (velocity)", r2, r1);
  mass_diagonal(Vp, geom, r1);
  dev.mass_diagonal(Vp, r2);
  cmp("mass_diagonal (pressure)", r2, r1);
  {  // a stage-2-shaped RHS: two terms per list, pressure term, Dirichlet data at t = 0.3
    const Field u2 = rnd(Vu.n_dofs(), 4), p2 = rnd(Vp.n_dofs(), 5);
    MomentumRhs<dim> spec;
    spec.mass = {{7.1, &x}};
    spec.visc = {{0.004, &x}, {0.002, &u2}};
    spec.adv = {{0.3, &x, &w}, {0.2, &u2, &u2}};
    spec.pres = {{1.0, &p2}};
    spec.dir_visc_coef = 0.006;
    spec.dir_adv_coef = 0.5;
    spec.dir_w = &w;
    spec.time = 0.3;
    spec.bc = &bc;
    momentum_rhs(Vu, Vp, geom, spec, r1);
    dev.momentum_rhs(spec, r2);
    cmp("momentum_rhs", r2, r1);
    dev.set_boundary(bc, 0.0);
  }
  pressure_rhs(Vu, Vp, geom, 3.3, x, 2.3, &xp, &bc, r1);
  dev.pressure_rhs(3.3, x, 2.3, &xp, r2);
  cmp("pressure_rhs", r2, r1);
  {
    const double e1 = kinetic_energy(Vu, geom, x), e2 = dev.kinetic_energy(x);
    const double e = std::abs(e2 - e1) / std::abs(e1);
    std::printf("  %-28s rel     %.3e (tol 1e-12)\n", "kinetic_energy", e);
    bad += !(e <= 1e-12);
  }
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
  {  // the generic LinearOp-shaped overloads: cg_solve / gmres_solve(n, DeviceOp, b, s, M, x)
    dgb_adapter::DeviceJacobi Mdp(dev.ctx(), hd);
    Field xg(Vp.n_dofs(), 0.0);
    auto g = dev.cg_solve(Vp.n_dofs(), dgb_adapter::DeviceOp<dim>::pressure_helmholtz(2.3), xp.data(), s, &Mdp,
                          xg.data());
    std::printf("  cg_solve(DeviceOp)  ref %d  dev %d\n", rc.iterations, g.iterations);
    bad += std::abs(rc.iterations - g.iterations) > 1;
    cmp("cg_solve(DeviceOp) solution", xg, xr, 1e-8);
    // momentum GMRES: reference gmres_solve with its LinearOp vs the adapter (both Jacobi)
    Field md, ym;
    momentum_diagonal(Vu, geom, m, md);
    JacobiPreconditioner Mu(md);
    SolverSettings sg;
    sg.restart = 20;
    Field bu = rnd(Vu.n_dofs(), 6), xur(Vu.n_dofs(), 0.0), xud(Vu.n_dofs(), 0.0), xug(Vu.n_dofs(), 0.0);
    auto rg = gmres_solve(
        Vu.n_dofs(), [&](const double* a, double* b) {
          apply_momentum(Vu, geom, m, Field(a, a + Vu.n_dofs()), ym);
          std::copy(ym.begin(), ym.end(), b);
        },
        bu.data(), sg, &Mu, xur.data());
    auto dg = dev.gmres_momentum(m, bu, sg, true, xud);
    dgb_adapter::DeviceJacobi Mdu(dev.ctx(), md);
    auto gg = dev.gmres_solve(Vu.n_dofs(), dgb_adapter::DeviceOp<dim>::momentum(m), bu.data(), sg, &Mdu, xug.data());
    std::printf("  gmres iterations  ref %d  gmres_momentum %d  gmres_solve(DeviceOp) %d\n", rg.iterations,
                dg.iterations, gg.iterations);
    bad += std::abs(rg.iterations - dg.iterations) > 1 || std::abs(rg.iterations - gg.iterations) > 1;
    cmp("gmres_momentum solution", xud, xur, 1e-8);
    cmp("gmres_solve(DeviceOp) solution", xug, xur, 1e-8);
    // a zero diagonal is reported as the reference does (SolverError naming the dof)
    Field zd(Vp.n_dofs(), 1.0);
    zd[3] = 0.0;
    try {
      dgb_adapter::DeviceJacobi bad_m(dev.ctx(), zd);
      std::printf("  zero diagonal NOT rejected\n");
      ++bad;
    } catch (const SolverError& e) {
      std::printf("  zero diagonal rejected: %s\n", e.what());
    }
  }
  {  // one TR-BDF2 step: the restated reference driver vs the device step through the adapter
    oracle_trbdf2::StepParams P;
    P.dt = 1e-3;
    P.Re = 100.0;
    oracle_trbdf2::StepStats st;
    Field u0;
    Vu.interpolate([&](const std::array<double, dim>& xx, double* out) { bc.entries[0].value(xx, 0.0, out); }, u0);
    Field p0(Vp.n_dofs(), 0.0), u1r, p1r, u1d, p1d;
    oracle_trbdf2::trbdf2_step(Vu, Vp, geom, bc, P, u0, u0, p0, u1r, p1r, st);
    dgb_step_params dp{};
    dp.dt = P.dt, dp.Re = P.Re, dp.c = P.c, dp.time = 0.0, dp.restart = P.restart;
    dp.tol_mom = P.tol_mom, dp.tol_p = P.tol_p, dp.tol_mass = P.tol_mass, dp.max_iter = P.max_iter;
    dp.first_step = 1;
    const auto its = dev.trbdf2_step(dp, u0, u0, p0, u1d, p1d);
    const int ref_its[8] = {st.gmres_its[0], st.gmres_its[1], st.cg_its[0], st.cg_its[1],
                            st.mass_its[0], st.mass_its[1], st.mass_its[2], st.mass_its[3]};
    int dmax = 0;
    for (int i = 0; i < 8; ++i) dmax = std::max(dmax, std::abs(its[i] - ref_its[i]));
    std::printf("  trbdf2_step iterations: max |dev - ref| = %d\n", dmax);
    bad += dmax > 1;
    cmp("trbdf2_step velocity", u1d, u1r, 1e-9);
    double mr = 0, md2 = 0;
    for (size_t i = 0; i < p1r.size(); ++i) mr += p1r[i], md2 += p1d[i];
    mr /= p1r.size(), md2 /= p1d.size();
    for (auto& v : p1r) v -= mr;
    for (auto& v : p1d) v -= md2;
    cmp("trbdf2_step pressure (mean-free)", p1d, p1r, 1e-9);
  }
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
  std::printf("2D 3x3 distorted, cells 0 and 4 refined (hanging faces), Q2/Q1\n");
  bad += run<2>(3, 0.04, 2, {0, 4});
  std::printf("3D 2^3 Cartesian, cell 0 refined (hanging faces), Q2/Q1\n");
  bad += run<3>(2, 0.0, 2, {0});
  std::printf(bad ? "ADAPTER PARITY FAILED (%d)\n" : "adapter parity ok\n", bad);
  return bad ? 1 : 0;
}
