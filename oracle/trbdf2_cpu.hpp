// Restated TR-BDF2 step on the CPU — TEST INFRASTRUCTURE (the parity oracle).
//
// The reference's driver (`src/schemes.cpp`, named at proj/CMakeLists.txt:25)
// is missing from the tree, so the "reference CPU implementation" of a full
// step is this restatement.  It calls ONLY unmodified reference functions
// (forms.hpp / krylov.hpp) and follows SURVEY.md Appendix A, which derives the
// stage -> operator coefficient map from SPEC.md:345-452, PAPER.md:90-180,
// 475-491 and the free-stream pin proj/tests/test_forms.cpp:369-422.
// The device driver (paper_2107_07776_b200/csrc/context.cu, Context::trbdf2_step) performs exactly
// the same sequence of operator / solver calls.
#pragma once

#include "forms.hpp"
#include "krylov.hpp"

#include <algorithm>
#include <cmath>
#include <vector>

namespace oracle_trbdf2 {

using dgns::Field;

struct StepParams {
  double dt = 1e-3;
  double Re = 100.0;
  double c = 1e3;         // artificial sound speed
  double time = 0.0;      // t^n
  int restart = 50;       // GMRES restart (krylov.hpp:28; cfg3 uses 30)
  double tol_mom = 1e-10;
  double tol_p = 1e-10;
  double tol_mass = 1e-12;
  int max_iter = 10000;
  bool first_step = true;   // n = 0: w1 = u^0
  // trbdf2_step_fixedpoint: each predictor solve is iterated with the
  // advecting field replaced by the latest iterate until the max-norm increment < fp_tol
  bool fixed_point = false;
  double fp_tol = 1e-8;
  int fp_max_iter = 100;
};

struct StepStats {
  int fp_its[2] = {0, 0};     // fixed-point re-solves per stage (0 without fixed_point)
  int gmres_its[2] = {0, 0};  // summed over the stage's predictor solves
  int cg_its[2] = {0, 0};
  int mass_its[4] = {0, 0, 0, 0};
  double gmres_res[2] = {0, 0};
  double cg_res[2] = {0, 0};
};

// y = a*x + b*y
inline void lincomb(double a, const Field& x, double b, const Field& y, Field& out) {
  out.resize(x.size());
  for (std::size_t i = 0; i < x.size(); ++i) out[i] = a * x[i] + b * y[i];
}

/// Solve M_u ut = pressure_gradient_rhs(p) (CG + Jacobi(mass_diagonal), rel 1e-12, x0 = 0).
template <int dim>
int projected_gradient(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
                       const dgns::GeometryCache<dim>& geom, const Field& p,
                       const StepParams& P, Field& ut) {
  Field g;
  dgns::pressure_gradient_rhs(Vu, Vp, geom, p, g);
  Field md;
  dgns::mass_diagonal(Vu, geom, md);
  const dgns::JacobiPreconditioner M(md);
  dgns::SolverSettings s;
  s.rel_tol = P.tol_mass;
  s.max_iter = P.max_iter;
  ut.assign(Vu.n_dofs(), 0.0);
  Field tmp;
  auto res = dgns::cg_solve(
      Vu.n_dofs(), [&](const double* x, double* y) {
        Field xx(x, x + Vu.n_dofs());
        dgns::apply_mass(Vu, geom, xx, tmp);
        std::copy(tmp.begin(), tmp.end(), y);
      },
      g.data(), s, &M, ut.data());
  return res.iterations;
}

/// One stage.  alpha = gamma (stage 1) or 1-gamma (stage 2).
template <int dim>
void stage(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
           const dgns::GeometryCache<dim>& geom, const dgns::BoundaryTable<dim>& bc,
           const dgns::MomentumCtx<dim>& ctx, const dgns::MomentumRhs<dim>& rhs, Field& w, double alpha,
           const Field& u_guess, const Field& p_old, const StepParams& P, Field& u_new,
           Field& p_new, StepStats& st, int si) {
  const int nu = Vu.n_dofs(), np = Vp.n_dofs();
  // momentum: u*
  Field F;
  dgns::momentum_rhs(Vu, Vp, geom, rhs, F);
  Field diag;
  dgns::momentum_diagonal(Vu, geom, ctx, diag);
  const dgns::JacobiPreconditioner Mu(diag);
  dgns::SolverSettings sm;
  sm.rel_tol = P.tol_mom;
  sm.restart = P.restart;
  sm.max_iter = P.max_iter;
  Field ustar = u_guess;
  Field tmp;
  auto rg = dgns::gmres_solve(
      nu, [&](const double* x, double* y) {
        Field xx(x, x + nu);
        dgns::apply_momentum(Vu, geom, ctx, xx, tmp);
        std::copy(tmp.begin(), tmp.end(), y);
      },
      F.data(), sm, &Mu, ustar.data());
  st.gmres_its[si] = rg.iterations;
  st.gmres_res[si] = rg.residual;
  // fixed point (decision FP1): w is the field every advecting-field pointer of
  // ctx / rhs refers to; it becomes the latest iterate, then RHS, diagonal and solve again
  // (initial guess: the latest iterate) until max |u*_i - u*_{i-1}| < fp_tol
  for (int it = 0; P.fixed_point && it < P.fp_max_iter; ++it) {
    w = ustar;
    dgns::momentum_rhs(Vu, Vp, geom, rhs, F);
    dgns::momentum_diagonal(Vu, geom, ctx, diag);
    const dgns::JacobiPreconditioner Mf(diag);
    Field prev = ustar;
    auto rf = dgns::gmres_solve(
        nu, [&](const double* x, double* y) {
          Field xx(x, x + nu);
          dgns::apply_momentum(Vu, geom, ctx, xx, tmp);
          std::copy(tmp.begin(), tmp.end(), y);
        },
        F.data(), sm, &Mf, ustar.data());
    st.gmres_its[si] += rf.iterations;
    st.gmres_res[si] = rf.residual;
    st.fp_its[si] = it + 1;
    double inc = 0.0;
    for (int i = 0; i < nu; ++i) inc = std::max(inc, std::abs(ustar[i] - prev[i]));
    if (inc < P.fp_tol) break;
  }

  const double adt = alpha * P.dt;
  // u** = u* + alpha dt M^-1 G p_old
  Field ut_old;
  st.mass_its[2 * si] = projected_gradient(Vu, Vp, geom, p_old, P, ut_old);
  Field uss(nu);
  for (int i = 0; i < nu; ++i) uss[i] = ustar[i] + adt * ut_old[i];

  // pressure Helmholtz
  const double mass_coef = 1.0 / (P.c * P.c * adt * adt);
  Field prhs;
  dgns::pressure_rhs(Vu, Vp, geom, 1.0 / adt, uss, mass_coef, &p_old, &bc, prhs);
  Field hd;
  dgns::helmholtz_diagonal(Vp, geom, mass_coef, hd);
  const dgns::JacobiPreconditioner Mp(hd);
  dgns::SolverSettings sp;
  sp.rel_tol = P.tol_p;
  sp.max_iter = P.max_iter;
  p_new = p_old;
  auto rc = dgns::cg_solve(
      np, [&](const double* x, double* y) {
        Field xx(x, x + np);
        dgns::apply_pressure_helmholtz(Vp, geom, mass_coef, xx, tmp);
        std::copy(tmp.begin(), tmp.end(), y);
      },
      prhs.data(), sp, &Mp, p_new.data());
  st.cg_its[si] = rc.iterations;
  st.cg_res[si] = rc.residual;

  // u = u** - alpha dt M^-1 G p_new
  Field ut_new;
  st.mass_its[2 * si + 1] = projected_gradient(Vu, Vp, geom, p_new, P, ut_new);
  u_new.resize(nu);
  for (int i = 0; i < nu; ++i) u_new[i] = uss[i] - adt * ut_new[i];
}

/// One TR-BDF2 step: (u^{n-1}, u^n, p^n) -> (u^{n+1}, p^{n+1}).
template <int dim>
void trbdf2_step(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
                 const dgns::GeometryCache<dim>& geom, const dgns::BoundaryTable<dim>& bc,
                 const StepParams& P, const Field& u_nm1, const Field& u_n, const Field& p_n,
                 Field& u_np1, Field& p_np1, StepStats& st) {
  const double g = 2.0 - std::sqrt(2.0);
  const double dt = P.dt, Re = P.Re;

  // ---- stage 1 (alpha = gamma) ----
  Field w1;
  if (P.first_step)
    w1 = u_n;
  else
    lincomb(1.0 + g / (2.0 * (1.0 - g)), u_n, -g / (2.0 * (1.0 - g)), u_nm1, w1);
  dgns::MomentumCtx<dim> c1;
  c1.mass_coef = 1.0 / (g * dt);
  c1.visc_coef = 1.0 / (2.0 * Re);
  c1.adv_coef = 0.5;
  c1.skew_coef = 0.0;
  c1.advecting = &w1;
  c1.bc = &bc;
  dgns::MomentumRhs<dim> r1;
  r1.mass = {{1.0 / (g * dt), &u_n}};
  r1.visc = {{1.0 / (2.0 * Re), &u_n}};
  r1.adv = {{0.5, &u_n, &w1}};
  r1.pres = {{1.0, &p_n}};
  r1.dir_visc_coef = 1.0 / (2.0 * Re);
  r1.dir_adv_coef = 0.5;
  r1.dir_w = &w1;
  r1.time = P.time + g * dt;
  r1.bc = &bc;
  Field u_g, p_g;
  stage(Vu, Vp, geom, bc, c1, r1, w1, g, u_n, p_n, P, u_g, p_g, st, 0);

  // ---- stage 2 (alpha = 1 - gamma) ----
  const double a33 = 1.0 / (2.0 - g);
  const double a31 = (1.0 - g) / (2.0 * (2.0 - g));
  const double a32 = a31;
  Field w2;
  lincomb(1.0 + (1.0 - g) / g, u_g, -(1.0 - g) / g, u_n, w2);
  dgns::MomentumCtx<dim> c2;
  c2.mass_coef = 1.0 / ((1.0 - g) * dt);
  c2.visc_coef = a33 / Re;
  c2.adv_coef = a33;
  c2.skew_coef = 0.0;
  c2.advecting = &w2;
  c2.bc = &bc;
  dgns::MomentumRhs<dim> r2;
  r2.mass = {{1.0 / ((1.0 - g) * dt), &u_g}};
  r2.visc = {{a32 / Re, &u_g}, {a31 / Re, &u_n}};
  r2.adv = {{a32, &u_g, &u_g}, {a31, &u_n, &u_n}};
  r2.pres = {{1.0, &p_g}};
  r2.dir_visc_coef = a33 / Re;
  r2.dir_adv_coef = a33;
  r2.dir_w = &w2;
  r2.time = P.time + dt;
  r2.bc = &bc;
  stage(Vu, Vp, geom, bc, c2, r2, w2, 1.0 - g, u_g, p_g, P, u_np1, p_np1, st, 1);
}


// ---------------------------------------------------------------------------
// The two baseline projection schemes of PAPER.md:182-232 / SPEC.md:391-405
// (bcg_step, gq_bdf2_step), restated with the same reference calls.  Decisions
// (DESIGN.md "Baseline schemes"): BCG solves its fully nonlinear predictor by fixed
// point with w_0 = u^n, w_{i+1} = (u*_i + u^n) / 2, and uses the increment-form
// Helmholtz (14) as printed; GQ-BDF2 uses the consistent BDF2 weights 3/(2dt) with the
// 2/3 dt projection throughout (the printed /dt in Eqs. (15)-(16) read as the effective
// step 2dt/3), advecting field 2u^n - u^{n-1}, skew coefficient -1/2 (the conservative
// C_LF of forms.cpp minus 1/2 (div w) u gives (w.grad)u + 1/2 (div w) u), and takes its
// first step (no u^{n-1}) with BCG.
// its: [gmres, 0, cg, 0, mass-cg (pre), mass-cg (post), 0, 0, fixed-point re-solves, 0]

/// Predictor GMRES with Jacobi(momentum_diagonal), initial guess x.
template <int dim>
dgns::SolveResult predictor(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
                            const dgns::GeometryCache<dim>& geom, const dgns::MomentumCtx<dim>& ctx,
                            const dgns::MomentumRhs<dim>& rhs, const StepParams& P, Field& x) {
  const int nu = Vu.n_dofs();
  Field F, diag, tmp;
  dgns::momentum_rhs(Vu, Vp, geom, rhs, F);
  dgns::momentum_diagonal(Vu, geom, ctx, diag);
  const dgns::JacobiPreconditioner M(diag);
  dgns::SolverSettings sm;
  sm.rel_tol = P.tol_mom;
  sm.restart = P.restart;
  sm.max_iter = P.max_iter;
  return dgns::gmres_solve(
      nu, [&](const double* xx, double* y) {
        Field v(xx, xx + nu);
        dgns::apply_momentum(Vu, geom, ctx, v, tmp);
        std::copy(tmp.begin(), tmp.end(), y);
      },
      F.data(), sm, &M, x.data());
}

/// Bell-Colella-Glaz step.
template <int dim>
void bcg_step(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
              const dgns::GeometryCache<dim>& geom, const dgns::BoundaryTable<dim>& bc, const StepParams& P,
              const Field& u_n, const Field& p_n, Field& u_np1, Field& p_np1, int* its) {
  const int nu = Vu.n_dofs(), np = Vp.n_dofs();
  const double dt = P.dt, Re = P.Re;
  for (int i = 0; i < 10; ++i) its[i] = 0;
  Field w = u_n;
  dgns::MomentumCtx<dim> c;
  c.mass_coef = 1.0 / dt;
  c.visc_coef = 1.0 / (2.0 * Re);
  c.adv_coef = 0.5;
  c.skew_coef = 0.0;
  c.advecting = &w;
  c.bc = &bc;
  dgns::MomentumRhs<dim> r;
  r.mass = {{1.0 / dt, &u_n}};
  r.visc = {{1.0 / (2.0 * Re), &u_n}};
  r.adv = {{0.5, &u_n, &w}};
  r.pres = {{1.0, &p_n}};
  r.dir_visc_coef = 1.0 / (2.0 * Re);
  r.dir_adv_coef = 0.5;
  r.dir_w = &w;
  r.time = P.time + dt;
  r.bc = &bc;
  Field ustar = u_n;
  its[0] = predictor(Vu, Vp, geom, c, r, P, ustar).iterations;
  for (int it = 0; it < P.fp_max_iter; ++it) {  // fully nonlinear: w = (u* + u^n) / 2
    lincomb(0.5, ustar, 0.5, u_n, w);
    Field prev = ustar;
    its[0] += predictor(Vu, Vp, geom, c, r, P, ustar).iterations;
    its[8] = it + 1;
    double inc = 0.0;
    for (int i = 0; i < nu; ++i) inc = std::max(inc, std::abs(ustar[i] - prev[i]));
    if (inc < P.fp_tol) break;
  }
  // increment-form Helmholtz (14): (mc M + K) dp = (1/dt) B(u*), dp0 = 0
  const double mass_coef = 1.0 / (P.c * P.c * dt * dt);
  Field prhs, hd, tmp;
  dgns::pressure_rhs(Vu, Vp, geom, 1.0 / dt, ustar, mass_coef, nullptr, &bc, prhs);
  dgns::helmholtz_diagonal(Vp, geom, mass_coef, hd);
  const dgns::JacobiPreconditioner Mp(hd);
  dgns::SolverSettings sp;
  sp.rel_tol = P.tol_p;
  sp.max_iter = P.max_iter;
  Field dp(np, 0.0);
  its[2] = dgns::cg_solve(
               np, [&](const double* x, double* y) {
                 Field xx(x, x + np);
                 dgns::apply_pressure_helmholtz(Vp, geom, mass_coef, xx, tmp);
                 std::copy(tmp.begin(), tmp.end(), y);
               },
               prhs.data(), sp, &Mp, dp.data())
               .iterations;
  Field ut;
  its[5] = projected_gradient(Vu, Vp, geom, dp, P, ut);
  u_np1.resize(nu);
  for (int i = 0; i < nu; ++i) u_np1[i] = ustar[i] - dt * ut[i];
  p_np1.resize(np);
  for (int i = 0; i < np; ++i) p_np1[i] = p_n[i] + dp[i];
}

/// Guermond-Quartapelle BDF2 step; first step (first_step) = BCG.
template <int dim>
void gq_bdf2_step(const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
                  const dgns::GeometryCache<dim>& geom, const dgns::BoundaryTable<dim>& bc, const StepParams& P,
                  const Field& u_nm1, const Field& u_n, const Field& p_n, Field& u_np1, Field& p_np1, int* its) {
  if (P.first_step) {
    bcg_step(Vu, Vp, geom, bc, P, u_n, p_n, u_np1, p_np1, its);
    return;
  }
  for (int i = 0; i < 10; ++i) its[i] = 0;
  const double dt = P.dt, Re = P.Re;
  Field w;
  lincomb(2.0, u_n, -1.0, u_nm1, w);
  dgns::MomentumCtx<dim> c;
  c.mass_coef = 3.0 / (2.0 * dt);
  c.visc_coef = 1.0 / Re;
  c.adv_coef = 1.0;
  c.skew_coef = -0.5;
  c.advecting = &w;
  c.bc = &bc;
  dgns::MomentumRhs<dim> r;
  r.mass = {{2.0 / dt, &u_n}, {-1.0 / (2.0 * dt), &u_nm1}};
  r.pres = {{1.0, &p_n}};
  r.dir_visc_coef = 1.0 / Re;
  r.dir_adv_coef = 1.0;
  r.dir_w = &w;
  r.time = P.time + dt;
  r.bc = &bc;
  StepParams Q = P;
  Q.fixed_point = false;
  StepStats st;
  stage(Vu, Vp, geom, bc, c, r, w, 2.0 / 3.0, u_n, p_n, Q, u_np1, p_np1, st, 0);
  its[0] = st.gmres_its[0];
  its[2] = st.cg_its[0];
  its[4] = st.mass_its[0];
  its[5] = st.mass_its[1];
}

}  // namespace oracle_trbdf2
