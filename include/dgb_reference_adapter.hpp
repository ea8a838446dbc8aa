// dgb_reference_adapter.hpp — drop-in binding of the reference's operator /
// solver API (proj/src/forms.hpp, krylov.hpp) onto libdgb.so (include/dgb.h).
//
// A maintainer of the reference adds this header and links libdgb.so; call
// sites keep their signatures and semantics:
//
//   dgns::apply_momentum(Vu, geom, ctx, x, out)        forms.hpp:111-113
//   dgns::momentum_diagonal(Vu, geom, ctx, diag)       forms.hpp:114-116
//   dgns::apply_pressure_helmholtz(Vp, geom, mc, x, y) forms.hpp:126-128
//   dgns::helmholtz_diagonal(Vp, geom, mc, diag)       forms.hpp:129-131
//   dgns::apply_mass / mass_diagonal                   forms.hpp:105-109
//   dgns::momentum_rhs                                 forms.hpp:118-120
//   dgns::divergence_functional / pressure_rhs /
//         pressure_gradient_rhs                        forms.hpp:136-150
//   dgns::kinetic_energy                               forms.hpp:168-170
//   dgns::JacobiPreconditioner                         krylov.hpp:40-48
//   dgns::cg_solve / gmres_solve                       krylov.hpp:58-66
//   the TR-BDF2 step (reference schemes.cpp is missing)
//
// become  dgb_adapter::Device dev(mesh, Vu, Vp);  dev.apply_momentum(ctx, x, out); ...
//
// Solvers.  The reference passes the operator as a host closure (LinearOp =
// std::function<void(const double*, double*)>, krylov.hpp:22).  A host closure
// cannot run inside the device-resident Krylov loop (no host round trip per
// iteration), so the adapter's cg_solve / gmres_solve keep the reference's
// signature with the closure replaced by a DeviceOp naming the operator
// (DeviceOp::momentum(ctx), ::pressure_helmholtz(mc), ::mass(V)) and the
// preconditioner by a DeviceJacobi built from the same diagonal Field
// (JacobiPreconditioner semantics: SolverError naming a zero-diagonal dof).
// Outputs are resized and overwritten like the reference (out.assign(n, 0)),
// errors are re-raised as the reference's exception types (SolverError with the
// residual history, std::runtime_error for a missing advecting field).
// Host Fields are staged through persistent device buffers; keep fields on the
// device (Device::DeviceField) inside time loops to avoid PCIe traffic.
#pragma once

#include <algorithm>
#include <array>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "dgb.h"
#include "forms.hpp"
#include "krylov.hpp"
#include "mesh.hpp"
#include "space.hpp"

namespace dgb_adapter {

inline void check(int status) {
  if (status == DGB_OK) return;
  const std::string msg = dgb_last_error();
  if (status == DGB_E_MISSING_FIELD) throw std::runtime_error(msg);
  if (status == DGB_E_NO_CONVERGENCE || status == DGB_E_BREAKDOWN || status == DGB_E_NOT_SPD ||
      status == DGB_E_ZERO_DIAG)
    throw dgns::SolverError(msg, {});
  throw std::runtime_error("dgb: " + msg);
}

class DeviceField {
 public:
  DeviceField(dgb_ctx* c, size_t n) : ctx_(c), n_(n) { check(dgb_alloc(c, n, &p_)); }
  ~DeviceField() { dgb_free(ctx_, p_); }
  DeviceField(const DeviceField&) = delete;
  DeviceField& operator=(const DeviceField&) = delete;
  void upload(const dgns::Field& f) { check(dgb_copy_h2d(ctx_, p_, f.data(), n_)); }
  void download(dgns::Field& f) const {
    f.resize(n_);
    check(dgb_copy_d2h(ctx_, f.data(), p_, n_));
  }
  double* get() const { return p_; }
  size_t size() const { return n_; }

 private:
  dgb_ctx* ctx_;
  size_t n_;
  double* p_ = nullptr;
};

/// The operator a device solve applies (stands in for krylov.hpp:22's LinearOp).
template <int dim>
struct DeviceOp {
  dgb_operator op{};
  const dgns::Field* advecting = nullptr;
  static DeviceOp momentum(const dgns::MomentumCtx<dim>& m) {
    DeviceOp o;
    o.op.op = DGB_OP_MOMENTUM;
    o.op.coefs[0] = m.mass_coef;
    o.op.coefs[1] = m.visc_coef;
    o.op.coefs[2] = m.adv_coef;
    o.op.coefs[3] = m.skew_coef;
    o.advecting = m.advecting;
    return o;
  }
  static DeviceOp pressure_helmholtz(double mass_coef) {
    DeviceOp o;
    o.op.op = DGB_OP_PRESSURE;
    o.op.coefs[0] = mass_coef;
    return o;
  }
  /// mass operator of the velocity (n_comp == dim) or pressure space
  static DeviceOp mass(const dgns::FunctionSpace<dim>& V) {
    DeviceOp o;
    o.op.op = V.n_comp() == dim ? DGB_OP_MASS_U : DGB_OP_MASS_P;
    return o;
  }
};

/// JacobiPreconditioner (krylov.hpp:40-48) on the device: inv_diag = 1 / diag, built
/// from the same host diagonal; throws SolverError naming the first zero-diagonal dof.
class DeviceJacobi {
 public:
  DeviceJacobi(dgb_ctx* ctx, const std::vector<double>& diag) : inv_(ctx, diag.size()) {
    inv_.upload(diag);
    check(dgb_jacobi_inverse(ctx, diag.size(), inv_.get(), inv_.get()));
  }
  const double* get() const { return inv_.get(); }
  std::size_t size() const { return inv_.size(); }

 private:
  DeviceField inv_;
};

/// Device context built from the reference's host objects (Mesh + spaces).
template <int dim>
class Device {
 public:
  Device(const dgns::Mesh<dim>& mesh, const dgns::FunctionSpace<dim>& Vu, const dgns::FunctionSpace<dim>& Vp,
         int device = 0) {
    // active cells become the context's cells (reference active order, space.hpp:5-8)
    const int nv = dgns::Mesh<dim>::n_vertices_per_cell, nf = 2 * dim;
    std::vector<double> verts(mesh.vertices.size() * dim);
    for (size_t v = 0; v < mesh.vertices.size(); ++v)
      for (int d = 0; d < dim; ++d) verts[v * dim + d] = mesh.vertices[v][d];
    std::vector<int> cells, bids;
    for (int c : mesh.active_cells()) {
      for (int v = 0; v < nv; ++v) cells.push_back(mesh.cells[c].v[v]);
      for (int f = 0; f < nf; ++f) bids.push_back(mesh.cells[c].boundary_id[f]);
    }
    // hanging subfaces of a refined mesh (FaceInfo::hanging, mesh.cpp:344-375): the fine
    // owner, the coarse neighbour and the subface's embedding into the coarse cell
    std::vector<int> hang;
    std::vector<double> emb;
    for (const auto& f : mesh.faces().interior) {
      if (!f.hanging) continue;
      hang.insert(hang.end(), {mesh.active_index(f.cell_in), f.face_in, mesh.active_index(f.cell_out), f.face_out});
      for (int d = 0; d < dim; ++d) emb.push_back(f.emb_out.origin[d]);
      for (int t = 0; t < dim - 1; ++t)
        for (int d = 0; d < dim; ++d) emb.push_back(f.emb_out.tangent[t][d]);
    }
    if (hang.empty())
      check(dgb_ctx_create_mesh(dim, (int)mesh.vertices.size(), verts.data(), mesh.n_active(), cells.data(),
                                bids.data(), Vu.degree(), Vp.degree(), device, &ctx_));
    else
      check(dgb_ctx_create_mesh_hanging(dim, (int)mesh.vertices.size(), verts.data(), mesh.n_active(), cells.data(),
                                        bids.data(), (int)hang.size() / 4, hang.data(), emb.data(), Vu.degree(),
                                        Vp.degree(), device, &ctx_));
    nu_ = Vu.n_dofs();
    np_ = Vp.n_dofs();
  }
  ~Device() {
    x_u_.reset(), w_u_.reset(), y_u_.reset(), x_p_.reset(), y_p_.reset(), d_.reset(), b_.reset(), s_.reset();
    dgb_ctx_destroy(ctx_);
  }
  dgb_ctx* ctx() const { return ctx_; }

  /// BoundaryTable (forms.hpp:29-51): types + Dirichlet data tabulated at time t.  The
  /// table's std::functions may depend on t, so device steps re-evaluate them at every
  /// stage time (dgb_set_dirichlet_time_dependent); bc must outlive the Device's use of
  /// it, like the reference's non-owning MomentumRhs::bc.  Pass time_dependent = false
  /// for time-independent data (one tabulation, no host work inside steps).
  void set_boundary(const dgns::BoundaryTable<dim>& bc, double t, bool time_dependent = true) {
    check(dgb_set_dirichlet_time_dependent(ctx_, time_dependent ? 1 : 0));
    for (const auto& [id, e] : bc.entries) {
      check(dgb_set_boundary_type(ctx_, id, e.type == dgns::BcType::outlet ? DGB_BC_OUTLET : DGB_BC_DIRICHLET));
      if (e.value) {
        const auto* fn = &e.value;
        check(dgb_set_dirichlet_fn(
            ctx_, id,
            [](const double* x, double tt, double* out, void* user) {
              std::array<double, dim> xx;
              for (int d = 0; d < dim; ++d) xx[d] = x[d];
              (*static_cast<const decltype(fn)>(user))(xx, tt, out);
            },
            const_cast<void*>(static_cast<const void*>(fn)), t));
      }
    }
  }

  void apply_momentum(const dgns::MomentumCtx<dim>& m, const dgns::Field& x, dgns::Field& out) {
    const double coefs[4] = {m.mass_coef, m.visc_coef, m.adv_coef, m.skew_coef};
    up(x_u_, x, nu_);
    const double* w = nullptr;
    if (m.advecting) {
      up(w_u_, *m.advecting, nu_);
      w = w_u_->get();
    }
    check(dgb_momentum_apply(ctx_, coefs, w, x_u_->get(), y_u()->get()));
    y_u_->download(out);
  }
  void momentum_diagonal(const dgns::MomentumCtx<dim>& m, dgns::Field& diag) {
    const double coefs[4] = {m.mass_coef, m.visc_coef, m.adv_coef, m.skew_coef};
    const double* w = nullptr;
    if (m.advecting) {
      up(w_u_, *m.advecting, nu_);
      w = w_u_->get();
    }
    check(dgb_momentum_diag(ctx_, coefs, w, y_u()->get()));
    y_u_->download(diag);
  }
  void apply_pressure_helmholtz(double mc, const dgns::Field& x, dgns::Field& out) {
    up(x_p_, x, np_);
    check(dgb_pressure_apply(ctx_, mc, x_p_->get(), y_p()->get()));
    y_p_->download(out);
  }
  void helmholtz_diagonal(double mc, dgns::Field& diag) {
    check(dgb_helmholtz_diag(ctx_, mc, y_p()->get()));
    y_p_->download(diag);
  }
  /// apply_mass / mass_diagonal (forms.hpp:105-109) on the velocity or pressure space
  void apply_mass(const dgns::FunctionSpace<dim>& V, const dgns::Field& x, dgns::Field& out) {
    const int sp = space(V);
    up(sp ? x_p_ : x_u_, x, sp ? np_ : nu_);
    DeviceField* y = sp ? y_p() : y_u();
    check(dgb_mass_apply(ctx_, sp, (sp ? x_p_ : x_u_)->get(), y->get()));
    y->download(out);
  }
  void mass_diagonal(const dgns::FunctionSpace<dim>& V, dgns::Field& diag) {
    const int sp = space(V);
    DeviceField* y = sp ? y_p() : y_u();
    check(dgb_mass_diag(ctx_, sp, y->get()));
    y->download(diag);
  }
  /// momentum_rhs (forms.hpp:118-120): every field of the spec is staged on the device;
  /// the Dirichlet data of spec.bc is tabulated at spec.time.
  void momentum_rhs(const dgns::MomentumRhs<dim>& spec, dgns::Field& out) {
    if (spec.mass.size() > 4 || spec.visc.size() > 4 || spec.adv.size() > 4 || spec.pres.size() > 4)
      throw std::invalid_argument("dgb: at most 4 terms per MomentumRhs list");
    if (spec.bc) set_boundary(*spec.bc, spec.time);
    std::vector<std::unique_ptr<DeviceField>> keep;
    auto stage = [&](const dgns::Field* f, size_t n) -> const double* {
      if (!f) return nullptr;
      keep.push_back(std::make_unique<DeviceField>(ctx_, n));
      keep.back()->upload(*f);
      return keep.back()->get();
    };
    dgb_rhs_desc d{};
    d.n_mass = (int)spec.mass.size();
    d.n_visc = (int)spec.visc.size();
    d.n_adv = (int)spec.adv.size();
    d.n_pres = (int)spec.pres.size();
    for (int i = 0; i < d.n_mass; ++i) d.mass_coef[i] = spec.mass[i].coef, d.mass_f[i] = stage(spec.mass[i].f, nu_);
    for (int i = 0; i < d.n_visc; ++i) d.visc_coef[i] = spec.visc[i].coef, d.visc_f[i] = stage(spec.visc[i].f, nu_);
    for (int i = 0; i < d.n_adv; ++i) {
      d.adv_coef[i] = spec.adv[i].coef;
      d.adv_f[i] = stage(spec.adv[i].f, nu_);
      d.adv_w[i] = stage(spec.adv[i].w, nu_);
    }
    for (int i = 0; i < d.n_pres; ++i) d.pres_coef[i] = spec.pres[i].coef, d.pres_f[i] = stage(spec.pres[i].f, np_);
    d.dir_visc_coef = spec.dir_visc_coef;
    d.dir_adv_coef = spec.dir_adv_coef;
    d.dir_w = stage(spec.dir_w, nu_);
    check(dgb_momentum_rhs(ctx_, &d, y_u()->get()));
    y_u_->download(out);
  }
  /// pressure_rhs (forms.hpp:142-145): out = inv_adt B(u) + mass_coef M_p p_old
  void pressure_rhs(double inv_adt, const dgns::Field& u, double mass_coef, const dgns::Field* p_old,
                    dgns::Field& out) {
    up(x_u_, u, nu_);
    if (p_old) up(x_p_, *p_old, np_);
    check(dgb_pressure_rhs(ctx_, inv_adt, x_u_->get(), mass_coef, p_old ? x_p_->get() : nullptr, y_p()->get()));
    y_p_->download(out);
  }
  /// kinetic_energy (forms.hpp:168-170)
  double kinetic_energy(const dgns::Field& u) {
    up(x_u_, u, nu_);
    double e = 0.0;
    check(dgb_kinetic_energy(ctx_, x_u_->get(), &e));
    return e;
  }
  /// One TR-BDF2 step entirely on the device;
  /// returns the Krylov iteration counts (dgb_trbdf2_step order).  The boundary table
  /// must have been set (set_boundary) for the step's time.
  std::vector<int> trbdf2_step(const dgb_step_params& p, const dgns::Field& u_nm1, const dgns::Field& u_n,
                               const dgns::Field& p_n, dgns::Field& u_np1, dgns::Field& p_np1) {
    DeviceField a(ctx_, nu_), b(ctx_, nu_), c(ctx_, np_), du(ctx_, nu_), dp(ctx_, np_);
    a.upload(u_nm1);
    b.upload(u_n);
    c.upload(p_n);
    std::vector<int> its(10, 0);
    check(dgb_trbdf2_step(ctx_, &p, a.get(), b.get(), c.get(), du.get(), dp.get(), its.data()));
    du.download(u_np1);
    dp.download(p_np1);
    its.resize(p.fixed_point ? 10 : 8);
    return its;
  }

  void divergence_functional(const dgns::Field& u, dgns::Field& out) {
    up(x_u_, u, nu_);
    check(dgb_divergence(ctx_, x_u_->get(), y_p()->get()));
    y_p_->download(out);
  }
  void pressure_gradient_rhs(const dgns::Field& p, dgns::Field& out) {
    up(x_p_, p, np_);
    check(dgb_pressure_gradient(ctx_, x_p_->get(), y_u()->get()));
    y_u_->download(out);
  }

  /// cg_solve / gmres_solve (krylov.hpp:58-66) with the operator named by a DeviceOp
  /// and the preconditioner by a DeviceJacobi (null = unpreconditioned).  x is the
  /// initial guess on entry and the solution on return; SolverError (with the residual
  /// history) on non-convergence, breakdown or a non-SPD operator, as the reference.
  dgns::SolveResult cg_solve(std::size_t n, const DeviceOp<dim>& A, const double* b, const dgns::SolverSettings& s,
                             const DeviceJacobi* M, double* x) {
    return solve_op(n, A, b, s, M, x, false);
  }
  dgns::SolveResult gmres_solve(std::size_t n, const DeviceOp<dim>& A, const double* b,
                                const dgns::SolverSettings& s, const DeviceJacobi* M, double* x) {
    return solve_op(n, A, b, s, M, x, true);
  }

  /// cg_solve on the device pressure operator (krylov.hpp:58-60 semantics).
  dgns::SolveResult cg_pressure(double mc, const dgns::Field& b, const dgns::SolverSettings& s, bool jacobi,
                                dgns::Field& x) {
    dgb_operator op{};
    op.op = DGB_OP_PRESSURE;
    op.coefs[0] = mc;
    return solve(op, b, s, jacobi, x, np_, false);
  }
  /// gmres_solve on the device momentum operator (krylov.hpp:64-66 semantics).
  dgns::SolveResult gmres_momentum(const dgns::MomentumCtx<dim>& m, const dgns::Field& b,
                                   const dgns::SolverSettings& s, bool jacobi, dgns::Field& x) {
    dgb_operator op{};
    op.op = DGB_OP_MOMENTUM;
    op.coefs[0] = m.mass_coef;
    op.coefs[1] = m.visc_coef;
    op.coefs[2] = m.adv_coef;
    op.coefs[3] = m.skew_coef;
    if (m.advecting) {
      up(w_u_, *m.advecting, nu_);
      op.d_w = w_u_->get();
    }
    return solve(op, b, s, jacobi, x, nu_, true);
  }

 private:
  dgb_ctx* ctx_ = nullptr;
  size_t nu_ = 0, np_ = 0;
  std::unique_ptr<DeviceField> x_u_, w_u_, y_u_, x_p_, y_p_, d_, b_, s_;

  int space(const dgns::FunctionSpace<dim>& V) const { return V.n_comp() == dim ? 0 : 1; }
  dgns::SolveResult solve_op(std::size_t n, const DeviceOp<dim>& A, const double* b, const dgns::SolverSettings& s,
                             const DeviceJacobi* M, double* x, bool gmres) {
    dgb_operator op = A.op;
    std::unique_ptr<DeviceField> w;
    if (A.advecting) {
      w = std::make_unique<DeviceField>(ctx_, nu_);
      w->upload(*A.advecting);
      op.d_w = w->get();
    }
    DeviceField db(ctx_, n), dx(ctx_, n);
    check(dgb_copy_h2d(ctx_, db.get(), b, n));
    check(dgb_copy_h2d(ctx_, dx.get(), x, n));
    const dgb_solver_settings st{s.rel_tol, s.abs_tol, s.max_iter, s.restart};
    dgb_solve_result r{};
    std::vector<double> hist(std::max(1, s.max_iter));
    int hl = 0;
    const double* inv = M ? M->get() : nullptr;
    const int status = gmres ? dgb_gmres(ctx_, &op, &st, inv, db.get(), dx.get(), &r, hist.data(), (int)hist.size(), &hl)
                             : dgb_cg(ctx_, &op, &st, inv, db.get(), dx.get(), &r, hist.data(), (int)hist.size(), &hl);
    if (status == DGB_E_NO_CONVERGENCE || status == DGB_E_BREAKDOWN || status == DGB_E_NOT_SPD) {
      hist.resize(std::min<size_t>(hist.size(), hl));
      throw dgns::SolverError(dgb_last_error(), hist);
    }
    check(status);
    check(dgb_copy_d2h(ctx_, x, dx.get(), n));
    return {r.iterations, r.residual};
  }
  void up(std::unique_ptr<DeviceField>& f, const dgns::Field& h, size_t n) {
    if (!f) f = std::make_unique<DeviceField>(ctx_, n);
    f->upload(h);
  }
  DeviceField* y_u() {
    if (!y_u_) y_u_ = std::make_unique<DeviceField>(ctx_, nu_);
    return y_u_.get();
  }
  DeviceField* y_p() {
    if (!y_p_) y_p_ = std::make_unique<DeviceField>(ctx_, np_);
    return y_p_.get();
  }
  dgns::SolveResult solve(const dgb_operator& op, const dgns::Field& b, const dgns::SolverSettings& s, bool jacobi,
                          dgns::Field& x, size_t n, bool gmres) {
    d_ = std::make_unique<DeviceField>(ctx_, n);
    b_ = std::make_unique<DeviceField>(ctx_, n);
    s_ = std::make_unique<DeviceField>(ctx_, n);
    b_->upload(b);
    s_->upload(x);
    const double* inv = nullptr;
    if (jacobi) {
      if (op.op == DGB_OP_MOMENTUM)
        check(dgb_momentum_diag(ctx_, op.coefs, op.d_w, d_->get()));
      else
        check(dgb_helmholtz_diag(ctx_, op.coefs[0], d_->get()));
      check(dgb_jacobi_inverse(ctx_, n, d_->get(), d_->get()));
      inv = d_->get();
    }
    const dgb_solver_settings st{s.rel_tol, s.abs_tol, s.max_iter, s.restart};
    dgb_solve_result r{};
    std::vector<double> hist(std::max(1, s.max_iter));
    int hl = 0;
    const int status = gmres ? dgb_gmres(ctx_, &op, &st, inv, b_->get(), s_->get(), &r, hist.data(),
                                         (int)hist.size(), &hl)
                             : dgb_cg(ctx_, &op, &st, inv, b_->get(), s_->get(), &r, hist.data(),
                                      (int)hist.size(), &hl);
    if (status == DGB_E_NO_CONVERGENCE || status == DGB_E_BREAKDOWN || status == DGB_E_NOT_SPD) {
      hist.resize(std::min<size_t>(hist.size(), hl));
      throw dgns::SolverError(dgb_last_error(), hist);
    }
    check(status);
    s_->download(x);
    return {r.iterations, r.residual};
  }
};

}  // namespace dgb_adapter
