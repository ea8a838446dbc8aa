// C-ABI shim over the UNMODIFIED reference library — TEST INFRASTRUCTURE.
//
// Lets the Python tests / bench CPU-baseline legs drive the reference's own
// operator and solver code (proj/src/forms.hpp:105-170, krylov.hpp:22-66) on
// the same host arrays the device path receives.  Nothing in the product
// package links or loads this; it lives in oracle/_ref/libdgref.so.
#include "forms.hpp"
#include "kernels.hpp"
#include "krylov.hpp"
#include "mesh.hpp"
#include "space.hpp"
#include "support/dense_oracle.hpp"
#include "trbdf2_cpu.hpp"

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cstring>
#include <cmath>
#include <memory>
#include <random>
#include <string>
#include <thread>
#include <vector>

using namespace dgns;

extern "C" {
typedef void (*ref_bc_fn)(const double* x, double t, double* out, void* user);
}

namespace {

thread_local std::string g_err;

struct Base {
  virtual ~Base() = default;
  int ndim = 0;
  virtual void info(long long* out) = 0;
  virtual void set_bc(int id, int type, ref_bc_fn fn, void* user) = 0;
  virtual void momentum(const double* c, const double* w, const double* x, double* y) = 0;
  virtual void momentum_diag(const double* c, const double* w, double* d) = 0;
  virtual void pressure(double mc, const double* x, double* y) = 0;
  virtual void helmholtz_diag(double mc, double* d) = 0;
  virtual void laplace(int dir, const double* x, double* y) = 0;
  virtual void laplace_diag(int dir, double* d) = 0;
  virtual void mass(int space, const double* x, double* y) = 0;
  virtual void mass_diag(int space, double* d) = 0;
  virtual void momentum_rhs(int nm, const double* mc, const double* const* mf, int nv,
                            const double* vc, const double* const* vf, int na, const double* ac,
                            const double* const* af, const double* const* aw, int np,
                            const double* pc, const double* const* pf, double dvisc, double dadv,
                            const double* dir_w, double time, double* y) = 0;
  virtual void divergence(const double* u, double* y) = 0;
  virtual void pressure_rhs(double inv_adt, const double* u, double mc, const double* p_old,
                            double* y) = 0;
  virtual void pressure_gradient(const double* p, double* y) = 0;
  virtual double kinetic_energy(const double* u) = 0;
  virtual int solve(int op, int solver, const double* coefs, const double* w, const double* b,
                    double rel_tol, double abs_tol, int max_iter, int restart, int precond,
                    double* x, int* iters, double* resid, double* hist, int hist_cap,
                    int* hist_len) = 0;
  virtual void step(const double* params, const double* u_nm1, const double* u_n,
                    const double* p_n, double* u_np1, double* p_np1, int* its) = 0;
  virtual void scheme_step(int scheme, const double* params, const double* u_nm1, const double* u_n,
                           const double* p_n, double* u_np1, double* p_np1, int* its) = 0;
  virtual void faces(int* iface, double* imeas, int* bface, double* bmeas) = 0;
  virtual void cell_vertices(double* xv) = 0;
  virtual void mesh_arrays(double* xv, int* cv, int* bid, double* emb_out) = 0;
  virtual void bface_points(int rule, double* xq) = 0;
  virtual void interpolate_nodes(int space, double* xn) = 0;
  virtual void interpolate_fn(ref_bc_fn fn, void* user, double* u, int nthreads) = 0;
  virtual double bench(int op, const double* coefs, const double* w, const double* x, int nthreads,
                       int napplies) = 0;
  virtual void pair_setup(const double* c, const double* w, const double* x, double pmc, const double* xp) = 0;
  virtual void pair_run() = 0;
  virtual void dense_momentum(const double* c, const double* w, double* A) = 0;
  virtual void dense_scalar_sip(double mc, int dir, int rule, double* A) = 0;
};

template <int dim>
struct Ctx : Base {
  Mesh<dim> mesh;
  std::unique_ptr<GeometryCache<dim>> geom;
  std::unique_ptr<FunctionSpace<dim>> Vu, Vp;
  BoundaryTable<dim> bc;

  Ctx(Mesh<dim>&& m, int ku, int kp) : mesh(std::move(m)) {
    this->ndim = dim;
    geom = std::make_unique<GeometryCache<dim>>(mesh);
    Vu = std::make_unique<FunctionSpace<dim>>(mesh, ku, dim);
    Vp = std::make_unique<FunctionSpace<dim>>(mesh, kp, 1);
  }
  static Field F(const double* p, int n) { return Field(p, p + n); }
  int nu() const { return Vu->n_dofs(); }
  int np() const { return Vp->n_dofs(); }

  void info(long long* out) override {
    out[0] = mesh.n_active();
    out[1] = nu();
    out[2] = np();
    out[3] = static_cast<long long>(mesh.faces().interior.size());
    out[4] = static_cast<long long>(mesh.faces().boundary.size());
    out[5] = Vu->degree();
    out[6] = Vp->degree();
    out[7] = dim;
    out[8] = static_cast<long long>(mesh.vertices.size());
    int nh = 0;
    for (const auto& f : mesh.faces().interior) nh += f.hanging;
    out[9] = nh;
  }
  void set_bc(int id, int type, ref_bc_fn fn, void* user) override {
    auto& e = bc.entries[id];
    e.type = type == 1 ? BcType::outlet : BcType::dirichlet;
    if (fn)
      e.value = [fn, user](const std::array<double, dim>& x, double t, double* out) {
        fn(x.data(), t, out, user);
      };
    else
      e.value = nullptr;
  }
  MomentumCtx<dim> mctx(const double* c, const Field* w) {
    MomentumCtx<dim> m;
    m.mass_coef = c[0];
    m.visc_coef = c[1];
    m.adv_coef = c[2];
    m.skew_coef = c[3];
    m.advecting = w;
    m.bc = &bc;
    return m;
  }
  void momentum(const double* c, const double* w, const double* x, double* y) override {
    Field wf = w ? F(w, nu()) : Field();
    Field out;
    apply_momentum(*Vu, *geom, mctx(c, w ? &wf : nullptr), F(x, nu()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void momentum_diag(const double* c, const double* w, double* d) override {
    Field wf = w ? F(w, nu()) : Field();
    Field out;
    momentum_diagonal(*Vu, *geom, mctx(c, w ? &wf : nullptr), out);
    std::memcpy(d, out.data(), sizeof(double) * out.size());
  }
  void pressure(double mc, const double* x, double* y) override {
    Field out;
    apply_pressure_helmholtz(*Vp, *geom, mc, F(x, np()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void helmholtz_diag(double mc, double* d) override {
    Field out;
    helmholtz_diagonal(*Vp, *geom, mc, out);
    std::memcpy(d, out.data(), sizeof(double) * out.size());
  }
  void laplace(int dir, const double* x, double* y) override {
    Field out;
    apply_scalar_laplace(*Vp, *geom, dir != 0, F(x, np()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void laplace_diag(int dir, double* d) override {
    Field out;
    scalar_laplace_diagonal(*Vp, *geom, dir != 0, out);
    std::memcpy(d, out.data(), sizeof(double) * out.size());
  }
  void mass(int space, const double* x, double* y) override {
    const auto& V = space == 0 ? *Vu : *Vp;
    Field out;
    apply_mass(V, *geom, F(x, V.n_dofs()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void mass_diag(int space, double* d) override {
    const auto& V = space == 0 ? *Vu : *Vp;
    Field out;
    mass_diagonal(V, *geom, out);
    std::memcpy(d, out.data(), sizeof(double) * out.size());
  }
  void momentum_rhs(int nm, const double* mc, const double* const* mf, int nv, const double* vc,
                    const double* const* vf, int na, const double* ac, const double* const* af,
                    const double* const* aw, int npr, const double* pc, const double* const* pf,
                    double dvisc, double dadv, const double* dir_w, double time,
                    double* y) override {
    std::vector<std::unique_ptr<Field>> keep;
    auto hold = [&](const double* p, int n) {
      keep.push_back(std::make_unique<Field>(p, p + n));
      return keep.back().get();
    };
    MomentumRhs<dim> s;
    for (int i = 0; i < nm; ++i) s.mass.push_back({mc[i], hold(mf[i], nu())});
    for (int i = 0; i < nv; ++i) s.visc.push_back({vc[i], hold(vf[i], nu())});
    for (int i = 0; i < na; ++i) s.adv.push_back({ac[i], hold(af[i], nu()), hold(aw[i], nu())});
    for (int i = 0; i < npr; ++i) s.pres.push_back({pc[i], hold(pf[i], np())});
    s.dir_visc_coef = dvisc;
    s.dir_adv_coef = dadv;
    s.dir_w = dir_w ? hold(dir_w, nu()) : nullptr;
    s.time = time;
    s.bc = &bc;
    Field out;
    dgns::momentum_rhs(*Vu, *Vp, *geom, s, out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void divergence(const double* u, double* y) override {
    Field out;
    divergence_functional(*Vu, *Vp, *geom, F(u, nu()), &bc, out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void pressure_rhs(double inv_adt, const double* u, double mc, const double* p_old,
                    double* y) override {
    Field po = p_old ? F(p_old, np()) : Field();
    Field out;
    dgns::pressure_rhs(*Vu, *Vp, *geom, inv_adt, F(u, nu()), mc, p_old ? &po : nullptr, &bc, out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  void pressure_gradient(const double* p, double* y) override {
    Field out;
    pressure_gradient_rhs(*Vu, *Vp, *geom, F(p, np()), out);
    std::memcpy(y, out.data(), sizeof(double) * out.size());
  }
  double kinetic_energy(const double* u) override {
    return dgns::kinetic_energy(*Vu, *geom, F(u, nu()));
  }

  // op: 0 momentum(coefs, w), 1 pressure helmholtz(coefs[0]), 2 mass(u), 3 mass(p)
  // solver: 0 cg, 1 gmres.  precond: 0 none, 1 jacobi(exact diagonal)
  int solve(int op, int solver, const double* coefs, const double* w, const double* b,
            double rel_tol, double abs_tol, int max_iter, int restart, int precond, double* x,
            int* iters, double* resid, double* hist, int hist_cap, int* hist_len) override {
    const int n = (op == 0 || op == 2) ? nu() : np();
    Field wf = w ? F(w, nu()) : Field();
    const auto mc = mctx(coefs, w ? &wf : nullptr);
    Field tmp, diag;
    LinearOp A;
    if (op == 0) {
      A = [&](const double* xx, double* yy) {
        apply_momentum(*Vu, *geom, mc, F(xx, n), tmp);
        std::memcpy(yy, tmp.data(), sizeof(double) * n);
      };
      if (precond) momentum_diagonal(*Vu, *geom, mc, diag);
    } else if (op == 1) {
      A = [&](const double* xx, double* yy) {
        apply_pressure_helmholtz(*Vp, *geom, coefs[0], F(xx, n), tmp);
        std::memcpy(yy, tmp.data(), sizeof(double) * n);
      };
      if (precond) helmholtz_diagonal(*Vp, *geom, coefs[0], diag);
    } else {
      const auto& V = op == 2 ? *Vu : *Vp;
      A = [&](const double* xx, double* yy) {
        apply_mass(V, *geom, F(xx, n), tmp);
        std::memcpy(yy, tmp.data(), sizeof(double) * n);
      };
      if (precond) mass_diagonal(V, *geom, diag);
    }
    SolverSettings s;
    s.rel_tol = rel_tol;
    s.abs_tol = abs_tol;
    s.max_iter = max_iter;
    s.restart = restart;
    *hist_len = 0;
    try {
      std::unique_ptr<JacobiPreconditioner> M;
      if (precond) M = std::make_unique<JacobiPreconditioner>(diag);
      auto r = solver == 0 ? cg_solve(n, A, b, s, M.get(), x) : gmres_solve(n, A, b, s, M.get(), x);
      *iters = r.iterations;
      *resid = r.residual;
      return 0;
    } catch (const SolverError& e) {
      g_err = e.what();
      const int m = std::min<int>(hist_cap, static_cast<int>(e.history.size()));
      for (int i = 0; i < m; ++i) hist[i] = e.history[i];
      *hist_len = static_cast<int>(e.history.size());
      return 2;
    } catch (const std::exception& e) {
      g_err = e.what();
      return 1;
    }
  }

  // params: dt, Re, c, time, restart, tol_mom, tol_p, tol_mass, max_iter, first_step,
  //         fixed_point, fp_tol, fp_max_iter; its: 10 (the device order, + fixed-point counts)
  void step(const double* prm, const double* u_nm1, const double* u_n, const double* p_n,
            double* u_np1, double* p_np1, int* its) override {
    oracle_trbdf2::StepParams P;
    P.dt = prm[0];
    P.Re = prm[1];
    P.c = prm[2];
    P.time = prm[3];
    P.restart = static_cast<int>(prm[4]);
    P.tol_mom = prm[5];
    P.tol_p = prm[6];
    P.tol_mass = prm[7];
    P.max_iter = static_cast<int>(prm[8]);
    P.first_step = prm[9] != 0.0;
    P.fixed_point = prm[10] != 0.0;
    P.fp_tol = prm[11];
    P.fp_max_iter = static_cast<int>(prm[12]);
    oracle_trbdf2::StepStats st;
    Field un1, pn1;
    oracle_trbdf2::trbdf2_step(*Vu, *Vp, *geom, bc, P, F(u_nm1, nu()), F(u_n, nu()), F(p_n, np()),
                               un1, pn1, st);
    std::memcpy(u_np1, un1.data(), sizeof(double) * nu());
    std::memcpy(p_np1, pn1.data(), sizeof(double) * np());
    its[0] = st.gmres_its[0];
    its[1] = st.gmres_its[1];
    its[2] = st.cg_its[0];
    its[3] = st.cg_its[1];
    for (int i = 0; i < 4; ++i) its[4 + i] = st.mass_its[i];
    its[8] = st.fp_its[0];
    its[9] = st.fp_its[1];
  }

  // scheme 1 = BCG, 2 = GQ-BDF2 (params as step(); its: 10)
  void scheme_step(int scheme, const double* prm, const double* u_nm1, const double* u_n, const double* p_n,
                   double* u_np1, double* p_np1, int* its) override {
    oracle_trbdf2::StepParams P;
    P.dt = prm[0];
    P.Re = prm[1];
    P.c = prm[2];
    P.time = prm[3];
    P.restart = static_cast<int>(prm[4]);
    P.tol_mom = prm[5];
    P.tol_p = prm[6];
    P.tol_mass = prm[7];
    P.max_iter = static_cast<int>(prm[8]);
    P.first_step = prm[9] != 0.0;
    P.fp_tol = prm[11];
    P.fp_max_iter = static_cast<int>(prm[12]);
    Field un1, pn1;
    if (scheme == 1)
      oracle_trbdf2::bcg_step(*Vu, *Vp, *geom, bc, P, F(u_n, nu()), F(p_n, np()), un1, pn1, its);
    else
      oracle_trbdf2::gq_bdf2_step(*Vu, *Vp, *geom, bc, P, F(u_nm1 ? u_nm1 : u_n, nu()), F(u_n, nu()),
                                  F(p_n, np()), un1, pn1, its);
    std::memcpy(u_np1, un1.data(), sizeof(double) * nu());
    std::memcpy(p_np1, pn1.data(), sizeof(double) * np());
  }

  // interior: [cell_in, face_in, cell_out, face_out, hanging] per face (active indices)
  // boundary: [cell_in, face_in, boundary_id]
  // The active mesh as raw arrays (what a reference-side binding hands the device, see
  // INTEGRATION.md): every vertex [nverts][dim], active cells' vertex ids [n_active][2^dim]
  // and boundary ids [n_active][2dim] in active order, and for every interior face
  // (mesh.faces().interior order) its emb_out (mesh.hpp:28-36): origin[dim], then
  // tangent[t][dim] for t < dim-1  -> [n_interior][dim*dim].
  void mesh_arrays(double* xv, int* cv, int* bid, double* emb_out) override {
    for (size_t v = 0; v < mesh.vertices.size(); ++v)
      for (int d = 0; d < dim; ++d) xv[v * dim + d] = mesh.vertices[v][d];
    for (int a = 0; a < mesh.n_active(); ++a) {
      const auto& c = mesh.cells[mesh.active_cells()[a]];
      for (int v = 0; v < Mesh<dim>::n_vertices_per_cell; ++v) cv[(size_t)a * Mesh<dim>::n_vertices_per_cell + v] = c.v[v];
      for (int f = 0; f < Mesh<dim>::n_faces_per_cell; ++f)
        bid[(size_t)a * Mesh<dim>::n_faces_per_cell + f] = c.boundary_id[f];
    }
    const auto& fl = mesh.faces();
    for (size_t f = 0; f < fl.interior.size(); ++f) {
      const auto& e = fl.interior[f].emb_out;
      double* o = emb_out + f * dim * dim;
      for (int d = 0; d < dim; ++d) o[d] = e.origin[d];
      for (int t = 0; t < dim - 1; ++t)
        for (int d = 0; d < dim; ++d) o[dim + t * dim + d] = e.tangent[t][d];
    }
  }
  void faces(int* iface, double* imeas, int* bface, double* bmeas) override {
    const auto& fl = mesh.faces();
    for (size_t f = 0; f < fl.interior.size(); ++f) {
      const auto& fi = fl.interior[f];
      iface[5 * f + 0] = mesh.active_index(fi.cell_in);
      iface[5 * f + 1] = fi.face_in;
      iface[5 * f + 2] = mesh.active_index(fi.cell_out);
      iface[5 * f + 3] = fi.face_out;
      iface[5 * f + 4] = fi.hanging;
      imeas[f] = fi.measure;
    }
    for (size_t f = 0; f < fl.boundary.size(); ++f) {
      const auto& fi = fl.boundary[f];
      bface[3 * f + 0] = mesh.active_index(fi.cell_in);
      bface[3 * f + 1] = fi.face_in;
      bface[3 * f + 2] = fi.boundary_id;
      bmeas[f] = fi.measure;
    }
  }
  // Per active cell, the 2^dim vertex coordinates (lexicographic vertex order).
  void cell_vertices(double* xv) override {
    const int nv = Mesh<dim>::n_vertices_per_cell;
    for (int i = 0; i < mesh.n_active(); ++i) {
      const auto& c = mesh.cells[mesh.active_cells()[i]];
      for (int v = 0; v < nv; ++v)
        for (int d = 0; d < dim; ++d) xv[(static_cast<size_t>(i) * nv + v) * dim + d] = mesh.vertices[c.v[v]][d];
    }
  }
  void bface_points(int rule, double* xq) override {
    const auto& bfg = geom->boundary_faces(rule);
    size_t k = 0;
    for (const auto& fg : bfg)
      for (const auto& p : fg.xq)
        for (int d = 0; d < dim; ++d) xq[k++] = p[d];
  }
  // Physical coordinates of the nodal points of every cell (space 0: Vu nodes, 1: Vp nodes).
  void interpolate_nodes(int space, double* xn) override {
    const auto& V = space == 0 ? *Vu : *Vp;
    for (int i = 0; i < mesh.n_active(); ++i) {
      const int c = mesh.active_cells()[i];
      for (int j = 0; j < V.nb(); ++j) {
        const auto x = mesh.map_point(c, V.nodes()[j]);
        for (int d = 0; d < dim; ++d) xn[(static_cast<size_t>(i) * V.nb() + j) * dim + d] = x[d];
      }
    }
  }
  // FunctionSpace::interpolate (space.cpp:239-253) with a C callback, the cells split
  // over nthreads (each thread writes its own cells; same values as the serial loop).
  void interpolate_fn(ref_bc_fn fn, void* user, double* u, int nthreads) override {
    const int nc = mesh.n_active(), nb = Vu->nb();
    auto run = [&](int c0, int c1) {
      double tmp[3];
      for (int i = c0; i < c1; ++i) {
        const int c = mesh.active_cells()[i];
        const size_t off = static_cast<size_t>(i) * dim * nb;
        for (int j = 0; j < nb; ++j) {
          const auto x = mesh.map_point(c, Vu->nodes()[j]);
          fn(x.data(), 0.0, tmp, user);
          for (int comp = 0; comp < dim; ++comp) u[off + comp * nb + j] = tmp[comp];
        }
      }
    };
    nthreads = std::max(1, nthreads);
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t)
      th.emplace_back(run, static_cast<int>((long long)nc * t / nthreads),
                      static_cast<int>((long long)nc * (t + 1) / nthreads));
    for (auto& t : th) t.join();
  }
  // Throughput of the reference CPU apply: nthreads concurrent independent
  // applies (reference code is single-threaded; caches are warmed first so the
  // lazily-filled GeometryCache / trace tables are read-only during the run).
  double bench(int op, const double* c, const double* w, const double* x, int nthreads,
               int napplies) override {
    const int n = op == 0 ? nu() : np();
    Field wf = w ? F(w, nu()) : Field();
    Field xf = F(x, n);
    const auto m = mctx(c, w ? &wf : nullptr);
    auto one = [&](Field& out) {
      if (op == 0)
        apply_momentum(*Vu, *geom, m, xf, out);
      else
        apply_pressure_helmholtz(*Vp, *geom, c[0], xf, out);
    };
    {
      Field warm;
      one(warm);
    }
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < nthreads; ++t)
      th.emplace_back([&]() {
        Field out;
        for (int k = 0; k < napplies; ++k) one(out);
      });
    for (auto& t : th) t.join();
    const auto t1 = std::chrono::steady_clock::now();
    return std::chrono::duration<double>(t1 - t0).count();
  }
  // bench.py reference arm: one apply_momentum + one apply_pressure_helmholtz
  // (forms.cpp:389-604, 1090-1095) on inputs held by the context; outputs are
  // resized and zeroed by the callee every call, exactly as in the reference.
  Field pw, px, pxp, pyu, pyp;
  double pc[4] = {0, 0, 0, 0}, ppmc = 0.0;
  void pair_setup(const double* c, const double* w, const double* x, double pmc, const double* xp) override {
    std::copy(c, c + 4, pc);
    ppmc = pmc;
    pw = F(w, nu());
    px = F(x, nu());
    pxp = F(xp, np());
  }
  void pair_run() override {
    apply_momentum(*Vu, *geom, mctx(pc, &pw), px, pyu);
    apply_pressure_helmholtz(*Vp, *geom, ppmc, pxp, pyp);
  }
  void dense_momentum(const double* c, const double* w, double* A) override {
    Field wf = w ? F(w, nu()) : Field();
    const auto m = mctx(c, w ? &wf : nullptr);
    const auto M = oracle::momentum_matrix(*Vu, m, Vu->degree() + 1, Vu->degree() + 2);
    std::memcpy(A, M.a.data(), sizeof(double) * M.a.size());
  }
  void dense_scalar_sip(double mc, int dir, int rule, double* A) override {
    const auto M = oracle::scalar_sip_matrix(*Vp, mc, dir != 0, rule);
    std::memcpy(A, M.a.data(), sizeof(double) * M.a.size());
  }
};

template <int dim>
Base* make_cartesian(int n_el, double amp, unsigned seed, int ku, int kp, int refine_first) {
  std::array<double, dim> lo{}, hi{};
  hi.fill(1.0);
  Mesh<dim> m = generate_cartesian<dim>(n_el, lo, hi);
  if (amp != 0.0) distort(m, amp, seed);
  if (refine_first) m.refine_and_coarsen({0}, {});
  return new Ctx<dim>(std::move(m), ku, kp);
}
// generate_cartesian (+ distort), then one Mesh::refine_and_coarsen(refine_set, {})
// (mesh.hpp:125-128; the reference grows the set for 1-irregularity): hanging faces
template <int dim>
Base* make_refined(int n_el, double amp, unsigned seed, int ku, int kp, int n_ref, const int* refine) {
  std::array<double, dim> lo{}, hi{};
  hi.fill(1.0);
  Mesh<dim> m = generate_cartesian<dim>(n_el, lo, hi);
  if (amp != 0.0) distort(m, amp, seed);
  m.refine_and_coarsen(std::vector<int>(refine, refine + n_ref), {});
  return new Ctx<dim>(std::move(m), ku, kp);
}

// Same construction as import_text (mesh.cpp:793-817) from raw arrays: vertices
// [nv][dim], cell vertices [nc][2^dim], boundary ids [nc][2dim] (-1 interior), then
// Mesh::finalize().  (Avoids the iostream parse, which is fragile when the host
// process has already loaded another libstdc++.)
template <int dim>
Mesh<dim> mesh_from_arrays(int nv, const double* xv, int nc, const int* cv, const int* bid) {
  Mesh<dim> m;
  m.vertices.resize(nv);
  for (int v = 0; v < nv; ++v)
    for (int a = 0; a < dim; ++a) m.vertices[v][a] = xv[(size_t)v * dim + a];
  m.cells.resize(nc);
  for (int c = 0; c < nc; ++c) {
    for (int v = 0; v < Mesh<dim>::n_vertices_per_cell; ++v) {
      const int id = cv[(size_t)c * Mesh<dim>::n_vertices_per_cell + v];
      if (id < 0 || id >= nv) throw std::runtime_error("mesh arrays: bad cell vertex index");
      m.cells[c].v[v] = id;
    }
    for (int f = 0; f < Mesh<dim>::n_faces_per_cell; ++f)
      m.cells[c].boundary_id[f] = bid[(size_t)c * Mesh<dim>::n_faces_per_cell + f];
  }
  m.finalize();
  return m;
}

// A z-slab [0,1]^2 x [z0/n, (z0+nz)/n] of generate_cartesian<3>(n, 0, 1)
// (mesh.cpp:572-615): the same vertex coordinates lo + (hi-lo)*id/n, the same
// lexicographic vertex / cell order; the slab's own bottom / top faces carry
// boundary ids 4 / 5.  Every cell is bit-identical to the corresponding cell of
// the full mesh, so per-cell reference work equals the full config's.
Mesh<3> slab_mesh(int n, int z0, int nz) {
  if (n < 1 || nz < 1 || z0 < 0 || z0 + nz > n) throw std::invalid_argument("slab_mesh: bad extent");
  const int nx = n + 1, nzv = nz + 1;
  std::vector<double> xv(static_cast<size_t>(nx) * nx * nzv * 3);
  for (int k = 0; k < nzv; ++k)
    for (int j = 0; j < nx; ++j)
      for (int i = 0; i < nx; ++i) {
        double* p = &xv[3 * ((static_cast<size_t>(k) * nx + j) * nx + i)];
        p[0] = 0.0 + (1.0 - 0.0) * i / n;
        p[1] = 0.0 + (1.0 - 0.0) * j / n;
        p[2] = 0.0 + (1.0 - 0.0) * (z0 + k) / n;
      }
  const int nc = n * n * nz;
  std::vector<int> cv(static_cast<size_t>(nc) * 8), bid(static_cast<size_t>(nc) * 6, -1);
  for (int c = 0; c < nc; ++c) {
    const int ic[3] = {c % n, (c / n) % n, c / (n * n)};
    for (int b = 0; b < 8; ++b)
      cv[8 * c + b] = ((ic[2] + ((b >> 2) & 1)) * nx + ic[1] + ((b >> 1) & 1)) * nx + ic[0] + (b & 1);
    const int lim[3] = {n, n, nz};
    for (int d = 0; d < 3; ++d) {
      if (ic[d] == 0) bid[6 * c + 2 * d] = 2 * d;
      if (ic[d] == lim[d] - 1) bid[6 * c + 2 * d + 1] = 2 * d + 1;
    }
  }
  return mesh_from_arrays<3>(nx * nx * nzv, xv.data(), nc, cv.data(), bid.data());
}

}  // namespace

extern "C" {

// ---- synthetic inputs (BASELINE.json configs) ----------
// TEST INFRASTRUCTURE: a restatement of the frozen generator (mt19937_64; uniform
// = (x >> 11) * 2^-53; Box-Muller normal; modes lexicographic, last index fastest;
// a before phi; potential component 1, 2, 3) so that reference-only processes (the
// bench reference arm, the CPU phase of tools/full_step_parity.py) build the same
// inputs as the device path without loading libdgb.so.  Bit-identity with the
// product's generator (capi.cpp dgb_seeded_uniform / dgb_synth_*) is a CPU test
// (tests/test_oracle_inputs.py).
// The product compiles its generator as plain host code (no FMA contraction), so the
// restatement is compiled without contraction too: bit-identical values.
#pragma GCC push_options
#pragma GCC optimize("fp-contract=off")
void ref_seeded_uniform(unsigned long long seed, size_t n, double lo, double hi, double* out) {
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * ((double)(rng() >> 11) * 0x1.0p-53);
}
void ref_synth_init(int dim, unsigned long long seed, double scale, double* user) {
  std::mt19937_64 rng(seed);
  auto uni = [&]() { return (double)(rng() >> 11) * 0x1.0p-53; };
  const int nm = dim == 2 ? 16 : 64, ncomp = dim == 2 ? 1 : 3;
  user[0] = dim;
  user[1] = scale;
  user[2] = nm;
  int k = 3;
  for (int c = 0; c < ncomp; ++c)
    for (int m = 0; m < nm; ++m) {
      double k2 = 0.0;
      for (int d = 0, rem = m; d < dim; ++d, rem /= 4) {
        const int i = 1 + rem % 4;
        k2 += i * i;
      }
      const double u1 = uni(), u2 = uni();
      user[k++] = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2) / k2;
      user[k++] = 2.0 * M_PI * uni();
    }
}
// 2D: u = (dpsi/dy, -dpsi/dx); 3D: u = curl A.
void ref_synth_eval(const double* x, double /*t*/, double* out, void* user) {
  const double* u = static_cast<const double*>(user);
  const int dim = static_cast<int>(u[0]), nm = static_cast<int>(u[2]);
  const double scale = u[1], tp = 2.0 * M_PI;
  if (dim == 2) {
    double dx = 0.0, dy = 0.0;
    for (int m = 0; m < nm; ++m) {
      const int i0 = 1 + m / 4, i1 = 1 + m % 4;
      const double cth = std::cos(tp * (i0 * x[0] + i1 * x[1]) + u[4 + 2 * m]);
      dx += u[3 + 2 * m] * tp * i0 * cth;
      dy += u[3 + 2 * m] * tp * i1 * cth;
    }
    out[0] = scale * dy;
    out[1] = -scale * dx;
    return;
  }
  double G[3][3] = {};
  for (int c = 0; c < 3; ++c)
    for (int m = 0; m < nm; ++m) {
      const int i0 = 1 + m / 16, i1 = 1 + (m / 4) % 4, i2 = 1 + m % 4;
      const double a = u[3 + 2 * (c * nm + m)], ph = u[4 + 2 * (c * nm + m)];
      const double cth = a * tp * std::cos(tp * (i0 * x[0] + i1 * x[1] + i2 * x[2]) + ph);
      G[c][0] += i0 * cth;
      G[c][1] += i1 * cth;
      G[c][2] += i2 * cth;
    }
  out[0] = scale * (G[2][1] - G[1][2]);
  out[1] = scale * (G[0][2] - G[2][0]);
  out[2] = scale * (G[1][0] - G[0][1]);
}
#pragma GCC pop_options
void ref_interpolate_fn(void* h, ref_bc_fn fn, void* user, double* u, int nthreads) {
  static_cast<Base*>(h)->interpolate_fn(fn, user, u, nthreads);
}
// The reference's BLAS-1 kernels (kernels.hpp:34-43, the active backend: AVX2 on an
// AVX2 host, kernels_avx2.cpp:12-70) on host arrays.  op: 0 axpy (y += a x), 1 axpby
// (y = a x + b y), 2 scal (y *= a), 3 dot, 4 max_abs_diff; returns the scalar result.
double ref_kern(int op, size_t n, double a, double b, const double* x, double* y) {
  switch (op) {
    case 0: kern::axpy(n, a, x, y); return 0.0;
    case 1: kern::axpby(n, a, x, b, y); return 0.0;
    case 2: kern::scal(n, a, y); return 0.0;
    case 3: return kern::dot(n, x, y);
    default: return kern::max_abs_diff(n, x, y);
  }
}
void* ref_create_slab(int n, int z0, int nz, int ku, int kp) {
  try {
    return new Ctx<3>(slab_mesh(n, z0, nz), ku, kp);
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}

const char* ref_last_error() { return g_err.c_str(); }
const char* ref_backend() {
  static std::string s;
  s = kern::backend_name();
  return s.c_str();
}

void* ref_create_cartesian(int dim, int n_el, double amp, unsigned seed, int ku, int kp,
                           int refine_first) {
  try {
    if (dim == 2) return make_cartesian<2>(n_el, amp, seed, ku, kp, refine_first);
    if (dim == 3) return make_cartesian<3>(n_el, amp, seed, ku, kp, refine_first);
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
void* ref_create_refined(int dim, int n_el, double amp, unsigned seed, int ku, int kp, int n_ref,
                         const int* refine) {
  try {
    if (dim == 2) return make_refined<2>(n_el, amp, seed, ku, kp, n_ref, refine);
    if (dim == 3) return make_refined<3>(n_el, amp, seed, ku, kp, n_ref, refine);
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
void ref_mesh_arrays(void* h, double* xv, int* cv, int* bid, double* emb_out) {
  static_cast<Base*>(h)->mesh_arrays(xv, cv, bid, emb_out);
}
void* ref_create_from_text(const char* text, int ku, int kp) {
  try {
    const std::string s(text);
    const int d = mesh_file_dim(s);
    if (d == 2) return new Ctx<2>(import_text<2>(s), ku, kp);
    return new Ctx<3>(import_text<3>(s), ku, kp);
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
void* ref_create_from_arrays(int dim, int nv, const double* xv, int nc, const int* cv, const int* bid, int ku,
                             int kp) {
  try {
    if (dim == 2) return new Ctx<2>(mesh_from_arrays<2>(nv, xv, nc, cv, bid), ku, kp);
    if (dim == 3) return new Ctx<3>(mesh_from_arrays<3>(nv, xv, nc, cv, bid), ku, kp);
    g_err = "mesh arrays: dim must be 2 or 3";
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
void* ref_create_cylinder(int level, int ku, int kp) {
  try {
    return new Ctx<2>(generate_cylinder_channel(level), ku, kp);
  } catch (const std::exception& e) {
    g_err = e.what();
  }
  return nullptr;
}
void ref_destroy(void* h) { delete static_cast<Base*>(h); }
void ref_info(void* h, long long* out) { static_cast<Base*>(h)->info(out); }
void ref_set_bc(void* h, int id, int type, ref_bc_fn fn, void* user) {
  static_cast<Base*>(h)->set_bc(id, type, fn, user);
}
int ref_apply_momentum(void* h, const double* c, const double* w, const double* x, double* y) {
  try {
    static_cast<Base*>(h)->momentum(c, w, x, y);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
int ref_momentum_diagonal(void* h, const double* c, const double* w, double* d) {
  try {
    static_cast<Base*>(h)->momentum_diag(c, w, d);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
void ref_apply_pressure(void* h, double mc, const double* x, double* y) {
  static_cast<Base*>(h)->pressure(mc, x, y);
}
void ref_helmholtz_diagonal(void* h, double mc, double* d) {
  static_cast<Base*>(h)->helmholtz_diag(mc, d);
}
void ref_apply_laplace(void* h, int dir, const double* x, double* y) {
  static_cast<Base*>(h)->laplace(dir, x, y);
}
void ref_laplace_diagonal(void* h, int dir, double* d) { static_cast<Base*>(h)->laplace_diag(dir, d); }
void ref_apply_mass(void* h, int space, const double* x, double* y) {
  static_cast<Base*>(h)->mass(space, x, y);
}
void ref_mass_diagonal(void* h, int space, double* d) { static_cast<Base*>(h)->mass_diag(space, d); }
int ref_momentum_rhs(void* h, int nm, const double* mc, const double* const* mf, int nv,
                     const double* vc, const double* const* vf, int na, const double* ac,
                     const double* const* af, const double* const* aw, int np, const double* pc,
                     const double* const* pf, double dvisc, double dadv, const double* dir_w,
                     double time, double* y) {
  try {
    static_cast<Base*>(h)->momentum_rhs(nm, mc, mf, nv, vc, vf, na, ac, af, aw, np, pc, pf, dvisc,
                                        dadv, dir_w, time, y);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
void ref_divergence(void* h, const double* u, double* y) { static_cast<Base*>(h)->divergence(u, y); }
void ref_pressure_rhs(void* h, double inv_adt, const double* u, double mc, const double* p_old,
                      double* y) {
  static_cast<Base*>(h)->pressure_rhs(inv_adt, u, mc, p_old, y);
}
void ref_pressure_gradient(void* h, const double* p, double* y) {
  static_cast<Base*>(h)->pressure_gradient(p, y);
}
double ref_kinetic_energy(void* h, const double* u) { return static_cast<Base*>(h)->kinetic_energy(u); }
int ref_solve(void* h, int op, int solver, const double* coefs, const double* w, const double* b,
              double rel_tol, double abs_tol, int max_iter, int restart, int precond, double* x,
              int* iters, double* resid, double* hist, int hist_cap, int* hist_len) {
  return static_cast<Base*>(h)->solve(op, solver, coefs, w, b, rel_tol, abs_tol, max_iter, restart,
                                      precond, x, iters, resid, hist, hist_cap, hist_len);
}
int ref_trbdf2_step(void* h, const double* params, const double* u_nm1, const double* u_n,
                    const double* p_n, double* u_np1, double* p_np1, int* its) {
  try {
    static_cast<Base*>(h)->step(params, u_nm1, u_n, p_n, u_np1, p_np1, its);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
int ref_scheme_step(void* h, int scheme, const double* params, const double* u_nm1, const double* u_n,
                    const double* p_n, double* u_np1, double* p_np1, int* its) {
  try {
    static_cast<Base*>(h)->scheme_step(scheme, params, u_nm1, u_n, p_n, u_np1, p_np1, its);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
void ref_faces(void* h, int* iface, double* imeas, int* bface, double* bmeas) {
  static_cast<Base*>(h)->faces(iface, imeas, bface, bmeas);
}
void ref_cell_vertices(void* h, double* xv) { static_cast<Base*>(h)->cell_vertices(xv); }
void ref_bface_points(void* h, int rule, double* xq) { static_cast<Base*>(h)->bface_points(rule, xq); }
void ref_node_points(void* h, int space, double* xn) { static_cast<Base*>(h)->interpolate_nodes(space, xn); }
double ref_bench(void* h, int op, const double* c, const double* w, const double* x, int nthreads,
                 int napplies) {
  return static_cast<Base*>(h)->bench(op, c, w, x, nthreads, napplies);
}
void ref_pair_setup(void* h, const double* c, const double* w, const double* x, double pmc, const double* xp) {
  static_cast<Base*>(h)->pair_setup(c, w, x, pmc, xp);
}
// `rounds` rounds; in each, every context runs pair_run() once, the contexts taken
// from a shared counter by `nthreads` host threads (the reference is single-
// threaded: parallelism is across independent contexts).  times[r] = wall seconds
// of round r.
void ref_pair_rounds(void** hs, int nh, int nthreads, int rounds, double* times) {
  for (int r = 0; r < rounds; ++r) {
    std::atomic<int> next{0};
    const auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> th;
    for (int t = 0; t < std::max(1, nthreads); ++t)
      th.emplace_back([&]() {
        for (int i; (i = next.fetch_add(1)) < nh;) static_cast<Base*>(hs[i])->pair_run();
      });
    for (auto& t : th) t.join();
    times[r] = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  }
}
void ref_dense_momentum(void* h, const double* c, const double* w, double* A) {
  static_cast<Base*>(h)->dense_momentum(c, w, A);
}
void ref_dense_scalar_sip(void* h, double mc, int dir, int rule, double* A) {
  static_cast<Base*>(h)->dense_scalar_sip(mc, dir, rule, A);
}

}  // extern "C"
