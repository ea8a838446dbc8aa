// Device context: mesh + geometry resident in HBM, the operator tables for
// the two spaces, reduction scratch, Krylov workspaces, and the C++ methods
// behind the C-ABI (capi.cpp).
#pragma once

#include <cuda_runtime.h>

#include <string>
#include <utility>
#include <vector>

#include "../../include/dgb.h"
#include "dispatch.hpp"
#include "blas.cuh"
#include "host_setup.hpp"
#include "hang.hpp"

namespace dgb {

struct SolveOut {
  int iterations = 0;
  double residual = 0.0;
  std::vector<double> history;
};

struct MgHierarchy;
void mg_release(MgHierarchy* h);

class Context {
 public:
  int dim = 0, ku = 0, kp = 0, device = 0;
  HostMesh mesh;
  DevCtx dc;
  const OpTable* opu = nullptr;  // velocity-degree table
  const OpTable* opp = nullptr;  // scalar-degree table
  cudaStream_t own_stream = nullptr;
  int bctype_h[64] = {};
  long long launches = 0;
  bool use_fast = true;  // route axis-aligned 3D applies to fast_axis.cuh
  bool hang_fast_ok = false;  // refined mesh whose cells are all axis-aligned boxes: fast kernels + hang.cu
  HangState* hang_ = nullptr;  // hanging-subface supplement (refined meshes; hang.cu), else null

  ~Context();
  int init(HostMesh&& m, int ku, int kp, int device, std::string& err);

  size_t nu() const { return (size_t)mesh.ncells * dim * ipow(ku + 1, dim); }
  size_t np() const { return (size_t)mesh.ncells * ipow(kp + 1, dim); }
  static size_t ipow(int b, int e) {
    size_t r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
  }
  int nqf(int q1d) const { return dim == 3 ? q1d * q1d : q1d; }
  size_t n_bface() const { return mesh.bface.size() / 3; }

  // operators (status = DGB_*)
  int momentum(const double* coefs, const double* w, const double* x, double* y);
  int momentum_diag(const double* coefs, const double* w, double* d);
  int sip(double mc, int dir, const double* x, double* y);
  // host-buffer applies (blocking): H2D, apply, D2H pipelined over z-slabs when possible
  int apply_host(bool momentum_op, const double* coefs, double mc, const double* h_w, const double* h_x,
                 double* h_y);
  int sip_diag(double mc, int dir, double* d);
  int mass(int space, const double* x, double* y);
  int mass_diag(int space, double* d);
  int rhs(const dgb_rhs_desc& desc, double* y);
  int divergence(const double* u, double* y);
  int pressure_rhs(double inv_adt, const double* u, double mc, const double* p_old, double* y);
  int gradient(const double* p, double* y);
  int kinetic(const double* u, double* out);
  int apply_op(const dgb_operator& op, const double* x, double* y);
  size_t op_size(const dgb_operator& op) const;

  // vectors
  int dot(size_t n, const double* x, const double* y, double* out);
  int max_abs_diff(size_t n, const double* x, const double* y, double* out);
  int jacobi_inverse(size_t n, const double* d, double* inv);

  // solvers (krylov.cpp:43-207 control flow)
  int cg(const dgb_operator& op, const dgb_solver_settings& s, const double* inv, const double* b, double* x,
         SolveOut& out);
  int gmres(const dgb_operator& op, const dgb_solver_settings& s, const double* inv, const double* b, double* x,
            SolveOut& out);

  // pressure multigrid preconditioner (mg.cu; uniform Cartesian 3D meshes)
  bool mg_supported() const;
  int mg_setup(double mc);
  int mg_precondition(double mc, const double* r, double* z);
  int cg_mg(double mc, const dgb_solver_settings& s, const double* b, double* x, SolveOut& out);

  // TR-BDF2 step
  int trbdf2_step(const dgb_step_params& p, const double* u_nm1, const double* u_n, const double* p_n,
                  double* u_np1, double* p_np1, int* its);
  int projection_step(int scheme, const dgb_step_params& p, const double* u_nm1, const double* u_n,
                      const double* p_n, double* u_np1, double* p_np1, int* its);

  // Dirichlet data
  int set_dirichlet_table(const double* g);
  int set_dirichlet_fn(int id, dgb_bc_fn fn, void* user, double t);
  int tabulate_dirichlet(int id, dgb_bc_fn fn, void* user, double t);
  int dirichlet_at(double t);  // re-tabulate time-dependent data at t (no-op otherwise)
  std::pair<dgb_bc_fn, void*> bc_fn_[64] = {};
  bool g_time_dep_ = false;
  double g_time_ = 0.0;

  // device scratch helpers
  double* scratch_vec(int slot, size_t n);  // persistent per-slot device buffers
  int fail(int code, const std::string& msg);
  int cuda_fail(cudaError_t e, const char* where);
  int host_scalars(int n, double* out);  // copy d_res[0..n) to host (syncs)

  std::string err;
  cudaStream_t stream() const { return dc.stream; }
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;

 private:
  // device allocations owned by the context
  std::vector<void*> allocs_;
  void* dalloc(size_t bytes);
  double* d_partial_ = nullptr;  // reduction partials
  double* d_res_ = nullptr;      // reduction results (device)
  double* h_res_ = nullptr;      // pinned host mirror
  long long* d_bad_ = nullptr;
  double* d_gtab_ = nullptr;
  std::vector<double> gtab_h_;
  std::vector<std::pair<double*, size_t>> slots_;
  std::vector<double*> gm_basis_;  // GMRES basis slots (offset into gm_raw_)
  std::vector<double*> gm_raw_;    // their allocations
  CgState* d_cg_ = nullptr;         // device-resident CG scalars
  CgState* h_cg_ = nullptr;         // pinned: [0..1] polled status, [2] staging
  double* d_hist_ = nullptr;        // device residual history
  size_t hist_cap_ = 0;
  double* h_gm_ = nullptr;          // pinned GMRES Hessenberg column
  size_t h_gm_cap_ = 0;
  cudaEvent_t poll_ev_[2] = {nullptr, nullptr};
  // host-buffer pipeline: two copy streams + per-slab events
  static constexpr int kMaxSlabs = 32;
  cudaStream_t cp_in_ = nullptr, cp_out_ = nullptr;
  cudaStream_t cap_stream_ = nullptr;  // CUDA-graph capture of the CG batches
  cudaEvent_t ev_start_ = nullptr, ev_in_[kMaxSlabs] = {}, ev_k_[kMaxSlabs] = {};
  size_t gm_n_ = 0;
  int ensure_geometry();
  MgHierarchy* mg_ = nullptr;
  mutable int mg_topo_n_ = -1;  // Cartesian topology size (0: none), computed on first use
  mutable double mg_side_ = 0.0;
  int mg_level_apply(int l, const double* x, double* y);
  int mg_smooth(int l, const double* b, double* x, bool zero_start);
  int mg_restrict(int l, const double* r_fine, double* r_coarse);
  int mg_prolong_add(int l, const double* x_coarse, double* x_fine);
  int mg_vcycle(int l, const double* b, double* x);
  int mg_lambda_max(int l, double& lmax);
};

}  // namespace dgb

// opaque handle of the C-ABI
struct dgb_ctx {
  dgb::Context c;
};

// Every entry point that touches device state runs on the context's device and
// restores the caller's current device on return (a context created on
// device N and used while another device is current).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(const dgb_ctx* h) {
    if (h && cudaGetDevice(&prev) == cudaSuccess && prev != h->c.device) cudaSetDevice(h->c.device);
    else prev = -1;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

