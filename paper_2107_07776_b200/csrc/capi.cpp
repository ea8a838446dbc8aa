// extern "C" entry points of libdgb.so (declared in include/dgb.h).
// Each call maps a reference operator / solver entry point onto the device
// context; exceptions never cross the boundary (status codes + last error).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <random>
#include <string>
#include <vector>

#include "../../include/dgb.h"
#include "blas.cuh"
#include "context.hpp"

using dgb::Context;


static thread_local std::string g_last_error;

static int ret(dgb_ctx* h, int status) {
  if (status != DGB_OK) g_last_error = h ? h->c.err : std::string("error");
  return status;
}
static int bad(const char* msg) {
  g_last_error = msg;
  return DGB_E_ARG;
}
#define NEED(cond, msg) \
  if (!(cond)) return bad(msg)


extern "C" {

const char* dgb_last_error(void) { return g_last_error.c_str(); }
const char* dgb_version(void) { return "dgb 0.1 sm_100a fp64 (element-centric matrix-free DG, TR-BDF2)"; }

static int finish_create(dgb::HostMesh&& m, int ku, int kp, int device, const std::string& merr, dgb_ctx** out) {
  if (m.ncells == 0) {
    g_last_error = merr.empty() ? "mesh construction failed" : merr;
    return merr.find("unsupported") != std::string::npos ? DGB_E_UNSUPPORTED : DGB_E_ARG;
  }
  dgb_ctx* h = new (std::nothrow) dgb_ctx;
  if (!h) return bad("out of host memory");
  std::string err;
  const int st = h->c.init(std::move(m), ku, kp, device, err);
  if (st != DGB_OK) {
    g_last_error = err;
    delete h;
    return st;
  }
  *out = h;
  return DGB_OK;
}

int dgb_ctx_create_cartesian(int dim, int n_el, double amp, unsigned seed, int ku, int kp, int device,
                             dgb_ctx** out) {
  NEED(out, "null out");
  NEED(dim == 2 || dim == 3, "dim must be 2 or 3");
  NEED(n_el >= 1, "n_el must be >= 1");
  std::string err;
  dgb::HostMesh m = dgb::make_cartesian(dim, n_el, amp, seed, err);
  return finish_create(std::move(m), ku, kp, device, err, out);
}

int dgb_ctx_create_mesh(int dim, int nverts, const double* verts, int ncells, const int* cell_vertices,
                        const int* boundary_ids, int ku, int kp, int device, dgb_ctx** out) {
  NEED(out && verts && cell_vertices, "null argument");
  NEED(dim == 2 || dim == 3, "dim must be 2 or 3");
  NEED(nverts > 0 && ncells > 0, "empty mesh");
  std::string err;
  dgb::HostMesh m = dgb::make_from_arrays(dim, nverts, verts, ncells, cell_vertices, boundary_ids, err);
  return finish_create(std::move(m), ku, kp, device, err, out);
}

int dgb_ctx_create_mesh_hanging(int dim, int nverts, const double* verts, int ncells, const int* cell_vertices,
                                const int* boundary_ids, int n_hang, const int* hang_faces, const double* hang_emb,
                                int ku, int kp, int device, dgb_ctx** out) {
  NEED(out && verts && cell_vertices, "null argument");
  NEED(dim == 2 || dim == 3, "dim must be 2 or 3");
  NEED(nverts > 0 && ncells > 0, "empty mesh");
  NEED(n_hang >= 0 && (n_hang == 0 || (hang_faces && hang_emb)), "hanging faces: bad record arrays");
  std::string err;
  dgb::HostMesh m = dgb::make_from_arrays(dim, nverts, verts, ncells, cell_vertices, boundary_ids, err, n_hang,
                                          hang_faces, hang_emb);
  return finish_create(std::move(m), ku, kp, device, err, out);
}

void dgb_ctx_destroy(dgb_ctx* h) {
  DevGuard guard_(h);
  delete h;
}

int dgb_ctx_info(dgb_ctx* h, long long* info) {
  DevGuard guard_(h);
  NEED(h && info, "null argument");
  const Context& c = h->c;
  for (int i = 0; i < 16; ++i) info[i] = 0;
  info[0] = c.mesh.ncells;
  info[1] = (long long)c.nu();
  info[2] = (long long)c.np();
  info[3] = (long long)(c.mesh.iface.size() / 4);
  info[4] = (long long)c.n_bface();
  info[5] = c.ku;
  info[6] = c.kp;
  info[7] = c.dim;
  info[8] = c.mesh.affine ? 1 : 0;
  info[9] = c.nqf(c.ku + 2);
  info[10] = c.device;
  info[11] = c.mesh.n_hang();
  return DGB_OK;
}

int dgb_set_stream(dgb_ctx* h, void* s) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  // NULL selects the legacy default stream (what torch's default current stream is)
  h->c.dc.stream = static_cast<cudaStream_t>(s);
  return DGB_OK;
}
void* dgb_get_stream(dgb_ctx* h) { return h ? static_cast<void*>(h->c.dc.stream) : nullptr; }

int dgb_sync(dgb_ctx* h) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  const cudaError_t e = cudaStreamSynchronize(h->c.dc.stream);
  if (e != cudaSuccess) return ret(h, h->c.cuda_fail(e, "dgb_sync"));
  return DGB_OK;
}

int dgb_set_boundary_type(dgb_ctx* h, int id, int type) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  NEED(id >= 0 && id < 64, "boundary id must be in [0, 64)");
  NEED(type == DGB_BC_DIRICHLET || type == DGB_BC_OUTLET, "bad boundary type");
  h->c.bctype_h[id] = type;
  if (type == DGB_BC_OUTLET)
    h->c.dc.ug.outlet_mask |= 1ull << id;
  else
    h->c.dc.ug.outlet_mask &= ~(1ull << id);
  const cudaError_t e = cudaMemcpyAsync(const_cast<int*>(h->c.dc.mesh.bctype), h->c.bctype_h, sizeof(h->c.bctype_h),
                                        cudaMemcpyHostToDevice, h->c.dc.stream);
  if (e != cudaSuccess) return ret(h, h->c.cuda_fail(e, "dgb_set_boundary_type"));
  cudaStreamSynchronize(h->c.dc.stream);
  return DGB_OK;
}
int dgb_set_debug(dgb_ctx* h, int flags) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  h->c.dc.mesh.poison = (flags & DGB_DEBUG_POISON_SMEM) ? 1 : 0;
  return DGB_OK;
}
int dgb_set_cell_range(dgb_ctx* h, int cell0, int cell1) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  NEED(cell0 >= 0 && (cell1 < 0 || (cell1 >= cell0 && cell1 <= h->c.mesh.ncells)), "bad cell range");
  // refined meshes: the subface kernels always cover every hanging face, so only the whole mesh
  NEED(!h->c.hang_ || (cell0 == 0 && (cell1 < 0 || cell1 == h->c.mesh.ncells)),
       "cell ranges are not defined on meshes with hanging faces");
  h->c.dc.mesh.cell0 = cell0;
  h->c.dc.mesh.cell1 = cell1;
  return DGB_OK;
}
int dgb_set_dirichlet_time_dependent(dgb_ctx* h, int enable) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  h->c.g_time_dep_ = enable != 0;
  return DGB_OK;
}
int dgb_set_dirichlet_table(dgb_ctx* h, const double* g) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  return ret(h, h->c.set_dirichlet_table(g));
}
int dgb_set_dirichlet_fn(dgb_ctx* h, int id, dgb_bc_fn fn, void* user, double t) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  return ret(h, h->c.set_dirichlet_fn(id, fn, user, t));
}
int dgb_boundary_points(dgb_ctx* h, int q1d, double* xq) {
  DevGuard guard_(h);
  NEED(h && xq, "null argument");
  NEED(q1d >= 1 && q1d <= 12, "bad rule");
  std::vector<double> v;
  dgb::boundary_points(h->c.mesh, q1d, v);
  std::memcpy(xq, v.data(), v.size() * sizeof(double));
  return DGB_OK;
}
int dgb_node_points(dgb_ctx* h, int space, double* xn) {
  DevGuard guard_(h);
  NEED(h && xn, "null argument");
  const Context& c = h->c;
  const int deg = space == DGB_SPACE_U ? c.ku : c.kp;
  const std::vector<double> nodes = dgb::gauss_lobatto(deg + 1);
  const int n1 = deg + 1;
  const int nb = c.dim == 2 ? n1 * n1 : n1 * n1 * n1;
  double ref[3], x[3];
  for (int cell = 0; cell < c.mesh.ncells; ++cell)
    for (int j = 0; j < nb; ++j) {
      int rem = j;
      for (int d = 0; d < c.dim; ++d) {
        ref[d] = nodes[rem % n1];
        rem /= n1;
      }
      dgb::map_point(c.mesh, cell, ref, x);
      for (int d = 0; d < c.dim; ++d) xn[((size_t)cell * nb + j) * c.dim + d] = x[d];
    }
  return DGB_OK;
}
int dgb_face_lists(dgb_ctx* h, int* interior, int* boundary) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  if (interior) std::memcpy(interior, h->c.mesh.iface.data(), h->c.mesh.iface.size() * sizeof(int));
  if (boundary) std::memcpy(boundary, h->c.mesh.bface.data(), h->c.mesh.bface.size() * sizeof(int));
  return DGB_OK;
}

// ------------------------------------------------------------------ memory
int dgb_alloc(dgb_ctx* h, size_t n, double** p) {
  DevGuard guard_(h);
  NEED(h && p, "null argument");
  cudaSetDevice(h->c.device);
  const cudaError_t e = cudaMalloc(reinterpret_cast<void**>(p), (n ? n : 1) * sizeof(double));
  if (e != cudaSuccess) return ret(h, h->c.cuda_fail(e, "dgb_alloc"));
  return DGB_OK;
}
int dgb_free(dgb_ctx* h, double* p) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  cudaStreamSynchronize(h->c.dc.stream);
  cudaFree(p);
  return DGB_OK;
}
static int cpy(dgb_ctx* h, void* dst, const void* src, size_t n, cudaMemcpyKind k, bool sync) {
  const cudaError_t e = cudaMemcpyAsync(dst, src, n * sizeof(double), k, h->c.dc.stream);
  if (e != cudaSuccess) return ret(h, h->c.cuda_fail(e, "copy"));
  if (sync) cudaStreamSynchronize(h->c.dc.stream);
  return DGB_OK;
}
int dgb_copy_h2d(dgb_ctx* h, double* d, const double* s, size_t n) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  return cpy(h, d, s, n, cudaMemcpyHostToDevice, true);
}
int dgb_copy_d2h(dgb_ctx* h, double* d, const double* s, size_t n) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  return cpy(h, d, s, n, cudaMemcpyDeviceToHost, true);
}
int dgb_copy_d2d(dgb_ctx* h, double* d, const double* s, size_t n) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  return cpy(h, d, s, n, cudaMemcpyDeviceToDevice, false);
}
int dgb_fill(dgb_ctx* h, double* x, double v, size_t n);

// ------------------------------------------------------------------ operators
int dgb_momentum_apply(dgb_ctx* h, const double* coefs, const double* w, const double* x, double* y) {
  DevGuard guard_(h);
  NEED(h && coefs && x && y, "null argument");
  NEED(x != y, "x and y must not alias");
  return ret(h, h->c.momentum(coefs, w, x, y));
}
int dgb_momentum_apply_host(dgb_ctx* h, const double* coefs, const double* h_w, const double* h_x, double* h_y) {
  DevGuard guard_(h);
  NEED(h && coefs && h_x && h_y, "null argument");
  NEED(h_x != h_y, "x and y must not alias");
  return ret(h, h->c.apply_host(true, coefs, 0.0, h_w, h_x, h_y));
}
int dgb_pressure_apply_host(dgb_ctx* h, double mc, const double* h_x, double* h_y) {
  DevGuard guard_(h);
  NEED(h && h_x && h_y, "null argument");
  NEED(h_x != h_y, "x and y must not alias");
  return ret(h, h->c.apply_host(false, nullptr, mc, nullptr, h_x, h_y));
}
int dgb_momentum_diag(dgb_ctx* h, const double* coefs, const double* w, double* d) {
  DevGuard guard_(h);
  NEED(h && coefs && d, "null argument");
  return ret(h, h->c.momentum_diag(coefs, w, d));
}
int dgb_pressure_apply(dgb_ctx* h, double mc, const double* x, double* y) {
  DevGuard guard_(h);
  NEED(h && x && y, "null argument");
  NEED(x != y, "x and y must not alias");
  return ret(h, h->c.sip(mc, 0, x, y));
}
int dgb_helmholtz_diag(dgb_ctx* h, double mc, double* d) {
  DevGuard guard_(h);
  NEED(h && d, "null argument");
  return ret(h, h->c.sip_diag(mc, 0, d));
}
int dgb_laplace_apply(dgb_ctx* h, int dir, const double* x, double* y) {
  DevGuard guard_(h);
  NEED(h && x && y, "null argument");
  NEED(x != y, "x and y must not alias");
  return ret(h, h->c.sip(0.0, dir != 0, x, y));
}
int dgb_laplace_diag(dgb_ctx* h, int dir, double* d) {
  DevGuard guard_(h);
  NEED(h && d, "null argument");
  return ret(h, h->c.sip_diag(0.0, dir != 0, d));
}
int dgb_mass_apply(dgb_ctx* h, int space, const double* x, double* y) {
  DevGuard guard_(h);
  NEED(h && x && y, "null argument");
  NEED(space == DGB_SPACE_U || space == DGB_SPACE_P, "bad space");
  return ret(h, h->c.mass(space, x, y));
}
int dgb_mass_diag(dgb_ctx* h, int space, double* d) {
  DevGuard guard_(h);
  NEED(h && d, "null argument");
  NEED(space == DGB_SPACE_U || space == DGB_SPACE_P, "bad space");
  return ret(h, h->c.mass_diag(space, d));
}
int dgb_momentum_rhs(dgb_ctx* h, const dgb_rhs_desc* desc, double* out) {
  DevGuard guard_(h);
  NEED(h && desc && out, "null argument");
  return ret(h, h->c.rhs(*desc, out));
}
int dgb_divergence(dgb_ctx* h, const double* u, double* out) {
  DevGuard guard_(h);
  NEED(h && u && out, "null argument");
  return ret(h, h->c.divergence(u, out));
}
int dgb_pressure_rhs(dgb_ctx* h, double inv_adt, const double* u, double mc, const double* p_old, double* out) {
  DevGuard guard_(h);
  NEED(h && u && out, "null argument");
  return ret(h, h->c.pressure_rhs(inv_adt, u, mc, p_old, out));
}
int dgb_pressure_gradient(dgb_ctx* h, const double* p, double* out) {
  DevGuard guard_(h);
  NEED(h && p && out, "null argument");
  return ret(h, h->c.gradient(p, out));
}
int dgb_kinetic_energy(dgb_ctx* h, const double* u, double* result) {
  DevGuard guard_(h);
  NEED(h && u && result, "null argument");
  return ret(h, h->c.kinetic(u, result));
}

int dgb_l2_norm(dgb_ctx* h, int space, const double* x, double* result) {
  DevGuard guard_(h);
  NEED(h && x && result, "null argument");
  NEED(space == DGB_SPACE_U || space == DGB_SPACE_P, "space must be 0 or 1");
  dgb::Context& c = h->c;
  const size_t n = space == DGB_SPACE_U ? c.nu() : c.np();
  double* mx = c.scratch_vec(19, n);
  NEED(mx, "out of device memory");
  int code = c.mass(space, x, mx);
  if (code == DGB_OK) code = c.dot(n, x, mx, result);
  if (code == DGB_OK) *result = std::sqrt(std::max(*result, 0.0));
  return ret(h, code);
}
int dgb_check_steady(dgb_ctx* h, const double* un, const double* uo, double tol, int* steady, double* diff) {
  DevGuard guard_(h);
  NEED(h && un && uo && steady && diff, "null argument");
  const int code = h->c.max_abs_diff(h->c.nu(), un, uo, diff);
  *steady = code == DGB_OK && *diff < tol;
  return ret(h, code);
}
int dgb_stability_params(dgb_ctx* h, double dt, double Re, double U, double* C, double* mu) {
  DevGuard guard_(h);
  NEED(h && C && mu, "null argument");
  NEED(Re > 0.0, "Re must be positive");
  const auto& d = h->c.mesh.cell_diam;
  double H = d.empty() ? 0.0 : d[0];
  for (double v : d) H = std::min(H, v);
  NEED(H > 0.0, "empty mesh");
  const double k = h->c.ku;
  *C = k * U * dt / H;
  *mu = k * k * dt / (Re * H * H);
  return DGB_OK;
}

// ------------------------------------------------------------------ vectors
int dgb_axpy(dgb_ctx* h, size_t n, double a, const double* x, double* y) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  ++h->c.launches;
  const cudaError_t e = dgb::v_axpy(h->c.dc.stream, n, a, x, y);
  return e == cudaSuccess ? DGB_OK : ret(h, h->c.cuda_fail(e, "dgb_axpy"));
}
int dgb_axpby(dgb_ctx* h, size_t n, double a, const double* x, double b, double* y) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  ++h->c.launches;
  const cudaError_t e = dgb::v_axpby(h->c.dc.stream, n, a, x, b, y);
  return e == cudaSuccess ? DGB_OK : ret(h, h->c.cuda_fail(e, "dgb_axpby"));
}
int dgb_scal(dgb_ctx* h, size_t n, double a, double* x) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  ++h->c.launches;
  const cudaError_t e = dgb::v_scal(h->c.dc.stream, n, a, x);
  return e == cudaSuccess ? DGB_OK : ret(h, h->c.cuda_fail(e, "dgb_scal"));
}
int dgb_fill(dgb_ctx* h, double* x, double v, size_t n) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  ++h->c.launches;
  const cudaError_t e = dgb::v_fill(h->c.dc.stream, n, v, x);
  return e == cudaSuccess ? DGB_OK : ret(h, h->c.cuda_fail(e, "dgb_fill"));
}
int dgb_dot(dgb_ctx* h, size_t n, const double* x, const double* y, double* result) {
  DevGuard guard_(h);
  NEED(h && result, "null argument");
  return ret(h, h->c.dot(n, x, y, result));
}
int dgb_norm(dgb_ctx* h, size_t n, const double* x, double* result) {
  DevGuard guard_(h);
  NEED(h && result, "null argument");
  double s = 0.0;
  const int st = h->c.dot(n, x, x, &s);
  if (st != DGB_OK) return ret(h, st);
  *result = std::sqrt(s);
  return DGB_OK;
}
int dgb_max_abs_diff(dgb_ctx* h, size_t n, const double* x, const double* y, double* result) {
  DevGuard guard_(h);
  NEED(h && result, "null argument");
  return ret(h, h->c.max_abs_diff(n, x, y, result));
}

// ------------------------------------------------------------------ solvers
int dgb_jacobi_inverse(dgb_ctx* h, size_t n, const double* d, double* inv) {
  DevGuard guard_(h);
  NEED(h && d && inv, "null argument");
  return ret(h, h->c.jacobi_inverse(n, d, inv));
}
static int solve(dgb_ctx* h, bool gm, const dgb_operator* op, const dgb_solver_settings* s, const double* inv,
                 const double* b, double* x, dgb_solve_result* res, double* hist, int cap, int* hlen) {
  NEED(h && op && s && b && x && res, "null argument");
  dgb::SolveOut so;
  const int st = gm ? h->c.gmres(*op, *s, inv, b, x, so) : h->c.cg(*op, *s, inv, b, x, so);
  res->iterations = so.iterations;
  res->residual = so.residual;
  if (hlen) *hlen = (int)so.history.size();
  if (hist)
    for (int i = 0; i < cap && i < (int)so.history.size(); ++i) hist[i] = so.history[i];
  return ret(h, st);
}
int dgb_cg(dgb_ctx* h, const dgb_operator* op, const dgb_solver_settings* s, const double* inv, const double* b,
           double* x, dgb_solve_result* res, double* hist, int cap, int* hlen) {
  DevGuard guard_(h);
  return solve(h, false, op, s, inv, b, x, res, hist, cap, hlen);
}
int dgb_gmres(dgb_ctx* h, const dgb_operator* op, const dgb_solver_settings* s, const double* inv, const double* b,
              double* x, dgb_solve_result* res, double* hist, int cap, int* hlen) {
  DevGuard guard_(h);
  return solve(h, true, op, s, inv, b, x, res, hist, cap, hlen);
}

int dgb_pressure_cg_mg(dgb_ctx* h, double mc, const dgb_solver_settings* s, const double* b, double* x,
                       dgb_solve_result* res) {
  DevGuard guard_(h);
  NEED(h && s && b && x && res, "null argument");
  dgb::SolveOut out;
  const int code = h->c.cg_mg(mc, *s, b, x, out);
  res->iterations = out.iterations;
  res->residual = out.residual;
  return ret(h, code);
}
int dgb_pressure_mg_vcycle(dgb_ctx* h, double mc, const double* r, double* z) {
  DevGuard guard_(h);
  NEED(h && r && z, "null argument");
  return ret(h, h->c.mg_precondition(mc, r, z));
}

int dgb_projection_step(dgb_ctx* h, int scheme, const dgb_step_params* p, const double* u_nm1, const double* u_n,
                        const double* p_n, double* u_np1, double* p_np1, int* its) {
  DevGuard guard_(h);
  NEED(h && p && u_n && p_n && u_np1 && p_np1 && its, "null argument");
  NEED(scheme >= DGB_SCHEME_TRBDF2 && scheme <= DGB_SCHEME_GQ_BDF2, "unknown scheme");
  NEED(p->first_step || u_nm1 || scheme == DGB_SCHEME_BCG, "u_nm1 required after the first step");
  return ret(h, h->c.projection_step(scheme, *p, u_nm1, u_n, p_n, u_np1, p_np1, its));
}
int dgb_trbdf2_step(dgb_ctx* h, const dgb_step_params* p, const double* u_nm1, const double* u_n,
                    const double* p_n, double* u_np1, double* p_np1, int* its) {
  DevGuard guard_(h);
  NEED(h && p && u_n && p_n && u_np1 && p_np1 && its, "null argument");
  NEED(p->first_step || u_nm1, "u_nm1 required after the first step");
  return ret(h, h->c.trbdf2_step(*p, u_nm1, u_n, p_n, u_np1, p_np1, its));
}

// ------------------------------------------------------------------ synthetic inputs
int dgb_seeded_uniform(unsigned long long seed, size_t n, double lo, double hi, double* out) {
  NEED(out || n == 0, "null out");
  std::mt19937_64 rng(seed);
  for (size_t i = 0; i < n; ++i) out[i] = lo + (hi - lo) * ((double)(rng() >> 11) * 0x1.0p-53);
  return DGB_OK;
}

// user layout: [0] dim, [1] scale, [2] nmodes, then per potential component c and
// mode: (a, phi); modes lexicographic over {1..4}^dim, last index fastest.
int dgb_synth_init(int dim, unsigned long long seed, double scale, double* user) {
  NEED(user, "null user");
  NEED(dim == 2 || dim == 3, "dim must be 2 or 3");
  std::mt19937_64 rng(seed);
  auto uni = [&]() { return (double)(rng() >> 11) * 0x1.0p-53; };
  const int nm = dim == 2 ? 16 : 64;
  const int ncomp = dim == 2 ? 1 : 3;
  user[0] = dim;
  user[1] = scale;
  user[2] = nm;
  int k = 3;
  for (int c = 0; c < ncomp; ++c)
    for (int m = 0; m < nm; ++m) {
      int idx[3];
      int rem = m;
      for (int d = dim - 1; d >= 0; --d) {
        idx[d] = 1 + rem % 4;
        rem /= 4;
      }
      double k2 = 0.0;
      for (int d = 0; d < dim; ++d) k2 += idx[d] * idx[d];
      const double u1 = uni(), u2 = uni();
      const double normal = std::sqrt(-2.0 * std::log(1.0 - u1)) * std::cos(2.0 * M_PI * u2);  // Box-Muller
      user[k++] = normal / k2;
      user[k++] = 2.0 * M_PI * uni();
    }
  return DGB_OK;
}

void dgb_synth_eval(const double* x, double /*t*/, double* out, void* user) {
  const double* u = static_cast<const double*>(user);
  const int dim = (int)u[0];
  const double scale = u[1];
  const int nm = (int)u[2];
  const double tp = 2.0 * M_PI;
  if (dim == 2) {  // u = (dpsi/dy, -dpsi/dx)
    double dx = 0.0, dy = 0.0;
    for (int m = 0; m < nm; ++m) {
      const int i0 = 1 + (m / 4), i1 = 1 + (m % 4);
      const double a = u[3 + 2 * m], ph = u[4 + 2 * m];
      const double cth = std::cos(tp * (i0 * x[0] + i1 * x[1]) + ph);
      dx += a * tp * i0 * cth;
      dy += a * tp * i1 * cth;
    }
    out[0] = scale * dy;
    out[1] = -scale * dx;
    return;
  }
  double G[3][3] = {};  // G[c][j] = dA_c / dx_j
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

int dgb_interpolate_synth(dgb_ctx* h, const double* user, double* hu) {
  DevGuard guard_(h);
  NEED(h && user && hu, "null argument");
  const Context& c = h->c;
  const int n1 = c.ku + 1;
  const int nb = c.dim == 2 ? n1 * n1 : n1 * n1 * n1;
  const std::vector<double> nodes = dgb::gauss_lobatto(n1);
  double ref[3], x[3], v[3];
  for (int cell = 0; cell < c.mesh.ncells; ++cell)
    for (int j = 0; j < nb; ++j) {
      int rem = j;
      for (int d = 0; d < c.dim; ++d) {
        ref[d] = nodes[rem % n1];
        rem /= n1;
      }
      dgb::map_point(c.mesh, cell, ref, x);
      dgb_synth_eval(x, 0.0, v, const_cast<double*>(user));
      for (int comp = 0; comp < c.dim; ++comp) hu[(size_t)cell * c.dim * nb + comp * nb + j] = v[comp];
    }
  return DGB_OK;
}

// ------------------------------------------------------------------ measurement
int dgb_timer_start(dgb_ctx* h) {
  DevGuard guard_(h);
  NEED(h, "null ctx");
  cudaEventRecord(h->c.ev0, h->c.dc.stream);
  return DGB_OK;
}
int dgb_timer_stop(dgb_ctx* h, float* ms) {
  DevGuard guard_(h);
  NEED(h && ms, "null argument");
  cudaEventRecord(h->c.ev1, h->c.dc.stream);
  cudaEventSynchronize(h->c.ev1);
  const cudaError_t e = cudaEventElapsedTime(ms, h->c.ev0, h->c.ev1);
  if (e != cudaSuccess) return ret(h, h->c.cuda_fail(e, "dgb_timer_stop"));
  return DGB_OK;
}
long long dgb_launch_count(dgb_ctx* h) {
  DevGuard guard_(h); return h ? h->c.launches : 0; }

}  // extern "C"

// ------------------------------------------------------------------ host-only inspection
// Builds the host mesh exactly as context creation does (no GPU needed) and
// returns sizes / face lists / measures, so the host setup can be checked
// against the reference's Mesh on CPU-only machines.
extern "C" int dgb_host_mesh_cartesian(int dim, int n_el, double amp, unsigned seed, long long* sizes,
                                       int* iface, int* bface, double* cell_measure, double* face_measure,
                                       double* vertices) {
  NEED(sizes, "null sizes");
  std::string err;
  dgb::HostMesh m = dgb::make_cartesian(dim, n_el, amp, seed, err);
  if (m.ncells == 0) return bad(err.c_str());
  sizes[0] = m.ncells;
  sizes[1] = (long long)(m.iface.size() / 4);
  sizes[2] = (long long)(m.bface.size() / 3);
  sizes[3] = m.affine ? 1 : 0;
  sizes[4] = (long long)(m.vertices.size() / dim);
  if (iface) std::memcpy(iface, m.iface.data(), m.iface.size() * sizeof(int));
  if (bface) std::memcpy(bface, m.bface.data(), m.bface.size() * sizeof(int));
  if (cell_measure) std::memcpy(cell_measure, m.cell_measure.data(), m.cell_measure.size() * sizeof(double));
  if (face_measure) std::memcpy(face_measure, m.face_measure.data(), m.face_measure.size() * sizeof(double));
  if (vertices) std::memcpy(vertices, m.vertices.data(), m.vertices.size() * sizeof(double));
  return DGB_OK;
}

// 1D tables used by the kernels: B[q][n], D[q][n], dE[2][n], w[q]
extern "C" int dgb_host_tables(int n, int q, double* B, double* D, double* dE, double* w) {
  NEED(n >= 2 && n <= 8 && q >= 1 && q <= 12, "bad sizes");
  dgb::host_tab(n, q, B, D, dE);
  dgb::host_w(q, w);
  return DGB_OK;
}

// Route axis-aligned 3D applies to the fast kernels (1, default) or force the
// generic kernels (0).  Both are parity-tested against the reference.
extern "C" int dgb_set_fast_path(dgb_ctx* h, int enable) {
  NEED(h, "null ctx");
  // refined meshes: the fast kernels only where their cells are axis-aligned (hang_fast_ok)
  h->c.use_fast = enable != 0 && (!h->c.hang_ || h->c.hang_fast_ok);
  return DGB_OK;
}
extern "C" int dgb_hanging_mode(dgb_ctx* h) { return h ? dgb::hang_mode(h->c.hang_) : 0; }
// 1: axis-aligned fast kernels (fast_axis.cuh), 2: deformed 3D fast kernels (fast_deformed.cuh), 0: generic
extern "C" int dgb_fast_path_active(dgb_ctx* h) {
  if (!h || !h->c.use_fast || h->c.dim != 3) return 0;
  return h->c.dc.axis ? 1 : (!h->c.dc.affine ? 2 : 0);
}
