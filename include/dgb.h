/* dgb.h — C-ABI of the B200 DG / TR-BDF2 hot path (libdgb.so).
 *
 * Drop-in boundary for the reference's operator/solver interface
 * (/root/reference/proj/src/forms.hpp, krylov.hpp).  Every entry point takes
 * plain pointers and sizes; field pointers named d_* are DEVICE pointers in the
 * reference DoF layout (space.hpp:5-8):
 *     dof = cell * (n_comp * nb) + comp * nb + node,  node lexicographic, x fastest,
 * on Gauss-Lobatto nodes.  Outputs are overwritten (the reference zeroes them,
 * e.g. forms.cpp:394 `out.assign(n, 0)`), inputs and outputs never alias.
 * All calls return a status code; dgb_last_error() has the message.
 * Work is enqueued on the context stream; results are complete after
 * dgb_sync() (or any call that returns host scalars).
 */
#ifndef DGB_H
#define DGB_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct dgb_ctx dgb_ctx;

enum {
  DGB_OK = 0,
  DGB_E_ARG = 1,            /* bad argument / shape                              */
  DGB_E_NO_CONVERGENCE = 2, /* SolverError "no convergence" (krylov.cpp:64,128)  */
  DGB_E_BREAKDOWN = 3,      /* SolverError "breakdown, <r,z> = 0" (krylov.cpp:78) */
  DGB_E_NOT_SPD = 4,        /* SolverError "<p,Ap> <= 0" (krylov.cpp:89)          */
  DGB_E_ZERO_DIAG = 5,      /* JacobiPreconditioner zero diagonal (krylov.cpp:30) */
  DGB_E_CUDA = 6,           /* CUDA runtime failure                              */
  DGB_E_UNSUPPORTED = 7,    /* configuration outside the device path             */
  DGB_E_MISSING_FIELD = 8   /* runtime_error "advecting field missing" (forms.cpp:499) */
};

/* Boundary condition types (forms.hpp:27 BcType). */
enum { DGB_BC_DIRICHLET = 0, DGB_BC_OUTLET = 1 };
/* Spaces: velocity (n_comp = dim, degree ku) and pressure (scalar, degree kp). */
enum { DGB_SPACE_U = 0, DGB_SPACE_P = 1 };

/* Thread-local message of the last failing call (any context). */
const char* dgb_last_error(void);
/* Build identification, e.g. "dgb sm_100a fp64". */
const char* dgb_version(void);

/* ------------------------------------------------------------------ context */
/* Unit-box Cartesian mesh generate_cartesian<dim>(n_el, 0, 1) (mesh.cpp:571-616),
 * optionally distort(mesh, amp, seed) (mesh.cpp:618-646); spaces FunctionSpace(mesh,
 * ku, dim) and FunctionSpace(mesh, kp, 1) (space.cpp:188-203). */
int dgb_ctx_create_cartesian(int dim, int n_el, double distort_amp, unsigned distort_seed, int ku,
                             int kp, int device, dgb_ctx** out);
/* Conforming mesh from raw arrays: vertices [nverts][dim], cell vertices
 * [ncells][2^dim] (lexicographic, mesh.hpp:6-7), boundary ids [ncells][2dim]
 * (-1 = interior; local face 2*axis+side).  Every interior face must pair
 * opposite sides with identical corner order (Cartesian topology). */
int dgb_ctx_create_mesh(int dim, int nverts, const double* verts, int ncells, const int* cell_vertices,
                        const int* boundary_ids, int ku, int kp, int device, dgb_ctx** out);
/* Mesh with hanging faces (1-irregular refinement: Mesh::refine_and_coarsen, mesh.hpp:125-128;
 * subface records mesh.cpp:344-375).  The arrays are the active cells as above plus, for
 * every hanging subface (FaceInfo with hanging == true, mesh.hpp:46-57; its cell_in is the
 * fine cell): hang_faces [n_hang][4] = fine cell, fine face, coarse cell, coarse face (active
 * indices), hang_emb [n_hang][dim*dim] = emb_out.origin[dim] then emb_out.tangent[t][dim],
 * t < dim-1 (the subface in the coarse cell's reference coordinates).  Conforming faces
 * must pair as in dgb_ctx_create_mesh.  Such meshes run the generic kernels plus the
 * subface kernels (hang.cu); the fast paths and the pressure multigrid are off. */
int dgb_ctx_create_mesh_hanging(int dim, int nverts, const double* verts, int ncells, const int* cell_vertices,
                                const int* boundary_ids, int n_hang, const int* hang_faces, const double* hang_emb,
                                int ku, int kp, int device, dgb_ctx** out);
void dgb_ctx_destroy(dgb_ctx* ctx);
/* info[16]: ncells, n_u, n_p, n_interior_faces, n_boundary_faces, ku, kp, dim, affine,
 *           nqf_bdry (points per boundary face at rule ku+2), device, n_hanging_subfaces, 0... */
int dgb_ctx_info(dgb_ctx* ctx, long long* info);
/* Use an external cudaStream_t (NULL = the legacy default stream); a new context uses its own stream. */
int dgb_set_stream(dgb_ctx* ctx, void* cuda_stream);
void* dgb_get_stream(dgb_ctx* ctx);
int dgb_sync(dgb_ctx* ctx);

/* Boundary table (forms.hpp:29-51): type per boundary id (default Dirichlet). */
int dgb_set_boundary_type(dgb_ctx* ctx, int boundary_id, int type);
/* Dirichlet data g tabulated at the boundary-face quadrature points of rule ku+2,
 * host array [n_boundary_faces][nqf][dim] in the reference boundary-face order
 * (mesh.cpp:316-327).  NULL clears (g = 0). */
int dgb_set_dirichlet_table(dgb_ctx* ctx, const double* g_host);
/* Callback form of BoundaryTable::Entry::value: tabulates g(x, t) for every
 * boundary face with this id and uploads it. */
typedef void (*dgb_bc_fn)(const double* x, double t, double* out, void* user);
int dgb_set_dirichlet_fn(dgb_ctx* ctx, int boundary_id, dgb_bc_fn fn, void* user, double t);
/* Time-dependent Dirichlet data (MomentumRhs::time, forms.cpp:1061-1062): with enable != 0
 * the callbacks registered by dgb_set_dirichlet_fn (kept, non-owning: fn / user must stay
 * valid) are re-evaluated at every stage time t* inside dgb_trbdf2_step /
 * dgb_projection_step (t^n + gamma dt, t^n + dt).  Off by default: BASELINE data is
 * time-independent and one tabulation serves every step. */
int dgb_set_dirichlet_time_dependent(dgb_ctx* ctx, int enable);
/* Multi-GPU z-slabs (paper_2107_07776_b200/slabs.py): the fast 3D operator
 * applies (momentum, pressure / Laplacian) compute only cells [cell0, cell1) of the
 * context (the rank's owned cells; the others are ghost cells whose values the halo
 * exchange supplies) and leave the other rows of the output untouched.  cell1 < 0 =
 * all cells (the default).  Other kernels (and the momentum apply at k = 4, which has
 * no axis-aligned fast kernel) compute every cell.  Meshes with hanging faces accept only
 * the whole mesh (DGB_E_ARG otherwise): their subface kernels always cover every subface. */
int dgb_set_cell_range(dgb_ctx* ctx, int cell0, int cell1);
/* Debug switches.  DGB_DEBUG_POISON_SMEM: every operator kernel first fills its dynamic
 * shared memory with NaN, so a stage reading a value no earlier stage of the launch wrote
 * (an uninitialised read / missing barrier) changes the result (tests/test_gpu_race.py). */
enum { DGB_DEBUG_POISON_SMEM = 1 };
int dgb_set_debug(dgb_ctx* ctx, int flags);
/* Physical coordinates of boundary-face quadrature points of rule q1d,
 * [n_boundary_faces][nqf][dim] (GeometryCache::boundary_faces().xq). */
int dgb_boundary_points(dgb_ctx* ctx, int q1d, double* xq_host);
/* Physical coordinates of the nodal points of a space, [ncells][nb][dim]. */
int dgb_node_points(dgb_ctx* ctx, int space, double* xn_host);
/* Host copies of the face lists: interior [n][4] = cell_in, face_in, cell_out,
 * face_out; boundary [n][3] = cell, face, boundary_id (reference order). */
int dgb_face_lists(dgb_ctx* ctx, int* interior, int* boundary);

/* ------------------------------------------------------------------ memory */
int dgb_alloc(dgb_ctx* ctx, size_t n_doubles, double** d_ptr);
int dgb_free(dgb_ctx* ctx, double* d_ptr);
int dgb_copy_h2d(dgb_ctx* ctx, double* d_dst, const double* h_src, size_t n);
int dgb_copy_d2h(dgb_ctx* ctx, double* h_dst, const double* d_src, size_t n);
int dgb_copy_d2d(dgb_ctx* ctx, double* d_dst, const double* d_src, size_t n);
int dgb_fill(dgb_ctx* ctx, double* d_x, double value, size_t n);

/* ------------------------------------------------------------------ operators */
/* coefs = {mass, visc, adv, skew} (MomentumCtx, forms.hpp:56-64).  d_w may be NULL
 * only when adv == skew == 0. */
/* replaces apply_momentum (forms.hpp:111-113, forms.cpp:389-604) */
int dgb_momentum_apply(dgb_ctx* ctx, const double* coefs, const double* d_w, const double* d_x, double* d_y);
/* replaces momentum_diagonal (forms.hpp:114-116, forms.cpp:606-810) */
int dgb_momentum_diag(dgb_ctx* ctx, const double* coefs, const double* d_w, double* d_diag);
/* replaces apply_pressure_helmholtz (forms.hpp:126-128, forms.cpp:1090-1095) */
int dgb_pressure_apply(dgb_ctx* ctx, double mass_coef, const double* d_x, double* d_y);
/* Host-buffer variants (blocking; the result is in h_y on return): the same operators
 * on HOST arrays, the reference's calling convention (apply_momentum(V, geom, ctx, x,
 * out) with host Fields).  On uniform Cartesian 3D meshes the host->device copies, the
 * apply and the device->host copy are pipelined over z-slabs on separate streams
 * (overlap needs page-locked buffers); otherwise copy in / apply / copy out. */
int dgb_momentum_apply_host(dgb_ctx* ctx, const double* coefs, const double* h_w, const double* h_x, double* h_y);
int dgb_pressure_apply_host(dgb_ctx* ctx, double mass_coef, const double* h_x, double* h_y);
/* replaces helmholtz_diagonal (forms.hpp:129-131, forms.cpp:1097-1102) */
int dgb_helmholtz_diag(dgb_ctx* ctx, double mass_coef, double* d_diag);
/* replaces apply_scalar_laplace / scalar_laplace_diagonal on the scalar space (forms.hpp:157-162) */
int dgb_laplace_apply(dgb_ctx* ctx, int dirichlet_bdry, const double* d_x, double* d_y);
int dgb_laplace_diag(dgb_ctx* ctx, int dirichlet_bdry, double* d_diag);
/* replaces apply_mass / mass_diagonal (forms.hpp:105-109) */
int dgb_mass_apply(dgb_ctx* ctx, int space, const double* d_x, double* d_y);
int dgb_mass_diag(dgb_ctx* ctx, int space, double* d_diag);

/* MomentumRhs (forms.hpp:89-100): up to 4 terms per list; pressure fields live
 * in the pressure space.  Dirichlet data comes from the context's table. */
typedef struct {
  int n_mass, n_visc, n_adv, n_pres;
  double mass_coef[4], visc_coef[4], adv_coef[4], pres_coef[4];
  const double* mass_f[4];
  const double* visc_f[4];
  const double* adv_f[4];
  const double* adv_w[4];
  const double* pres_f[4];
  double dir_visc_coef, dir_adv_coef;
  const double* dir_w;
} dgb_rhs_desc;
/* replaces momentum_rhs (forms.hpp:118-120, forms.cpp:816-1084) */
int dgb_momentum_rhs(dgb_ctx* ctx, const dgb_rhs_desc* desc, double* d_out);
/* replaces divergence_functional (forms.hpp:136-139, forms.cpp:1118-1197) */
int dgb_divergence(dgb_ctx* ctx, const double* d_u, double* d_out);
/* replaces pressure_rhs (forms.hpp:142-145, forms.cpp:1199-1210); d_p_old may be NULL */
int dgb_pressure_rhs(dgb_ctx* ctx, double inv_adt, const double* d_u, double mass_coef,
                     const double* d_p_old, double* d_out);
/* replaces pressure_gradient_rhs (forms.hpp:149-150, forms.cpp:1212-1233) */
int dgb_pressure_gradient(dgb_ctx* ctx, const double* d_p, double* d_out);
/* replaces kinetic_energy (forms.hpp:168-170, forms.cpp:1239-1260) */
int dgb_kinetic_energy(dgb_ctx* ctx, const double* d_u, double* result);
/* On-device diagnostics: */
/* L2 norm sqrt(x^T M x) of a field of the velocity (space 0) or pressure (space 1) space. */
int dgb_l2_norm(dgb_ctx* ctx, int space, const double* d_x, double* result);
/* check_steady: *steady = max |u_new - u_old| < tol; *diff = that max. */
int dgb_check_steady(dgb_ctx* ctx, const double* d_u_new, const double* d_u_old, double tol, int* steady,
                     double* diff);
/* compute_stability_params: C = k U dt / H, mu = k^2 dt / (Re H^2),
 * H = min cell diameter (GeometryCache::min_diam, space.hpp:64), k = velocity degree. */
int dgb_stability_params(dgb_ctx* ctx, double dt, double Re, double U, double* C, double* mu);

/* ------------------------------------------------------------------ vector kernels */
/* kern::axpy/axpby/scal/dot/max_abs_diff (kernels.hpp:34-43) on device vectors.
 * axpy = fma(a, x, y) and axpby = fma(a, x, b*y) elementwise, bit-identical to the
 * reference's AVX2 backend (kernels_avx2.cpp:12-33); dot / norm reassociate the sum
 * (single-pass block reduction).  dgb_norm = sqrt(dot(x, x)) (the 2-norm the solvers
 * use, krylov.cpp:54-56; SURVEY 8(b) "fused dgb_axpy/axpby/dot/norm"). */
int dgb_axpy(dgb_ctx* ctx, size_t n, double a, const double* d_x, double* d_y);
int dgb_axpby(dgb_ctx* ctx, size_t n, double a, const double* d_x, double b, double* d_y);
int dgb_scal(dgb_ctx* ctx, size_t n, double a, double* d_x);
int dgb_dot(dgb_ctx* ctx, size_t n, const double* d_x, const double* d_y, double* result);
int dgb_max_abs_diff(dgb_ctx* ctx, size_t n, const double* d_x, const double* d_y, double* result);
int dgb_norm(dgb_ctx* ctx, size_t n, const double* d_x, double* result);

/* ------------------------------------------------------------------ solvers */
/* SolverSettings (krylov.hpp:24-29) */
typedef struct {
  double rel_tol;
  double abs_tol;
  int max_iter;
  int restart;
} dgb_solver_settings;
/* SolveResult (krylov.hpp:50-53) */
typedef struct {
  int iterations;
  double residual;
} dgb_solve_result;
/* The operator a solver applies (the reference passes a LinearOp closure,
 * krylov.hpp:22): op = DGB_OP_* with its parameters. */
enum { DGB_OP_MOMENTUM = 0, DGB_OP_PRESSURE = 1, DGB_OP_MASS_U = 2, DGB_OP_MASS_P = 3, DGB_OP_LAPLACE = 4 };
typedef struct {
  int op;
  double coefs[4];     /* momentum coefs, or coefs[0] = pressure mass_coef */
  const double* d_w;   /* advecting field (momentum) */
  int dirichlet_bdry;  /* laplace */
} dgb_operator;
/* JacobiPreconditioner (krylov.hpp:40-48): d_inv = 1/d_diag; DGB_E_ZERO_DIAG names the dof. */
int dgb_jacobi_inverse(dgb_ctx* ctx, size_t n, const double* d_diag, double* d_inv);
/* cg_solve / gmres_solve (krylov.hpp:58-66): d_x is initial guess and result;
 * d_inv_diag NULL = unpreconditioned.  Any 8-byte-aligned d_inv_diag is accepted
 * (GMRES copies one that is not 16-byte aligned to an aligned scratch vector first:
 * its Gram-Schmidt pass reads it as double2).  On DGB_E_NO_CONVERGENCE / BREAKDOWN /
 * NOT_SPD the residual history (SolverError::history) is copied to hist_host
 * (up to hist_cap entries) and its full length stored in *hist_len. */
int dgb_cg(dgb_ctx* ctx, const dgb_operator* op, const dgb_solver_settings* s, const double* d_inv_diag,
           const double* d_b, double* d_x, dgb_solve_result* res, double* hist_host, int hist_cap,
           int* hist_len);
int dgb_gmres(dgb_ctx* ctx, const dgb_operator* op, const dgb_solver_settings* s, const double* d_inv_diag,
              const double* d_b, double* d_x, dgb_solve_result* res, double* hist_host, int hist_cap,
              int* hist_len);

/* Pressure solve (mass_coef M + K_SIP) x = b by CG preconditioned with a hybrid
 * multigrid V-cycle (DG Q_kp -> continuous Q1 levels, Chebyshev-Jacobi smoothing, dense
 * coarsest solve).  Same stopping rule as dgb_cg; not
 * part of the reference (which uses Jacobi): iteration counts differ, solutions agree to
 * the solver tolerance.  DGB_E_UNSUPPORTED unless the mesh is a uniform Cartesian 3D grid. */
int dgb_pressure_cg_mg(dgb_ctx* ctx, double mass_coef, const dgb_solver_settings* s, const double* d_b,
                       double* d_x, dgb_solve_result* res);
/* z = B r: one application of that V-cycle (symmetric positive definite). */
int dgb_pressure_mg_vcycle(dgb_ctx* ctx, double mass_coef, const double* d_r, double* d_z);

/* ------------------------------------------------------------------ TR-BDF2 */
/* One step of the TR-BDF2 projection scheme,
 * entirely on the device.  its[8] = gmres stage 1/2, cg stage 1/2, mass-cg x4
 * (its[10] with fixed_point: + fixed-point re-solves of stage 1/2). */
typedef struct {
  double dt, Re, c, time;
  int restart;
  double tol_mom, tol_p, tol_mass;
  int max_iter;
  int first_step;
  /* pressure preconditioner: 0 = Jacobi (the reference's, krylov.cpp:27-41; iteration-count
   * parity), 1 = hybrid multigrid V-cycle (dgb_pressure_cg_mg; uniform Cartesian 3D meshes) */
  int pressure_precond;
  /* trbdf2_step_fixedpoint: each momentum predictor solve is repeated
   * with the advecting field replaced by the latest iterate until the max-norm increment
   * is below fp_tol (at most fp_max_iter re-solves); its[] then needs 10 entries:
   * its[8], its[9] = re-solves of stage 1 / 2 (its[0], its[1] sum all GMRES iterations). */
  int fixed_point;
  double fp_tol;
  int fp_max_iter;
} dgb_step_params;
/* The two baseline projection schemes the paper compares against (PAPER.md:182-232,
 * SPEC.md:391-405): DGB_SCHEME_BCG (Bell-Colella-Glaz, fully nonlinear Crank-Nicolson
 * predictor solved by fixed point, increment-form Helmholtz) and DGB_SCHEME_GQ_BDF2
 * (Guermond-Quartapelle BDF2; its first step, first_step != 0, is a BCG step).  Same
 * params; its[10] = [gmres, 0, cg, 0, mass-cg (pre), mass-cg (post), 0, 0, fixed-point
 * re-solves, 0].  DGB_SCHEME_TRBDF2 = dgb_trbdf2_step. */
enum { DGB_SCHEME_TRBDF2 = 0, DGB_SCHEME_BCG = 1, DGB_SCHEME_GQ_BDF2 = 2 };
int dgb_projection_step(dgb_ctx* ctx, int scheme, const dgb_step_params* p, const double* d_u_nm1,
                        const double* d_u_n, const double* d_p_n, double* d_u_np1, double* d_p_np1, int* its);
int dgb_trbdf2_step(dgb_ctx* ctx, const dgb_step_params* p, const double* d_u_nm1, const double* d_u_n,
                    const double* d_p_n, double* d_u_np1, double* d_p_np1, int* its);

/* ------------------------------------------------------------------ synthetic inputs */
/* mt19937_64(seed), U[lo,hi) via (x >> 11) * 2^-53. */
int dgb_seeded_uniform(unsigned long long seed, size_t n, double lo, double hi, double* h_out);
/* Curl of a random stream function / vector potential (BASELINE configs):
 * fills *user (opaque, >= 512 doubles) for dgb_synth_eval. */
int dgb_synth_init(int dim, unsigned long long seed, double scale, double* user);
void dgb_synth_eval(const double* x, double t, double* out, void* user);
/* Nodal interpolation of the synthetic field into the velocity space (host array). */
int dgb_interpolate_synth(dgb_ctx* ctx, const double* user, double* h_u);
/* Same on the device (fp64 cos on the GPU; agrees with the host version to rounding). */
int dgb_interpolate_synth_device(dgb_ctx* ctx, const double* user, double* d_u);
/* Host-only helpers (no GPU needed): the context's mesh setup and 1D tables. */
int dgb_host_mesh_cartesian(int dim, int n_el, double amp, unsigned seed, long long* sizes, int* iface,
                            int* bface, double* cell_measure, double* face_measure, double* vertices);
int dgb_host_tables(int n, int q, double* B, double* D, double* dE, double* w);

/* ------------------------------------------------------------------ measurement */
/* Milliseconds of the last kernel launch timed with dgb_timer_* (CUDA events on the ctx stream). */
int dgb_timer_start(dgb_ctx* ctx);
int dgb_timer_stop(dgb_ctx* ctx, float* ms);
/* fp64 DFMA peak microbenchmark on the context device (TFLOP/s). */
int dgb_fp64_peak(dgb_ctx* ctx, double* tflops);
/* the same through the FP64 tensor-core instruction (DMMA, mma.sync m8n8k4.f64): the pipe's upper peak. */
int dgb_fp64_peak_dmma(dgb_ctx* ctx, double* tflops);
/* Fast 3D kernels on (default) / off (generic kernels); and which apply:
 * 1 = axis-aligned (fast_axis.cuh), 2 = deformed (fast_deformed.cuh), 0 = generic only. */
int dgb_set_fast_path(dgb_ctx* ctx, int enable);
int dgb_fast_path_active(dgb_ctx* ctx);
/* Subface kernels of a refined mesh (hang.cu): 0 = no hanging faces, 1 = dense embedded-point
 * tables (any dim / geometry), 2 = sum-factorised (3D, every subface between axis-aligned boxes). */
int dgb_hanging_mode(dgb_ctx* ctx);
/* number of device kernels this context launched so far */
long long dgb_launch_count(dgb_ctx* ctx);

#ifdef __cplusplus
}
#endif
#endif /* DGB_H */
