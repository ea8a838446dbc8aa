// Plain-C++ view of the device context consumed by the operator launchers,
// plus the per-dimension operator tables (defined in ops_d2.cu / ops_d3.cu so
// the two dimensions compile as parallel translation units).
#pragma once

#include <cuda_runtime.h>

namespace dgb {

constexpr int kMaxRule = 8;
constexpr int kMaxTerms = 4;

struct MeshArgs {
  int ncells = 0;
  const int* nbr = nullptr;      // [ncells][2dim]: neighbour, or -1 - boundary_id
  const double* pen = nullptr;   // [ncells][2dim]: interior mean |F|/|K|, boundary |F|/|K|
  const int* bctype = nullptr;   // [64]: 0 dirichlet, 1 outlet
  const int* bslot = nullptr;    // [ncells][2dim]: boundary-face index (reference order) or -1
  const int* skip = nullptr;     // device flag: nonzero -> the launch is a no-op (device-side Krylov exit)
  int cell0 = 0, cell1 = -1;     // fast kernels: process cells [cell0, cell1) only (-1: ncells)
  int poison = 0;                // debug (dgb_set_debug): fill dynamic shared memory with NaN first
};

#ifdef __CUDACC__
// Debug check for reads of shared memory that no stage of this launch wrote (the
// uninitialised-read half of a race detector; compute-sanitizer is not available on the
// GPU pool): every CTA first fills its dynamic shared memory with a NaN pattern, so a
// stage that consumed a value before its producer stored it changes the result
// (tests/test_gpu_race.py compares poisoned and clean launches bit for bit).
// (out of line, so the check costs the hot kernels no registers when it is off)
__device__ __noinline__ inline void dgb_poison_smem(double* sm) {
  unsigned nbytes;
  asm volatile("mov.u32 %0, %%dynamic_smem_size;" : "=r"(nbytes));
  for (unsigned i = threadIdx.x; i < nbytes / 8; i += blockDim.x) sm[i] = __longlong_as_double(0x7ff8dead0000beefll);
  __syncthreads();
}
#define DGB_POISON_SMEM(m, sm) \
  if ((m).poison) dgb_poison_smem(sm)
#endif

struct GeoArgs {
  const double* aff = nullptr;    // affine: per cell {Jinv, detJ, per face {n, ds}}
  const double* qcell = nullptr;  // per-qp cell geometry for this rule
  const double* qface = nullptr;  // per-qp face geometry for this rule
  const int* nbr = nullptr;
};

struct MomCoef {
  double mass, visc, adv, skew;
};

struct RhsArgs {
  int nm = 0, nv = 0, na = 0, np = 0;
  double mc[kMaxTerms], vc[kMaxTerms], ac[kMaxTerms], pc[kMaxTerms];
  const double* mf[kMaxTerms];
  const double* vf[kMaxTerms];
  const double* af[kMaxTerms];
  const double* aw[kMaxTerms];
  const double* pf[kMaxTerms];
  double dvisc = 0.0, dadv = 0.0;
  const double* dir_w = nullptr;
  const double* gtab = nullptr;  // [n_bface][NQF(rule k+2)][DIM], reference boundary-face order
  int accumulate = 0;            // y += result (blocks without Dirichlet faces skip when only data terms)
};

// Uniform structured (generate_cartesian, lexicographic cells, equal h): neighbours,
// boundary ids and geometry follow from the cell index, so the fast kernels need
// no mesh-table loads (n == 0: use the tables).
struct UniformGrid {
  int n = 0;
  unsigned magic = 0, shift = 0;  // x / n == (umulhi(x, magic) + ((x - umulhi) >> 1)) >> (shift - 1), x < 2^32
  double ih = 0.0, detJ = 0.0, pen_int = 0.0, pen_bdry = 0.0;
  unsigned long long outlet_mask = 0;
};
// round-up multiplier for exact unsigned division by n >= 1 (Granlund-Montgomery)
inline void uniform_grid_set_divisor(UniformGrid& g, int n) {
  unsigned l = 0;
  while ((1ull << l) < (unsigned long long)n) ++l;
  g.n = n;
  g.shift = l;
  g.magic = (unsigned)(((1ull << 32) * ((1ull << l) - (unsigned long long)n)) / (unsigned long long)n + 1);
}

struct DevCtx {
  int dim = 0, ku = 0, kp = 0, ncells = 0;
  bool affine = true;
  bool axis = false;  // affine with diagonal Jinv on every cell (fast_axis.cuh)
  bool axis2 = false;  // the same in 2D (fast_sip2)
  UniformGrid ug;
  MeshArgs mesh;
  const double* aff = nullptr;
  const double* qcell[kMaxRule] = {};
  const double* qface[kMaxRule] = {};
  // compact per-qp geometry for the deformed fast kernels (fast_deformed.cuh):
  // per cell SoA: cell [7][qx][qy][qz] {detJw Jinv Jinv^T (xx, xy, xz, yy, yz, zz), detJw};
  // face [6][7][qp + Q qq] {Jinv n (3), Jinv_nbr n (3), w ds}
  const double* qcm[kMaxRule] = {};
  const double* qfn[kMaxRule] = {};
  // pass-B (advection) records of the deformed momentum kernel, per cell SoA:
  // detJ w Jinv [9][Q^3] and n ds w [6 faces][3][Q^2] (rule k_u+2 only)
  const double* qadv[kMaxRule] = {};
  const double* qfw[kMaxRule] = {};
  cudaStream_t stream = nullptr;
};

struct OpTable {
  cudaError_t (*momentum)(const DevCtx&, MomCoef, const double* w, const double* x, double* y);
  cudaError_t (*momentum_diag)(const DevCtx&, MomCoef, const double* w, double* y);
  cudaError_t (*rhs)(const DevCtx&, const RhsArgs&, double* y);
  cudaError_t (*sip)(const DevCtx&, double mc, int dir, const double* x, double* y);
  cudaError_t (*sip_diag)(const DevCtx&, double mc, int dir, double* y);
  cudaError_t (*mass)(const DevCtx&, int space, const double* x, double* y);
  cudaError_t (*mass_diag)(const DevCtx&, int space, double* y);
  cudaError_t (*gradient)(const DevCtx&, const double* p, double* y);
  cudaError_t (*divergence)(const DevCtx&, const double* u, double* y);
  cudaError_t (*kinetic)(const DevCtx&, const double* u, double* partial, int* nblocks);
  cudaError_t (*tables)();
};

// fast axis-aligned 3D kernels (fast_d3.cu); cudaErrorNotSupported when not applicable
cudaError_t fast_sip3(const DevCtx& c, double mc, int dir, const double* x, double* y);
// 2D axis-aligned scalar SIP, one thread per cell (fast_axis.cuh k_sip_axis2)
cudaError_t fast_sip2(const DevCtx& c, double mc, int dir, const double* x, double* y);
// deformed (per-qp geometry) 3D meshes (fast_deformed.cuh)
cudaError_t fast_sip3_qp(const DevCtx& c, double mc, int dir, const double* x, double* y);
cudaError_t fast_mass3_qp(const DevCtx& c, int pressure, const double* x, double* y);
cudaError_t fast_momentum3(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y);
cudaError_t fast_momentum3_qp(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y);
cudaError_t fast_momentum_diag3(const DevCtx& c, MomCoef co, const double* w, double* y);
cudaError_t fast_momentum_diag3_qp(const DevCtx& c, MomCoef co, const double* w, double* y);
cudaError_t fast_divergence3(const DevCtx& c, const double* u, double* y);
// deformed 3D meshes: divergence functional and (inside fast_rhs3_qp) the weak pressure gradient
cudaError_t fast_divergence3_qp(const DevCtx& c, const double* u, double* y);
cudaError_t fast_sip_diag3(const DevCtx& c, double mc, int dir, double* y);
cudaError_t fast_sip_diag3_qp(const DevCtx& c, double mc, int dir, double* y);
struct CgState;
// CG apply on the axis-aligned scalar SIP operator with <p, q> fused (fast_axis.cuh
// k_sip_axis<.., CGF>): q = A p, block partials, alpha written to st by the last block
cudaError_t fast_sip3_cg(const DevCtx& c, double mc, int dir, const double* p, double* q, double* partial,
                         CgState* st);
int fast_sip3_cg_blocks(const DevCtx& c);  // number of partials fast_sip3_cg writes (0: unsupported)
// stage right-hand side (momentum_rhs) on axis-aligned 3D meshes; ptmp: pressure-space scratch
cudaError_t fast_rhs3(const DevCtx& c, const RhsArgs& ra, double* y, double* ptmp);
// stage right-hand side on deformed 3D meshes (RHS-mode k_momentum_qp + generic pressure / data terms)
cudaError_t fast_rhs3_qp(const DevCtx& c, const RhsArgs& ra, double* y);

// defined in ops_d{2,3}_k{1..4}.cu
#define DGB_DECL_OPS(D, K) const OpTable& ops_d##D##_k##K();
DGB_DECL_OPS(2, 1) DGB_DECL_OPS(2, 2) DGB_DECL_OPS(2, 3) DGB_DECL_OPS(2, 4)
DGB_DECL_OPS(3, 1) DGB_DECL_OPS(3, 2) DGB_DECL_OPS(3, 3) DGB_DECL_OPS(3, 4)
#undef DGB_DECL_OPS
/// operator table for dimension dim and space degree k (1..4); nullptr if unsupported
inline const OpTable* ops_for(int dim, int k) {
  if (dim == 2) {
    switch (k) {
      case 1: return &ops_d2_k1();
      case 2: return &ops_d2_k2();
      case 3: return &ops_d2_k3();
      case 4: return &ops_d2_k4();
    }
  } else if (dim == 3) {
    switch (k) {
      case 1: return &ops_d3_k1();
      case 2: return &ops_d3_k2();
      case 3: return &ops_d3_k3();
      case 4: return &ops_d3_k4();
    }
  }
  return nullptr;
}

}  // namespace dgb
