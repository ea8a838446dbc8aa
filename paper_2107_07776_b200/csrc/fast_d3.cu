// Axis-aligned affine 3D fast kernels (fast_axis.cuh) + their launchers.
#include "fast_axis.cuh"
#include "fast_deformed.cuh"

#include <cstdlib>
#include <vector>

#include "blas.cuh"

namespace dgb {

void host_tab(int N, int Q, double* B, double* D, double* dE);
void host_w(int Q, double* w);

void host_ftab(int N, int Q, double* M, double* K, double* B, double* D, double* dE, double* w) {
  host_tab(N, Q, B, D, dE);
  host_w(Q, w);
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < N; ++j) {
      double m = 0.0, k = 0.0;
      for (int q = 0; q < Q; ++q) {
        m += w[q] * B[q * N + i] * B[q * N + j];
        k += w[q] * D[q * N + i] * D[q * N + j];
      }
      M[i * N + j] = m;
      K[i * N + j] = k;
    }
}

// mixed velocity / pressure 1D tables (rule k+1): Mvp = sum_q w phi_i psi_j, G1 = sum_q w phi_i' psi_j
static void host_ptab(int K, double* Mvp, double* G1, double* Dpv) {
  const int N = K + 1, NP = K, Q = K + 1;
  std::vector<double> Bn(Q * N), Dn(Q * N), En(2 * N), Bp(Q * NP), Dp(Q * NP), Ep(2 * NP), w(Q);
  host_tab(N, Q, Bn.data(), Dn.data(), En.data());
  host_tab(NP, Q, Bp.data(), Dp.data(), Ep.data());
  host_w(Q, w.data());
  for (int i = 0; i < N; ++i)
    for (int j = 0; j < NP; ++j) {
      double mv = 0.0, g = 0.0;
      for (int q = 0; q < Q; ++q) {
        mv += w[q] * Bn[q * N + i] * Bp[q * NP + j];
        g += w[q] * Dn[q * N + i] * Bp[q * NP + j];
      }
      Mvp[i * NP + j] = mv;
      G1[i * NP + j] = g;
    }
  for (int i = 0; i < NP; ++i)
    for (int j = 0; j < N; ++j) {
      double dv = 0.0;
      for (int q = 0; q < Q; ++q) dv += w[q] * Dp[q * NP + i] * Bn[q * N + j];
      Dpv[i * N + j] = dv;
    }
}
template <int K>
static cudaError_t ensure_ptab() {
  static int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return cudaSuccess;
  PTab<K> t;
  host_ptab(K, &t.Mvp[0][0], &t.G1[0][0], &t.Dpv[0][0]);
  const cudaError_t e = cudaMemcpyToSymbol(c_pt<K>, &t, sizeof(t));
  if (e == cudaSuccess) done_dev = dev;
  return e;
}

// cells a fast launch covers (a z-slab range for the host-buffer pipelines)
static int fast_cells(const DevCtx& c) {
  const int c1 = c.mesh.cell1 < 0 ? c.ncells : c.mesh.cell1;
  return c1 - c.mesh.cell0;
}

template <class KernelT>
static cudaError_t set_smem(KernelT kern, size_t smem) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

// Uniform Cartesian grids, pressure degrees 1 and 2, whole-mesh applies: the
// thread-per-cell kernel (DGB_SIP_CELL=0 in the environment keeps k_sip_axis)
template <int KP>
static bool sip_cell_applies(const DevCtx& c) {
  static const bool off = [] {
    const char* v = std::getenv("DGB_SIP_CELL");
    return v && v[0] == '0';
  }();
  const long long n = c.ug.n, layer = n * n;
  // the whole mesh or a range of whole z-layers (dgb_set_cell_range: slabs, host-buffer pipeline)
  return KP <= 2 && !off && n > 1 && n * layer == (long long)c.ncells && c.mesh.cell0 % layer == 0 &&
         (c.mesh.cell1 < 0 || c.mesh.cell1 % layer == 0);
}
template <int KP>
static int sip_cell_grid(const DevCtx& c) {
  using G = SipCellCfg<KP>;
  const int n = c.ug.n, layer = n * n;
  const int nz = (c.mesh.cell1 < 0 ? n : c.mesh.cell1 / layer) - c.mesh.cell0 / layer;
  return ((n + G::TX - 1) / G::TX) * ((n + G::TY - 1) / G::TY) * ((nz + G::TZ - 1) / G::TZ);
}

template <int KP, bool CGF = false>
static cudaError_t run_sip_axis(const DevCtx& c, double mc, int dir, const double* x, double* y,
                                SipCgArgs cg = SipCgArgs()) {
  using G = SipAxisCfg<KP>;
  cudaError_t e = ensure_ftab<KP + 1, KP + 1>();
  if (e != cudaSuccess) return e;
  if constexpr (KP <= 2) {
    if (sip_cell_applies<KP>(c)) {
      using S = SipCellCfg<KP>;
      if ((e = set_smem(k_sip_cell<KP, CGF>, S::SMEM)) != cudaSuccess) return e;
      k_sip_cell<KP, CGF><<<sip_cell_grid<KP>(c), S::T, S::SMEM, c.stream>>>(c.mesh, c.ug, mc, dir, x, y, cg);
      return cudaGetLastError();
    }
  }
  const int grid = (fast_cells(c) + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_sip_axis<KP, true, CGF>, G::SMEM)) != cudaSuccess) return e;
    k_sip_axis<KP, true, CGF><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, x, y, cg);
  } else {
    if ((e = set_smem(k_sip_axis<KP, false, CGF>, G::SMEM)) != cudaSuccess) return e;
    k_sip_axis<KP, false, CGF><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, x, y, cg);
  }
  return cudaGetLastError();
}

template <int K, int MODE, bool RHS = false>
static cudaError_t launch_momentum_axis(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y,
                                        int acc = 0) {
  constexpr int CC = MomAxisTune<K, MODE>::C, TH = MomAxisTune<K, MODE>::T;
  using G = MomAxisCfg<K, CC, TH, MODE>;
  cudaError_t e;
  const int grid = (fast_cells(c) + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_momentum_axis<K, CC, TH, MODE, true, RHS>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_axis<K, CC, TH, MODE, true, RHS><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, x, w, y, acc);
  } else {
    if ((e = set_smem(k_momentum_axis<K, CC, TH, MODE, false, RHS>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_axis<K, CC, TH, MODE, false, RHS><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, x, w, y, acc);
  }
  return cudaGetLastError();
}

template <int K>
static cudaError_t run_momentum_axis(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  cudaError_t e = ensure_ftab<K + 1, K + 2>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 1>();
  if (e != cudaSuccess) return e;
  if (MomAxisTune<K, 0>::SPLIT && co.adv != 0.0 && (co.mass != 0.0 || co.visc != 0.0)) {
    e = launch_momentum_axis<K, 1>(c, co, w, x, y);   // mass + viscous -> y
    if (e != cudaSuccess) return e;
    return launch_momentum_axis<K, 2>(c, co, w, x, y);  // + advection
  }
  return launch_momentum_axis<K, 0>(c, co, w, x, y);
}

// Stage right-hand side (forms.cpp:816-1084) as a sum of fast launches:
//   one RHS-mode momentum launch per distinct (field, advecting field) pair
//   (mass + consistency-only viscous + central advective terms, coefficients
//   merged per field), the weak pressure gradient of sum_i pc_i p_i, and the
//   boundary-data terms through the generic kernel (only blocks that own a
//   Dirichlet face do work).
template <int K>
static cudaError_t run_rhs_axis(const DevCtx& c, const RhsArgs& ra, double* y, double* ptmp) {
  cudaError_t e = ensure_ftab<K + 1, K + 2>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 1>();
  if (e == cudaSuccess && ra.np > 0) e = ensure_ptab<K>();
  if (e != cudaSuccess) return e;
  struct Call {
    const double* x;
    const double* w;
    MomCoef co;
  };
  std::vector<Call> calls;
  auto find = [&](const double* x, const double* w, bool need_w) -> Call& {
    for (Call& cl : calls)
      if (cl.x == x && (!need_w || cl.w == w || cl.w == nullptr)) {
        if (need_w) cl.w = w;
        return cl;
      }
    calls.push_back(Call{x, need_w ? w : nullptr, MomCoef{0.0, 0.0, 0.0, 0.0}});
    return calls.back();
  };
  for (int i = 0; i < ra.na; ++i) find(ra.af[i], ra.aw[i], true).co.adv -= ra.ac[i];
  for (int i = 0; i < ra.nm; ++i) find(ra.mf[i], nullptr, false).co.mass += ra.mc[i];
  for (int i = 0; i < ra.nv; ++i) find(ra.vf[i], nullptr, false).co.visc -= ra.vc[i];
  const size_t nu = (size_t)c.ncells * 3 * (K + 1) * (K + 1) * (K + 1);
  if (calls.empty()) {
    if ((e = cudaMemsetAsync(y, 0, nu * sizeof(double), c.stream)) != cudaSuccess) return e;
  }
  for (size_t i = 0; i < calls.size(); ++i) {
    const Call& cl = calls[i];
    e = launch_momentum_axis<K, 0, true>(c, cl.co, cl.w ? cl.w : cl.x, cl.x, y, i > 0 ? 1 : 0);
    if (e != cudaSuccess) return e;
  }
  if (ra.np > 0) {
    const size_t np = (size_t)c.ncells * K * K * K;
    if ((e = v_scale_copy(c.stream, np, ra.pc[0], ra.pf[0], ptmp)) != cudaSuccess) return e;
    for (int i = 1; i < ra.np; ++i)
      if ((e = v_axpy(c.stream, np, ra.pc[i], ra.pf[i], ptmp)) != cudaSuccess) return e;
    using G = PGradCfg<K>;
    const int grid = (c.ncells + G::C - 1) / G::C;
    if (c.ug.n > 0) {
      if ((e = set_smem(k_pgrad_axis<K, true>, G::SMEM)) != cudaSuccess) return e;
      k_pgrad_axis<K, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, ptmp, y);
    } else {
      if ((e = set_smem(k_pgrad_axis<K, false>, G::SMEM)) != cudaSuccess) return e;
      k_pgrad_axis<K, false><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, ptmp, y);
    }
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  if (ra.dvisc != 0.0 || ra.dadv != 0.0) {
    RhsArgs rd;
    rd.dvisc = ra.dvisc;
    rd.dadv = ra.dadv;
    rd.dir_w = ra.dir_w;
    rd.gtab = ra.gtab;
    rd.accumulate = 1;
    const OpTable* ops = ops_for(3, K);
    if (!ops) return cudaErrorNotSupported;
    return ops->rhs(c, rd, y);
  }
  return cudaSuccess;
}

// Deformed 3D meshes: the stage right-hand side as RHS-mode k_momentum_qp launches (one
// per distinct (field, advecting field) pair, coefficients merged per field: mass,
// consistency-only viscous, central advective terms), then the pressure and boundary-data
// terms through the generic kernel (accumulating).
template <int K>
static cudaError_t run_rhs_qp(const DevCtx& c, const RhsArgs& ra, double* y) {
  cudaError_t e = ensure_ftab<K + 1, K + 1>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 2>();
  if (e != cudaSuccess) return e;
  using G = MomQpCfg<K>;
  const double *gcA = c.qcm[K + 1], *gfA = c.qfn[K + 1], *gadv = c.qadv[K + 2], *gfw = c.qfw[K + 2];
  if (!gcA || !gfA || !gadv || !gfw) return cudaErrorNotSupported;
  struct Call {
    const double* x;
    const double* w;
    MomCoef co;
  };
  std::vector<Call> calls;
  auto find = [&](const double* x, const double* w, bool need_w) -> Call& {
    for (Call& cl : calls)
      if (cl.x == x && (!need_w || cl.w == w || cl.w == nullptr)) {
        if (need_w) cl.w = w;
        return cl;
      }
    calls.push_back(Call{x, need_w ? w : nullptr, MomCoef{0.0, 0.0, 0.0, 0.0}});
    return calls.back();
  };
  for (int i = 0; i < ra.na; ++i) find(ra.af[i], ra.aw[i], true).co.adv -= ra.ac[i];
  for (int i = 0; i < ra.nm; ++i) find(ra.mf[i], nullptr, false).co.mass += ra.mc[i];
  for (int i = 0; i < ra.nv; ++i) find(ra.vf[i], nullptr, false).co.visc -= ra.vc[i];
  const size_t nu = (size_t)c.ncells * 3 * (K + 1) * (K + 1) * (K + 1);
  if (calls.empty() && (e = cudaMemsetAsync(y, 0, nu * sizeof(double), c.stream)) != cudaSuccess) return e;
  if ((e = set_smem(k_momentum_qp<K, true>, G::SMEM)) != cudaSuccess) return e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  for (size_t i = 0; i < calls.size(); ++i) {
    const Call& cl = calls[i];
    k_momentum_qp<K, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, gcA, gfA, gadv, gfw, cl.co, cl.x,
                                                            cl.w ? cl.w : cl.x, y, i > 0 ? 1 : 0);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  // two accumulating launches of the generic kernel: the pressure terms over every cell,
  // then the boundary-data terms, whose blocks without a Dirichlet face exit at once
  // (one launch carrying both runs the data path's stages in every block: 32.7 ms at cfg4
  // against 14.5 + 3.4 ms)
  const OpTable* ops = ops_for(3, K);
  bool pres_done = ra.np == 0;
  if constexpr (K >= 2) {  // weak pressure gradient on the fast kernel (pressure degree K - 1)
    const double *ga1 = c.qadv[K + 1], *gw1 = c.qfw[K + 1];
    if (!pres_done && c.kp == K - 1 && ga1 && gw1 && (e = ensure_ftab<K, K + 1>()) == cudaSuccess) {
      using M = MixQpCfg<K>;
      if ((e = set_smem(k_pgrad_qp<K>, M::G_SMEM)) != cudaSuccess) return e;
      PresTerms pt;
      pt.n = ra.np;
      for (int i = 0; i < ra.np; ++i) {
        pt.c[i] = ra.pc[i];
        pt.f[i] = ra.pf[i];
      }
      k_pgrad_qp<K><<<(c.ncells + M::C - 1) / M::C, M::T, M::G_SMEM, c.stream>>>(c.mesh, ga1, gw1, pt, y);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
      pres_done = true;
    }
  }
  if (!pres_done) {
    RhsArgs rd;
    rd.np = ra.np;
    for (int i = 0; i < ra.np; ++i) {
      rd.pc[i] = ra.pc[i];
      rd.pf[i] = ra.pf[i];
    }
    rd.accumulate = 1;
    if (!ops) return cudaErrorNotSupported;
    if ((e = ops->rhs(c, rd, y)) != cudaSuccess) return e;
  }
  if (ra.dvisc != 0.0 || ra.dadv != 0.0) {
    RhsArgs rd;
    rd.dvisc = ra.dvisc;
    rd.dadv = ra.dadv;
    rd.dir_w = ra.dir_w;
    rd.gtab = ra.gtab;
    rd.accumulate = 1;
    if (!ops) return cudaErrorNotSupported;
    return ops->rhs(c, rd, y);
  }
  return cudaSuccess;
}
template <int K>
static cudaError_t run_div_qp(const DevCtx& c, const double* u, double* y) {
  const double *ga1 = c.qadv[K + 1], *gw1 = c.qfw[K + 1];
  if (!ga1 || !gw1) return cudaErrorNotSupported;
  cudaError_t e = ensure_ftab<K + 1, K + 1>();
  if (e == cudaSuccess) e = ensure_ftab<K, K + 1>();
  if (e != cudaSuccess) return e;
  using M = MixQpCfg<K>;
  if ((e = set_smem(k_div_qp<K>, M::D_SMEM)) != cudaSuccess) return e;
  k_div_qp<K><<<(c.ncells + M::C - 1) / M::C, M::T, M::D_SMEM, c.stream>>>(c.mesh, ga1, gw1, u, y);
  return cudaGetLastError();
}
cudaError_t fast_divergence3_qp(const DevCtx& c, const double* u, double* y) {
  if (c.dim != 3 || c.affine || c.kp != c.ku - 1) return cudaErrorNotSupported;
  switch (c.ku) {
    case 2: return run_div_qp<2>(c, u, y);
    case 3: return run_div_qp<3>(c, u, y);
    case 4: return run_div_qp<4>(c, u, y);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast_rhs3_qp(const DevCtx& c, const RhsArgs& ra, double* y) {
  if (c.dim != 3 || c.affine) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_rhs_qp<1>(c, ra, y);
    case 2: return run_rhs_qp<2>(c, ra, y);
    case 3: return run_rhs_qp<3>(c, ra, y);
    case 4: return run_rhs_qp<4>(c, ra, y);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast_rhs3(const DevCtx& c, const RhsArgs& ra, double* y, double* ptmp) {
  if ((c.kp != c.ku - 1 && ra.np > 0) || !ptmp) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_rhs_axis<1>(c, ra, y, ptmp);
    case 2: return run_rhs_axis<2>(c, ra, y, ptmp);
    case 3: return run_rhs_axis<3>(c, ra, y, ptmp);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast_sip3(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  switch (c.kp) {
    case 1: return run_sip_axis<1>(c, mc, dir, x, y);
    case 2: return run_sip_axis<2>(c, mc, dir, x, y);
    case 3: return run_sip_axis<3>(c, mc, dir, x, y);
  }
  return cudaErrorNotSupported;
}

int fast_sip3_cg_blocks(const DevCtx& c) {
  if (c.kp == 1 && sip_cell_applies<1>(c)) return sip_cell_grid<1>(c) * (SipCellCfg<1>::T / 32);
  if (c.kp == 2 && sip_cell_applies<2>(c)) return sip_cell_grid<2>(c) * (SipCellCfg<2>::T / 32);
  switch (c.kp) {
    case 1: return (c.ncells + SipAxisCfg<1>::C - 1) / SipAxisCfg<1>::C * (SipAxisCfg<1>::T / 32);
    case 2: return (c.ncells + SipAxisCfg<2>::C - 1) / SipAxisCfg<2>::C * (SipAxisCfg<2>::T / 32);
    case 3: return (c.ncells + SipAxisCfg<3>::C - 1) / SipAxisCfg<3>::C * (SipAxisCfg<3>::T / 32);
  }
  return 0;
}

cudaError_t fast_sip3_cg(const DevCtx& c, double mc, int dir, const double* p, double* q, double* partial,
                         CgState* st) {
  SipCgArgs a;
  a.partial = partial;
  a.st = st;
  switch (c.kp) {
    case 1: return run_sip_axis<1, true>(c, mc, dir, p, q, a);
    case 2: return run_sip_axis<2, true>(c, mc, dir, p, q, a);
    case 3: return run_sip_axis<3, true>(c, mc, dir, p, q, a);
  }
  return cudaErrorNotSupported;
}

template <int K>
static cudaError_t run_momentum_diag_axis(const DevCtx& c, MomCoef co, const double* w, double* y) {
  cudaError_t e = ensure_ftab<K + 1, K + 2>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 1>();
  if (e != cudaSuccess) return e;
  using G = MomDiagCfg<K>;
  const int grid = (c.ncells + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_momentum_diag_axis<K, true>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_diag_axis<K, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, w, y);
  } else {
    if ((e = set_smem(k_momentum_diag_axis<K, false>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_diag_axis<K, false><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, w, y);
  }
  return cudaGetLastError();
}

cudaError_t fast_momentum_diag3(const DevCtx& c, MomCoef co, const double* w, double* y) {
  if (co.skew != 0.0 || (co.adv != 0.0 && w == nullptr)) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_momentum_diag_axis<1>(c, co, w, y);
    case 2: return run_momentum_diag_axis<2>(c, co, w, y);
    case 3: return run_momentum_diag_axis<3>(c, co, w, y);
  }
  return cudaErrorNotSupported;
}

template <int K>
static cudaError_t run_div_axis(const DevCtx& c, const double* u, double* y) {
  cudaError_t e = ensure_ptab<K>();
  if (e != cudaSuccess) return e;
  using G = DivCfg<K>;
  const int grid = (c.ncells + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_div_axis<K, true>, G::SMEM)) != cudaSuccess) return e;
    k_div_axis<K, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, u, y);
  } else {
    if ((e = set_smem(k_div_axis<K, false>, G::SMEM)) != cudaSuccess) return e;
    k_div_axis<K, false><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, u, y);
  }
  return cudaGetLastError();
}
cudaError_t fast_divergence3(const DevCtx& c, const double* u, double* y) {
  if (c.kp != c.ku - 1) return cudaErrorNotSupported;
  switch (c.ku) {
    case 2: return run_div_axis<2>(c, u, y);
    case 3: return run_div_axis<3>(c, u, y);
    case 4: return run_div_axis<4>(c, u, y);
  }
  return cudaErrorNotSupported;
}

template <int KP>
static cudaError_t run_sip_diag_axis(const DevCtx& c, double mc, int dir, double* y) {
  cudaError_t e = ensure_ftab<KP + 1, KP + 1>();
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + 15) / 16;
  if (c.ug.n > 0)
    k_sip_diag_axis<KP, true><<<grid, 128, 0, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, y);
  else
    k_sip_diag_axis<KP, false><<<grid, 128, 0, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, y);
  return cudaGetLastError();
}
cudaError_t fast_sip_diag3(const DevCtx& c, double mc, int dir, double* y) {
  switch (c.kp) {
    case 1: return run_sip_diag_axis<1>(c, mc, dir, y);
    case 2: return run_sip_diag_axis<2>(c, mc, dir, y);
    case 3: return run_sip_diag_axis<3>(c, mc, dir, y);
  }
  return cudaErrorNotSupported;
}

template <int KP>
static cudaError_t run_sip_qp(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  cudaError_t e = ensure_ftab<KP + 1, KP + 2>();
  if (e != cudaSuccess) return e;
  using G = SipQpCfg<KP>;
  const double* gc = c.qcm[KP + 2];
  const double* gf = c.qfn[KP + 2];
  if (!gc || !gf) return cudaErrorNotSupported;
  if ((e = set_smem(k_sip_qp<KP>, G::SMEM)) != cudaSuccess) return e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  k_sip_qp<KP><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, gc, gf, mc, dir, x, y);
  return cudaGetLastError();
}
template <int N, int Q, int NC>
static cudaError_t run_mass_qp(const DevCtx& c, const double* x, double* y) {
  const cudaError_t e = ensure_ftab<N, Q>();
  if (e != cudaSuccess) return e;
  const double* gc = c.qcm[Q];
  if (!gc) return cudaErrorNotSupported;
  using G = MassQpCfg<N, Q, NC>;
  k_mass_qp<N, Q, NC><<<(c.ncells + G::W - 1) / G::W, G::T, 0, c.stream>>>(c.mesh, gc, x, y);
  return cudaGetLastError();
}
// deformed mass: velocity (N = ku+1, rule ku+1, 3 components), pressure (N = kp+1, rule kp+2)
cudaError_t fast_mass3_qp(const DevCtx& c, int pressure, const double* x, double* y) {
  if (c.dim != 3 || c.affine) return cudaErrorNotSupported;
  if (!pressure) {
    switch (c.ku) {
      case 1: return run_mass_qp<2, 2, 3>(c, x, y);
      case 2: return run_mass_qp<3, 3, 3>(c, x, y);
      case 3: return run_mass_qp<4, 4, 3>(c, x, y);
      case 4: return run_mass_qp<5, 5, 3>(c, x, y);
    }
  } else {
    switch (c.kp) {
      case 1: return run_mass_qp<2, 3, 1>(c, x, y);
      case 2: return run_mass_qp<3, 4, 1>(c, x, y);
      case 3: return run_mass_qp<4, 5, 1>(c, x, y);
    }
  }
  return cudaErrorNotSupported;
}
template <int KP>
static cudaError_t run_sip_axis2(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  const cudaError_t e = ensure_ftab<KP + 1, KP + 1>();
  if (e != cudaSuccess) return e;
  k_sip_axis2<KP><<<(c.ncells + 127) / 128, 128, 0, c.stream>>>(c.mesh, c.aff, mc, dir, x, y);
  return cudaGetLastError();
}
cudaError_t fast_sip2(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  if (c.dim != 2 || !c.axis2 || !c.aff) return cudaErrorNotSupported;
  switch (c.kp) {
    case 1: return run_sip_axis2<1>(c, mc, dir, x, y);
    case 2: return run_sip_axis2<2>(c, mc, dir, x, y);
    case 3: return run_sip_axis2<3>(c, mc, dir, x, y);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast_sip3_qp(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  if (c.dim != 3 || c.affine) return cudaErrorNotSupported;
  switch (c.kp) {
    case 1: return run_sip_qp<1>(c, mc, dir, x, y);
    case 2: return run_sip_qp<2>(c, mc, dir, x, y);
    case 3: return run_sip_qp<3>(c, mc, dir, x, y);
  }
  return cudaErrorNotSupported;
}

template <int K>
static cudaError_t run_momentum_qp(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  cudaError_t e = ensure_ftab<K + 1, K + 1>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 2>();
  if (e != cudaSuccess) return e;
  using G = MomQpCfg<K>;
  const double *gcA = c.qcm[K + 1], *gfA = c.qfn[K + 1], *gadv = c.qadv[K + 2], *gfw = c.qfw[K + 2];
  if (!gcA || !gfA || !gadv || !gfw) return cudaErrorNotSupported;
  if ((e = set_smem(k_momentum_qp<K>, G::SMEM)) != cudaSuccess) return e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  k_momentum_qp<K><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, gcA, gfA, gadv, gfw, co, x, w ? w : x, y);
  return cudaGetLastError();
}
template <int K>
static cudaError_t run_momentum_diag_qp(const DevCtx& c, MomCoef co, const double* w, double* y) {
  cudaError_t e = ensure_ftab<K + 1, K + 1>();
  if (e == cudaSuccess) e = ensure_ftab<K + 1, K + 2>();
  if (e != cudaSuccess) return e;
  using G = MomDiagQpCfg<K>;
  const double *gcA = c.qcm[K + 1], *gfA = c.qfn[K + 1], *gadv = c.qadv[K + 2], *gfw = c.qfw[K + 2];
  if (!gcA || !gfA || !gadv || !gfw) return cudaErrorNotSupported;
  if ((e = set_smem(k_momentum_diag_qp<K>, G::SMEM)) != cudaSuccess) return e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  k_momentum_diag_qp<K><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, gcA, gfA, gadv, gfw, co, w, y);
  return cudaGetLastError();
}
template <int KP>
static cudaError_t run_sip_diag_qp(const DevCtx& c, double mc, int dir, double* y) {
  cudaError_t e = ensure_ftab<KP + 1, KP + 2>();
  if (e != cudaSuccess) return e;
  using G = MomDiagQpCfg<KP, true>;
  const double *gc = c.qcm[KP + 2], *gf = c.qfn[KP + 2];
  if (!gc || !gf) return cudaErrorNotSupported;
  if ((e = set_smem(k_momentum_diag_qp<KP, true>, G::SMEM)) != cudaSuccess) return e;
  MomCoef co{};
  co.mass = mc;
  co.visc = 1.0;
  const int grid = (c.ncells + G::C - 1) / G::C;
  k_momentum_diag_qp<KP, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, gc, gf, nullptr, nullptr, co, nullptr, y,
                                                                  dir);
  return cudaGetLastError();
}
// deformed 3D meshes: the scalar SIP diagonal through the momentum-diagonal stages
cudaError_t fast_sip_diag3_qp(const DevCtx& c, double mc, int dir, double* y) {
  if (c.dim != 3 || c.affine) return cudaErrorNotSupported;
  switch (c.kp) {
    case 1: return run_sip_diag_qp<1>(c, mc, dir, y);
    case 2: return run_sip_diag_qp<2>(c, mc, dir, y);
    case 3: return run_sip_diag_qp<3>(c, mc, dir, y);
  }
  return cudaErrorNotSupported;
}
// deformed 3D meshes: the exact momentum diagonal, sum-factorised (fast_deformed.cuh)
cudaError_t fast_momentum_diag3_qp(const DevCtx& c, MomCoef co, const double* w, double* y) {
  if (c.dim != 3 || c.affine || co.skew != 0.0 || (co.adv != 0.0 && w == nullptr)) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_momentum_diag_qp<1>(c, co, w, y);
    case 2: return run_momentum_diag_qp<2>(c, co, w, y);
    case 3: return run_momentum_diag_qp<3>(c, co, w, y);
    case 4: return run_momentum_diag_qp<4>(c, co, w, y);
  }
  return cudaErrorNotSupported;
}

// deformed (non-affine) 3D meshes: pass A + LF advection with per-qp geometry (fast_deformed.cuh)
cudaError_t fast_momentum3_qp(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  if (c.dim != 3 || c.affine || co.skew != 0.0 || (co.adv != 0.0 && w == nullptr)) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_momentum_qp<1>(c, co, w, x, y);
    case 2: return run_momentum_qp<2>(c, co, w, x, y);
    case 3: return run_momentum_qp<3>(c, co, w, x, y);
    case 4: return run_momentum_qp<4>(c, co, w, x, y);
  }
  return cudaErrorNotSupported;
}

cudaError_t fast_momentum3(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  if (co.skew != 0.0 || w == nullptr) return cudaErrorNotSupported;
  switch (c.ku) {
    case 1: return run_momentum_axis<1>(c, co, w, x, y);
    case 2: return run_momentum_axis<2>(c, co, w, x, y);
    case 3: return run_momentum_axis<3>(c, co, w, x, y);
  }
  return cudaErrorNotSupported;
}

}  // namespace dgb
