// Runtime (dim, degree, geometry-kind) -> template dispatch for the generic
// operator kernels.  Included by ops_d2.cu / ops_d3.cu with DGB_DIM defined,
// so the two dimensions compile in parallel translation units.
#pragma once

#include "dg_ops_rhs.cuh"

namespace dgb {

inline GeoArgs geo_for(const DevCtx& c, int Q) {
  GeoArgs g;
  g.aff = c.aff;
  g.qcell = (Q >= 0 && Q < kMaxRule) ? c.qcell[Q] : nullptr;
  g.qface = (Q >= 0 && Q < kMaxRule) ? c.qface[Q] : nullptr;
  g.nbr = c.mesh.nbr;
  return g;
}

template <class KernelT>
inline cudaError_t prep(KernelT kern, size_t smem) {
  if (smem > 48 * 1024) return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  return cudaSuccess;
}

template <int DIM, int K, bool AFF>
cudaError_t run_momentum(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  using L = MomLayout<DIM, K>;
  auto kern = AFF ? k_momentum<DIM, K, GeoAff> : k_momentum<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, mom_threads<K>(), L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 1), geo_for(c, K + 2), co, x, w, y);
  return cudaGetLastError();
}

template <int DIM, int K, bool AFF>
cudaError_t run_momentum_diag(const DevCtx& c, MomCoef co, const double* w, double* y) {
  using L = MomDiagLayout<DIM, K>;
  auto kern = AFF ? k_momentum_diag<DIM, K, GeoAff> : k_momentum_diag<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + MomLayout<DIM, K>::CB - 1) / MomLayout<DIM, K>::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 1), geo_for(c, K + 2), co, w, y);
  return cudaGetLastError();
}

template <int DIM, int K, bool AFF>
cudaError_t run_rhs(const DevCtx& c, const RhsArgs& ra, double* y) {
  using L = RhsLayout<DIM, K>;
  auto kern = AFF ? k_momentum_rhs<DIM, K, GeoAff> : k_momentum_rhs<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 1), geo_for(c, K + 2), ra, y);
  return cudaGetLastError();
}

template <int DIM, int KP, bool AFF>
cudaError_t run_sip(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  using L = SipLayout<DIM, KP>;
  auto kern = AFF ? k_sip<DIM, KP, GeoAff> : k_sip<DIM, KP, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, KP + 2), mc, dir, x, y);
  return cudaGetLastError();
}

template <int DIM, int KP, bool AFF>
cudaError_t run_sip_diag(const DevCtx& c, double mc, int dir, double* y) {
  auto kern = AFF ? k_sip_diag<DIM, KP, GeoAff> : k_sip_diag<DIM, KP, GeoQp>;
  const long long n = (long long)c.ncells * Elem<DIM, KP + 1, KP + 2>::NB;
  const int grid = (int)((n + kThreads - 1) / kThreads);
  kern<<<grid, kThreads, 0, c.stream>>>(c.mesh, geo_for(c, KP + 2), mc, dir, y);
  return cudaGetLastError();
}

template <int DIM, int N, int Q, int NCOMP, bool AFF>
cudaError_t run_mass(const DevCtx& c, const double* x, double* y) {
  using L = CellLayout<DIM, N, Q>;
  auto kern = AFF ? k_mass<DIM, N, Q, NCOMP, GeoAff> : k_mass<DIM, N, Q, NCOMP, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, Q), x, y);
  return cudaGetLastError();
}

template <int DIM, int N, int Q, int NCOMP, bool AFF>
cudaError_t run_mass_diag(const DevCtx& c, double* y) {
  auto kern = AFF ? k_mass_diag<DIM, N, Q, NCOMP, GeoAff> : k_mass_diag<DIM, N, Q, NCOMP, GeoQp>;
  const long long n = (long long)c.ncells * Elem<DIM, N, Q>::NB;
  const int grid = (int)((n + kThreads - 1) / kThreads);
  kern<<<grid, kThreads, 0, c.stream>>>(c.mesh, geo_for(c, Q), y);
  return cudaGetLastError();
}

template <int DIM, int K, bool AFF>
cudaError_t run_gradient(const DevCtx& c, const double* p, double* y) {
  using L = GradLayout<DIM, K>;
  auto kern = AFF ? k_gradient<DIM, K, GeoAff> : k_gradient<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 1), p, y);
  return cudaGetLastError();
}

template <int DIM, int K, bool AFF>
cudaError_t run_divergence(const DevCtx& c, const double* u, double* y) {
  using L = DivLayout<DIM, K>;
  auto kern = AFF ? k_divergence<DIM, K, GeoAff> : k_divergence<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 1), u, y);
  return cudaGetLastError();
}

template <int DIM, int K, bool AFF>
cudaError_t run_kinetic(const DevCtx& c, const double* u, double* partial, int* nblocks) {
  using L = CellLayout<DIM, K + 1, K + 2>;
  auto kern = AFF ? k_kinetic<DIM, K, GeoAff> : k_kinetic<DIM, K, GeoQp>;
  cudaError_t e = prep(kern, L::SMEM);
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + L::CB - 1) / L::CB;
  *nblocks = grid;
  if (partial == nullptr) return cudaSuccess;  // size query
  kern<<<grid, kThreads, L::SMEM, c.stream>>>(c.mesh, geo_for(c, K + 2), u, partial);
  return cudaGetLastError();
}

// ---------------------------------------------------------------------------
// Per-(dim, degree) operator table.  Velocity-space ops use the table of the
// velocity degree ku, scalar-space ops (sip, sip_diag, mass(space 1)) the
// table of the scalar degree kp.  One translation unit per (dim, degree).
// ---------------------------------------------------------------------------
template <int DIM, int K>
struct DegreeOps {
  static cudaError_t momentum(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
    return c.affine ? run_momentum<DIM, K, true>(c, co, w, x, y) : run_momentum<DIM, K, false>(c, co, w, x, y);
  }
  static cudaError_t momentum_diag(const DevCtx& c, MomCoef co, const double* w, double* y) {
    return c.affine ? run_momentum_diag<DIM, K, true>(c, co, w, y) : run_momentum_diag<DIM, K, false>(c, co, w, y);
  }
  static cudaError_t rhs(const DevCtx& c, const RhsArgs& ra, double* y) {
    if constexpr (K < 2) {
      return cudaErrorNotSupported;
    } else {
      if (c.kp != c.ku - 1 && ra.np > 0) return cudaErrorNotSupported;
      return c.affine ? run_rhs<DIM, K, true>(c, ra, y) : run_rhs<DIM, K, false>(c, ra, y);
    }
  }
  static cudaError_t sip(const DevCtx& c, double mc, int dir, const double* x, double* y) {
    return c.affine ? run_sip<DIM, K, true>(c, mc, dir, x, y) : run_sip<DIM, K, false>(c, mc, dir, x, y);
  }
  static cudaError_t sip_diag(const DevCtx& c, double mc, int dir, double* y) {
    return c.affine ? run_sip_diag<DIM, K, true>(c, mc, dir, y) : run_sip_diag<DIM, K, false>(c, mc, dir, y);
  }
  // space 0: velocity (degree K, rule K+1, DIM components); 1: scalar (degree K, rule K+2)
  static cudaError_t mass(const DevCtx& c, int space, const double* x, double* y) {
    if (space == 0)
      return c.affine ? run_mass<DIM, K + 1, K + 1, DIM, true>(c, x, y) : run_mass<DIM, K + 1, K + 1, DIM, false>(c, x, y);
    return c.affine ? run_mass<DIM, K + 1, K + 2, 1, true>(c, x, y) : run_mass<DIM, K + 1, K + 2, 1, false>(c, x, y);
  }
  static cudaError_t mass_diag(const DevCtx& c, int space, double* y) {
    if (space == 0)
      return c.affine ? run_mass_diag<DIM, K + 1, K + 1, DIM, true>(c, y) : run_mass_diag<DIM, K + 1, K + 1, DIM, false>(c, y);
    return c.affine ? run_mass_diag<DIM, K + 1, K + 2, 1, true>(c, y) : run_mass_diag<DIM, K + 1, K + 2, 1, false>(c, y);
  }
  static cudaError_t gradient(const DevCtx& c, const double* p, double* y) {
    if constexpr (K < 2) {
      return cudaErrorNotSupported;
    } else {
      if (c.kp != c.ku - 1) return cudaErrorNotSupported;
      return c.affine ? run_gradient<DIM, K, true>(c, p, y) : run_gradient<DIM, K, false>(c, p, y);
    }
  }
  static cudaError_t divergence(const DevCtx& c, const double* u, double* y) {
    if constexpr (K < 2) {
      return cudaErrorNotSupported;
    } else {
      if (c.kp != c.ku - 1) return cudaErrorNotSupported;
      return c.affine ? run_divergence<DIM, K, true>(c, u, y) : run_divergence<DIM, K, false>(c, u, y);
    }
  }
  static cudaError_t kinetic(const DevCtx& c, const double* u, double* partial, int* nblocks) {
    return c.affine ? run_kinetic<DIM, K, true>(c, u, partial, nblocks) : run_kinetic<DIM, K, false>(c, u, partial, nblocks);
  }
  static cudaError_t tables() {
    cudaError_t e = ensure_tab<K + 1, K + 1>();
    if (e == cudaSuccess) e = ensure_tab<K + 1, K + 2>();
    if constexpr (K >= 2)
      if (e == cudaSuccess) e = ensure_tab<K, K + 1>();
    return e;
  }
  static const OpTable& table() {
    static const OpTable t = {momentum, momentum_diag, rhs,      sip,        sip_diag, mass,
                              mass_diag, gradient,     divergence, kinetic, tables};
    return t;
  }
};

}  // namespace dgb
