// Axis-aligned affine 3D fast kernels (fast_axis.cuh) + their launchers.
#include "fast_axis.cuh"

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

template <class KernelT>
static cudaError_t set_smem(KernelT kern, size_t smem) {
  return cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
}

template <int KP>
static cudaError_t run_sip_axis(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  using G = SipAxisCfg<KP>;
  cudaError_t e = ensure_ftab<KP + 1, KP + 1>();
  if (e != cudaSuccess) return e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_sip_axis<KP, true>, G::SMEM)) != cudaSuccess) return e;
    k_sip_axis<KP, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, x, y);
  } else {
    if ((e = set_smem(k_sip_axis<KP, false>, G::SMEM)) != cudaSuccess) return e;
    k_sip_axis<KP, false><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, mc, dir, x, y);
  }
  return cudaGetLastError();
}

template <int K, int MODE>
static cudaError_t launch_momentum_axis(const DevCtx& c, MomCoef co, const double* w, const double* x, double* y) {
  constexpr int CC = MomAxisTune<K, MODE>::C, TH = MomAxisTune<K, MODE>::T;
  using G = MomAxisCfg<K, CC, TH, MODE>;
  cudaError_t e;
  const int grid = (c.ncells + G::C - 1) / G::C;
  if (c.ug.n > 0) {
    if ((e = set_smem(k_momentum_axis<K, CC, TH, MODE, true>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_axis<K, CC, TH, MODE, true><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, x, w, y);
  } else {
    if ((e = set_smem(k_momentum_axis<K, CC, TH, MODE, false>, G::SMEM)) != cudaSuccess) return e;
    k_momentum_axis<K, CC, TH, MODE, false><<<grid, G::T, G::SMEM, c.stream>>>(c.mesh, c.ug, c.aff, co, x, w, y);
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

cudaError_t fast_sip3(const DevCtx& c, double mc, int dir, const double* x, double* y) {
  switch (c.kp) {
    case 1: return run_sip_axis<1>(c, mc, dir, x, y);
    case 2: return run_sip_axis<2>(c, mc, dir, x, y);
    case 3: return run_sip_axis<3>(c, mc, dir, x, y);
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
