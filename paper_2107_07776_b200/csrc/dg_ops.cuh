// Matrix-free DG operator kernels (generic path: any dim/degree, affine or
// per-quadrature-point geometry).  One CTA owns CB cells; every cell
// integrates its volume terms and ALL of its faces (element-centric: each
// interior face is evaluated once from each side, so every output dof is
// written by exactly one CTA — no atomics, no colouring, deterministic).
//
// Reference correspondence (proj/src/forms.cpp):
//   k_momentum        apply_momentum        :389-604
//   k_sip             scalar_sip_apply      :148-243 (apply_pressure_helmholtz :1090,
//                                                     apply_scalar_laplace :1104)
//   k_mass            apply_mass            :337-360
//   k_gradient        pressure_gradient_rhs :1212-1233
//   k_divergence      divergence_functional :1118-1197
//   k_momentum_rhs    momentum_rhs          :816-1084
//   k_kinetic         kinetic_energy        :1239-1260
//   k_*_diag          momentum_diagonal :606-810, scalar_sip_diagonal :246-329,
//                     mass_diagonal :362-383
//
// Element-centric sign convention: the reference evaluates each interior face
// once from the owner with the owner->neighbour normal (forms.cpp:443-461,
// :555-573).  Re-deriving both sides' contributions with the normal pointing
// OUT of the cell doing the work gives the same formula on both sides (see
// DESIGN.md "Element-centric faces"), which is what the pointwise code uses.
#pragma once

#include "dg_element.cuh"

namespace dgb {

constexpr int kThreads = 256;
// generic momentum kernel: threads per block and shared-memory budget per block
// (tools/tune_gmom.sh overrides; measured best: k = 4 (cfg4) 64 threads / 48 KB: 45.8 -> 39.9 ms)
#ifdef DGB_GMOM_T
template <int K> constexpr int mom_threads() { return DGB_GMOM_T; }
template <int K> constexpr int mom_smem_kb() { return DGB_GMOM_KB; }
#else
template <int K> constexpr int mom_threads() { return K == 4 ? 64 : 256; }
template <int K> constexpr int mom_smem_kb() { return K == 4 ? 48 : 96; }
#endif

__device__ __forceinline__ bool is_outlet(const MeshArgs& m, int nb) {
  const int bid = -1 - nb;
  return bid >= 0 && bid < 64 && m.bctype[bid] == 1;
}

template <int DIM>
__device__ __forceinline__ double dotn(const double* a, const double* n) {
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) s = fma(a[d], n[d], s);
  return s;
}

// load a component block of nc cells: dst[c*cs + i] = src[(c0+c)*stride + off + i]
template <int NB>
__device__ __forceinline__ void load_block(double* dst, int cs, const double* __restrict__ src, int c0,
                                           int stride, int off, int nc) {
  for (int idx = threadIdx.x; idx < nc * NB; idx += blockDim.x) {
    const int c = idx / NB, i = idx - c * NB;
    dst[c * cs + i] = src[(size_t)(c0 + c) * stride + off + i];
  }
}
// neighbour blocks for face f (zeros on boundary faces)
template <int NB, int DIM>
__device__ __forceinline__ void load_nbr(double* dst, int cs, const double* __restrict__ src,
                                         const MeshArgs& m, int c0, int f, int stride, int off, int nc) {
  for (int idx = threadIdx.x; idx < nc * NB; idx += blockDim.x) {
    const int c = idx / NB, i = idx - c * NB;
    const int nb = m.nbr[(size_t)(c0 + c) * 2 * DIM + f];
    dst[c * cs + i] = nb >= 0 ? src[(size_t)nb * stride + off + i] : 0.0;
  }
}
template <int NB>
__device__ __forceinline__ void store_block(const double* srcs, int cs, double* __restrict__ dst, int c0,
                                            int stride, int off, int nc) {
  for (int idx = threadIdx.x; idx < nc * NB; idx += blockDim.x) {
    const int c = idx / NB, i = idx - c * NB;
    dst[(size_t)(c0 + c) * stride + off + i] = srcs[c * cs + i];
  }
}
__device__ __forceinline__ void zero(double* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0.0;
}

// ===========================================================================
// Momentum operator: y = mass M x + visc A_sip x + adv C_lf(w) x + skew (div w) x
// ===========================================================================
template <int DIM, int K>
struct MomLayout {
  static constexpr int N = K + 1, QA = K + 1, QB = K + 2, NF = 2 * DIM;
  using EA = Elem<DIM, N, QA>;
  using EB = Elem<DIM, N, QB>;
  static constexpr int NB = EA::NB;
  static constexpr int SCR = EA::SCR > EB::SCR ? EA::SCR : EB::SCR;
  static constexpr int QBK = EA::QB > EB::QB ? EA::QB : EB::QB;
  static constexpr int FBK = EA::FB > EB::FB ? EA::FB : EB::FB;
  static constexpr int WQ = (DIM + 1) * EB::NQ;       // w values + div w at rule-B points
  static constexpr int WF = NF * 2 * DIM * EB::NQF;    // w traces, both sides, every face
  static constexpr int PER_CELL = NB * (2 + NF) + SCR + QBK + 2 * FBK + WQ + WF;
  static constexpr int CB_RAW = (mom_smem_kb<K>() * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 16 ? 16 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

// w values (and div w) at rule-B cell points + traces on every face (both sides)
template <int DIM, int K, template <int, int> class Geo>
__device__ void momentum_w_phase(const MeshArgs& m, const GeoArgs& gB, bool skew, const double* __restrict__ w,
                                 int c0, int nc, double* U, double* UN, double* SCR, double* QBK, double* FBS,
                                 double* FBN, double* WQ, double* WF) {
  using L = MomLayout<DIM, K>;
  using EB = typename L::EB;
  constexpr int NB = L::NB, NQ = EB::NQ, NQF = EB::NQF, NF = L::NF;
  const Geo<DIM, L::QB> geo(gB);
  if (skew) zero(WQ, nc * L::WQ);  // div w accumulates
  __syncthreads();
  for (int d = 0; d < DIM; ++d) {
    load_block<NB>(U, NB, w, c0, DIM * NB, d * NB, nc);
    __syncthreads();
    if (skew)
      EB::template eval_cell<true>(U, NB, SCR, QBK, nc);
    else
      EB::template eval_cell<false>(U, NB, SCR, QBK, nc);
    for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
      const int c = idx / NQ, q = idx - c * NQ;
      const double* qb = QBK + c * L::QBK;
      double* wq = WQ + c * L::WQ;
      wq[d * NQ + q] = qb[q];
      if (skew) {
        double Ji[DIM * DIM], jxw;
        geo.cell(c0 + c, q, Ji, jxw);
        double gr[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = qb[(1 + a) * NQ + q];
        double g = 0.0;  // d w_d / d x_d
#pragma unroll
        for (int a = 0; a < DIM; ++a) g = fma(Ji[a * DIM + d], gr[a], g);
        wq[DIM * NQ + q] += g;
      }
    }
    __syncthreads();
    for (int f = 0; f < NF; ++f) {
      load_nbr<NB, DIM>(UN, NB, w, m, c0, f, DIM * NB, d * NB, nc);
      __syncthreads();
      EB::template eval_face_rt<false>(f, U, NB, SCR, FBS, nc);
      EB::template eval_face_rt<false>(f ^ 1, UN, NB, SCR, FBN, nc);
      for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
        const int c = idx / NQF, t = idx - c * NQF;
        double* wf = WF + c * L::WF + ((f * 2) * DIM + d) * NQF;
        wf[t] = FBS[c * L::FBK + t];
        wf[DIM * NQF + t] = FBN[c * L::FBK + t];
      }
      __syncthreads();
    }
  }
}

template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(mom_threads<K>()) k_momentum(MeshArgs m, GeoArgs gA, GeoArgs gB, MomCoef co,
                                                       const double* __restrict__ x,
                                                       const double* __restrict__ w, double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  using L = MomLayout<DIM, K>;
  using EA = typename L::EA;
  using EB = typename L::EB;
  constexpr int NB = L::NB, NF = L::NF, CB = L::CB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* UNB = U + CB * NB;         // NF neighbour blocks
  double* OUT = UNB + CB * NF * NB;
  double* SCR = OUT + CB * NB;
  double* QBK = SCR + CB * L::SCR;
  double* FBS = QBK + CB * L::QBK;
  double* FBN = FBS + CB * L::FBK;
  double* WQ = FBN + CB * L::FBK;
  double* WF = WQ + CB * L::WQ;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const bool passA = co.mass != 0.0 || co.visc != 0.0;
  const bool passB = co.adv != 0.0 || co.skew != 0.0;
  const bool skew = co.skew != 0.0;
  const double sfac = (double)((K + 1) * (K + 1));  // sip_sigma (deg+1)^2 (forms.hpp:175)

  if (passB) momentum_w_phase<DIM, K, Geo>(m, gB, skew, w, c0, nc, U, UNB, SCR, QBK, FBS, FBN, WQ, WF);

  const Geo<DIM, L::QA> geoA(gA);
  const Geo<DIM, L::QB> geoB(gB);
  for (int comp = 0; comp < DIM; ++comp) {
    load_block<NB>(U, NB, x, c0, DIM * NB, comp * NB, nc);
    for (int f = 0; f < NF; ++f) load_nbr<NB, DIM>(UNB + f * NB, NF * NB, x, m, c0, f, DIM * NB, comp * NB, nc);
    zero(OUT, nc * NB);
    __syncthreads();
    // ---------------- pass A: mass + viscous (rule k+1), forms.cpp:397-495
    if (passA) {
      constexpr int NQ = EA::NQ;
      if (co.visc != 0.0)
        EA::template eval_cell<true>(U, NB, SCR, QBK, nc);
      else
        EA::template eval_cell<false>(U, NB, SCR, QBK, nc);
      for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
        const int c = idx / NQ, q = idx - c * NQ;
        double* qb = QBK + c * EA::QB;
        double Ji[DIM * DIM], jxw;
        geoA.cell(c0 + c, q, Ji, jxw);
        const double v = qb[q];
        double gr[DIM], g[DIM], s[DIM], r[DIM];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = co.visc != 0.0 ? qb[(1 + a) * NQ + q] : 0.0;
        to_phys<DIM>(Ji, gr, g);
#pragma unroll
        for (int d = 0; d < DIM; ++d) s[d] = co.visc * g[d] * jxw;
        to_ref<DIM>(Ji, s, r);
        qb[q] = co.mass * v * jxw;
#pragma unroll
        for (int a = 0; a < DIM; ++a) qb[(1 + a) * NQ + q] = r[a];
      }
      __syncthreads();
      EA::template integrate_cell<true, true>(QBK, SCR, OUT, NB, nc);
      if (co.visc != 0.0) {
        constexpr int NQF = EA::NQF;
        for (int f = 0; f < NF; ++f) {
          EA::template eval_face_rt<true>(f, U, NB, SCR, FBS, nc);
          EA::template eval_face_rt<true>(f ^ 1, UNB + f * NB, NF * NB, SCR, FBN, nc);
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            double* fs = FBS + c * EA::FB;
            const double* fo = FBN + c * EA::FB;
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoA.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            double gr[DIM], g[DIM], s[DIM], r[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) gr[a] = fs[(1 + a) * NQF + t];
            to_phys<DIM>(Ji, gr, g);
            const double dn_s = dotn<DIM>(g, n);
            const double us = fs[t];
            double fv = 0.0, ssym = 0.0;
            if (nb >= 0) {  // interior (forms.cpp:443-461)
#pragma unroll
              for (int a = 0; a < DIM; ++a) gr[a] = fo[(1 + a) * NQF + t];
              to_phys<DIM>(Jo, gr, g);
              const double dn_o = dotn<DIM>(g, n);
              const double ju = us - fo[t];
              const double C = sfac * m.pen[(size_t)(c0 + c) * NF + f];
              fv = co.visc * (-0.5 * (dn_s + dn_o) + C * ju) * wds;
              ssym = -co.visc * 0.5 * ju * wds;
            } else if (!is_outlet(m, nb)) {  // Dirichlet boundary (forms.cpp:469-493)
              const double sK = sfac * m.pen[(size_t)(c0 + c) * NF + f];
              fv = co.visc * (-dn_s + 2.0 * sK * us) * wds;
              ssym = -co.visc * us * wds;
            }
#pragma unroll
            for (int d = 0; d < DIM; ++d) s[d] = ssym * n[d];
            to_ref<DIM>(Ji, s, r);
            fs[t] = fv;
#pragma unroll
            for (int a = 0; a < DIM; ++a) fs[(1 + a) * NQF + t] = r[a];
          }
          __syncthreads();
          EA::template integrate_face_rt<true>(f, FBS, SCR, OUT, NB, nc);
        }
      }
    }
    // ---------------- pass B: advection + skew (rule k+2), forms.cpp:498-602
    if (passB) {
      constexpr int NQ = EB::NQ;
      EB::template eval_cell<false>(U, NB, SCR, QBK, nc);
      for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
        const int c = idx / NQ, q = idx - c * NQ;
        double* qb = QBK + c * L::QBK;
        const double* wq = WQ + c * L::WQ;
        double Ji[DIM * DIM], jxw;
        geoB.cell(c0 + c, q, Ji, jxw);
        const double u = qb[q];
        double s[DIM], r[DIM];
#pragma unroll
        for (int d = 0; d < DIM; ++d) s[d] = -co.adv * u * wq[d * NQ + q] * jxw;
        to_ref<DIM>(Ji, s, r);
        qb[q] = skew ? co.skew * wq[DIM * NQ + q] * u * jxw : 0.0;
#pragma unroll
        for (int a = 0; a < DIM; ++a) qb[(1 + a) * NQ + q] = r[a];
      }
      __syncthreads();
      EB::template integrate_cell<true, true>(QBK, SCR, OUT, NB, nc);
      if (co.adv != 0.0) {
        constexpr int NQF = EB::NQF;
        for (int f = 0; f < NF; ++f) {
          EB::template eval_face_rt<false>(f, U, NB, SCR, FBS, nc);
          EB::template eval_face_rt<false>(f ^ 1, UNB + f * NB, NF * NB, SCR, FBN, nc);
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            double* fs = FBS + c * L::FBK;
            const double* fo = FBN + c * L::FBK;
            const double* wf = WF + c * L::WF + (f * 2) * DIM * NQF;
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoB.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            double ws[DIM], wo[DIM];
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
              ws[d] = wf[d * NQF + t];
              wo[d] = wf[(DIM + d) * NQF + t];
            }
            const double wn_s = dotn<DIM>(ws, n);
            const double us = fs[t];
            double fv;
            if (nb >= 0) {  // Lax-Friedrichs (forms.cpp:555-573)
              const double wn_o = dotn<DIM>(wo, n);
              const double lam = fmax(fabs(wn_s), fabs(wn_o));
              fv = co.adv * (0.5 * (us * wn_s + fo[t] * wn_o) + 0.5 * lam * (us - fo[t])) * wds;
            } else {  // forms.cpp:592-599
              const double coef = is_outlet(m, nb) ? wn_s : fabs(wn_s);
              fv = co.adv * coef * us * wds;
            }
            fs[t] = fv;
          }
          __syncthreads();
          EB::template integrate_face_rt<false>(f, FBS, SCR, OUT, NB, nc);
        }
      }
    }
    store_block<NB>(OUT, NB, y, c0, DIM * NB, comp * NB, nc);
    __syncthreads();
  }
}

// ===========================================================================
// Scalar SIP: y = mass_coef M x + interior SIP (+ homogeneous Dirichlet terms)
// ===========================================================================
template <int DIM, int KP>
struct SipLayout {
  static constexpr int N = KP + 1, Q = KP + 2, NF = 2 * DIM;
  using E = Elem<DIM, N, Q>;
  static constexpr int NB = E::NB;
  static constexpr int PER_CELL = NB * (2 + NF) + E::SCR + E::QB + 2 * E::FB;
  static constexpr int CB_RAW = (64 * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 32 ? 32 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

template <int DIM, int KP, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads, 2) k_sip(MeshArgs m, GeoArgs gq, double mass_coef, int dir_bdry,
                                                  const double* __restrict__ x, double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  using L = SipLayout<DIM, KP>;
  using E = typename L::E;
  constexpr int NB = L::NB, NF = L::NF, CB = L::CB, NQ = E::NQ, NQF = E::NQF;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* UNB = U + CB * NB;
  double* OUT = UNB + CB * NF * NB;
  double* SCR = OUT + CB * NB;
  double* QBK = SCR + CB * E::SCR;
  double* FBS = QBK + CB * E::QB;
  double* FBN = FBS + CB * E::FB;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const double sfac = (double)((KP + 1) * (KP + 1));
  const Geo<DIM, L::Q> geo(gq);

  load_block<NB>(U, NB, x, c0, NB, 0, nc);
  for (int f = 0; f < NF; ++f) load_nbr<NB, DIM>(UNB + f * NB, NF * NB, x, m, c0, f, NB, 0, nc);
  __syncthreads();
  // cells (forms.cpp:161-173)
  E::template eval_cell<true>(U, NB, SCR, QBK, nc);
  for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
    const int c = idx / NQ, q = idx - c * NQ;
    double* qb = QBK + c * E::QB;
    double Ji[DIM * DIM], jxw;
    geo.cell(c0 + c, q, Ji, jxw);
    double gr[DIM], g[DIM], r[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) gr[a] = qb[(1 + a) * NQ + q];
    to_phys<DIM>(Ji, gr, g);
#pragma unroll
    for (int d = 0; d < DIM; ++d) g[d] *= jxw;
    to_ref<DIM>(Ji, g, r);
    qb[q] = mass_coef * qb[q] * jxw;
#pragma unroll
    for (int a = 0; a < DIM; ++a) qb[(1 + a) * NQ + q] = r[a];
  }
  __syncthreads();
  E::template integrate_cell<true, false>(QBK, SCR, OUT, NB, nc);
  // faces (forms.cpp:179-242)
  for (int f = 0; f < NF; ++f) {
    E::template eval_face_rt<true>(f, U, NB, SCR, FBS, nc);
    E::template eval_face_rt<true>(f ^ 1, UNB + f * NB, NF * NB, SCR, FBN, nc);
    for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
      const int c = idx / NQF, t = idx - c * NQF;
      const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
      double* fs = FBS + c * E::FB;
      const double* fo = FBN + c * E::FB;
      double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
      geo.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
      double gr[DIM], g[DIM], s[DIM], r[DIM];
#pragma unroll
      for (int a = 0; a < DIM; ++a) gr[a] = fs[(1 + a) * NQF + t];
      to_phys<DIM>(Ji, gr, g);
      const double dn_s = dotn<DIM>(g, n);
      const double us = fs[t];
      double fv = 0.0, ssym = 0.0;
      if (nb >= 0) {
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = fo[(1 + a) * NQF + t];
        to_phys<DIM>(Jo, gr, g);
        const double dn_o = dotn<DIM>(g, n);
        const double ju = us - fo[t];
        const double C = sfac * m.pen[(size_t)(c0 + c) * NF + f];
        fv = (-0.5 * (dn_s + dn_o) + C * ju) * wds;
        ssym = -0.5 * ju * wds;
      } else if (dir_bdry) {
        const double sK = sfac * m.pen[(size_t)(c0 + c) * NF + f];
        fv = (-dn_s + 2.0 * sK * us) * wds;
        ssym = -us * wds;
      }
#pragma unroll
      for (int d = 0; d < DIM; ++d) s[d] = ssym * n[d];
      to_ref<DIM>(Ji, s, r);
      fs[t] = fv;
#pragma unroll
      for (int a = 0; a < DIM; ++a) fs[(1 + a) * NQF + t] = r[a];
    }
    __syncthreads();
    E::template integrate_face_rt<true>(f, FBS, SCR, OUT, NB, nc);
  }
  store_block<NB>(OUT, NB, y, c0, NB, 0, nc);
}

// ===========================================================================
// Mass (nc components, degree N-1, rule Q), forms.cpp:337-360
// ===========================================================================
template <int DIM, int N, int Q>
struct CellLayout {
  using E = Elem<DIM, N, Q>;
  static constexpr int PER_CELL = 2 * E::NB + E::SCR + E::QB;
  static constexpr int CB_RAW = (48 * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 32 ? 32 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

template <int DIM, int N, int Q, int NCOMP, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_mass(MeshArgs m, GeoArgs gq, const double* __restrict__ x,
                                                   double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  using L = CellLayout<DIM, N, Q>;
  using E = typename L::E;
  constexpr int NB = E::NB, NQ = E::NQ, CB = L::CB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* OUT = U + CB * NB;
  double* SCR = OUT + CB * NB;
  double* QBK = SCR + CB * E::SCR;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const Geo<DIM, Q> geo(gq);
  for (int comp = 0; comp < NCOMP; ++comp) {
    load_block<NB>(U, NB, x, c0, NCOMP * NB, comp * NB, nc);
    __syncthreads();
    E::template eval_cell<false>(U, NB, SCR, QBK, nc);
    for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
      const int c = idx / NQ, q = idx - c * NQ;
      double Ji[DIM * DIM], jxw;
      geo.cell(c0 + c, q, Ji, jxw);
      QBK[c * E::QB + q] *= jxw;
    }
    __syncthreads();
    E::template integrate_cell<false, false>(QBK, SCR, OUT, NB, nc);
    store_block<NB>(OUT, NB, y, c0, NCOMP * NB, comp * NB, nc);
    __syncthreads();
  }
}

// ===========================================================================
// Kinetic energy partials: sum 1/2 |u|^2 detJw at rule k+2 (forms.cpp:1239-1260)
// ===========================================================================
template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_kinetic(MeshArgs m, GeoArgs gq, const double* __restrict__ u,
                                                      double* __restrict__ partial) {
  constexpr int N = K + 1, Q = K + 2;
  using L = CellLayout<DIM, N, Q>;
  using E = typename L::E;
  constexpr int NB = E::NB, NQ = E::NQ, CB = L::CB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* SCR = U + 2 * CB * NB;
  double* QBK = SCR + CB * E::SCR;
  __shared__ double red[kThreads / 32];
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const Geo<DIM, Q> geo(gq);
  double acc = 0.0;
  for (int comp = 0; comp < DIM; ++comp) {
    load_block<NB>(U, NB, u, c0, DIM * NB, comp * NB, nc);
    __syncthreads();
    E::template eval_cell<false>(U, NB, SCR, QBK, nc);
    for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
      const int c = idx / NQ, q = idx - c * NQ;
      double Ji[DIM * DIM], jxw;
      geo.cell(c0 + c, q, Ji, jxw);
      const double v = QBK[c * E::QB + q];
      acc += 0.5 * v * v * jxw;
    }
    __syncthreads();
  }
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = acc;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int i = 0; i < (int)(blockDim.x >> 5); ++i) s += red[i];
    partial[blockIdx.x] = s;
  }
}

// ===========================================================================
// Gradient coupling: y_u = (grad p, phi) cellwise at rule k_u+1 (forms.cpp:1212-1233)
// ===========================================================================
template <int DIM, int K>
struct GradLayout {
  using EP = Elem<DIM, K, K + 1>;  // pressure basis (degree K-1), rule K+1
  using EU = Elem<DIM, K + 1, K + 1>;
  static constexpr int SCR = EP::SCR > EU::SCR ? EP::SCR : EU::SCR;
  static constexpr int PER_CELL = EP::NB + EU::NB + SCR + 2 * EU::QB;
  static constexpr int CB_RAW = (48 * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 32 ? 32 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_gradient(MeshArgs m, GeoArgs gq, const double* __restrict__ p,
                                                       double* __restrict__ y) {
  using L = GradLayout<DIM, K>;
  using EP = typename L::EP;
  using EU = typename L::EU;
  constexpr int CB = L::CB, NQ = EU::NQ;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* P = sm;
  double* OUT = P + CB * EP::NB;
  double* SCR = OUT + CB * EU::NB;
  double* GP = SCR + CB * L::SCR;  // pressure grads (physical) at qps
  double* QBK = GP + CB * EU::QB;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const Geo<DIM, K + 1> geo(gq);
  load_block<EP::NB>(P, EP::NB, p, c0, EP::NB, 0, nc);
  __syncthreads();
  EP::template eval_cell<true>(P, EP::NB, SCR, GP, nc);  // EP::QB == EU::QB (same rule)
  for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
    const int c = idx / NQ, q = idx - c * NQ;
    double* gp = GP + c * EU::QB;
    double Ji[DIM * DIM], jxw;
    geo.cell(c0 + c, q, Ji, jxw);
    double gr[DIM], g[DIM];
#pragma unroll
    for (int a = 0; a < DIM; ++a) gr[a] = gp[(1 + a) * NQ + q];
    to_phys<DIM>(Ji, gr, g);
#pragma unroll
    for (int a = 0; a < DIM; ++a) gp[(1 + a) * NQ + q] = g[a] * jxw;
  }
  __syncthreads();
  for (int comp = 0; comp < DIM; ++comp) {
    for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
      const int c = idx / NQ, q = idx - c * NQ;
      QBK[c * EU::QB + q] = GP[c * EU::QB + (1 + comp) * NQ + q];
    }
    __syncthreads();
    EU::template integrate_cell<false, false>(QBK, SCR, OUT, EU::NB, nc);
    store_block<EU::NB>(OUT, EU::NB, y, c0, DIM * EU::NB, comp * EU::NB, nc);
    __syncthreads();
  }
}

// ===========================================================================
// Divergence functional: y_p = (u, grad q) - sum_F <{u}.n, [q]>  (forms.cpp:1118-1197)
// ===========================================================================
template <int DIM, int K>
struct DivLayout {
  static constexpr int NF = 2 * DIM;
  using EP = Elem<DIM, K, K + 1>;
  using EU = Elem<DIM, K + 1, K + 1>;
  static constexpr int SCR = EP::SCR > EU::SCR ? EP::SCR : EU::SCR;
  static constexpr int FBK = EU::FB;
  static constexpr int PER_CELL = (1 + NF) * EU::NB + EP::NB + SCR + EU::QB + DIM * EU::NQ + 2 * DIM * EU::NQF + 2 * FBK;
  static constexpr int CB_RAW = (64 * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 32 ? 32 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_divergence(MeshArgs m, GeoArgs gq, const double* __restrict__ u,
                                                         double* __restrict__ y) {
  using L = DivLayout<DIM, K>;
  using EP = typename L::EP;
  using EU = typename L::EU;
  constexpr int CB = L::CB, NF = L::NF, NQ = EU::NQ, NQF = EU::NQF, NBU = EU::NB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* UNB = U + CB * NBU;
  double* OUT = UNB + CB * NF * NBU;
  double* SCR = OUT + CB * EP::NB;
  double* QBK = SCR + CB * L::SCR;
  double* UQ = QBK + CB * EU::QB;      // u_d at cell qps
  double* UF = UQ + CB * DIM * NQ;     // u_d traces, self + nbr
  double* FBS = UF + CB * 2 * DIM * NQF;
  double* FBN = FBS + CB * L::FBK;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const Geo<DIM, K + 1> geo(gq);
  zero(OUT, nc * EP::NB);
  for (int d = 0; d < DIM; ++d) {
    load_block<NBU>(U, NBU, u, c0, DIM * NBU, d * NBU, nc);
    __syncthreads();
    EU::template eval_cell<false>(U, NBU, SCR, QBK, nc);
    for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
      const int c = idx / NQ, q = idx - c * NQ;
      UQ[c * DIM * NQ + d * NQ + q] = QBK[c * EU::QB + q];
    }
    __syncthreads();
  }
  for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
    const int c = idx / NQ, q = idx - c * NQ;
    double Ji[DIM * DIM], jxw, s[DIM], r[DIM];
    geo.cell(c0 + c, q, Ji, jxw);
#pragma unroll
    for (int d = 0; d < DIM; ++d) s[d] = UQ[c * DIM * NQ + d * NQ + q] * jxw;
    to_ref<DIM>(Ji, s, r);
    double* qb = QBK + c * EP::QB;
    qb[q] = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) qb[(1 + a) * NQ + q] = r[a];
  }
  __syncthreads();
  EP::template integrate_cell<true, true>(QBK, SCR, OUT, EP::NB, nc);
  for (int f = 0; f < NF; ++f) {
    for (int d = 0; d < DIM; ++d) {
      load_block<NBU>(U, NBU, u, c0, DIM * NBU, d * NBU, nc);
      load_nbr<NBU, DIM>(UNB, NBU, u, m, c0, f, DIM * NBU, d * NBU, nc);
      __syncthreads();
      EU::template eval_face_rt<false>(f, U, NBU, SCR, FBS, nc);
      EU::template eval_face_rt<false>(f ^ 1, UNB, NBU, SCR, FBN, nc);
      for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
        const int c = idx / NQF, t = idx - c * NQF;
        UF[c * 2 * DIM * NQF + d * NQF + t] = FBS[c * L::FBK + t];
        UF[c * 2 * DIM * NQF + (DIM + d) * NQF + t] = FBN[c * L::FBK + t];
      }
      __syncthreads();
    }
    for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
      const int c = idx / NQF, t = idx - c * NQF;
      const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
      double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
      geo.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
      const double* uf = UF + c * 2 * DIM * NQF;
      double un = 0.0;
      if (nb >= 0) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) un += 0.5 * (uf[d * NQF + t] + uf[(DIM + d) * NQF + t]) * n[d];
      } else if (!is_outlet(m, nb)) {
#pragma unroll
        for (int d = 0; d < DIM; ++d) un += uf[d * NQF + t] * n[d];
      }
      FBS[c * EP::FB + t] = -un * wds;
    }
    __syncthreads();
    EP::template integrate_face_rt<false>(f, FBS, SCR, OUT, EP::NB, nc);
  }
  store_block<EP::NB>(OUT, EP::NB, y, c0, EP::NB, 0, nc);
}

}  // namespace dgb
