// Stage right-hand side and exact operator diagonals (once per TR-BDF2 stage).
//
//   k_momentum_rhs   momentum_rhs          proj/src/forms.cpp:816-1084
//   k_momentum_diag  momentum_diagonal     forms.cpp:606-810
//   k_sip_diag       scalar_sip_diagonal   forms.cpp:246-329
//   k_mass_diag      mass_diagonal         forms.cpp:362-383
//
// The diagonals are exact (the same quadrature sums as the reference), one
// thread per (cell, basis function), with the 1D tables staged in shared
// memory; advecting-field values at the quadrature points come from the
// sum-factorised evaluation shared with the apply kernels.
#pragma once

#include "dg_ops.cuh"

namespace dgb {

template <int DIM, int K>
struct RhsLayout {
  static constexpr int N = K + 1, QA = K + 1, QB = K + 2, NF = 2 * DIM;
  using EA = Elem<DIM, N, QA>;
  using EB = Elem<DIM, N, QB>;
  using EP = Elem<DIM, K, QA>;  // pressure space (degree K-1) at the velocity rule
  static constexpr int NB = EA::NB, NBP = EP::NB;
  static constexpr int SCR = EA::SCR > EB::SCR ? (EA::SCR > EP::SCR ? EA::SCR : EP::SCR)
                                               : (EB::SCR > EP::SCR ? EB::SCR : EP::SCR);
  static constexpr int QBK = EA::QB > EB::QB ? EA::QB : EB::QB;
  static constexpr int FBK = EA::FB > EB::FB ? EA::FB : EB::FB;
  static constexpr int WQ = DIM * EB::NQ;
  static constexpr int WF = 3 * DIM * EB::NQF;  // self, nbr, dir_w self
  static constexpr int PER_CELL = 3 * NB + 2 * NBP + SCR + 2 * QBK + 3 * FBK + WQ + WF;
  static constexpr int CB_RAW = (96 * 1024 / 8) / PER_CELL;
  static constexpr int CB = CB_RAW < 1 ? 1 : (CB_RAW > 16 ? 16 : CB_RAW);
  static constexpr size_t SMEM = (size_t)CB * PER_CELL * sizeof(double);
};

template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_momentum_rhs(MeshArgs m, GeoArgs gA, GeoArgs gB, RhsArgs ra,
                                                           double* __restrict__ y) {
  using L = RhsLayout<DIM, K>;
  using EA = typename L::EA;
  using EB = typename L::EB;
  using EP = typename L::EP;
  constexpr int NB = L::NB, NBP = L::NBP, NF = L::NF, CB = L::CB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* UN = U + CB * NB;
  double* OUT = UN + CB * NB;
  double* P = OUT + CB * NB;
  double* PN = P + CB * NBP;
  double* SCR = PN + CB * NBP;
  double* TQ = SCR + CB * L::SCR;  // test block (cell)
  double* EQ = TQ + CB * L::QBK;   // evaluation block (cell)
  double* FBS = EQ + CB * L::QBK;
  double* FBN = FBS + CB * L::FBK;
  double* FT = FBN + CB * L::FBK;
  double* WQ = FT + CB * L::FBK;
  double* WF = WQ + CB * L::WQ;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const double sfac = (double)((K + 1) * (K + 1));
  const bool any_dir = ra.dvisc != 0.0 || ra.dadv != 0.0;
  if (ra.accumulate && ra.nm + ra.nv + ra.na + ra.np == 0) {
    // boundary-data terms only: blocks without a Dirichlet face contribute nothing
    bool any = false;
    for (int i = 0; i < nc * NF; ++i) {
      const int nb = m.nbr[(size_t)c0 * NF + i];
      any = any || (nb < 0 && !is_outlet(m, nb));
    }
    if (!any) return;
  }
  const Geo<DIM, L::QA> geoA(gA);
  const Geo<DIM, L::QB> geoB(gB);

  for (int comp = 0; comp < DIM; ++comp) {
    zero(OUT, nc * NB);
    // ------------------------------------------------ rule k+1 cell terms (:824-857)
    zero(TQ, nc * EA::QB);
    __syncthreads();
    {
      constexpr int NQ = EA::NQ;
      for (int ti = 0; ti < ra.nm + ra.nv; ++ti) {
        const bool visc = ti >= ra.nm;
        const double coef = visc ? ra.vc[ti - ra.nm] : ra.mc[ti];
        const double* f = visc ? ra.vf[ti - ra.nm] : ra.mf[ti];
        load_block<NB>(U, NB, f, c0, DIM * NB, comp * NB, nc);
        __syncthreads();
        if (visc)
          EA::template eval_cell<true>(U, NB, SCR, EQ, nc);
        else
          EA::template eval_cell<false>(U, NB, SCR, EQ, nc);
        for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
          const int c = idx / NQ, q = idx - c * NQ;
          const double* eq = EQ + c * EA::QB;
          double* tq = TQ + c * EA::QB;
          double Ji[DIM * DIM], jxw;
          geoA.cell(c0 + c, q, Ji, jxw);
          if (!visc) {
            tq[q] += coef * eq[q] * jxw;
          } else {
            double gr[DIM], g[DIM], r[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) gr[a] = eq[(1 + a) * NQ + q];
            to_phys<DIM>(Ji, gr, g);
#pragma unroll
            for (int d = 0; d < DIM; ++d) g[d] *= -coef * jxw;
            to_ref<DIM>(Ji, g, r);
#pragma unroll
            for (int a = 0; a < DIM; ++a) tq[(1 + a) * NQ + q] += r[a];
          }
        }
        __syncthreads();
      }
      for (int ti = 0; ti < ra.np; ++ti) {
        load_block<NBP>(P, NBP, ra.pf[ti], c0, NBP, 0, nc);
        __syncthreads();
        EP::template eval_cell<false>(P, NBP, SCR, EQ, nc);
        for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
          const int c = idx / NQ, q = idx - c * NQ;
          double* tq = TQ + c * EA::QB;
          double Ji[DIM * DIM], jxw;
          geoA.cell(c0 + c, q, Ji, jxw);
          double s[DIM], r[DIM];
#pragma unroll
          for (int d = 0; d < DIM; ++d) s[d] = d == comp ? ra.pc[ti] * EQ[c * EA::QB + q] * jxw : 0.0;
          to_ref<DIM>(Ji, s, r);
#pragma unroll
          for (int a = 0; a < DIM; ++a) tq[(1 + a) * NQ + q] += r[a];
        }
        __syncthreads();
      }
      EA::template integrate_cell<true, true>(TQ, SCR, OUT, NB, nc);
    }
    // ------------------------------------------------ rule k+1 face terms (:859-952)
    if (ra.nv + ra.np > 0) {
      constexpr int NQF = EA::NQF;
      for (int f = 0; f < NF; ++f) {
        zero(FT, nc * EA::FB);
        __syncthreads();
        for (int ti = 0; ti < ra.nv; ++ti) {
          load_block<NB>(U, NB, ra.vf[ti], c0, DIM * NB, comp * NB, nc);
          load_nbr<NB, DIM>(UN, NB, ra.vf[ti], m, c0, f, DIM * NB, comp * NB, nc);
          __syncthreads();
          EA::template eval_face_rt<true>(f, U, NB, SCR, FBS, nc);
          EA::template eval_face_rt<true>(f ^ 1, UN, NB, SCR, FBN, nc);
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            if (nb < 0 && is_outlet(m, nb)) continue;
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoA.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            const double* fs = FBS + c * EA::FB;
            const double* fo = FBN + c * EA::FB;
            double gr[DIM], g[DIM];
#pragma unroll
            for (int a = 0; a < DIM; ++a) gr[a] = fs[(1 + a) * NQF + t];
            to_phys<DIM>(Ji, gr, g);
            const double dn_s = dotn<DIM>(g, n);
            double fv;
            if (nb >= 0) {
#pragma unroll
              for (int a = 0; a < DIM; ++a) gr[a] = fo[(1 + a) * NQF + t];
              to_phys<DIM>(Jo, gr, g);
              fv = ra.vc[ti] * 0.5 * (dn_s + dotn<DIM>(g, n)) * wds;
            } else {
              fv = ra.vc[ti] * dn_s * wds;
            }
            FT[c * EA::FB + t] += fv;
          }
          __syncthreads();
        }
        for (int ti = 0; ti < ra.np; ++ti) {
          load_block<NBP>(P, NBP, ra.pf[ti], c0, NBP, 0, nc);
          load_nbr<NBP, DIM>(PN, NBP, ra.pf[ti], m, c0, f, NBP, 0, nc);
          __syncthreads();
          EP::template eval_face_rt<false>(f, P, NBP, SCR, FBS, nc);
          EP::template eval_face_rt<false>(f ^ 1, PN, NBP, SCR, FBN, nc);
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            if (nb < 0 && is_outlet(m, nb)) continue;
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoA.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            const double ps = FBS[c * EA::FB + t];
            const double pv = nb >= 0 ? 0.5 * (ps + FBN[c * EA::FB + t]) : ps;
            FT[c * EA::FB + t] -= ra.pc[ti] * pv * n[comp] * wds;
          }
          __syncthreads();
        }
        EA::template integrate_face_rt<false>(f, FT, SCR, OUT, NB, nc);
      }
    }
    // ------------------------------------------------ rule k+2: advection + boundary data (:955-1083)
    if (ra.na > 0 || any_dir) {
      constexpr int NQ = EB::NQ, NQF = EB::NQF;
      if (ra.na > 0) {
        zero(TQ, nc * L::QBK);
        __syncthreads();
        for (int ti = 0; ti < ra.na; ++ti) {
          for (int d = 0; d < DIM; ++d) {
            load_block<NB>(U, NB, ra.aw[ti], c0, DIM * NB, d * NB, nc);
            __syncthreads();
            EB::template eval_cell<false>(U, NB, SCR, EQ, nc);
            for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
              const int c = idx / NQ, q = idx - c * NQ;
              WQ[c * L::WQ + d * NQ + q] = EQ[c * L::QBK + q];
            }
            __syncthreads();
          }
          load_block<NB>(U, NB, ra.af[ti], c0, DIM * NB, comp * NB, nc);
          __syncthreads();
          EB::template eval_cell<false>(U, NB, SCR, EQ, nc);
          for (int idx = threadIdx.x; idx < nc * NQ; idx += blockDim.x) {
            const int c = idx / NQ, q = idx - c * NQ;
            double Ji[DIM * DIM], jxw;
            geoB.cell(c0 + c, q, Ji, jxw);
            const double fval = EQ[c * L::QBK + q];
            double s[DIM], r[DIM];
#pragma unroll
            for (int d = 0; d < DIM; ++d) s[d] = ra.ac[ti] * fval * WQ[c * L::WQ + d * NQ + q] * jxw;
            to_ref<DIM>(Ji, s, r);
#pragma unroll
            for (int a = 0; a < DIM; ++a) TQ[c * L::QBK + (1 + a) * NQ + q] += r[a];
          }
          __syncthreads();
        }
        EB::template integrate_cell<true, true>(TQ, SCR, OUT, NB, nc);
      }
      for (int f = 0; f < NF; ++f) {
        zero(FT, nc * L::FBK);
        __syncthreads();
        for (int ti = 0; ti < ra.na; ++ti) {
          for (int d = 0; d < DIM; ++d) {
            load_block<NB>(U, NB, ra.aw[ti], c0, DIM * NB, d * NB, nc);
            load_nbr<NB, DIM>(UN, NB, ra.aw[ti], m, c0, f, DIM * NB, d * NB, nc);
            __syncthreads();
            EB::template eval_face_rt<false>(f, U, NB, SCR, FBS, nc);
            EB::template eval_face_rt<false>(f ^ 1, UN, NB, SCR, FBN, nc);
            for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
              const int c = idx / NQF, t = idx - c * NQF;
              WF[c * L::WF + d * NQF + t] = FBS[c * L::FBK + t];
              WF[c * L::WF + (DIM + d) * NQF + t] = FBN[c * L::FBK + t];
            }
            __syncthreads();
          }
          load_block<NB>(U, NB, ra.af[ti], c0, DIM * NB, comp * NB, nc);
          load_nbr<NB, DIM>(UN, NB, ra.af[ti], m, c0, f, DIM * NB, comp * NB, nc);
          __syncthreads();
          EB::template eval_face_rt<false>(f, U, NB, SCR, FBS, nc);
          EB::template eval_face_rt<false>(f ^ 1, UN, NB, SCR, FBN, nc);
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoB.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            const double* wf = WF + c * L::WF;
            double ws[DIM], wo[DIM];
#pragma unroll
            for (int d = 0; d < DIM; ++d) {
              ws[d] = wf[d * NQF + t];
              wo[d] = wf[(DIM + d) * NQF + t];
            }
            const double wn_s = dotn<DIM>(ws, n);
            const double fs = FBS[c * L::FBK + t];
            double fv;
            if (nb >= 0)
              fv = ra.ac[ti] * 0.5 * (fs * wn_s + FBN[c * L::FBK + t] * dotn<DIM>(wo, n)) * wds;
            else
              fv = ra.ac[ti] * fs * wn_s * wds;
            FT[c * L::FBK + t] -= fv;
          }
          __syncthreads();
        }
        if (any_dir) {
          if (ra.dadv != 0.0) {
            for (int d = 0; d < DIM; ++d) {
              load_block<NB>(U, NB, ra.dir_w, c0, DIM * NB, d * NB, nc);
              __syncthreads();
              EB::template eval_face_rt<false>(f, U, NB, SCR, FBS, nc);
              for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
                const int c = idx / NQF, t = idx - c * NQF;
                WF[c * L::WF + (2 * DIM + d) * NQF + t] = FBS[c * L::FBK + t];
              }
              __syncthreads();
            }
          }
          for (int idx = threadIdx.x; idx < nc * NQF; idx += blockDim.x) {
            const int c = idx / NQF, t = idx - c * NQF;
            const int nb = m.nbr[(size_t)(c0 + c) * NF + f];
            if (nb >= 0 || is_outlet(m, nb)) continue;
            double Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
            geoB.face(c0 + c, f, nb, t, Ji, Jo, n, wds);
            const int b = m.bslot[(size_t)(c0 + c) * NF + f];
            const double g = ra.gtab ? ra.gtab[((size_t)b * NQF + t) * DIM + comp] : 0.0;
            const double sK = sfac * m.pen[(size_t)(c0 + c) * NF + f];
            double* ft = FT + c * L::FBK;
            double fv = 0.0;
            if (ra.dvisc != 0.0) {
              fv += ra.dvisc * 2.0 * sK * g * wds;
              double s[DIM], r[DIM];
#pragma unroll
              for (int d = 0; d < DIM; ++d) s[d] = -ra.dvisc * g * n[d] * wds;
              to_ref<DIM>(Ji, s, r);
#pragma unroll
              for (int a = 0; a < DIM; ++a) ft[(1 + a) * NQF + t] += r[a];
            }
            if (ra.dadv != 0.0) {
              double ws[DIM];
#pragma unroll
              for (int d = 0; d < DIM; ++d) ws[d] = WF[c * L::WF + (2 * DIM + d) * NQF + t];
              const double wn = dotn<DIM>(ws, n);
              fv += ra.dadv * (fabs(wn) - wn) * g * wds;
            }
            ft[t] += fv;
          }
          __syncthreads();
        }
        EB::template integrate_face_rt<true>(f, FT, SCR, OUT, NB, nc);
      }
    }
    if (ra.accumulate) {
      for (int idx = threadIdx.x; idx < nc * NB; idx += blockDim.x) {
        const int c = idx / NB, i = idx - c * NB;
        y[(size_t)(c0 + c) * DIM * NB + comp * NB + i] += OUT[c * NB + i];
      }
    } else {
      store_block<NB>(OUT, NB, y, c0, DIM * NB, comp * NB, nc);
    }
    __syncthreads();
  }
}

// ===========================================================================
// Diagonals
// ===========================================================================
// shared-memory copy of one (N, Q) table: B[Q][N], D[Q][N], dE[2][N]
template <int N, int Q>
__device__ __forceinline__ void stage_tab(double* s) {
  const double* src = &c_tab<N, Q>.B[0][0];
  constexpr int n = 2 * Q * N + 2 * N;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s[i] = src[i];
}
template <int N, int Q>
struct STab {
  const double* s;
  __device__ double B(int q, int i) const { return s[q * N + i]; }
  __device__ double D(int q, int i) const { return s[Q * N + q * N + i]; }
  __device__ double E(int side, int i) const { return s[2 * Q * N + side * N + i]; }
  static constexpr int SIZE = 2 * Q * N + 2 * N;
};

// value and reference gradient of basis function (i0,i1,i2) at cell point (q0,q1,q2)
template <int DIM, int N, int Q>
__device__ __forceinline__ void basis_cell(const STab<N, Q>& t, const int* ii, int q, double& phi, double* gr) {
  int qq[3] = {q % Q, (q / Q) % Q, DIM == 3 ? q / (Q * Q) : 0};
  double b[3], d[3];
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    b[k] = t.B(qq[k], ii[k]);
    d[k] = t.D(qq[k], ii[k]);
  }
  phi = b[0] * b[1] * (DIM == 3 ? b[2] : 1.0);
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double g = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) g *= (k == a) ? d[k] : b[k];
    gr[a] = g;
  }
}
// same at face point t of local face f (canonical embedding)
template <int DIM, int N, int Q>
__device__ __forceinline__ void basis_face(const STab<N, Q>& tb, const int* ii, int f, int t, double& phi,
                                           double* gr) {
  const int A = f / 2, S = f % 2;
  const bool on = ii[A] == (S ? N - 1 : 0);
  double b[3], d[3];
  int rem = t;
#pragma unroll
  for (int k = 0; k < DIM; ++k) {
    if (k == A) {
      b[k] = on ? 1.0 : 0.0;
      d[k] = tb.E(S, ii[k]);
    } else {
      const int qk = rem % Q;
      rem /= Q;
      b[k] = tb.B(qk, ii[k]);
      d[k] = tb.D(qk, ii[k]);
    }
  }
  phi = b[0] * b[1] * (DIM == 3 ? b[2] : 1.0);
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double g = 1.0;
#pragma unroll
    for (int k = 0; k < DIM; ++k) g *= (k == a) ? d[k] : b[k];
    gr[a] = g;
  }
}
template <int DIM, int N>
__device__ __forceinline__ void basis_digits(int i, int* ii) {
  ii[0] = i % N;
  ii[1] = (i / N) % N;
  ii[2] = DIM == 3 ? i / (N * N) : 0;
}

template <int DIM, int K>
struct MomDiagLayout {
  using L = MomLayout<DIM, K>;
  static constexpr int TABS = STab<K + 1, K + 1>::SIZE + STab<K + 1, K + 2>::SIZE;
  static constexpr size_t SMEM = L::SMEM + TABS * sizeof(double);
};

template <int DIM, int K, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_momentum_diag(MeshArgs m, GeoArgs gA, GeoArgs gB, MomCoef co,
                                                            const double* __restrict__ w, double* __restrict__ y) {
  using L = MomLayout<DIM, K>;
  using EB = typename L::EB;
  constexpr int N = K + 1, QA = K + 1, QB = K + 2, NB = L::NB, NF = L::NF, CB = L::CB;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  double* U = sm;
  double* UNB = U + CB * NB;
  double* OUT = UNB + CB * NF * NB;
  double* SCR = OUT + CB * NB;
  double* QBK = SCR + CB * L::SCR;
  double* FBS = QBK + CB * L::QBK;
  double* FBN = FBS + CB * L::FBK;
  double* WQ = FBN + CB * L::FBK;
  double* WF = WQ + CB * L::WQ;
  double* TA = WF + CB * L::WF;
  double* TB = TA + STab<N, QA>::SIZE;
  const int c0 = blockIdx.x * CB;
  const int nc = min(CB, m.ncells - c0);
  const bool passB = co.adv != 0.0 || co.skew != 0.0;
  const double sfac = (double)((K + 1) * (K + 1));
  stage_tab<N, QA>(TA);
  stage_tab<N, QB>(TB);
  if (passB) momentum_w_phase<DIM, K, Geo>(m, gB, co.skew != 0.0, w, c0, nc, U, UNB, SCR, QBK, FBS, FBN, WQ, WF);
  __syncthreads();
  const STab<N, QA> ta{TA};
  const STab<N, QB> tb{TB};
  const Geo<DIM, QA> geoA(gA);
  const Geo<DIM, QB> geoB(gB);
  for (int idx = threadIdx.x; idx < nc * NB; idx += blockDim.x) {
    const int c = idx / NB, i = idx - c * NB;
    const int cell = c0 + c;
    int ii[3];
    basis_digits<DIM, N>(i, ii);
    double s = 0.0;
    // cell, rule k+1 (:616-637)
    for (int q = 0; q < Elem<DIM, N, QA>::NQ; ++q) {
      double phi, gr[DIM], g[DIM], Ji[DIM * DIM], jxw;
      basis_cell<DIM, N, QA>(ta, ii, q, phi, gr);
      geoA.cell(cell, q, Ji, jxw);
      to_phys<DIM>(Ji, gr, g);
      double g2 = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) g2 += g[d] * g[d];
      s += (co.mass * phi * phi + co.visc * g2) * jxw;
    }
    if (passB) {  // :639-674
      constexpr int NQ = EB::NQ;
      const double* wq = WQ + c * L::WQ;
      for (int q = 0; q < NQ; ++q) {
        double phi, gr[DIM], g[DIM], Ji[DIM * DIM], jxw;
        basis_cell<DIM, N, QB>(tb, ii, q, phi, gr);
        geoB.cell(cell, q, Ji, jxw);
        to_phys<DIM>(Ji, gr, g);
        double wg = 0.0;
#pragma unroll
        for (int d = 0; d < DIM; ++d) wg += wq[d * NQ + q] * g[d];
        s += -co.adv * phi * wg * jxw;
        // div w is only computed (and the slot only initialised) when skew != 0
        if (co.skew != 0.0) s += co.skew * wq[DIM * NQ + q] * phi * phi * jxw;
      }
    }
    for (int f = 0; f < NF; ++f) {
      const int nb = m.nbr[(size_t)cell * NF + f];
      if (co.visc != 0.0 && !(nb < 0 && is_outlet(m, nb))) {  // :677-737
        const double pen = sfac * m.pen[(size_t)cell * NF + f];
        for (int t = 0; t < Elem<DIM, N, QA>::NQF; ++t) {
          double phi, gr[DIM], g[DIM], Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
          basis_face<DIM, N, QA>(ta, ii, f, t, phi, gr);
          geoA.face(cell, f, nb, t, Ji, Jo, n, wds);
          to_phys<DIM>(Ji, gr, g);
          const double dn = dotn<DIM>(g, n);
          if (nb >= 0)
            s += co.visc * (-phi * dn + pen * phi * phi) * wds;
          else
            s += co.visc * (-2.0 * phi * dn + 2.0 * pen * phi * phi) * wds;
        }
      }
      if (co.adv != 0.0) {  // :740-809
        constexpr int NQF = EB::NQF;
        const double* wf = WF + c * L::WF + (f * 2) * DIM * NQF;
        for (int t = 0; t < NQF; ++t) {
          double phi, gr[DIM], Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
          basis_face<DIM, N, QB>(tb, ii, f, t, phi, gr);
          geoB.face(cell, f, nb, t, Ji, Jo, n, wds);
          double ws[DIM], wo[DIM];
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            ws[d] = wf[d * NQF + t];
            wo[d] = wf[(DIM + d) * NQF + t];
          }
          const double wn_s = dotn<DIM>(ws, n);
          if (nb >= 0) {
            const double lam = fmax(fabs(wn_s), fabs(dotn<DIM>(wo, n)));
            s += co.adv * (0.5 * wn_s + 0.5 * lam) * phi * phi * wds;
          } else {
            const double coef = is_outlet(m, nb) ? wn_s : fabs(wn_s);
            s += co.adv * coef * phi * phi * wds;
          }
        }
      }
    }
#pragma unroll
    for (int comp = 0; comp < DIM; ++comp) y[(size_t)cell * DIM * NB + comp * NB + i] = s;
  }
}

template <int DIM, int KP, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_sip_diag(MeshArgs m, GeoArgs gq, double mass_coef, int dir_bdry,
                                                       double* __restrict__ y) {
  constexpr int N = KP + 1, Q = KP + 2, NF = 2 * DIM;
  using E = Elem<DIM, N, Q>;
  __shared__ double TT[STab<N, Q>::SIZE];
  stage_tab<N, Q>(TT);
  __syncthreads();
  const STab<N, Q> tb{TT};
  const Geo<DIM, Q> geo(gq);
  const double sfac = (double)((KP + 1) * (KP + 1));
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)m.ncells * E::NB;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int cell = (int)(idx / E::NB), i = (int)(idx % E::NB);
    int ii[3];
    basis_digits<DIM, N>(i, ii);
    double s = 0.0;
    for (int q = 0; q < E::NQ; ++q) {  // forms.cpp:257-271
      double phi, gr[DIM], g[DIM], Ji[DIM * DIM], jxw;
      basis_cell<DIM, N, Q>(tb, ii, q, phi, gr);
      geo.cell(cell, q, Ji, jxw);
      to_phys<DIM>(Ji, gr, g);
      double g2 = 0.0;
#pragma unroll
      for (int d = 0; d < DIM; ++d) g2 += g[d] * g[d];
      s += (mass_coef * phi * phi + g2) * jxw;
    }
    for (int f = 0; f < NF; ++f) {  // :273-328
      const int nb = m.nbr[(size_t)cell * NF + f];
      if (nb < 0 && !dir_bdry) continue;
      const double pen = sfac * m.pen[(size_t)cell * NF + f];
      for (int t = 0; t < E::NQF; ++t) {
        double phi, gr[DIM], g[DIM], Ji[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
        basis_face<DIM, N, Q>(tb, ii, f, t, phi, gr);
        geo.face(cell, f, nb, t, Ji, Jo, n, wds);
        to_phys<DIM>(Ji, gr, g);
        const double dn = dotn<DIM>(g, n);
        if (nb >= 0)
          s += (-phi * dn + pen * phi * phi) * wds;
        else
          s += (-2.0 * phi * dn + 2.0 * pen * phi * phi) * wds;
      }
    }
    y[idx] = s;
  }
}

template <int DIM, int N, int Q, int NCOMP, template <int, int> class Geo>
__global__ void __launch_bounds__(kThreads) k_mass_diag(MeshArgs m, GeoArgs gq, double* __restrict__ y) {
  using E = Elem<DIM, N, Q>;
  __shared__ double TT[STab<N, Q>::SIZE];
  stage_tab<N, Q>(TT);
  __syncthreads();
  const STab<N, Q> tb{TT};
  const Geo<DIM, Q> geo(gq);
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)m.ncells * E::NB;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int cell = (int)(idx / E::NB), i = (int)(idx % E::NB);
    int ii[3];
    basis_digits<DIM, N>(i, ii);
    double s = 0.0;
    for (int q = 0; q < E::NQ; ++q) {
      double phi, gr[DIM], Ji[DIM * DIM], jxw;
      basis_cell<DIM, N, Q>(tb, ii, q, phi, gr);
      geo.cell(cell, q, Ji, jxw);
      s += phi * phi * jxw;
    }
#pragma unroll
    for (int comp = 0; comp < NCOMP; ++comp) y[(size_t)cell * NCOMP * E::NB + comp * E::NB + i] = s;
  }
}

}  // namespace dgb
