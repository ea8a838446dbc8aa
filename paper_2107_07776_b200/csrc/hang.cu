// Hanging-face supplement of the generic operator kernels (see hang.hpp).
//
// Reference correspondence (proj/src):
//   subface records / emb_out        mesh.cpp:344-375 (FaceInfo, mesh.hpp:28-64)
//   subface geometry (w_ds, normal,  space.cpp:100-150: w_ds and the normal from the
//     Jinv_in / Jinv_out)              owner (fine) side, Jinv_out at emb_out points
//   traces through the embedding     space.cpp:216-237 (trace_table keyed by embedding)
//   penalty                          forms.cpp:111-121 (mean of both sides, |F| = fine face)
//   momentum faces                   forms.cpp:443-461 (viscous), :555-573 (Lax-Friedrichs)
//   scalar SIP faces                 forms.cpp:179-242
//   momentum / SIP diagonals         forms.cpp:677-809, :273-328
//   stage RHS interior faces         forms.cpp:859-952 (viscous, pressure), :1010-1048 (advective)
//   divergence interior faces        forms.cpp:1160-1190
// Every integrand is the element-centric one of dg_ops.cuh / dg_ops_rhs.cuh written
// for the side doing the work (normal out of that side), evaluated once per side.
#include "hang.hpp"

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <map>
#include <vector>

#include "dg_common.cuh"

namespace dgb {

namespace {

constexpr int kHK = 4;  // table kinds: velocity basis @ rule ku+1, @ ku+2, pressure @ kp+2, @ ku+1
constexpr int kHR = 3;  // rule kinds: A = ku+1, B = ku+2, S = kp+2
__host__ __device__ constexpr int rule_of(int kind) { return kind == 1 ? 1 : (kind == 2 ? 2 : 0); }
constexpr int kThr = 128;

struct HangDev {
  int n = 0, nbu = 0, nbp = 0, nqm = 0;
  double sfu = 0.0, sfp = 0.0;  // (k+1)^2 of the velocity / pressure space (forms.hpp:175-177)
  const int* rec = nullptr;     // [n][4] fine cell, fine face, coarse cell, coarse face
  const double* pen = nullptr;  // [n] mean |F|/|K|
  const double* tab = nullptr;
  const long long* toff = nullptr;  // [kHK][n][2] table offsets (side 0 = fine, 1 = coarse)
  int nqf[kHR] = {};
  const double* geo[kHR] = {};  // [n][nqf][2 dim^2 + dim + 1]: Jinv_in, Jinv_out, n (fine -> coarse), w_ds
  int ntouch = 0;
  const int* tcell = nullptr;  // touched cells
  const int* tptr = nullptr;   // [ntouch + 1]
  const int* tent = nullptr;   // contribution blocks (2 h + side) per touched cell, ascending
  double* contrib = nullptr;   // [n][2][block]
};

__device__ __forceinline__ const double* htab(const HangDev& H, int kind, int h, int s) {
  return H.tab + H.toff[((size_t)kind * H.n + h) * 2 + s];
}

// geometry of subface point t seen from side s (normal out of side s)
template <int DIM>
__device__ __forceinline__ void hgeo(const HangDev& H, int r, int h, int t, int s, double* Js, double* Jo, double* n,
                                     double& wds) {
  constexpr int GS = 2 * DIM * DIM + DIM + 1;
  const double* g = H.geo[r] + ((size_t)h * H.nqf[r] + t) * GS;
#pragma unroll
  for (int i = 0; i < DIM * DIM; ++i) {
    Js[i] = g[(s ? DIM * DIM : 0) + i];
    Jo[i] = g[(s ? 0 : DIM * DIM) + i];
  }
#pragma unroll
  for (int d = 0; d < DIM; ++d) n[d] = s ? -g[2 * DIM * DIM + d] : g[2 * DIM * DIM + d];
  wds = g[2 * DIM * DIM + DIM];
}

template <int DIM>
__device__ __forceinline__ double hdot(const double* a, const double* b) {
  double s = 0.0;
#pragma unroll
  for (int d = 0; d < DIM; ++d) s = fma(a[d], b[d], s);
  return s;
}

// u_s[i] = f[cell_s * stride + off + i] for both sides
__device__ __forceinline__ void hload(double* u, int ust, const double* __restrict__ f, const int* cell, int stride,
                                      int off, int nb) {
  for (int idx = threadIdx.x; idx < 2 * nb; idx += blockDim.x) {
    const int s = idx >= nb, i = idx - s * nb;
    u[s * ust + i] = f[(size_t)cell[s] * stride + off + i];
  }
}
// E_s[k nq + t] = sum_i T_s[(k nq + t) nb + i] u_s[i], k < nk, both sides
__device__ __forceinline__ void heval(const double* T0, const double* T1, int nq, int nb, int nk, const double* u,
                                      int ust, double* E, int est) {
  const int per = nk * nq;
  for (int idx = threadIdx.x; idx < 2 * per; idx += blockDim.x) {
    const int s = idx >= per, r = idx - s * per;
    const double* row = (s ? T1 : T0) + (size_t)r * nb;
    const double* us = u + s * ust;
    double a = 0.0;
    for (int i = 0; i < nb; ++i) a = fma(row[i], us[i], a);
    E[s * est + r] = a;
  }
}
// out_s[i] += sum_{k < nk, t} T_s[(k nq + t) nb + i] I_s[k nq + t], both sides
__device__ __forceinline__ void hinteg(const double* T0, const double* T1, int nq, int nb, int nk, const double* I,
                                       int ist, double* out, int ost) {
  for (int idx = threadIdx.x; idx < 2 * nb; idx += blockDim.x) {
    const int s = idx >= nb, i = idx - s * nb;
    const double* T = s ? T1 : T0;
    const double* in = I + s * ist;
    double a = out[s * ost + i];
    for (int r = 0; r < nk * nq; ++r) a = fma(T[(size_t)r * nb + i], in[r], a);
    out[s * ost + i] = a;
  }
}
__device__ __forceinline__ void hzero(double* p, int n) {
  for (int i = threadIdx.x; i < n; i += blockDim.x) p[i] = 0.0;
}

// shared-memory carve-up common to the kernels
template <int DIM>
struct HSmem {
  double *U, *OUT, *E, *I, *W;
  int ust, ost, est, wst;
  __device__ HSmem(double* sm, const HangDev& H, int oblk) {
    ust = H.nbu > H.nbp ? H.nbu : H.nbp;
    ost = oblk;
    est = (1 + DIM) * H.nqm;
    wst = DIM * H.nqm;
    U = sm;
    OUT = U + 2 * ust;
    E = OUT + 2 * ost;
    I = E + 2 * est;
    W = I + 2 * est;
  }
  static size_t bytes(const HangDev& H, int oblk) {
    const int ust = H.nbu > H.nbp ? H.nbu : H.nbp;
    return sizeof(double) * (size_t)(2 * ust + 2 * oblk + 4 * (1 + DIM) * H.nqm + 2 * DIM * H.nqm);
  }
};

// advecting-field traces W_s[d nq + t] at the subface points of table kind `kind`
template <int DIM>
__device__ void hwtrace(const HangDev& H, HSmem<DIM>& S, int kind, int h, const int* cell, int nbu,
                        const double* __restrict__ w) {
  const int nq = H.nqf[rule_of(kind)];
  for (int d = 0; d < DIM; ++d) {
    hload(S.U, S.ust, w, cell, DIM * nbu, d * nbu, nbu);
    __syncthreads();
    heval(htab(H, kind, h, 0), htab(H, kind, h, 1), nq, nbu, 1, S.U, S.ust, S.W + d * nq, S.wst);
    __syncthreads();
  }
}

template <int DIM>
__device__ void hstore(const HangDev& H, const HSmem<DIM>& S, int h, int blk) {
  for (int idx = threadIdx.x; idx < 2 * blk; idx += blockDim.x) {
    const int s = idx >= blk, r = idx - s * blk;
    H.contrib[(size_t)(2 * h + s) * blk + r] = S.OUT[s * S.ost + r];
  }
}

// ------------------------------------------------------------------ momentum apply
template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_momentum(HangDev H, MomCoef co, const double* __restrict__ w,
                                                        const double* __restrict__ x) {
  extern __shared__ double sm[];
  const int h = blockIdx.x, nb = H.nbu;
  HSmem<DIM> S(sm, H, DIM * nb);
  const int cell[2] = {H.rec[4 * h], H.rec[4 * h + 2]};
  hzero(S.OUT, 2 * S.ost);
  const double C = H.sfu * H.pen[h];
  __syncthreads();
  if (co.visc != 0.0) {  // forms.cpp:443-461
    const int nq = H.nqf[0];
    for (int comp = 0; comp < DIM; ++comp) {
      hload(S.U, S.ust, x, cell, DIM * nb, comp * nb, nb);
      __syncthreads();
      heval(htab(H, 0, h, 0), htab(H, 0, h, 1), nq, nb, 1 + DIM, S.U, S.ust, S.E, S.est);
      __syncthreads();
      for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {
        const int s = idx >= nq, t = idx - s * nq;
        const double* Es = S.E + s * S.est;
        const double* Eo = S.E + (1 - s) * S.est;
        double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, gr[DIM], g[DIM], sv[DIM], r[DIM];
        hgeo<DIM>(H, 0, h, t, s, Js, Jo, n, wds);
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = Es[(1 + a) * nq + t];
        to_phys<DIM>(Js, gr, g);
        const double dn_s = hdot<DIM>(g, n);
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = Eo[(1 + a) * nq + t];
        to_phys<DIM>(Jo, gr, g);
        const double dn_o = hdot<DIM>(g, n);
        const double ju = Es[t] - Eo[t];
        const double fv = co.visc * (-0.5 * (dn_s + dn_o) + C * ju) * wds;
        const double ssym = -co.visc * 0.5 * ju * wds;
#pragma unroll
        for (int d = 0; d < DIM; ++d) sv[d] = ssym * n[d];
        to_ref<DIM>(Js, sv, r);
        double* Is = S.I + s * S.est;
        Is[t] = fv;
#pragma unroll
        for (int a = 0; a < DIM; ++a) Is[(1 + a) * nq + t] = r[a];
      }
      __syncthreads();
      hinteg(htab(H, 0, h, 0), htab(H, 0, h, 1), nq, nb, 1 + DIM, S.I, S.est, S.OUT + comp * nb, S.ost);
      __syncthreads();
    }
  }
  if (co.adv != 0.0) {  // forms.cpp:555-573
    const int nq = H.nqf[1];
    hwtrace<DIM>(H, S, 1, h, cell, nb, w);
    for (int comp = 0; comp < DIM; ++comp) {
      hload(S.U, S.ust, x, cell, DIM * nb, comp * nb, nb);
      __syncthreads();
      heval(htab(H, 1, h, 0), htab(H, 1, h, 1), nq, nb, 1, S.U, S.ust, S.E, S.est);
      __syncthreads();
      for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {
        const int s = idx >= nq, t = idx - s * nq;
        double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, ws[DIM], wo[DIM];
        hgeo<DIM>(H, 1, h, t, s, Js, Jo, n, wds);
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          ws[d] = S.W[s * S.wst + d * nq + t];
          wo[d] = S.W[(1 - s) * S.wst + d * nq + t];
        }
        const double wn_s = hdot<DIM>(ws, n), wn_o = hdot<DIM>(wo, n);
        const double us = S.E[s * S.est + t], uo = S.E[(1 - s) * S.est + t];
        const double lam = fmax(fabs(wn_s), fabs(wn_o));
        S.I[s * S.est + t] = co.adv * (0.5 * (us * wn_s + uo * wn_o) + 0.5 * lam * (us - uo)) * wds;
      }
      __syncthreads();
      hinteg(htab(H, 1, h, 0), htab(H, 1, h, 1), nq, nb, 1, S.I, S.est, S.OUT + comp * nb, S.ost);
      __syncthreads();
    }
  }
  hstore<DIM>(H, S, h, DIM * nb);
}

// ------------------------------------------------------------------ momentum diagonal
template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_momentum_diag(HangDev H, MomCoef co, const double* __restrict__ w) {
  extern __shared__ double sm[];
  const int h = blockIdx.x, nb = H.nbu;
  HSmem<DIM> S(sm, H, nb);
  const int cell[2] = {H.rec[4 * h], H.rec[4 * h + 2]};
  const double C = H.sfu * H.pen[h];
  if (co.adv != 0.0) hwtrace<DIM>(H, S, 1, h, cell, nb, w);
  for (int idx = threadIdx.x; idx < 2 * nb; idx += blockDim.x) {
    const int s = idx >= nb, i = idx - s * nb;
    double sum = 0.0;
    if (co.visc != 0.0) {  // forms.cpp:677-737
      const int nq = H.nqf[0];
      const double* T = htab(H, 0, h, s);
      for (int t = 0; t < nq; ++t) {
        double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, gr[DIM], g[DIM];
        hgeo<DIM>(H, 0, h, t, s, Js, Jo, n, wds);
        const double phi = T[(size_t)t * nb + i];
#pragma unroll
        for (int a = 0; a < DIM; ++a) gr[a] = T[(size_t)((1 + a) * nq + t) * nb + i];
        to_phys<DIM>(Js, gr, g);
        const double dn = hdot<DIM>(g, n);
        sum += co.visc * (-phi * dn + C * phi * phi) * wds;
      }
    }
    if (co.adv != 0.0) {  // forms.cpp:740-809
      const int nq = H.nqf[1];
      const double* T = htab(H, 1, h, s);
      for (int t = 0; t < nq; ++t) {
        double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, ws[DIM], wo[DIM];
        hgeo<DIM>(H, 1, h, t, s, Js, Jo, n, wds);
#pragma unroll
        for (int d = 0; d < DIM; ++d) {
          ws[d] = S.W[s * S.wst + d * nq + t];
          wo[d] = S.W[(1 - s) * S.wst + d * nq + t];
        }
        const double wn_s = hdot<DIM>(ws, n);
        const double lam = fmax(fabs(wn_s), fabs(hdot<DIM>(wo, n)));
        const double phi = T[(size_t)t * nb + i];
        sum += co.adv * (0.5 * wn_s + 0.5 * lam) * phi * phi * wds;
      }
    }
    H.contrib[(size_t)(2 * h + s) * nb + i] = sum;
  }
}

// ------------------------------------------------------------------ scalar SIP apply / diagonal
template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_sip(HangDev H, const double* __restrict__ x) {
  extern __shared__ double sm[];
  const int h = blockIdx.x, nb = H.nbp, nq = H.nqf[2];
  HSmem<DIM> S(sm, H, nb);
  const int cell[2] = {H.rec[4 * h], H.rec[4 * h + 2]};
  const double C = H.sfp * H.pen[h];
  hzero(S.OUT, 2 * S.ost);
  hload(S.U, S.ust, x, cell, nb, 0, nb);
  __syncthreads();
  heval(htab(H, 2, h, 0), htab(H, 2, h, 1), nq, nb, 1 + DIM, S.U, S.ust, S.E, S.est);
  __syncthreads();
  for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {  // forms.cpp:179-242
    const int s = idx >= nq, t = idx - s * nq;
    const double* Es = S.E + s * S.est;
    const double* Eo = S.E + (1 - s) * S.est;
    double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, gr[DIM], g[DIM], sv[DIM], r[DIM];
    hgeo<DIM>(H, 2, h, t, s, Js, Jo, n, wds);
#pragma unroll
    for (int a = 0; a < DIM; ++a) gr[a] = Es[(1 + a) * nq + t];
    to_phys<DIM>(Js, gr, g);
    const double dn_s = hdot<DIM>(g, n);
#pragma unroll
    for (int a = 0; a < DIM; ++a) gr[a] = Eo[(1 + a) * nq + t];
    to_phys<DIM>(Jo, gr, g);
    const double dn_o = hdot<DIM>(g, n);
    const double ju = Es[t] - Eo[t];
    const double ssym = -0.5 * ju * wds;
#pragma unroll
    for (int d = 0; d < DIM; ++d) sv[d] = ssym * n[d];
    to_ref<DIM>(Js, sv, r);
    double* Is = S.I + s * S.est;
    Is[t] = (-0.5 * (dn_s + dn_o) + C * ju) * wds;
#pragma unroll
    for (int a = 0; a < DIM; ++a) Is[(1 + a) * nq + t] = r[a];
  }
  __syncthreads();
  hinteg(htab(H, 2, h, 0), htab(H, 2, h, 1), nq, nb, 1 + DIM, S.I, S.est, S.OUT, S.ost);
  __syncthreads();
  hstore<DIM>(H, S, h, nb);
}

template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_sip_diag(HangDev H) {
  const int h = blockIdx.x, nb = H.nbp, nq = H.nqf[2];
  const double C = H.sfp * H.pen[h];
  for (int idx = threadIdx.x; idx < 2 * nb; idx += blockDim.x) {  // forms.cpp:273-328
    const int s = idx >= nb, i = idx - s * nb;
    const double* T = htab(H, 2, h, s);
    double sum = 0.0;
    for (int t = 0; t < nq; ++t) {
      double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, gr[DIM], g[DIM];
      hgeo<DIM>(H, 2, h, t, s, Js, Jo, n, wds);
      const double phi = T[(size_t)t * nb + i];
#pragma unroll
      for (int a = 0; a < DIM; ++a) gr[a] = T[(size_t)((1 + a) * nq + t) * nb + i];
      to_phys<DIM>(Js, gr, g);
      sum += (-phi * hdot<DIM>(g, n) + C * phi * phi) * wds;
    }
    H.contrib[(size_t)(2 * h + s) * nb + i] = sum;
  }
}

// ------------------------------------------------------------------ divergence functional
template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_divergence(HangDev H, const double* __restrict__ u) {
  extern __shared__ double sm[];
  const int h = blockIdx.x, nbu = H.nbu, nbp = H.nbp, nq = H.nqf[0];
  HSmem<DIM> S(sm, H, nbp);
  const int cell[2] = {H.rec[4 * h], H.rec[4 * h + 2]};
  hzero(S.OUT, 2 * S.ost);
  hwtrace<DIM>(H, S, 0, h, cell, nbu, u);
  for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {  // forms.cpp:1160-1190
    const int s = idx >= nq, t = idx - s * nq;
    double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
    hgeo<DIM>(H, 0, h, t, s, Js, Jo, n, wds);
    double un = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d)
      un += 0.5 * (S.W[s * S.wst + d * nq + t] + S.W[(1 - s) * S.wst + d * nq + t]) * n[d];
    S.I[s * S.est + t] = -un * wds;
  }
  __syncthreads();
  hinteg(htab(H, 3, h, 0), htab(H, 3, h, 1), nq, nbp, 1, S.I, S.est, S.OUT, S.ost);
  __syncthreads();
  hstore<DIM>(H, S, h, nbp);
}

// ------------------------------------------------------------------ stage RHS (explicit interior-face terms)
template <int DIM>
__global__ void __launch_bounds__(kThr) k_hang_rhs(HangDev H, RhsArgs ra) {
  extern __shared__ double sm[];
  const int h = blockIdx.x, nb = H.nbu, nbp = H.nbp;
  HSmem<DIM> S(sm, H, DIM * nb);
  const int cell[2] = {H.rec[4 * h], H.rec[4 * h + 2]};
  hzero(S.OUT, 2 * S.ost);
  __syncthreads();
  for (int comp = 0; comp < DIM; ++comp) {
    if (ra.nv + ra.np > 0) {  // rule k+1: {grad f} n and {p} n (forms.cpp:859-952)
      const int nq = H.nqf[0];
      hzero(S.I, 2 * S.est);
      __syncthreads();
      for (int ti = 0; ti < ra.nv; ++ti) {
        hload(S.U, S.ust, ra.vf[ti], cell, DIM * nb, comp * nb, nb);
        __syncthreads();
        heval(htab(H, 0, h, 0), htab(H, 0, h, 1), nq, nb, 1 + DIM, S.U, S.ust, S.E, S.est);
        __syncthreads();
        for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {
          const int s = idx >= nq, t = idx - s * nq;
          const double* Es = S.E + s * S.est;
          const double* Eo = S.E + (1 - s) * S.est;
          double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, gr[DIM], g[DIM];
          hgeo<DIM>(H, 0, h, t, s, Js, Jo, n, wds);
#pragma unroll
          for (int a = 0; a < DIM; ++a) gr[a] = Es[(1 + a) * nq + t];
          to_phys<DIM>(Js, gr, g);
          const double dn_s = hdot<DIM>(g, n);
#pragma unroll
          for (int a = 0; a < DIM; ++a) gr[a] = Eo[(1 + a) * nq + t];
          to_phys<DIM>(Jo, gr, g);
          S.I[s * S.est + t] += ra.vc[ti] * 0.5 * (dn_s + hdot<DIM>(g, n)) * wds;
        }
        __syncthreads();
      }
      for (int ti = 0; ti < ra.np; ++ti) {
        hload(S.U, S.ust, ra.pf[ti], cell, nbp, 0, nbp);
        __syncthreads();
        heval(htab(H, 3, h, 0), htab(H, 3, h, 1), nq, nbp, 1, S.U, S.ust, S.E, S.est);
        __syncthreads();
        for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {
          const int s = idx >= nq, t = idx - s * nq;
          double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds;
          hgeo<DIM>(H, 0, h, t, s, Js, Jo, n, wds);
          const double pv = 0.5 * (S.E[s * S.est + t] + S.E[(1 - s) * S.est + t]);
          S.I[s * S.est + t] -= ra.pc[ti] * pv * n[comp] * wds;
        }
        __syncthreads();
      }
      hinteg(htab(H, 0, h, 0), htab(H, 0, h, 1), nq, nb, 1, S.I, S.est, S.OUT + comp * nb, S.ost);
      __syncthreads();
    }
    if (ra.na > 0) {  // rule k+2: central advective flux (forms.cpp:1010-1048)
      const int nq = H.nqf[1];
      hzero(S.I, 2 * S.est);
      __syncthreads();
      for (int ti = 0; ti < ra.na; ++ti) {
        hwtrace<DIM>(H, S, 1, h, cell, nb, ra.aw[ti]);
        hload(S.U, S.ust, ra.af[ti], cell, DIM * nb, comp * nb, nb);
        __syncthreads();
        heval(htab(H, 1, h, 0), htab(H, 1, h, 1), nq, nb, 1, S.U, S.ust, S.E, S.est);
        __syncthreads();
        for (int idx = threadIdx.x; idx < 2 * nq; idx += blockDim.x) {
          const int s = idx >= nq, t = idx - s * nq;
          double Js[DIM * DIM], Jo[DIM * DIM], n[DIM], wds, ws[DIM], wo[DIM];
          hgeo<DIM>(H, 1, h, t, s, Js, Jo, n, wds);
#pragma unroll
          for (int d = 0; d < DIM; ++d) {
            ws[d] = S.W[s * S.wst + d * nq + t];
            wo[d] = S.W[(1 - s) * S.wst + d * nq + t];
          }
          const double fs = S.E[s * S.est + t], fo = S.E[(1 - s) * S.est + t];
          S.I[s * S.est + t] -= ra.ac[ti] * 0.5 * (fs * hdot<DIM>(ws, n) + fo * hdot<DIM>(wo, n)) * wds;
        }
        __syncthreads();
      }
      hinteg(htab(H, 1, h, 0), htab(H, 1, h, 1), nq, nb, 1, S.I, S.est, S.OUT + comp * nb, S.ost);
      __syncthreads();
    }
  }
  hstore<DIM>(H, S, h, DIM * nb);
}

// ------------------------------------------------------------------ axis-aligned 3D subfaces (sum-factorised)
// Refined meshes whose cells are all axis-aligned boxes (the line-split fast kernels'
// meshes): the face normal is +-e_a, so only the trace and the reference normal
// derivative of both sides enter, the subface is the whole fine face, and its embedding
// into the coarse face is an offset (0 or 1/2 per tangential axis) + a scaling by 1/2.
// The dense embedded-point tables collapse to 1D tables (fine side: the basis at the
// Gauss points; coarse side: the basis at o + xi / 2) applied along the two tangential
// axes: ~6 k FMA per momentum subface instead of ~100 k, no table streaming.  Both sides'
// integrands differ by a sign only (normal out of the side doing the work), so each
// integrand field is evaluated once and tested through each side's own tables.
// One thread per (subface, component) for the momentum apply, per subface for the
// scalar SIP apply; same per-(subface, side) contribution blocks + k_hang_scatter.
template <int N, int Q>
struct HAxTab {
  double B[3][Q][N];  // basis at the Gauss points xi, at xi / 2, at 1/2 + xi / 2
  double w[Q];
  double dE[2][N];    // basis derivatives at 0, 1
};
struct HAxDev {
  const int4* rec = nullptr;     // fine cell, coarse cell, code = a | s_f << 2 | o_p << 3 | o_q << 4, unused
  const double4* geo = nullptr;  // 1/h_a fine, 1/h_a coarse, |fine face|, mean |F|/|K|
  const double* tab[3] = {};     // HAxTab<Nu, Nu>, HAxTab<Nu, Nu + 1>, HAxTab<Np, Np + 1>
};

template <int N>
__device__ __forceinline__ void hax_strides(int a, int& sl, int& sp, int& sq) {
  sl = a == 0 ? 1 : (a == 1 ? N : N * N);
  sp = a == 0 ? N : 1;
  sq = a == 2 ? N : N * N;
}
template <class T>
__device__ __forceinline__ const T& hax_load_tab(double* sm, const double* __restrict__ g) {
  for (int i = threadIdx.x; i < (int)(sizeof(T) / sizeof(double)); i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  return *reinterpret_cast<const T*>(sm);
}
// face-layer values t[p + N q] and reference normal derivatives g[p + N q] on face (a, s)
template <int N>
__device__ __forceinline__ void hax_face(const double* __restrict__ u, int a, int s, const double* dEs, double* t,
                                         double* g) {
  int sl, sp, sq;
  hax_strides<N>(a, sl, sp, sq);
  const int L = s ? N - 1 : 0;
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int p = 0; p < N; ++p) {
      const double* b = u + p * sp + q * sq;
      double gg = 0.0, tt = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double v = b[l * sl];
        gg = fma(dEs[l], v, gg);
        tt = l == L ? v : tt;
      }
      t[p + N * q] = tt;
      g[p + N * q] = gg;
    }
}
template <int N>
__device__ __forceinline__ void hax_trace(const double* __restrict__ u, int a, int s, double* t) {
  int sl, sp, sq;
  hax_strides<N>(a, sl, sp, sq);
  const double* b = u + (s ? N - 1 : 0) * sl;
#pragma unroll
  for (int q = 0; q < N; ++q)
#pragma unroll
    for (int p = 0; p < N; ++p) t[p + N * q] = b[p * sp + q * sq];
}
// out[tp + Q tq] += sgn sum_{p, q} Bp[tp][p] Bq[tq][q] f[p + N q]
template <int N, int Q>
__device__ __forceinline__ void hax_interp(const double (*Bp)[N], const double (*Bq)[N], const double* f, double sgn,
                                           double* out) {
#pragma unroll
  for (int tq = 0; tq < Q; ++tq) {
    double r[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      double a = 0.0;
#pragma unroll
      for (int q = 0; q < N; ++q) a = fma(Bq[tq][q], f[p + N * q], a);
      r[p] = sgn * a;
    }
#pragma unroll
    for (int tp = 0; tp < Q; ++tp) {
      double a = out[tp + Q * tq];
#pragma unroll
      for (int p = 0; p < N; ++p) a = fma(Bp[tp][p], r[p], a);
      out[tp + Q * tq] = a;
    }
  }
}
// out[p + N q] = sum_{tp, tq} Bp[tp][p] Bq[tq][q] F[tp + Q tq]
template <int N, int Q>
__device__ __forceinline__ void hax_back(const double (*Bp)[N], const double (*Bq)[N], const double* F, double* out) {
#pragma unroll
  for (int i = 0; i < N * N; ++i) out[i] = 0.0;
#pragma unroll
  for (int tq = 0; tq < Q; ++tq) {
    double z[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      double a = 0.0;
#pragma unroll
      for (int tp = 0; tp < Q; ++tp) a = fma(Bp[tp][p], F[tp + Q * tq], a);
      z[p] = a;
    }
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int p = 0; p < N; ++p) out[p + N * q] = fma(Bq[tq][q], z[p], out[p + N * q]);
  }
}
// The SIP face terms of one scalar field across one subface (forms.cpp:179-242 /
// :443-461 with n = +-e_a): writes both sides' contribution blocks
//   fine:   V_f (value test, face layer) + dE G_f (normal-derivative test)
//   coarse: the same through the embedded tables, V_c = -I_c^T F
template <int N, int Q>
__device__ __forceinline__ void hax_sip_field(const HAxTab<N, Q>& T, int code, double4 ge, double C, double scale,
                                              const double* __restrict__ uf, const double* __restrict__ uc,
                                              double* __restrict__ of, double* __restrict__ oc) {
  const int a = code & 3, sf = (code >> 2) & 1, op = (code >> 3) & 1, oq = (code >> 4) & 1;
  const double sg = sf ? 1.0 : -1.0, ihf = ge.x, ihc = ge.y, area = ge.z;
  const double (*B0)[N] = T.B[0];
  const double (*Bp)[N] = T.B[1 + op];
  const double (*Bq)[N] = T.B[1 + oq];
  double F[Q * Q], J[Q * Q];
#pragma unroll
  for (int i = 0; i < Q * Q; ++i) F[i] = J[i] = 0.0;
  {
    double t[N * N], g[N * N];
    hax_face<N>(uf, a, sf, T.dE[sf], t, g);
#pragma unroll
    for (int i = 0; i < N * N; ++i) g[i] = fma(-0.5 * sg * ihf, g[i], C * t[i]);
    hax_interp<N, Q>(B0, B0, g, 1.0, F);
    hax_interp<N, Q>(B0, B0, t, 1.0, J);
    hax_face<N>(uc, a, 1 - sf, T.dE[1 - sf], t, g);
#pragma unroll
    for (int i = 0; i < N * N; ++i) g[i] = fma(-0.5 * sg * ihc, g[i], -C * t[i]);
    hax_interp<N, Q>(Bp, Bq, g, 1.0, F);
    hax_interp<N, Q>(Bp, Bq, t, -1.0, J);
  }
#pragma unroll
  for (int tq = 0; tq < Q; ++tq)
#pragma unroll
    for (int tp = 0; tp < Q; ++tp) {
      const double wds = scale * area * T.w[tp] * T.w[tq];
      F[tp + Q * tq] *= wds;
      J[tp + Q * tq] *= -0.5 * wds;
    }
  int sl, sp, sq;
  hax_strides<N>(a, sl, sp, sq);
  double V[N * N], G[N * N];
#pragma unroll
  for (int side = 0; side < 2; ++side) {
    hax_back<N, Q>(side ? Bp : B0, side ? Bq : B0, F, V);
    hax_back<N, Q>(side ? Bp : B0, side ? Bq : B0, J, G);
    const int s = side ? 1 - sf : sf, L = s ? N - 1 : 0;
    const double vs = side ? -1.0 : 1.0, gs = sg * (side ? ihc : ihf);
    double* o = side ? oc : of;
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int p = 0; p < N; ++p)
#pragma unroll
        for (int l = 0; l < N; ++l)
          o[l * sl + p * sp + q * sq] = fma(T.dE[s][l], gs * G[p + N * q], l == L ? vs * V[p + N * q] : 0.0);
  }
}

constexpr int kAxThr = 64;

template <int NP>
__global__ void __launch_bounds__(kAxThr) k_hax_sip(HangDev H, HAxDev A, const double* __restrict__ x) {
  constexpr int Q = NP + 1, NB = NP * NP * NP;
  using T = HAxTab<NP, Q>;
  __shared__ double stab[sizeof(T) / sizeof(double)];
  const T& tab = hax_load_tab<T>(stab, A.tab[2]);
  const int h = blockIdx.x * kAxThr + threadIdx.x;
  if (h >= H.n) return;
  const int4 rc = A.rec[h];
  const double4 ge = A.geo[h];
  hax_sip_field<NP, Q>(tab, rc.z, ge, H.sfp * ge.w, 1.0, x + (size_t)rc.x * NB, x + (size_t)rc.y * NB,
                       H.contrib + (size_t)(2 * h) * NB, H.contrib + (size_t)(2 * h + 1) * NB);
}

template <int N>
__global__ void __launch_bounds__(kAxThr) k_hax_momentum(HangDev H, HAxDev A, MomCoef co, const double* __restrict__ w,
                                                         const double* __restrict__ x) {
  constexpr int QA = N, QB = N + 1, NB = N * N * N, NF = N * N;
  using TA = HAxTab<N, QA>;
  using TB = HAxTab<N, QB>;
  __shared__ double stab[(sizeof(TA) + sizeof(TB)) / sizeof(double)];
  const TA& ta = hax_load_tab<TA>(stab, A.tab[0]);
  const TB& tb = hax_load_tab<TB>(stab + sizeof(TA) / sizeof(double), A.tab[1]);
  const int idx = blockIdx.x * kAxThr + threadIdx.x;
  if (idx >= 3 * H.n) return;
  const int h = idx / 3, comp = idx - 3 * h;
  const int4 rc = A.rec[h];
  const double4 ge = A.geo[h];
  const int code = rc.z;
  const double* uf = x + (size_t)rc.x * 3 * NB + comp * NB;
  const double* uc = x + (size_t)rc.y * 3 * NB + comp * NB;
  double* of = H.contrib + (size_t)(2 * h) * 3 * NB + comp * NB;
  double* oc = H.contrib + (size_t)(2 * h + 1) * 3 * NB + comp * NB;
  if (co.visc != 0.0) {  // forms.cpp:443-461
    hax_sip_field<N, QA>(ta, code, ge, H.sfu * ge.w, co.visc, uf, uc, of, oc);
  } else {
#pragma unroll
    for (int i = 0; i < NB; ++i) of[i] = oc[i] = 0.0;
  }
  if (co.adv != 0.0) {  // forms.cpp:555-573 (Lax-Friedrichs), rule k+2
    const int a = code & 3, sf = (code >> 2) & 1, op = (code >> 3) & 1, oq = (code >> 4) & 1;
    const double sg = sf ? 1.0 : -1.0, area = ge.z;
    const double (*B0)[N] = tb.B[0];
    const double (*Bp)[N] = tb.B[1 + op];
    const double (*Bq)[N] = tb.B[1 + oq];
    double tf[NF], tc[NF], wf[NF], wc[NF], Vf[NF], Vc[NF];
    hax_trace<N>(uf, a, sf, tf);
    hax_trace<N>(uc, a, 1 - sf, tc);
    hax_trace<N>(w + (size_t)rc.x * 3 * NB + a * NB, a, sf, wf);
    hax_trace<N>(w + (size_t)rc.y * 3 * NB + a * NB, a, 1 - sf, wc);
#pragma unroll
    for (int i = 0; i < NF; ++i) Vf[i] = Vc[i] = 0.0;
#pragma unroll
    for (int tq = 0; tq < QB; ++tq) {
      double ruf[N], rwf[N], ruc[N], rwc[N];
#pragma unroll
      for (int p = 0; p < N; ++p) {
        double s0 = 0.0, s1 = 0.0, s2 = 0.0, s3 = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          s0 = fma(B0[tq][q], tf[p + N * q], s0);
          s1 = fma(B0[tq][q], wf[p + N * q], s1);
          s2 = fma(Bq[tq][q], tc[p + N * q], s2);
          s3 = fma(Bq[tq][q], wc[p + N * q], s3);
        }
        ruf[p] = s0;
        rwf[p] = s1;
        ruc[p] = s2;
        rwc[p] = s3;
      }
      double I[QB];
#pragma unroll
      for (int tp = 0; tp < QB; ++tp) {
        double us = 0.0, ws = 0.0, uo = 0.0, wo = 0.0;
#pragma unroll
        for (int p = 0; p < N; ++p) {
          us = fma(B0[tp][p], ruf[p], us);
          ws = fma(B0[tp][p], rwf[p], ws);
          uo = fma(Bp[tp][p], ruc[p], uo);
          wo = fma(Bp[tp][p], rwc[p], wo);
        }
        const double wn_s = sg * ws, wn_o = sg * wo;
        const double lam = fmax(fabs(wn_s), fabs(wn_o));
        I[tp] = co.adv * (0.5 * (us * wn_s + uo * wn_o) + 0.5 * lam * (us - uo)) * (area * tb.w[tp] * tb.w[tq]);
      }
#pragma unroll
      for (int p = 0; p < N; ++p) {
        double zf = 0.0, zc = 0.0;
#pragma unroll
        for (int tp = 0; tp < QB; ++tp) {
          zf = fma(B0[tp][p], I[tp], zf);
          zc = fma(Bp[tp][p], I[tp], zc);
        }
#pragma unroll
        for (int q = 0; q < N; ++q) {
          Vf[p + N * q] = fma(B0[tq][q], zf, Vf[p + N * q]);
          Vc[p + N * q] = fma(-Bq[tq][q], zc, Vc[p + N * q]);
        }
      }
    }
    int sl, sp, sq;
    hax_strides<N>(a, sl, sp, sq);
    double* bf = of + (sf ? N - 1 : 0) * sl;
    double* bc = oc + (sf ? 0 : N - 1) * sl;
#pragma unroll
    for (int q = 0; q < N; ++q)
#pragma unroll
      for (int p = 0; p < N; ++p) {
        bf[p * sp + q * sq] += Vf[p + N * q];
        bc[p * sp + q * sq] += Vc[p + N * q];
      }
  }
}

// ------------------------------------------------------------------ deterministic scatter
// y[cell][rep][blk] += sum of the cell's contribution blocks, in ascending (subface, side) order
__global__ void __launch_bounds__(kThr) k_hang_scatter(HangDev H, int blk, int rep, double* __restrict__ y) {
  const int j = blockIdx.x, cell = H.tcell[j], e0 = H.tptr[j], e1 = H.tptr[j + 1];
  for (int idx = threadIdx.x; idx < blk * rep; idx += blockDim.x) {
    const int r = idx % blk;
    double s = 0.0;
    for (int e = e0; e < e1; ++e) s += H.contrib[(size_t)H.tent[e] * blk + r];
    y[(size_t)cell * blk * rep + idx] += s;
  }
}

}  // namespace

struct HangState {
  int dim = 0, ku = 0, kp = 0;
  HangDev d;
  bool axis = false;  // every subface joins two axis-aligned boxes: the sum-factorised kernels apply
  HAxDev ax;
  std::vector<void*> allocs;
};

void hang_release(HangState* h) {
  if (!h) return;
  for (void* p : h->allocs) cudaFree(p);
  delete h;
}

namespace {
// basis (N GL nodes per axis, x fastest) and reference gradients at the embedded points
// of the Q-point face rule: T[(1+dim)][nqf][N^dim]  (tabulate_basis, lagrange.cpp:52-90)
void tabulate_embedded(int dim, int N, int Q, const double* emb, std::vector<double>& T) {
  const std::vector<double> nodes = gauss_lobatto(N);
  const Rule1D r = gauss_legendre(Q);
  const int nqf = dim == 2 ? Q : Q * Q;
  const int nb = dim == 2 ? N * N : N * N * N;
  T.assign((size_t)(1 + dim) * nqf * nb, 0.0);
  std::vector<double> val, der;
  for (int t = 0; t < nqf; ++t) {
    double ref[3];
    embed_point(dim, emb, r, t, ref);
    double va[3][8], da[3][8];
    for (int a = 0; a < dim; ++a) {
      lagrange_tables(nodes, {ref[a]}, val, der);
      for (int j = 0; j < N; ++j) {
        va[a][j] = val[j];
        da[a][j] = der[j];
      }
    }
    for (int i = 0; i < nb; ++i) {
      const int ii[3] = {i % N, (i / N) % N, dim == 3 ? i / (N * N) : 0};
      double v = 1.0;
      for (int a = 0; a < dim; ++a) v *= va[a][ii[a]];
      T[(size_t)t * nb + i] = v;
      for (int a = 0; a < dim; ++a) {
        double g = 1.0;
        for (int b = 0; b < dim; ++b) g *= b == a ? da[b][ii[b]] : va[b][ii[b]];
        T[((size_t)(1 + a) * nqf + t) * nb + i] = g;
      }
    }
  }
}
template <class T>
T* upload(HangState* hs, const std::vector<T>& v) {
  void* p = nullptr;
  if (cudaMalloc(&p, std::max<size_t>(1, v.size()) * sizeof(T)) != cudaSuccess) return nullptr;
  hs->allocs.push_back(p);
  if (!v.empty() && cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice) != cudaSuccess)
    return nullptr;
  return static_cast<T*>(p);
}
}  // namespace

namespace {
template <int N, int Q>
void fill_hax_tab(std::vector<double>& out) {
  HAxTab<N, Q> t;
  const std::vector<double> nodes = gauss_lobatto(N);
  const Rule1D r = gauss_legendre(Q);
  std::vector<double> val, der;
  for (int k = 0; k < 3; ++k) {
    std::vector<double> pts(Q);
    for (int q = 0; q < Q; ++q) pts[q] = k == 0 ? r.x[q] : 0.5 * (k - 1) + 0.5 * r.x[q];
    lagrange_tables(nodes, pts, val, der);
    for (int q = 0; q < Q; ++q)
      for (int j = 0; j < N; ++j) t.B[k][q][j] = val[(size_t)q * N + j];
  }
  for (int q = 0; q < Q; ++q) t.w[q] = r.w[q];
  lagrange_tables(nodes, {0.0, 1.0}, val, der);
  for (int e = 0; e < 2; ++e)
    for (int j = 0; j < N; ++j) t.dE[e][j] = der[(size_t)e * N + j];
  const double* p = reinterpret_cast<const double*>(&t);
  out.assign(p, p + sizeof(t) / sizeof(double));
}
void fill_hax_tab(int N, int Q, std::vector<double>& out) {
  if (Q == N) {
    if (N == 2) return fill_hax_tab<2, 2>(out);
    if (N == 3) return fill_hax_tab<3, 3>(out);
    if (N == 4) return fill_hax_tab<4, 4>(out);
    if (N == 5) return fill_hax_tab<5, 5>(out);
  } else {
    if (N == 2) return fill_hax_tab<2, 3>(out);
    if (N == 3) return fill_hax_tab<3, 4>(out);
    if (N == 4) return fill_hax_tab<4, 5>(out);
    if (N == 5) return fill_hax_tab<5, 6>(out);
  }
  out.clear();
}

// Axis-aligned boxes on both sides of every subface, opposite faces of one axis, identity
// orientation, embedding = offset {0, 1/2} + tangents e_p / 2, e_q / 2: the
// sum-factorised subface kernels apply.  Anything else keeps the dense-table kernels.
void hang_setup_axis(HangState* hs, const HostMesh& m, const std::vector<double>& pen) {
  const int n = m.n_hang();
  std::vector<int4> rec(n);
  std::vector<double4> geo(n);
  const double ref[3] = {0.5, 0.5, 0.5};
  auto near = [](double a, double b) { return std::abs(a - b) <= 1e-12; };
  for (int h = 0; h < n; ++h) {
    const int K = m.hrec[4 * h], f = m.hrec[4 * h + 1], Nc = m.hrec[4 * h + 2], fc = m.hrec[4 * h + 3];
    const int a = f / 2, sf = f % 2;
    if (fc != (f ^ 1)) return;
    double Jf[9], Jc[9];
    jacobian(m, K, ref, Jf);
    jacobian(m, Nc, ref, Jc);
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 3; ++j)
        if (i != j && (std::abs(Jf[3 * i + j]) > 1e-13 * std::abs(Jf[4 * i]) ||
                       std::abs(Jc[3 * i + j]) > 1e-13 * std::abs(Jc[4 * i])))
          return;
    if (Jf[4 * a] <= 0.0 || Jc[4 * a] <= 0.0) return;
    const double* e = &m.hemb[(size_t)h * 9];
    const int tp = a == 0 ? 1 : 0, tq = a == 2 ? 1 : 2;
    int o[2];
    for (int k = 0; k < 2; ++k) {
      const int ax = k == 0 ? tp : tq;
      for (int d = 0; d < 3; ++d)
        if (!near(e[3 + 3 * k + d], d == ax ? 0.5 : 0.0)) return;
      if (near(e[ax], 0.0))
        o[k] = 0;
      else if (near(e[ax], 0.5))
        o[k] = 1;
      else
        return;
    }
    if (!near(e[a], (double)(fc % 2))) return;
    rec[h] = make_int4(K, Nc, a | (sf << 2) | (o[0] << 3) | (o[1] << 4), 0);
    geo[h] = make_double4(1.0 / Jf[4 * a], 1.0 / Jc[4 * a], m.face_measure[(size_t)K * 6 + f], pen[h]);
  }
  std::vector<double> t0, t1, t2;
  fill_hax_tab(hs->ku + 1, hs->ku + 1, t0);
  fill_hax_tab(hs->ku + 1, hs->ku + 2, t1);
  fill_hax_tab(hs->kp + 1, hs->kp + 2, t2);
  if (t0.empty() || t1.empty() || t2.empty()) return;
  hs->ax.rec = upload(hs, rec);
  hs->ax.geo = upload(hs, geo);
  hs->ax.tab[0] = upload(hs, t0);
  hs->ax.tab[1] = upload(hs, t1);
  hs->ax.tab[2] = upload(hs, t2);
  hs->axis = hs->ax.rec && hs->ax.geo && hs->ax.tab[0] && hs->ax.tab[1] && hs->ax.tab[2];
}
}  // namespace

HangState* hang_setup(const HostMesh& m, int ku, int kp, std::string& err) {
  const int n = m.n_hang();
  if (n == 0) return nullptr;
  const int dim = m.dim, nf = m.nf_cell();
  auto ipow = [](int b, int e) {
    int r = 1;
    for (int i = 0; i < e; ++i) r *= b;
    return r;
  };
  HangState* hs = new HangState;
  hs->dim = dim;
  HangDev& H = hs->d;
  H.n = n;
  H.nbu = ipow(ku + 1, dim);
  H.nbp = ipow(kp + 1, dim);
  H.sfu = (double)((ku + 1) * (ku + 1));
  H.sfp = (double)((kp + 1) * (kp + 1));
  const int rule[kHR] = {ku + 1, ku + 2, kp + 2};
  const int basisN[kHK] = {ku + 1, ku + 1, kp + 1, kp + 1};
  H.nqm = 0;
  for (int r = 0; r < kHR; ++r) {
    H.nqf[r] = ipow(rule[r], dim - 1);
    H.nqm = std::max(H.nqm, H.nqf[r]);
  }
  // tables, deduplicated by (kind, embedding)
  std::vector<double> tab;
  std::vector<long long> toff((size_t)kHK * n * 2);
  std::map<std::vector<long long>, long long> seen;
  std::vector<double> T;
  for (int k = 0; k < kHK; ++k)
    for (int h = 0; h < n; ++h)
      for (int s = 0; s < 2; ++s) {
        double emb[9];
        if (s == 0)
          canonical_embedding(dim, m.hrec[4 * h + 1], emb);
        else
          std::copy(&m.hemb[(size_t)h * dim * dim], &m.hemb[(size_t)(h + 1) * dim * dim], emb);
        std::vector<long long> key{k};
        for (int i = 0; i < dim * dim; ++i) key.push_back(std::llround(emb[i] * 1e12));
        auto it = seen.find(key);
        if (it == seen.end()) {
          tabulate_embedded(dim, basisN[k], rule[rule_of(k)], emb, T);
          it = seen.emplace(key, (long long)tab.size()).first;
          tab.insert(tab.end(), T.begin(), T.end());
        }
        toff[((size_t)k * n + h) * 2 + s] = it->second;
      }
  // subface geometry per rule (space.cpp:100-150) and penalties (forms.cpp:111-121)
  const int GS = 2 * dim * dim + dim + 1;
  std::vector<double> geo[kHR], pen(n);
  for (int r = 0; r < kHR; ++r) {
    const Rule1D rr = gauss_legendre(rule[r]);
    geo[r].assign((size_t)n * H.nqf[r] * GS, 0.0);
    for (int h = 0; h < n; ++h) {
      const int K = m.hrec[4 * h], f = m.hrec[4 * h + 1], Nc = m.hrec[4 * h + 2];
      double ein[9];
      canonical_embedding(dim, f, ein);
      for (int t = 0; t < H.nqf[r]; ++t) {
        double* o = &geo[r][((size_t)h * H.nqf[r] + t) * GS];
        double ref[3], J[9], J2[9];
        embed_point(dim, ein, rr, t, ref);
        jacobian(m, K, ref, J);
        invert(dim, J, o);
        double nn[3], ds;
        face_frame(dim, f, J, o, nn, ds);
        embed_point(dim, &m.hemb[(size_t)h * dim * dim], rr, t, ref);
        jacobian(m, Nc, ref, J2);
        invert(dim, J2, o + dim * dim);
        for (int d = 0; d < dim; ++d) o[2 * dim * dim + d] = nn[d];
        double w = 1.0;
        int rem = t;
        for (int k = 0; k < dim - 1; ++k) {
          w *= rr.w[rem % rule[r]];
          rem /= rule[r];
        }
        o[2 * dim * dim + dim] = ds * w;
      }
    }
  }
  for (int h = 0; h < n; ++h) {
    const int K = m.hrec[4 * h], f = m.hrec[4 * h + 1], Nc = m.hrec[4 * h + 2];
    const double fm = m.face_measure[(size_t)K * nf + f];
    pen[h] = 0.5 * (fm / m.cell_measure[K] + fm / m.cell_measure[Nc]);
  }
  // scatter lists: contribution blocks (2h + side) per cell, ascending
  std::map<int, std::vector<int>> per;
  for (int h = 0; h < n; ++h)
    for (int s = 0; s < 2; ++s) per[m.hrec[4 * h + 2 * s]].push_back(2 * h + s);
  std::vector<int> tcell, tptr{0}, tent;
  for (auto& kv : per) {
    tcell.push_back(kv.first);
    tent.insert(tent.end(), kv.second.begin(), kv.second.end());
    tptr.push_back((int)tent.size());
  }
  H.ntouch = (int)tcell.size();
  const size_t blk = std::max<size_t>((size_t)dim * H.nbu, (size_t)H.nbp);
  std::vector<double> contrib((size_t)n * 2 * blk, 0.0);
  H.rec = upload(hs, m.hrec);
  H.pen = upload(hs, pen);
  H.tab = upload(hs, tab);
  H.toff = upload(hs, toff);
  for (int r = 0; r < kHR; ++r) H.geo[r] = upload(hs, geo[r]);
  H.tcell = upload(hs, tcell);
  H.tptr = upload(hs, tptr);
  H.tent = upload(hs, tent);
  H.contrib = upload(hs, contrib);
  bool ok = H.rec && H.pen && H.tab && H.toff && H.tcell && H.tptr && H.tent && H.contrib;
  for (int r = 0; r < kHR; ++r) ok = ok && H.geo[r];
  if (!ok) {
    err = "hanging faces: device allocation failed";
    hang_release(hs);
    return nullptr;
  }
  hs->ku = ku;
  hs->kp = kp;
  if (dim == 3 && m.affine && ku >= 1 && ku <= 4 && kp >= 1 && kp <= 3) hang_setup_axis(hs, m, pen);
  return hs;
}

namespace {
// DGB_HANG_AXIS=0 in the environment keeps the dense-table subface kernels (A/B, debugging)
bool hang_axis_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("DGB_HANG_AXIS");
    return !(v && v[0] == '0');
  }();
  return on;
}
template <class K>
cudaError_t hlaunch(cudaStream_t st, const HangState* h, K kern, size_t smem) {
  if (smem > 48 * 1024) {
    const cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}
cudaError_t scatter(cudaStream_t st, const HangState* h, int blk, int rep, double* y) {
  k_hang_scatter<<<h->d.ntouch, kThr, 0, st>>>(h->d, blk, rep, y);
  return cudaGetLastError();
}
}  // namespace

int hang_mode(const HangState* h) { return !h ? 0 : (h->axis && hang_axis_enabled() ? 2 : 1); }

#define HANG_DIM_DISPATCH(KERN, BLK, ...)                                                         \
  do {                                                                                            \
    const HangDev& H = h->d;                                                                      \
    if (h->dim == 2) {                                                                            \
      const size_t smem = HSmem<2>::bytes(H, BLK);                                                \
      cudaError_t e = hlaunch(st, h, KERN<2>, smem);                                              \
      if (e != cudaSuccess) return e;                                                             \
      KERN<2><<<H.n, kThr, smem, st>>>(H, __VA_ARGS__);                                           \
    } else {                                                                                      \
      const size_t smem = HSmem<3>::bytes(H, BLK);                                                \
      cudaError_t e = hlaunch(st, h, KERN<3>, smem);                                              \
      if (e != cudaSuccess) return e;                                                             \
      KERN<3><<<H.n, kThr, smem, st>>>(H, __VA_ARGS__);                                           \
    }                                                                                             \
    const cudaError_t e = cudaGetLastError();                                                     \
    if (e != cudaSuccess) return e;                                                               \
  } while (0)

cudaError_t hang_momentum(cudaStream_t st, const HangState* h, MomCoef co, const double* w, const double* x,
                          double* y) {
  if (!h || (co.visc == 0.0 && co.adv == 0.0)) return cudaSuccess;
  if (h->axis && hang_axis_enabled()) {
    const int grid = (3 * h->d.n + kAxThr - 1) / kAxThr;
    switch (h->ku) {
      case 1: k_hax_momentum<2><<<grid, kAxThr, 0, st>>>(h->d, h->ax, co, w, x); break;
      case 2: k_hax_momentum<3><<<grid, kAxThr, 0, st>>>(h->d, h->ax, co, w, x); break;
      case 3: k_hax_momentum<4><<<grid, kAxThr, 0, st>>>(h->d, h->ax, co, w, x); break;
      default: k_hax_momentum<5><<<grid, kAxThr, 0, st>>>(h->d, h->ax, co, w, x); break;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return scatter(st, h, 3 * h->d.nbu, 1, y);
  }
  HANG_DIM_DISPATCH(k_hang_momentum, h->dim * h->d.nbu, co, w, x);
  return scatter(st, h, h->dim * h->d.nbu, 1, y);
}
cudaError_t hang_momentum_diag(cudaStream_t st, const HangState* h, MomCoef co, const double* w, double* y) {
  if (!h || (co.visc == 0.0 && co.adv == 0.0)) return cudaSuccess;
  HANG_DIM_DISPATCH(k_hang_momentum_diag, h->d.nbu, co, w);
  return scatter(st, h, h->d.nbu, h->dim, y);
}
cudaError_t hang_sip(cudaStream_t st, const HangState* h, const double* x, double* y) {
  if (!h) return cudaSuccess;
  if (h->axis && hang_axis_enabled()) {
    const int grid = (h->d.n + kAxThr - 1) / kAxThr;
    switch (h->kp) {
      case 1: k_hax_sip<2><<<grid, kAxThr, 0, st>>>(h->d, h->ax, x); break;
      case 2: k_hax_sip<3><<<grid, kAxThr, 0, st>>>(h->d, h->ax, x); break;
      default: k_hax_sip<4><<<grid, kAxThr, 0, st>>>(h->d, h->ax, x); break;
    }
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
    return scatter(st, h, h->d.nbp, 1, y);
  }
  HANG_DIM_DISPATCH(k_hang_sip, h->d.nbp, x);
  return scatter(st, h, h->d.nbp, 1, y);
}
cudaError_t hang_sip_diag(cudaStream_t st, const HangState* h, double* y) {
  if (!h) return cudaSuccess;
  const HangDev& H = h->d;
  if (h->dim == 2)
    k_hang_sip_diag<2><<<H.n, kThr, 0, st>>>(H);
  else
    k_hang_sip_diag<3><<<H.n, kThr, 0, st>>>(H);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  return scatter(st, h, H.nbp, 1, y);
}
cudaError_t hang_rhs(cudaStream_t st, const HangState* h, const RhsArgs& ra, double* y) {
  if (!h || ra.nv + ra.np + ra.na == 0) return cudaSuccess;
  HANG_DIM_DISPATCH(k_hang_rhs, h->dim * h->d.nbu, ra);
  return scatter(st, h, h->dim * h->d.nbu, 1, y);
}
cudaError_t hang_divergence(cudaStream_t st, const HangState* h, const double* u, double* y) {
  if (!h) return cudaSuccess;
  HANG_DIM_DISPATCH(k_hang_divergence, h->d.nbp, u);
  return scatter(st, h, h->d.nbp, 1, y);
}

}  // namespace dgb
