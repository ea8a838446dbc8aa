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
  int dim = 0;
  HangDev d;
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
  return hs;
}

namespace {
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
