// Fast path for axis-aligned affine hexahedra (every BASELINE config except
// the deformed cfg4): Jinv = diag(1/h), constant per cell.
//
// On such cells every LINEAR term of the reference operators is integrated
// exactly by its Gauss rule (degree <= 2k integrands with >= k+1 points), so
// the rule can be replaced by the exact 1D matrices
//     M = B^T W B   (mass),   K = D^T W D   (stiffness),
// giving Kronecker-structured cell operators (mass + SIP volume terms) and
// nodal face terms with tangential mass matrices.  Results equal the
// reference's quadrature sums up to rounding.
// The advective (nonlinear) terms keep the reference's k+2 Gauss rule
// (forms.cpp:501) with sum factorisation; the LF face flux is evaluated at
// the face Gauss points (forms.cpp:555-573).
//
// Kernel structure: one CTA owns C cells; each stage is a flat loop of 1D
// "line" work items over all cells / components / faces, separated by
// __syncthreads(); element-centric faces (no atomics).
#pragma once

#include "dg_common.cuh"
#include "dispatch.hpp"

namespace dgb {

template <int N, int Q>
struct FTab {
  double M[N][N];   // exact 1D mass  (B^T W B)
  double K[N][N];   // exact 1D stiffness (D^T W D)
  double B[Q][N];   // basis at Gauss points
  double D[Q][N];   // derivatives at Gauss points
  double dE[2][N];  // derivatives at xi = 0, 1
  double w[Q];      // Gauss weights
};
template <int N, int Q>
__constant__ FTab<N, Q> c_ft;

void host_ftab(int N, int Q, double* M, double* K, double* B, double* D, double* dE, double* w);

template <int N, int Q>
static inline cudaError_t ensure_ftab() {
  static int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return cudaSuccess;
  FTab<N, Q> t;
  host_ftab(N, Q, &t.M[0][0], &t.K[0][0], &t.B[0][0], &t.D[0][0], &t.dE[0][0], t.w);
  const cudaError_t e = cudaMemcpyToSymbol(c_ft<N, Q>, &t, sizeof(t));
  if (e == cudaSuccess) done_dev = dev;
  return e;
}

// affine record (GeoAff layout): Jinv[9], detJ, faces...
constexpr int kAffStride3 = 9 + 1 + 6 * 4;

__device__ __forceinline__ bool fa_outlet(const MeshArgs& m, int nb) {
  const int bid = -1 - nb;
  return bid >= 0 && bid < 64 && m.bctype[bid] == 1;
}

// index of a cell node with coordinate `layer` along axis a and tangential coords (p, q)
// (p along the lower tangential axis, q along the upper)
template <int N>
__device__ __forceinline__ int face_node(int a, int layer, int p, int q) {
  if (a == 0) return layer + N * (p + N * q);
  if (a == 1) return p + N * (layer + N * q);
  return p + N * (q + N * layer);
}
template <int N>
__device__ __forceinline__ int axis_stride(int a) {
  return a == 0 ? 1 : (a == 1 ? N : N * N);
}

// ===========================================================================
// Scalar SIP (pressure Helmholtz / Laplacian), axis-aligned affine, 3D.
// ===========================================================================
template <int KP>
struct SipAxisCfg {
  static constexpr int N = KP + 1, Q = KP + 2, NB = N * N * N, NF = N * N;
  static constexpr int C = KP == 1 ? 64 : (KP == 2 ? 28 : 16);  // cells per CTA
  static constexpr int T = 256;
  // per-cell shared layout (doubles)
  static constexpr int O_U = 0, O_OUT = NB, O_A = 2 * NB, O_B = 3 * NB, O_C = 4 * NB, O_D = 5 * NB;
  static constexpr int O_F = 6 * NB;              // 6 faces x NF : F
  static constexpr int O_G = O_F + 6 * NF;        // GT
  static constexpr int O_F1 = O_G + 6 * NF;       // t1-stage outputs
  static constexpr int O_G1 = O_F1 + 6 * NF;
  static constexpr int O_GEO = O_G1 + 6 * NF;     // h0, h1, h2, detJ
  static constexpr int PER = O_GEO + 4;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int KP>
__global__ void __launch_bounds__(SipAxisCfg<KP>::T) k_sip_axis(MeshArgs m, const double* __restrict__ aff,
                                                                 double mc, int dir_bdry,
                                                                 const double* __restrict__ x,
                                                                 double* __restrict__ y) {
  using G = SipAxisCfg<KP>;
  constexpr int N = G::N, Q = G::Q, NB = G::NB, NF = G::NF, C = G::C, PER = G::PER;
  const FTab<N, Q>& tb = c_ft<N, Q>;
  extern __shared__ double sm[];
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const double sfac = (double)((KP + 1) * (KP + 1));
  const int tid = threadIdx.x;

  // S0: load cell values + geometry
  for (int idx = tid; idx < nc * NB; idx += G::T) {
    const int c = idx / NB, i = idx - c * NB;
    sm[c * PER + G::O_U + i] = x[(size_t)(c0 + c) * NB + i];
  }
  for (int c = tid; c < nc; c += G::T) {
    const double* r = aff + (size_t)(c0 + c) * kAffStride3;
    double* g = sm + c * PER + G::O_GEO;
    g[0] = 1.0 / r[0];
    g[1] = 1.0 / r[4];
    g[2] = 1.0 / r[8];
    g[3] = r[9];
  }
  __syncthreads();
  // S1: x-lines  UX = M u (O_A), KX = K u (O_B)
  for (int idx = tid; idx < nc * NF; idx += G::T) {
    const int c = idx / NF, jk = idx - c * NF;
    const double* u = sm + c * PER + G::O_U + jk * N;
    double v[N];
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = u[l];
    double* ux = sm + c * PER + G::O_A + jk * N;
    double* kx = sm + c * PER + G::O_B + jk * N;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(tb.M[i][l], v[l], s);
        t = fma(tb.K[i][l], v[l], t);
      }
      ux[i] = s;
      kx[i] = t;
    }
  }
  __syncthreads();
  // S2: y-lines  UY = M UX (O_D); T = mc' UY + cx M KX + cy K UX (O_C)
  for (int idx = tid; idx < nc * NF; idx += G::T) {
    const int c = idx / NF, r = idx - c * NF;
    const int i = r % N, k = r / N;
    const double* g = sm + c * PER + G::O_GEO;
    const double detJ = g[3];
    const double cm = mc * detJ, cx = detJ / (g[0] * g[0]), cy = detJ / (g[1] * g[1]);
    const int base = i + N * N * k;
    double a[N], b[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      a[l] = sm[c * PER + G::O_A + base + N * l];
      b[l] = sm[c * PER + G::O_B + base + N * l];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double uy = 0.0, mk = 0.0, ku = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        uy = fma(tb.M[j][l], a[l], uy);
        mk = fma(tb.M[j][l], b[l], mk);
        ku = fma(tb.K[j][l], a[l], ku);
      }
      sm[c * PER + G::O_D + base + N * j] = uy;
      sm[c * PER + G::O_C + base + N * j] = cm * uy + cx * mk + cy * ku;
    }
  }
  __syncthreads();
  // S3: z-lines  OUT = M T + cz K UY
  for (int idx = tid; idx < nc * NF; idx += G::T) {
    const int c = idx / NF, ij = idx - c * NF;
    const double* g = sm + c * PER + G::O_GEO;
    const double cz = g[3] / (g[2] * g[2]);
    double t[N], u[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      t[l] = sm[c * PER + G::O_C + ij + NF * l];
      u[l] = sm[c * PER + G::O_D + ij + NF * l];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0, q = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(tb.M[k][l], t[l], s);
        q = fma(tb.K[k][l], u[l], q);
      }
      sm[c * PER + G::O_OUT + ij + NF * k] = s + cz * q;
    }
  }
  // S4: face-node pointwise (all 6 faces), nodal SIP integrands (forms.cpp:196-213)
  for (int idx = tid; idx < nc * 6 * NF; idx += G::T) {
    const int c = idx / (6 * NF), r = idx - c * 6 * NF;
    const int f = r / NF, t = r - f * NF;
    const int a = f >> 1, s = f & 1, p = t % N, q = t / N;
    const int cell = c0 + c;
    const double* g = sm + c * PER + G::O_GEO;
    const int st = axis_stride<N>(a);
    const int b0 = face_node<N>(a, 0, p, q);
    const double* u = sm + c * PER + G::O_U + b0;
    double gs = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) gs = fma(tb.dE[s][l], u[l * st], gs);
    const double us = u[(s ? N - 1 : 0) * st];
    const double sgn = s ? 1.0 : -1.0;
    const double dns = sgn * gs / g[a];
    const int nb = m.nbr[(size_t)cell * 6 + f];
    double F = 0.0, GT = 0.0;
    if (nb >= 0) {
      const double* un = x + (size_t)nb * NB + b0;
      double go = 0.0, uo = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double v = __ldg(un + l * st);
        go = fma(tb.dE[1 - s][l], v, go);
        if (l == (s ? 0 : N - 1)) uo = v;
      }
      const double ho = 1.0 / __ldg(aff + (size_t)nb * kAffStride3 + 4 * a);
      const double dno = sgn * go / ho;
      const double Cp = sfac * m.pen[(size_t)cell * 6 + f];
      const double ju = us - uo;
      F = -0.5 * (dns + dno) + Cp * ju;
      GT = -0.5 * ju;
    } else if (dir_bdry) {
      const double sK = sfac * m.pen[(size_t)cell * 6 + f];
      F = -dns + 2.0 * sK * us;
      GT = -us;
    }
    sm[c * PER + G::O_F + f * NF + t] = F;
    sm[c * PER + G::O_G + f * NF + t] = GT;
  }
  __syncthreads();
  // S5: tangential mass along p (t1)
  for (int idx = tid; idx < nc * 6 * N; idx += G::T) {
    const int c = idx / (6 * N), r = idx - c * 6 * N;
    const int f = r / N, q = r - f * N;
    double a1[N], a2[N];
#pragma unroll
    for (int p = 0; p < N; ++p) {
      a1[p] = sm[c * PER + G::O_F + f * NF + p + N * q];
      a2[p] = sm[c * PER + G::O_G + f * NF + p + N * q];
    }
#pragma unroll
    for (int p = 0; p < N; ++p) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s1 = fma(tb.M[p][l], a1[l], s1);
        s2 = fma(tb.M[p][l], a2[l], s2);
      }
      sm[c * PER + G::O_F1 + f * NF + p + N * q] = s1;
      sm[c * PER + G::O_G1 + f * NF + p + N * q] = s2;
    }
  }
  __syncthreads();
  // S6: along q (t2), scale by face area (and sgn / h for the gradient test)
  for (int idx = tid; idx < nc * 6 * N; idx += G::T) {
    const int c = idx / (6 * N), r = idx - c * 6 * N;
    const int f = r / N, p = r - f * N;
    const int a = f >> 1;
    const double* g = sm + c * PER + G::O_GEO;
    const double A = g[3] / g[a];
    const double gsc = A * ((f & 1) ? 1.0 : -1.0) / g[a];
    double a1[N], a2[N];
#pragma unroll
    for (int q = 0; q < N; ++q) {
      a1[q] = sm[c * PER + G::O_F1 + f * NF + p + N * q];
      a2[q] = sm[c * PER + G::O_G1 + f * NF + p + N * q];
    }
#pragma unroll
    for (int q = 0; q < N; ++q) {
      double s1 = 0.0, s2 = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s1 = fma(tb.M[q][l], a1[l], s1);
        s2 = fma(tb.M[q][l], a2[l], s2);
      }
      sm[c * PER + G::O_F + f * NF + p + N * q] = A * s1;   // reuse F/G slots
      sm[c * PER + G::O_G + f * NF + p + N * q] = gsc * s2;
    }
  }
  __syncthreads();
  // S7: gather the 6 faces into every node and store
  for (int idx = tid; idx < nc * NB; idx += G::T) {
    const int c = idx / NB, i = idx - c * NB;
    const int ii[3] = {i % N, (i / N) % N, i / (N * N)};
    double acc = sm[c * PER + G::O_OUT + i];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      const int a = f >> 1, s = f & 1;
      const int p = a == 0 ? ii[1] : ii[0];
      const int q = a == 2 ? ii[1] : ii[2];
      const int t = p + N * q;
      const int la = ii[a];
      if (la == (s ? N - 1 : 0)) acc += sm[c * PER + G::O_F + f * NF + t];
      acc = fma(tb.dE[s][la], sm[c * PER + G::O_G + f * NF + t], acc);
    }
    y[(size_t)(c0 + c) * NB + i] = acc;
  }
}

}  // namespace dgb

namespace dgb {

// ===========================================================================
// Momentum operator, axis-aligned affine, 3D, skew = 0:
//   mass M x + visc A_sip x          (Kronecker / nodal-exact, rule k+1 equivalent)
// + adv C_lf(w) x                    (k+2 Gauss rule, sum factorisation)
// ===========================================================================
template <int K>
struct MomAxisCfg {
  static constexpr int N = K + 1, Q = K + 2, NB = N * N * N, NF = N * N, QN = Q * N, QQ = Q * Q;
  static constexpr int C = K == 2 ? 12 : 6;    // cells per CTA
  static constexpr int T = K == 2 ? 256 : 192;  // threads per CTA
  // persistent per-cell regions
  static constexpr int O_X = 0, O_W = 3 * NB, O_OUT = 6 * NB, O_GEO = 9 * NB, O_WORK = 9 * NB + 4;
  // phase A (Kronecker cell terms)
  static constexpr int A_UX = 0, A_KX = 3 * NB, A_T = 6 * NB, A_UY = 9 * NB, A_END = 12 * NB;
  // phase B (advection cell terms)
  static constexpr int B_R1 = 0;                 // XB (6 QNN) then TZ/TY/TX (9 QQN)
  static constexpr int B_R2 = 9 * QQ * N;        // YB (6 QQN) then SA/SB (6 QNN)
  static constexpr int B_END = B_R2 + 6 * QQ * N;
  // face phase (one axis = 2 faces at a time)
  static constexpr int F_F = 0;                  // [3][2][NF]  F   -> FM
  static constexpr int F_G = F_F + 6 * NF;       // [3][2][NF]  GT  -> GM
  static constexpr int F_V = F_G + 6 * NF;       // [8][2][NF]  US(3) UO(3) WS WO (nodal) -> FB [3][2][NF]
  static constexpr int F_M1 = F_V + 16 * NF;     // [6][2][NF]  mass along p
  static constexpr int F_V1 = F_M1 + 12 * NF;    // [8][2][QN]  values along p -> FLX [3][2][QQ] -> FL1 [3][2][QN]
  static constexpr int F_VQ = F_V1 + 16 * QN;    // [8][2][QQ]  values at face Gauss points
  static constexpr int F_END = F_VQ + 16 * QQ;
  static constexpr int WORK = A_END > B_END ? (A_END > F_END ? A_END : F_END) : (B_END > F_END ? B_END : F_END);
  static constexpr int PER = O_WORK + WORK;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int K>
__global__ void __launch_bounds__(MomAxisCfg<K>::T) k_momentum_axis(MeshArgs m, const double* __restrict__ aff,
                                                                    MomCoef co, const double* __restrict__ x,
                                                                    const double* __restrict__ w,
                                                                    double* __restrict__ y) {
  using G = MomAxisCfg<K>;
  constexpr int N = G::N, Q = G::Q, NB = G::NB, NF = G::NF, QN = G::QN, QQ = G::QQ, C = G::C, PER = G::PER;
  constexpr int TT = G::T;
  const FTab<N, Q>& tq = c_ft<N, Q>;      // k+2 rule: B, D, w (advection)
  const FTab<N, N>& ta = c_ft<N, N>;      // exact M, K, dE (rule-independent)
  extern __shared__ double sm[];
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x;
  const double sfac = (double)((K + 1) * (K + 1));
#define CELL(c) (sm + (c) * PER)
#define WK(c) (sm + (c) * PER + G::O_WORK)

  // ------------------------------------------------------------------ S0: load x, w, geometry
  for (int idx = tid; idx < nc * 3 * NB; idx += TT) {
    const int c = idx / (3 * NB), i = idx - c * 3 * NB;
    CELL(c)[G::O_X + i] = x[(size_t)(c0 + c) * 3 * NB + i];
    CELL(c)[G::O_W + i] = w[(size_t)(c0 + c) * 3 * NB + i];
  }
  for (int c = tid; c < nc; c += TT) {
    const double* r = aff + (size_t)(c0 + c) * kAffStride3;
    double* g = CELL(c) + G::O_GEO;
    g[0] = 1.0 / r[0];
    g[1] = 1.0 / r[4];
    g[2] = 1.0 / r[8];
    g[3] = r[9];
  }
  __syncthreads();

  // ------------------------------------------------------------------ pass A cell (Kronecker)
  // S1: x-lines UX = M u, KX = K u
  for (int idx = tid; idx < nc * 3 * NF; idx += TT) {
    const int c = idx / (3 * NF), r = idx - c * 3 * NF;  // r = comp*NF + jk
    const double* u = CELL(c) + G::O_X + r * N;
    double v[N];
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = u[l];
    double* ux = WK(c) + G::A_UX + r * N;
    double* kx = WK(c) + G::A_KX + r * N;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(ta.M[i][l], v[l], s);
        t = fma(ta.K[i][l], v[l], t);
      }
      ux[i] = s;
      kx[i] = t;
    }
  }
  __syncthreads();
  // S2: y-lines UY = M UX ; T = mass' UY + vx M KX + vy K UX
  for (int idx = tid; idx < nc * 3 * NF; idx += TT) {
    const int c = idx / (3 * NF), r = idx - c * 3 * NF;
    const int comp = r / NF, ik = r - comp * NF;
    const int i = ik % N, k = ik / N;
    const double* g = CELL(c) + G::O_GEO;
    const double cm = co.mass * g[3], vx = co.visc * g[3] / (g[0] * g[0]), vy = co.visc * g[3] / (g[1] * g[1]);
    const int base = comp * NB + i + NF * k;
    double a[N], b[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      a[l] = WK(c)[G::A_UX + base + N * l];
      b[l] = WK(c)[G::A_KX + base + N * l];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double uy = 0.0, mk = 0.0, ku = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        uy = fma(ta.M[j][l], a[l], uy);
        mk = fma(ta.M[j][l], b[l], mk);
        ku = fma(ta.K[j][l], a[l], ku);
      }
      WK(c)[G::A_UY + base + N * j] = uy;
      WK(c)[G::A_T + base + N * j] = cm * uy + vx * mk + vy * ku;
    }
  }
  __syncthreads();
  // S3: z-lines OUT = M T + vz K UY
  for (int idx = tid; idx < nc * 3 * NF; idx += TT) {
    const int c = idx / (3 * NF), r = idx - c * 3 * NF;
    const int comp = r / NF, ij = r - comp * NF;
    const double* g = CELL(c) + G::O_GEO;
    const double vz = co.visc * g[3] / (g[2] * g[2]);
    const int base = comp * NB + ij;
    double t[N], u[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      t[l] = WK(c)[G::A_T + base + NF * l];
      u[l] = WK(c)[G::A_UY + base + NF * l];
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = 0.0, q = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(ta.M[k][l], t[l], s);
        q = fma(ta.K[k][l], u[l], q);
      }
      CELL(c)[G::O_OUT + base + NF * k] = s + vz * q;
    }
  }
  __syncthreads();

  // ------------------------------------------------------------------ pass B cell (advection, rule k+2)
  // S4: x-lines for 6 fields (u0..2, w0..2): XB[f][(j,k)][qx]
  for (int idx = tid; idx < nc * 6 * NF; idx += TT) {
    const int c = idx / (6 * NF), r = idx - c * 6 * NF;  // r = f*NF + jk
    const double* in = CELL(c) + (r < 3 * NF ? G::O_X + r * N : G::O_W + (r - 3 * NF) * N);
    double v[N];
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = in[l];
    double* o = WK(c) + G::B_R1 + r * Q;
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) s = fma(tq.B[qx][l], v[l], s);
      o[qx] = s;
    }
  }
  __syncthreads();
  // S5: y-lines: YB[f][k][qy][qx]
  for (int idx = tid; idx < nc * 6 * QN; idx += TT) {
    const int c = idx / (6 * QN), r = idx - c * 6 * QN;
    const int f = r / QN, rk = r - f * QN;
    const int qx = rk % Q, k = rk / Q;
    const double* in = WK(c) + G::B_R1 + f * Q * NF + qx + Q * N * k;  // + Q*l
    double v[N];
#pragma unroll
    for (int l = 0; l < N; ++l) v[l] = in[Q * l];
    double* o = WK(c) + G::B_R2 + f * QQ * N + qx + QQ * k;  // + Q*qy
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      double s = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) s = fma(tq.B[qy][l], v[l], s);
      o[Q * qy] = s;
    }
  }
  __syncthreads();
  // S6: fused z: evaluate the 6 columns, pointwise flux, z-integration of the 3x3 gradient tests
  for (int idx = tid; idx < nc * QQ; idx += TT) {
    const int c = idx / QQ, qxy = idx - c * QQ;
    const double* g = CELL(c) + G::O_GEO;
    const double wxy = g[3] * tq.w[qxy % Q] * tq.w[qxy / Q];
    double col[6][Q];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      double v[N];
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = WK(c)[G::B_R2 + f * QQ * N + qxy + QQ * l];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(tq.B[qz][l], v[l], s);
        col[f][qz] = s;
      }
    }
    const double ih[3] = {-co.adv / g[0], -co.adv / g[1], -co.adv / g[2]};
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      double tz[N], ty[N], tx[N];
#pragma unroll
      for (int l = 0; l < N; ++l) tz[l] = ty[l] = tx[l] = 0.0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        const double uj = col[comp][qz] * wxy * tq.w[qz];
        const double rx = uj * col[3][qz] * ih[0];
        const double ry = uj * col[4][qz] * ih[1];
        const double rz = uj * col[5][qz] * ih[2];
#pragma unroll
        for (int l = 0; l < N; ++l) {
          tz[l] = fma(tq.D[qz][l], rz, tz[l]);
          ty[l] = fma(tq.B[qz][l], ry, ty[l]);
          tx[l] = fma(tq.B[qz][l], rx, tx[l]);
        }
      }
      double* o = WK(c) + G::B_R1 + comp * 3 * QQ * N + qxy;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        o[QQ * l] = tz[l];
        o[QQ * N + QQ * l] = ty[l];
        o[2 * QQ * N + QQ * l] = tx[l];
      }
    }
  }
  __syncthreads();
  // S7: y-lines: SA = B^T TZ + D^T TY, SB = B^T TX   -> [comp][l][j][qx]
  for (int idx = tid; idx < nc * 3 * QN; idx += TT) {
    const int c = idx / (3 * QN), r = idx - c * 3 * QN;
    const int comp = r / QN, rl = r - comp * QN;
    const int qx = rl % Q, l = rl / Q;
    const double* tzp = WK(c) + G::B_R1 + comp * 3 * QQ * N + qx + QQ * l;
    double vz[Q], vy[Q], vx[Q];
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      vz[qy] = tzp[Q * qy];
      vy[qy] = tzp[QQ * N + Q * qy];
      vx[qy] = tzp[2 * QQ * N + Q * qy];
    }
    double* sa = WK(c) + G::B_R2 + comp * 2 * QN * N + qx + QN * l;
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        a = fma(tq.B[qy][j], vz[qy], a);
        a = fma(tq.D[qy][j], vy[qy], a);
        b = fma(tq.B[qy][j], vx[qy], b);
      }
      sa[Q * j] = a;
      sa[QN * N + Q * j] = b;
    }
  }
  __syncthreads();
  // S8: x-lines: OUT += B^T SA + D^T SB
  for (int idx = tid; idx < nc * 3 * NF; idx += TT) {
    const int c = idx / (3 * NF), r = idx - c * 3 * NF;
    const int comp = r / NF, jl = r - comp * NF;
    const double* sa = WK(c) + G::B_R2 + comp * 2 * QN * N + Q * jl;
    double va[Q], vb[Q];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      va[qx] = sa[qx];
      vb[qx] = sa[QN * N + qx];
    }
    double* o = CELL(c) + G::O_OUT + comp * NB + N * jl;
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = o[i];
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        s = fma(tq.B[qx][i], va[qx], s);
        s = fma(tq.D[qx][i], vb[qx], s);
      }
      o[i] = s;
    }
  }
  __syncthreads();

  // ------------------------------------------------------------------ faces, one axis (2 faces) at a time
  for (int a = 0; a < 3; ++a) {
    const int st = axis_stride<N>(a);
    // S9: face-node pointwise: SIP integrands (nodal) + traces for the LF flux
    for (int idx = tid; idx < nc * 2 * NF; idx += TT) {
      const int c = idx / (2 * NF), r = idx - c * 2 * NF;
      const int s = r / NF, t = r - s * NF;  // local face s (side), node t
      const int f = 2 * a + s;
      const int p = t % N, q = t / N;
      const int cell = c0 + c;
      const double* g = CELL(c) + G::O_GEO;
      const int b0 = face_node<N>(a, 0, p, q);
      const int Ls = s ? N - 1 : 0, Lo = s ? 0 : N - 1;
      const double sgn = s ? 1.0 : -1.0;
      const int nb = m.nbr[(size_t)cell * 6 + f];
      double* wk = WK(c);
      const bool interior = nb >= 0;
      const bool outlet = !interior && fa_outlet(m, nb);
      const double ho = interior ? 1.0 / __ldg(aff + (size_t)nb * kAffStride3 + 4 * a) : 1.0;
      const double pen = sfac * m.pen[(size_t)cell * 6 + f];
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) {
        const double* u = CELL(c) + G::O_X + comp * NB + b0;
        double gs = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) gs = fma(ta.dE[s][l], u[l * st], gs);
        const double us = u[Ls * st];
        const double dns = sgn * gs / g[a];
        double F = 0.0, GT = 0.0, uo = 0.0;
        if (interior) {
          const double* un = x + (size_t)nb * 3 * NB + comp * NB + b0;
          double go = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) {
            const double v = __ldg(un + l * st);
            go = fma(ta.dE[1 - s][l], v, go);
            if (l == Lo) uo = v;
          }
          const double dno = sgn * go / ho;
          const double ju = us - uo;
          F = co.visc * (-0.5 * (dns + dno) + pen * ju);
          GT = -co.visc * 0.5 * ju;
        } else if (!outlet) {
          F = co.visc * (-dns + 2.0 * pen * us);
          GT = -co.visc * us;
        }
        wk[G::F_F + (comp * 2 + s) * NF + t] = F;
        wk[G::F_G + (comp * 2 + s) * NF + t] = GT;
        wk[G::F_V + (comp * 2 + s) * NF + t] = us;
        wk[G::F_V + ((3 + comp) * 2 + s) * NF + t] = uo;
      }
      wk[G::F_V + (6 * 2 + s) * NF + t] = CELL(c)[G::O_W + a * NB + b0 + Ls * st];
      wk[G::F_V + (7 * 2 + s) * NF + t] = interior ? __ldg(w + (size_t)nb * 3 * NB + a * NB + b0 + Lo * st) : 0.0;
    }
    __syncthreads();
    // S10: along p: mass for the 6 SIP fields, B for the 8 value fields
    for (int idx = tid; idx < nc * 2 * N * 14; idx += TT) {
      const int c = idx / (2 * N * 14), r = idx - c * 2 * N * 14;
      const int fld = r / (2 * N), r2 = r - fld * 2 * N;
      const int s = r2 / N, q = r2 - s * N;
      double* wk = WK(c);
      double v[N];
      if (fld < 6) {  // F0..2, GT0..2
        const double* in = wk + (fld < 3 ? G::F_F + (fld * 2 + s) * NF : G::F_G + ((fld - 3) * 2 + s) * NF) + N * q;
#pragma unroll
        for (int l = 0; l < N; ++l) v[l] = in[l];
        double* o = wk + G::F_M1 + (fld * 2 + s) * NF + N * q;
#pragma unroll
        for (int pp = 0; pp < N; ++pp) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(ta.M[pp][l], v[l], acc);
          o[pp] = acc;
        }
      } else {
        const int vf = fld - 6;
        const double* in = wk + G::F_V + (vf * 2 + s) * NF + N * q;
#pragma unroll
        for (int l = 0; l < N; ++l) v[l] = in[l];
        double* o = wk + G::F_V1 + (vf * 2 + s) * QN + Q * q;
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(tq.B[qp][l], v[l], acc);
          o[qp] = acc;
        }
      }
    }
    __syncthreads();
    // S11: along q: mass (scaled by the face area, and sgn/h for the gradient test) / B for values
    for (int idx = tid; idx < nc * 2 * (6 * N + 8 * Q); idx += TT) {
      const int c = idx / (2 * (6 * N + 8 * Q)), r = idx - c * 2 * (6 * N + 8 * Q);
      double* wk = WK(c);
      const double* g = CELL(c) + G::O_GEO;
      if (r < 2 * 6 * N) {
        const int fld = r / (2 * N), r2 = r - fld * 2 * N;
        const int s = r2 / N, pp = r2 - s * N;
        const double A = g[3] / g[a];
        const double scale = fld < 3 ? A : A * (s ? 1.0 : -1.0) / g[a];
        double v[N];
#pragma unroll
        for (int l = 0; l < N; ++l) v[l] = wk[G::F_M1 + (fld * 2 + s) * NF + pp + N * l];
        double* o = wk + (fld < 3 ? G::F_F + (fld * 2 + s) * NF : G::F_G + ((fld - 3) * 2 + s) * NF) + pp;
#pragma unroll
        for (int qq = 0; qq < N; ++qq) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(ta.M[qq][l], v[l], acc);
          o[N * qq] = scale * acc;
        }
      } else {
        const int r3 = r - 2 * 6 * N;
        const int vf = r3 / (2 * Q), r4 = r3 - vf * 2 * Q;
        const int s = r4 / Q, qp = r4 - s * Q;
        double v[N];
#pragma unroll
        for (int l = 0; l < N; ++l) v[l] = wk[G::F_V1 + (vf * 2 + s) * QN + qp + Q * l];
        double* o = wk + G::F_VQ + (vf * 2 + s) * QQ + qp;
#pragma unroll
        for (int qq = 0; qq < Q; ++qq) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(tq.B[qq][l], v[l], acc);
          o[Q * qq] = acc;
        }
      }
    }
    __syncthreads();
    // S12: LF flux at the face Gauss points (forms.cpp:555-573, boundary :592-599)
    for (int idx = tid; idx < nc * 2 * QQ; idx += TT) {
      const int c = idx / (2 * QQ), r = idx - c * 2 * QQ;
      const int s = r / QQ, gp = r - s * QQ;
      const int f = 2 * a + s;
      const int nb = m.nbr[(size_t)(c0 + c) * 6 + f];
      double* wk = WK(c);
      const double* g = CELL(c) + G::O_GEO;
      const double sgn = s ? 1.0 : -1.0;
      const double wq = co.adv * (g[3] / g[a]) * tq.w[gp % Q] * tq.w[gp / Q];
      const double wns = sgn * wk[G::F_VQ + (6 * 2 + s) * QQ + gp];
      double fl[3];
      if (nb >= 0) {
        const double wno = sgn * wk[G::F_VQ + (7 * 2 + s) * QQ + gp];
        const double lam = fmax(fabs(wns), fabs(wno));
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) {
          const double us = wk[G::F_VQ + (comp * 2 + s) * QQ + gp];
          const double uo = wk[G::F_VQ + ((3 + comp) * 2 + s) * QQ + gp];
          fl[comp] = wq * (0.5 * (us * wns + uo * wno) + 0.5 * lam * (us - uo));
        }
      } else {
        const double cf = fa_outlet(m, nb) ? wns : fabs(wns);
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) fl[comp] = wq * cf * wk[G::F_VQ + (comp * 2 + s) * QQ + gp];
      }
#pragma unroll
      for (int comp = 0; comp < 3; ++comp) wk[G::F_V1 + (comp * 2 + s) * QQ + gp] = fl[comp];  // FLX
    }
    __syncthreads();
    // S13: integrate along q (Q -> N): FL1 [3][2][Q x N] (into F_VQ region)
    for (int idx = tid; idx < nc * 6 * Q; idx += TT) {
      const int c = idx / (6 * Q), r = idx - c * 6 * Q;
      const int cs = r / Q, qp = r - cs * Q;  // cs = comp*2+s
      double* wk = WK(c);
      double v[Q];
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) v[qq] = wk[G::F_V1 + cs * QQ + qp + Q * qq];
      double* o = wk + G::F_VQ + cs * QN + qp;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double acc = 0.0;
#pragma unroll
        for (int qq = 0; qq < Q; ++qq) acc = fma(tq.B[qq][l], v[qq], acc);
        o[Q * l] = acc;
      }
    }
    __syncthreads();
    // S14: along p (Q -> N), add into FM (the value-test nodal integrand)
    for (int idx = tid; idx < nc * 6 * N; idx += TT) {
      const int c = idx / (6 * N), r = idx - c * 6 * N;
      const int cs = r / N, q = r - cs * N;
      double* wk = WK(c);
      double v[Q];
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) v[qp] = wk[G::F_VQ + cs * QN + qp + Q * q];
      double* o = wk + G::F_F + cs * NF + N * q;
#pragma unroll
      for (int pp = 0; pp < N; ++pp) {
        double acc = o[pp];
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) acc = fma(tq.B[qp][pp], v[qp], acc);
        o[pp] = acc;
      }
    }
    __syncthreads();
    // S15: gather both faces of this axis into every node
    for (int idx = tid; idx < nc * 3 * NB; idx += TT) {
      const int c = idx / (3 * NB), r = idx - c * 3 * NB;
      const int comp = r / NB, i = r - comp * NB;
      const int ii[3] = {i % N, (i / N) % N, i / NF};
      const int p = a == 0 ? ii[1] : ii[0];
      const int q = a == 2 ? ii[1] : ii[2];
      const int t = p + N * q;
      const int la = ii[a];
      const double* wk = WK(c);
      double acc = CELL(c)[G::O_OUT + r];
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        if (la == (s ? N - 1 : 0)) acc += wk[G::F_F + (comp * 2 + s) * NF + t];
        acc = fma(ta.dE[s][la], wk[G::F_G + (comp * 2 + s) * NF + t], acc);
      }
      if (a < 2)
        CELL(c)[G::O_OUT + r] = acc;
      else
        y[(size_t)(c0 + c) * 3 * NB + r] = acc;
    }
    __syncthreads();
  }
#undef CELL
#undef WK
}

}  // namespace dgb
