// Device building blocks shared by every DG kernel (sm_100a, fp64).
//
//  * 1D shape tables live in __constant__ memory per (N basis nodes, Q points),
//    so with fully unrolled compile-time indices every table read becomes a
//    constant-bank operand of the DFMA (no shared-memory traffic).
//  * Sum-factorised tensor contractions (`contract`) over cell tiles staged in
//    shared memory: one thread per 1D line, the line held in registers.
//    This replaces the reference's dense-table kern::contract_rows /
//    kern::project_rows (proj/src/kernels.cpp:41-57) used through Eval /
//    TestAcc (forms.cpp:16-109).
//  * Geometry policies: GeoAff (one record per affine cell, north-star item 3)
//    and GeoQp (per quadrature point, deformed cells).
#pragma once

#include <cuda_runtime.h>
#include <cstdint>

#include "dispatch.hpp"

namespace dgb {

// ---------------------------------------------------------------------------
// Constant tables
// ---------------------------------------------------------------------------
template <int N, int Q>
struct Tab {
  double B[Q][N];   // phi_j(x_q): GL-node Lagrange basis at Gauss points
  double D[Q][N];   // phi_j'(x_q)
  double dE[2][N];  // phi_j'(0), phi_j'(1): endpoint derivatives (face normal derivative)
};
template <int Q>
struct WTab {
  double w[Q];  // Gauss weights on [0,1]
};

template <int N, int Q>
__constant__ Tab<N, Q> c_tab;
template <int Q>
__constant__ WTab<Q> c_w;

// Host: fill + upload (once per process / device / translation unit).
void host_tab(int N, int Q, double* B, double* D, double* dE);
void host_w(int Q, double* w);

template <int N, int Q>
static inline cudaError_t ensure_tab() {  // static: one uploader per TU (each TU owns its __constant__ copy)
  static int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return cudaSuccess;
  Tab<N, Q> t;
  host_tab(N, Q, &t.B[0][0], &t.D[0][0], &t.dE[0][0]);
  WTab<Q> w;
  host_w(Q, w.w);
  cudaError_t e = cudaMemcpyToSymbol(c_tab<N, Q>, &t, sizeof(t));
  if (e == cudaSuccess) e = cudaMemcpyToSymbol(c_w<Q>, &w, sizeof(w));
  if (e == cudaSuccess) done_dev = dev;
  return e;
}

// ---------------------------------------------------------------------------
// Matrix accessors (compile-time indices -> constant-bank operands)
// ---------------------------------------------------------------------------
template <int N, int Q> struct MB  { __device__ __forceinline__ double operator()(int o, int i) const { return c_tab<N, Q>.B[o][i]; } };
template <int N, int Q> struct MD  { __device__ __forceinline__ double operator()(int o, int i) const { return c_tab<N, Q>.D[o][i]; } };
template <int N, int Q> struct MBt { __device__ __forceinline__ double operator()(int o, int i) const { return c_tab<N, Q>.B[i][o]; } };
template <int N, int Q> struct MDt { __device__ __forceinline__ double operator()(int o, int i) const { return c_tab<N, Q>.D[i][o]; } };
// 1 x N: normal derivative at side S; N x 1: its transpose
template <int N, int Q, int S> struct MEd  { __device__ __forceinline__ double operator()(int, int i) const { return c_tab<N, Q>.dE[S][i]; } };
template <int N, int Q, int S> struct MEdt { __device__ __forceinline__ double operator()(int o, int) const { return c_tab<N, Q>.dE[S][o]; } };
// 1 x N: pick the face layer of side S (GL nodes: phi_j(0)=delta_j0, phi_j(1)=delta_j,N-1)
template <int N, int S> struct MSel  { __device__ __forceinline__ double operator()(int, int i) const { return i == (S ? N - 1 : 0) ? 1.0 : 0.0; } };
template <int N, int S> struct MSelt { __device__ __forceinline__ double operator()(int o, int) const { return o == (S ? N - 1 : 0) ? 1.0 : 0.0; } };

// ---------------------------------------------------------------------------
// Contractions over per-cell tensors in shared memory, layout [z][y][x].
// out(.., o, ..) (+)= sum_i M(o, i) in(.., i, ..) along axis AX, for nc cells.
// ---------------------------------------------------------------------------
template <int AX, int X, int Y, int Z>
struct Ext {
  static constexpr int NI = AX == 0 ? X : (AX == 1 ? Y : Z);
  static constexpr int SIZE = X * Y * Z;
  static constexpr int NL = SIZE / NI;
};

template <int AX, int X, int Y, int Z, int NO>
__device__ __forceinline__ void line_offsets(int r, int& ib, int& ob) {
  constexpr int OX = AX == 0 ? NO : X, OY = AX == 1 ? NO : Y;
  if (AX == 0) {
    const int y = r % Y, z = r / Y;
    ib = y * X + z * X * Y;
    ob = y * OX + z * OX * OY;
  } else if (AX == 1) {
    const int x = r % X, z = r / X;
    ib = x + z * X * Y;
    ob = x + z * OX * OY;
  } else {
    const int x = r % X, y = r / X;
    ib = x + y * X;
    ob = x + y * OX;
  }
}

template <int AX, int X, int Y, int Z, int NO, bool ACC, class M>
__device__ __forceinline__ void contract(const double* __restrict__ in, int cs_in, double* __restrict__ out,
                                         int cs_out, int nc) {
  using E = Ext<AX, X, Y, Z>;
  constexpr int NI = E::NI, NL = E::NL;
  constexpr int OX = AX == 0 ? NO : X, OY = AX == 1 ? NO : Y;
  constexpr int IST = AX == 0 ? 1 : (AX == 1 ? X : X * Y);
  constexpr int OST = AX == 0 ? 1 : (AX == 1 ? OX : OX * OY);
  const M m;
  for (int idx = threadIdx.x; idx < nc * NL; idx += blockDim.x) {
    const int c = idx / NL, r = idx - c * NL;
    int ib, ob;
    line_offsets<AX, X, Y, Z, NO>(r, ib, ob);
    const double* ip = in + c * cs_in + ib;
    double* op = out + c * cs_out + ob;
    double v[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) v[i] = ip[i * IST];
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      double s = ACC ? op[o * OST] : 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) s = fma(m(o, i), v[i], s);
      op[o * OST] = s;
    }
  }
}

// out (+)= M1 in1 + M2 in2 along AX (same shapes)
template <int AX, int X, int Y, int Z, int NO, bool ACC, class M1, class M2>
__device__ __forceinline__ void contract2(const double* __restrict__ in1, const double* __restrict__ in2,
                                          int cs_in, double* __restrict__ out, int cs_out, int nc) {
  using E = Ext<AX, X, Y, Z>;
  constexpr int NI = E::NI, NL = E::NL;
  constexpr int OX = AX == 0 ? NO : X, OY = AX == 1 ? NO : Y;
  constexpr int IST = AX == 0 ? 1 : (AX == 1 ? X : X * Y);
  constexpr int OST = AX == 0 ? 1 : (AX == 1 ? OX : OX * OY);
  const M1 m1;
  const M2 m2;
  for (int idx = threadIdx.x; idx < nc * NL; idx += blockDim.x) {
    const int c = idx / NL, r = idx - c * NL;
    int ib, ob;
    line_offsets<AX, X, Y, Z, NO>(r, ib, ob);
    const double* ip1 = in1 + c * cs_in + ib;
    const double* ip2 = in2 + c * cs_in + ib;
    double* op = out + c * cs_out + ob;
    double v1[NI], v2[NI];
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      v1[i] = ip1[i * IST];
      v2[i] = ip2[i * IST];
    }
#pragma unroll
    for (int o = 0; o < NO; ++o) {
      double s = ACC ? op[o * OST] : 0.0;
#pragma unroll
      for (int i = 0; i < NI; ++i) s = fma(m1(o, i), v1[i], s);
#pragma unroll
      for (int i = 0; i < NI; ++i) s = fma(m2(o, i), v2[i], s);
      op[o * OST] = s;
    }
  }
}

// ---------------------------------------------------------------------------
// Geometry policies
// ---------------------------------------------------------------------------
template <int DIM, int Q>
struct GeoAff {
  static constexpr int STRIDE = DIM * DIM + 1 + 2 * DIM * (DIM + 1);
  const double* g;
  __device__ GeoAff(const GeoArgs& a) : g(a.aff) {}
  __device__ __forceinline__ void cell(int c, int q, double* Ji, double& jxw) const {
    const double* r = g + (size_t)c * STRIDE;
#pragma unroll
    for (int i = 0; i < DIM * DIM; ++i) Ji[i] = r[i];
    double w = c_w<Q>.w[q % Q] * c_w<Q>.w[(q / Q) % Q];
    if (DIM == 3) w *= c_w<Q>.w[q / (Q * Q)];
    jxw = r[DIM * DIM] * w;
  }
  // face qp t of local face f of cell c, neighbour nb (>=0 interior)
  __device__ __forceinline__ void face(int c, int f, int nb, int t, double* Ji, double* Jo, double* n,
                                       double& wds) const {
    const double* r = g + (size_t)c * STRIDE;
#pragma unroll
    for (int i = 0; i < DIM * DIM; ++i) Ji[i] = r[i];
    if (nb >= 0) {
      const double* ro = g + (size_t)nb * STRIDE;
#pragma unroll
      for (int i = 0; i < DIM * DIM; ++i) Jo[i] = ro[i];
    }
    const double* rf = r + DIM * DIM + 1 + f * (DIM + 1);
#pragma unroll
    for (int d = 0; d < DIM; ++d) n[d] = rf[d];
    double w = c_w<Q>.w[t % Q];
    if (DIM == 3) w *= c_w<Q>.w[t / Q];
    wds = rf[DIM] * w;
  }
};

template <int DIM, int Q>
struct GeoQp {
  static constexpr int NQ = DIM == 3 ? Q * Q * Q : Q * Q;
  static constexpr int NQF = DIM == 3 ? Q * Q : Q;
  static constexpr int CS = DIM * DIM + 1;
  static constexpr int FS = 2 * DIM * DIM + DIM + 1;
  const double* gc;
  const double* gf;
  __device__ GeoQp(const GeoArgs& a) : gc(a.qcell), gf(a.qface) {}
  __device__ __forceinline__ void cell(int c, int q, double* Ji, double& jxw) const {
    const double* r = gc + ((size_t)c * NQ + q) * CS;
#pragma unroll
    for (int i = 0; i < DIM * DIM; ++i) Ji[i] = r[i];
    jxw = r[DIM * DIM];
  }
  __device__ __forceinline__ void face(int c, int f, int nb, int t, double* Ji, double* Jo, double* n,
                                       double& wds) const {
    const double* r = gf + (((size_t)c * 2 * DIM + f) * NQF + t) * FS;
#pragma unroll
    for (int i = 0; i < DIM * DIM; ++i) Ji[i] = r[i];
    if (nb >= 0) {
#pragma unroll
      for (int i = 0; i < DIM * DIM; ++i) Jo[i] = r[DIM * DIM + i];
    }
#pragma unroll
    for (int d = 0; d < DIM; ++d) n[d] = r[2 * DIM * DIM + d];
    wds = r[2 * DIM * DIM + DIM];
  }
};

// physical gradient g_d = sum_a Jinv[a][d] gref_a  (forms.cpp:49-59)
template <int DIM>
__device__ __forceinline__ void to_phys(const double* Ji, const double* gr, double* g) {
#pragma unroll
  for (int d = 0; d < DIM; ++d) {
    double s = 0.0;
#pragma unroll
    for (int a = 0; a < DIM; ++a) s = fma(Ji[a * DIM + d], gr[a], s);
    g[d] = s;
  }
}
// reference-test integrand r_a = sum_d Jinv[a][d] s_d  (forms.cpp:97-103)
template <int DIM>
__device__ __forceinline__ void to_ref(const double* Ji, const double* s, double* r) {
#pragma unroll
  for (int a = 0; a < DIM; ++a) {
    double t = 0.0;
#pragma unroll
    for (int d = 0; d < DIM; ++d) t = fma(Ji[a * DIM + d], s[d], t);
    r[a] = t;
  }
}

}  // namespace dgb
