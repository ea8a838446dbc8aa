// Fast path for axis-aligned affine hexahedra (every BASELINE config except
// the deformed cfg4): Jinv = diag(1/h), constant per cell.
//
// Exactness.  On such cells every LINEAR term of the reference operators is
// integrated exactly by its Gauss rule (polynomial integrands of degree <= 2k
// per direction with >= k+1 points), so the rule can be replaced by the exact
// 1D matrices  M = B^T W B,  K = D^T W D  and the SIP operator (cell stiffness
// + interior-penalty / consistency / symmetry face terms, forms.cpp:148-243,
// :397-495) splits EXACTLY into 1D line operators along each direction:
//
//     A_sip u = sum_d (S_d (x) M (x) M) u,   S_d = 1D SIP operator along d
//                                            (stiffness + the two d-faces, which
//                                            read the neighbours' d-lines)
//     M u     = (M (x) M (x) M) u
//
// (tangential face integrals are the tangential mass matrices).  Results
// equal the reference's quadrature sums up to rounding.  The
// advective (nonlinear) terms keep the reference's k+2 Gauss rule
// (forms.cpp:501) with sum factorisation; the Lax-Friedrichs face flux is
// evaluated at the face Gauss points (forms.cpp:555-573).
//
// Kernel structure: one CTA owns C cells; every stage is a flat loop over 1D
// "line" work items (all cells / components / directions at once) separated
// by __syncthreads().  Element-centric faces: each cell integrates all of its
// faces, reading neighbour lines from global memory (L2), so every output DoF
// is written exactly once — no atomics, deterministic.  Shared-memory tensors
// use an odd x-pitch so line accesses are bank-conflict free.
#pragma once

#include <type_traits>

#include "blas.cuh"
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

// padded cell tensor: x-pitch odd
template <int N, int PXV = (N | 1)>
struct Pad {
  static constexpr int PX = PXV;
  static constexpr int PY = PX * N;
  static constexpr int CT = PY * N;
  __device__ __forceinline__ static int idx(int i, int j, int k) { return i + PX * j + PY * k; }
};

// per-cell face / geometry record kept in shared memory
struct CellInfo {
  double ih[3];    // 1/h_d  (Jinv diagonal)
  double detJ;
  double A[3];     // face areas detJ / h_d
  double pen[6];   // (deg+1)^2 * penalty ratio (interior mean / boundary own)
  double ihn[6];   // neighbour's 1/h_d across each face
  int nb[6];       // neighbour cell, or -1 - boundary id
  int type[6];     // 0 interior, 1 dirichlet, 2 outlet, 3 hanging slot (zero weight: the (cell, face)
                   // slot of a 1-irregular refined mesh, nbr = the cell itself; hang.cu adds its subfaces)
  // branch-free SIP face terms (see face_coefs):  F = cgs gs + cgo go + cus us + cuo uo,
  // GT = gus us + guo uo  (gs / go: own / neighbour reference normal derivative)
  double fc[6][6];
};
constexpr int kInfoDoubles = (sizeof(CellInfo) + 7) / 8;

__device__ __forceinline__ void load_info(CellInfo& ci, const MeshArgs& m, const double* __restrict__ aff, int cell,
                                          double sfac) {
  const double* r = aff + (size_t)cell * kAffStride3;
  ci.ih[0] = r[0];
  ci.ih[1] = r[4];
  ci.ih[2] = r[8];
  ci.detJ = r[9];
#pragma unroll
  for (int d = 0; d < 3; ++d) ci.A[d] = ci.detJ * ci.ih[d];
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int nb = m.nbr[(size_t)cell * 6 + f];
    ci.nb[f] = nb;
    ci.pen[f] = sfac * m.pen[(size_t)cell * 6 + f];
    if (nb >= 0) {
      ci.type[f] = nb == cell ? 3 : 0;
      ci.ihn[f] = __ldg(aff + (size_t)nb * kAffStride3 + 4 * (f >> 1));
    } else {
      const int bid = -1 - nb;
      ci.type[f] = (bid >= 0 && bid < 64 && m.bctype[bid] == 1) ? 2 : 1;
      ci.ihn[f] = 0.0;
    }
  }
}

__device__ __forceinline__ unsigned udiv_n(const UniformGrid& g, unsigned x) {
  if (g.shift == 0) return x;  // n == 1
  const unsigned t = __umulhi(x, g.magic);
  return (t + ((x - t) >> 1)) >> (g.shift - 1);
}
__device__ __forceinline__ int uniform_nbr(const UniformGrid& g, int cell, int f) {
  const int n = g.n, d = f >> 1, s = f & 1;
  const unsigned q1 = udiv_n(g, (unsigned)cell);
  const int co = d == 0 ? cell - n * (int)q1 : (d == 1 ? (int)q1 - n * (int)udiv_n(g, q1) : (int)udiv_n(g, q1));
  const int stride = d == 0 ? 1 : (d == 1 ? n : n * n);
  if (s == 0) return co == 0 ? -1 - f : cell - stride;
  return co == n - 1 ? -1 - f : cell + stride;
}
template <bool UNI>
__device__ __forceinline__ int cell_nbr(const MeshArgs& m, const UniformGrid& g, int cell, int f) {
  if (UNI) return uniform_nbr(g, cell, f);
  return m.nbr[(size_t)cell * 6 + f];
}
// All six neighbours of one cell at once (the uniform-grid coordinates take two
// divisions instead of two per face).
template <bool UNI>
__device__ __forceinline__ void cell_nbrs6(const MeshArgs& m, const UniformGrid& g, int cell, int nb[6]) {
  if (!UNI) {
#pragma unroll
    for (int f = 0; f < 6; ++f) nb[f] = m.nbr[(size_t)cell * 6 + f];
    return;
  }
  const int n = g.n;
  const unsigned q1 = udiv_n(g, (unsigned)cell), q2 = udiv_n(g, q1);
  const int co[3] = {cell - n * (int)q1, (int)q1 - n * (int)q2, (int)q2};
  const int stride[3] = {1, n, n * n};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    nb[2 * d] = co[d] == 0 ? -1 - 2 * d : cell - stride[d];
    nb[2 * d + 1] = co[d] == n - 1 ? -2 - 2 * d : cell + stride[d];
  }
}

// Parallel fill of the CellInfo records of nc cells: one thread per (cell, slot),
// slot 0..5 = faces, slot 6 = cell geometry (independent L2 loads in flight together).
template <int TT, bool UNI>
__device__ __forceinline__ void load_info_par(double* base, int per, int off, int nc, const MeshArgs& m,
                                              const UniformGrid& g, const double* __restrict__ aff, int c0,
                                              double sfac) {
  for (int idx = threadIdx.x; idx < nc * 7; idx += TT) {
    const int c = idx / 7, f = idx - c * 7;
    CellInfo& ci = *reinterpret_cast<CellInfo*>(base + c * per + off);
    const int cell = c0 + c;
    if (UNI) {  // no memory traffic: everything follows from the cell index
      if (f == 6) {
        ci.ih[0] = ci.ih[1] = ci.ih[2] = g.ih;
        ci.detJ = g.detJ;
        ci.A[0] = ci.A[1] = ci.A[2] = g.detJ * g.ih;
      } else {
        const int nb = uniform_nbr(g, cell, f);
        ci.nb[f] = nb;
        ci.pen[f] = sfac * (nb >= 0 ? g.pen_int : g.pen_bdry);
        ci.ihn[f] = nb >= 0 ? g.ih : 0.0;
        ci.type[f] = nb >= 0 ? 0 : (((g.outlet_mask >> f) & 1ull) ? 2 : 1);
      }
      continue;
    }
    if (f == 6) {
      const double* r = aff + (size_t)cell * kAffStride3;
      const double i0 = r[0], i1 = r[4], i2 = r[8], dj = r[9];
      ci.ih[0] = i0;
      ci.ih[1] = i1;
      ci.ih[2] = i2;
      ci.detJ = dj;
      ci.A[0] = dj * i0;
      ci.A[1] = dj * i1;
      ci.A[2] = dj * i2;
    } else {
      const int nb = m.nbr[(size_t)cell * 6 + f];
      const double pen = sfac * m.pen[(size_t)cell * 6 + f];
      int ty = 0;
      double ihn = 0.0;
      if (nb >= 0) {
        ihn = __ldg(aff + (size_t)nb * kAffStride3 + 4 * (f >> 1));
        if (nb == cell) ty = 3;  // hanging slot
      } else {
        const int bid = -1 - nb;
        ty = (bid >= 0 && bid < 64 && m.bctype[bid] == 1) ? 2 : 1;
      }
      ci.nb[f] = nb;
      ci.pen[f] = pen;
      ci.type[f] = ty;
      ci.ihn[f] = ihn;
    }
  }
}

// Branch-free coefficients of the 1D SIP face terms (forms.cpp:196-213 interior,
// :232-240 / :481-490 boundary), per face of one cell; `dirichlet` selects whether
// non-interior faces carry Dirichlet-type terms (outlets never do when
// outlet_natural).
__device__ __forceinline__ void face_coefs(CellInfo& ci, int f, bool dirichlet, bool outlet_natural,
                                           bool consistency_only = false) {
  const int d = f >> 1, s = f & 1;
  const double ih = ci.ih[d];
  const double sg = s ? -1.0 : 1.0;  // right face: -1/2 (...) ; left face: +1/2 (...)
  double* c = ci.fc[f];
  for (int i = 0; i < 6; ++i) c[i] = 0.0;
  const int ty = ci.type[f];
  if (ty == 0) {
    c[0] = 0.5 * sg * ih;
    c[1] = 0.5 * sg * ci.ihn[f];
    if (!consistency_only) {
      c[2] = ci.pen[f];
      c[3] = -ci.pen[f];
      c[4] = -0.5;
      c[5] = 0.5;
    }
  } else if (ty != 3 && dirichlet && !(ty == 2 && outlet_natural)) {
    c[0] = sg * ih;
    if (!consistency_only) {
      c[2] = 2.0 * ci.pen[f];
      c[4] = -1.0;
    }
  }
}

// 8-byte asynchronous global -> shared copy (LDGSTS); many in flight per thread.
__device__ __forceinline__ void cp_async8(double* smem_dst, const double* gsrc) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(smem_dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sa), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;\n" ::: "memory"); }

// Branch-free 1D SIP line operator along compile-time direction D (coefficients from
// face_coefs); neighbour lines of non-interior faces are multiplied by zero.
template <int N, int D>
__device__ __forceinline__ void sip_line_bf(const FTab<N, N>& t, const CellInfo& ci, const double* u,
                                            const double* uL, const double* uR, double scale, double* out) {
  const double ih = ci.ih[D], sa = scale * ci.A[D];
  const double stiff = sa * ih;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) s = fma(t.K[i][l], u[l], s);
    out[i] = stiff * s;
  }
  double gsR = 0.0, goR = 0.0, gsL = 0.0, goL = 0.0;
#pragma unroll
  for (int l = 0; l < N; ++l) {
    gsR = fma(t.dE[1][l], u[l], gsR);
    goR = fma(t.dE[0][l], uR[l], goR);
    gsL = fma(t.dE[0][l], u[l], gsL);
    goL = fma(t.dE[1][l], uL[l], goL);
  }
  const double* cR = ci.fc[2 * D + 1];
  const double* cL = ci.fc[2 * D];
  const double FR = cR[0] * gsR + cR[1] * goR + cR[2] * u[N - 1] + cR[3] * uR[0];
  const double GR = cR[4] * u[N - 1] + cR[5] * uR[0];
  const double FL = cL[0] * gsL + cL[1] * goL + cL[2] * u[0] + cL[3] * uL[N - 1];
  const double GL = cL[4] * u[0] + cL[5] * uL[N - 1];
  out[N - 1] = fma(sa, FR, out[N - 1]);
  out[0] = fma(sa, FL, out[0]);
  const double g2R = stiff * GR, g2L = -stiff * GL;
#pragma unroll
  for (int i = 0; i < N; ++i) out[i] = fma(t.dE[1][i], g2R, fma(t.dE[0][i], g2L, out[i]));
}

// 1D SIP line operator along direction d (stiffness + both d-faces), times `scale`.
// u: own line; uL / uR: neighbour lines across faces 2d / 2d+1 (read only if interior).
// dirichlet: whether non-interior, non-outlet faces carry the Dirichlet-type terms
// (momentum: always; pressure Helmholtz: never (natural); Laplacian: flag).
template <int N>
__device__ __forceinline__ void sip_line(const FTab<N, N>& t, const CellInfo& ci, int d, const double* u,
                                         const double* uL, const double* uR, bool dirichlet, double scale,
                                         double* out) {
  const double ih = ci.ih[d], A = ci.A[d];
  const double stiff = scale * A * ih;
#pragma unroll
  for (int i = 0; i < N; ++i) {
    double s = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) s = fma(t.K[i][l], u[l], s);
    out[i] = stiff * s;
  }
  // right face (side 1, outward normal +e_d)
  {
    const int f = 2 * d + 1;
    const int ty = ci.type[f];
    double F = 0.0, GT = 0.0;
    double gs = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) gs = fma(t.dE[1][l], u[l], gs);
    const double us = u[N - 1];
    if (ty == 0) {
      double go = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) go = fma(t.dE[0][l], uR[l], go);
      const double ju = us - uR[0];
      F = -0.5 * (gs * ih + go * ci.ihn[f]) + ci.pen[f] * ju;
      GT = -0.5 * ju;
    } else if (ty == 1 && dirichlet) {
      F = -gs * ih + 2.0 * ci.pen[f] * us;
      GT = -us;
    }
    const double sa = scale * A;
    out[N - 1] = fma(sa, F, out[N - 1]);
    const double g2 = sa * ih * GT;
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = fma(t.dE[1][i], g2, out[i]);
  }
  // left face (side 0, outward normal -e_d)
  {
    const int f = 2 * d;
    const int ty = ci.type[f];
    double F = 0.0, GT = 0.0;
    double gs = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) gs = fma(t.dE[0][l], u[l], gs);
    const double us = u[0];
    if (ty == 0) {
      double go = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) go = fma(t.dE[1][l], uL[l], go);
      const double ju = us - uL[N - 1];
      F = 0.5 * (gs * ih + go * ci.ihn[f]) + ci.pen[f] * ju;
      GT = -0.5 * ju;
    } else if (ty == 1 && dirichlet) {
      F = gs * ih + 2.0 * ci.pen[f] * us;
      GT = -us;
    }
    const double sa = scale * A;
    out[0] = fma(sa, F, out[0]);
    const double g2 = -sa * ih * GT;
#pragma unroll
    for (int i = 0; i < N; ++i) out[i] = fma(t.dE[0][i], g2, out[i]);
  }
}

// ===========================================================================
// Scalar SIP, axis-aligned affine, 2D (BASELINE cfg1): the same exact line split
//   y = mc detJ (M (x) M) u + (S_x (x) M) u + (M (x) S_y) u
// one thread per cell (the 2D problems are small: the generic kernel's many CTA-wide
// stages made it latency-bound).  Node (i, j) at i + N j.
// ===========================================================================
constexpr int kAffStride2 = 4 + 1 + 4 * 3;
template <int KP>
__global__ void __launch_bounds__(128) k_sip_axis2(MeshArgs m, const double* __restrict__ aff, double mc, int dir_bdry,
                                                   const double* __restrict__ x, double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  constexpr int N = KP + 1, NB = N * N;
  const FTab<N, N>& ta = c_ft<N, N>;
  const int cell = blockIdx.x * blockDim.x + threadIdx.x;
  if (cell >= m.ncells) return;
  const double sfac = (double)(N * N);
  CellInfo ci;
  {
    const double* r = aff + (size_t)cell * kAffStride2;
    ci.ih[0] = r[0];
    ci.ih[1] = r[3];
    ci.ih[2] = 0.0;
    ci.detJ = r[4];
    ci.A[0] = ci.detJ * ci.ih[0];
    ci.A[1] = ci.detJ * ci.ih[1];
#pragma unroll
    for (int f = 0; f < 4; ++f) {
      const int nb = m.nbr[(size_t)cell * 4 + f];
      ci.nb[f] = nb;
      ci.pen[f] = sfac * m.pen[(size_t)cell * 4 + f];
      if (nb >= 0) {
        ci.type[f] = nb == cell ? 3 : 0;  // 3: hanging slot (zero weight)
        ci.ihn[f] = __ldg(aff + (size_t)nb * kAffStride2 + 3 * (f >> 1));
      } else {
        ci.type[f] = 1;  // the scalar operator treats every boundary id alike (walls / natural)
        ci.ihn[f] = 0.0;
      }
    }
  }
  const double* u0 = x + (size_t)cell * NB;
  double u[NB];
#pragma unroll
  for (int i = 0; i < NB; ++i) u[i] = __ldg(u0 + i);
  double out[NB];
  // mass: mc detJ (M (x) M) u
  const double cm = mc * ci.detJ;
#pragma unroll
  for (int j = 0; j < N; ++j)
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double t = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) t = fma(ta.M[i][a], u[a + N * b], t);
        s = fma(ta.M[j][b], t, s);
      }
      out[i + N * j] = cm * s;
    }
  const bool dir = dir_bdry != 0;
  // x-lines: S_x on each row, then M along y
  {
    double sx[NB];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double line[N], lL[N], lR[N], o[N];
#pragma unroll
      for (int i = 0; i < N; ++i) line[i] = u[i + N * j];
      const int nl = ci.nb[0], nr = ci.nb[1];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        lL[i] = nl >= 0 ? __ldg(x + (size_t)nl * NB + i + N * j) : 0.0;
        lR[i] = nr >= 0 ? __ldg(x + (size_t)nr * NB + i + N * j) : 0.0;
      }
      sip_line<N>(ta, ci, 0, line, lL, lR, dir, 1.0, o);
#pragma unroll
      for (int i = 0; i < N; ++i) sx[i + N * j] = o[i];
    }
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int b = 0; b < N; ++b) s = fma(ta.M[j][b], sx[i + N * b], s);
        out[i + N * j] += s;
      }
  }
  // y-lines: S_y on each column, then M along x
  {
    double sy[NB];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double line[N], lL[N], lR[N], o[N];
#pragma unroll
      for (int j = 0; j < N; ++j) line[j] = u[i + N * j];
      const int nl = ci.nb[2], nr = ci.nb[3];
#pragma unroll
      for (int j = 0; j < N; ++j) {
        lL[j] = nl >= 0 ? __ldg(x + (size_t)nl * NB + i + N * j) : 0.0;
        lR[j] = nr >= 0 ? __ldg(x + (size_t)nr * NB + i + N * j) : 0.0;
      }
      sip_line<N>(ta, ci, 1, line, lL, lR, dir, 1.0, o);
#pragma unroll
      for (int j = 0; j < N; ++j) sy[i + N * j] = o[j];
    }
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int a = 0; a < N; ++a) s = fma(ta.M[i][a], sy[a + N * j], s);
        out[i + N * j] += s;
      }
  }
  double* yo = y + (size_t)cell * NB;
#pragma unroll
  for (int i = 0; i < NB; ++i) yo[i] = out[i];
}

// ===========================================================================
// Scalar SIP (pressure Helmholtz / Laplacian), axis-aligned affine, 3D.
//   y = mc detJ (M M M) u + sum_d (S_d (x) M (x) M) u
// ===========================================================================
template <int KP>
struct SipAxisCfg {
  static constexpr int N = KP + 1, NB = N * N * N, NF = N * N;
  #ifndef DGB_SIP_PX3
#define DGB_SIP_PX3 3
#endif
  using P = Pad<N, N == 3 ? DGB_SIP_PX3 : (N | 1)>;
#ifndef DGB_SIP2_C  // tuning overrides for experiments (tools/tune_sip.sh)
#define DGB_SIP2_C 16
#define DGB_SIP2_T 128
#endif
  static constexpr int C = KP == 1 ? 32 : (KP == 2 ? DGB_SIP2_C : 8);  // cells per CTA
  static constexpr int T = KP == 1 ? 128 : (KP == 2 ? DGB_SIP2_T : 128);
  // cells per warp: a warp owns CPW cells after the staging barrier (per-cell stages then
  // sync with __syncwarp); chosen so the N^2-item line stages fill 32 lanes
  static constexpr int CPW = KP == 1 ? 8 : (KP == 2 ? 3 : 2);
  static constexpr bool WPG = C % CPW == 0 && T == 32 * (C / CPW);
#ifndef DGB_SIP2_CTPAD
#define DGB_SIP2_CTPAD 0
#endif
  static constexpr int CTS = P::CT + (KP == 2 ? DGB_SIP2_CTPAD : 0);  // array stride (KP = 2: padded)
  static constexpr int O_U = 0, O_SX = CTS, O_SY = 2 * CTS, O_SZ = 3 * CTS, O_UX = 4 * CTS;
  static constexpr int O_INFO = 5 * CTS;
  // KP = 1: the per-cell stride is 10 mod 16 doubles and the warp's line items run
  // cell-fastest (CF): the 8 cells of a warp then sit on distinct even bank pairs and the
  // second line of each half-warp on the odd ones — conflict-free line stages (bank
  // simulation: 178 -> 80 wavefronts per warp-group vs an ideal of 80; ncu had 45 % of
  // the kernel's shared wavefronts as conflicts)
  static constexpr bool CF = KP == 1 && WPG;
#ifndef DGB_SIP2_PERPAD  // KP = 2: cell-stride pad (tools/bank_sim_sip2.py: 1131 -> 1026 modelled wavefronts)
#define DGB_SIP2_PERPAD 6
#endif
  static constexpr int PER = CF ? O_INFO + kInfoDoubles + 1
                                : ((O_INFO + kInfoDoubles) | 1) + (KP == 2 ? DGB_SIP2_PERPAD : 0);
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
  // the cell-fastest (CF) layout is bank-conflict-free only for a cell stride of 10 mod 16
  // doubles (tools/bank_sim_sip1.py); a new CellInfo field must keep that
  static_assert(!CF || PER % 16 == 10, "SipAxisCfg: CF layout needs PER % 16 == 10");
};

// CGF: the CG apply q = A p with <p, q> fused into the epilogue (krylov.cpp:84-87):
// partial[block * warps + warp] = sum over the warp's DoFs of p q (alpha:
// cg_alpha_from_partials, a two-level reduction; a single-block finish at the tail of this
// kernel was slower).
struct SipCgArgs {
  double* partial = nullptr;
  CgState* st = nullptr;
};

template <int KP, bool UNI, bool CGF = false>
__global__ void __launch_bounds__(SipAxisCfg<KP>::T) k_sip_axis(MeshArgs m, UniformGrid ug, const double* __restrict__ aff,
                                                                 double mc, int dir_bdry,
                                                                 const double* __restrict__ x,
                                                                 double* __restrict__ y, SipCgArgs cg) {
  if (m.skip && *m.skip) return;
  using G = SipAxisCfg<KP>;
  using P = typename G::P;
  constexpr int N = G::N, NB = G::NB, NF = G::NF, C = G::C, PER = G::PER, TT = G::T;
  const FTab<N, N>& ta = c_ft<N, N>;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = m.cell0 + blockIdx.x * C;
  const int nc = min(C, (m.cell1 < 0 ? m.ncells : m.cell1) - c0);
  const int tid = threadIdx.x;
  const double sfac = (double)((KP + 1) * (KP + 1));
  constexpr bool WPG = G::WPG;
  constexpr int CPW = G::CPW;
  const int lane = tid & 31, wbase = (tid >> 5) * CPW;
  const int it0 = WPG ? lane : tid;
  constexpr int IST = WPG ? 32 : TT;
  const int gbase = WPG ? wbase : 0;
  const int gcnt = WPG ? max(0, min(CPW, nc - wbase)) : nc;
  // item -> (cell of the group, rest): cell-major, or cell-fastest for CF
  auto split = [&](int idx, int X, int& cl, int& r) {
    if (G::CF) {
      cl = gcnt == CPW ? idx % CPW : idx % gcnt;
      r = gcnt == CPW ? idx / CPW : idx / gcnt;
    } else {
      cl = idx / X;
      r = idx - cl * X;
    }
  };
#define CELL(c) (sm + (c) * PER)
#define INFO(c) (*reinterpret_cast<CellInfo*>(sm + (c) * PER + G::O_INFO))
#define SYNC_G()       \
  do {                 \
    if (WPG)           \
      __syncwarp();    \
    else               \
      __syncthreads(); \
  } while (0)

  // S0: cell values (padded) + per-cell info
  for (int idx = tid; idx < nc * NB; idx += TT) {
    const int c = idx / NB, i = idx - c * NB;
    cp_async8(CELL(c) + G::O_U + P::idx(i % N, (i / N) % N, i / NF), x + (size_t)(c0 + c) * NB + i);
  }
  load_info_par<TT, UNI>(sm, PER, G::O_INFO, nc, m, ug, aff, c0, sfac);
  cp_async_wait_all();
  __syncthreads();
  // the scalar operator ignores outlet ids: all boundary faces are natural, or all
  // Dirichlet when dir_bdry (forms.cpp:218-242)
  for (int idx = it0; idx < gcnt * 6; idx += IST) {
    CellInfo& ci = INFO(gbase + idx / 6);
    if (ci.type[idx % 6] == 2) ci.type[idx % 6] = 1;
  }
  SYNC_G();
  // A: all-direction lines: S_d on raw lines (+ neighbour lines), and Ux = M_x u
  for (int idx = it0; idx < gcnt * 3 * NF; idx += IST) {
    int cl, r;
    split(idx, 3 * NF, cl, r);
    const int c = gbase + cl;
    const int d = r / NF, tl = r - d * NF;
    const int p = tl % N, q = tl / N;
    const CellInfo& ci = INFO(c);
    const int st = d == 0 ? 1 : (d == 1 ? P::PX : P::PY);
    const int b0 = d == 0 ? P::idx(0, p, q) : (d == 1 ? P::idx(p, 0, q) : P::idx(p, q, 0));
    const int gst = d == 0 ? 1 : (d == 1 ? N : NF);
    const int g0 = d == 0 ? N * (p + N * q) : (d == 1 ? p + NF * q : p + N * q);
    double u[N], uL[N], uR[N], o[N];
#pragma unroll
    for (int l = 0; l < N; ++l) u[l] = CELL(c)[G::O_U + b0 + l * st];
    const int nl = ci.nb[2 * d], nr = ci.nb[2 * d + 1];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      uL[l] = nl >= 0 ? __ldg(x + (size_t)nl * NB + g0 + l * gst) : 0.0;
      uR[l] = nr >= 0 ? __ldg(x + (size_t)nr * NB + g0 + l * gst) : 0.0;
    }
    sip_line<N>(ta, ci, d, u, uL, uR, dir_bdry != 0, 1.0, o);
    double* so = CELL(c) + (d == 0 ? G::O_SX : (d == 1 ? G::O_SY : G::O_SZ)) + b0;
#pragma unroll
    for (int l = 0; l < N; ++l) so[l * st] = o[l];
    if (d == 0) {
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(ta.M[i][l], u[l], s);
        CELL(c)[G::O_UX + b0 + i] = s;
      }
    }
  }
  SYNC_G();
  // B: x-lines, in place: SY <- M_x SY, SZ <- M_x SZ
  for (int idx = it0; idx < gcnt * NF; idx += IST) {
    int cl, tl;
    split(idx, NF, cl, tl);
    const int c = gbase + cl;
    const int b0 = P::idx(0, tl % N, tl / N);
    double a[N], b[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      a[l] = CELL(c)[G::O_SY + b0 + l];
      b[l] = CELL(c)[G::O_SZ + b0 + l];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0, t = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(ta.M[i][l], a[l], s);
        t = fma(ta.M[i][l], b[l], t);
      }
      CELL(c)[G::O_SY + b0 + i] = s;
      CELL(c)[G::O_SZ + b0 + i] = t;
    }
  }
  SYNC_G();
  // C: y-lines: SX <- M_y (SX + mc detJ UX) + SY ; SZ <- M_y SZ
  for (int idx = it0; idx < gcnt * NF; idx += IST) {
    int cl, tl;
    split(idx, NF, cl, tl);
    const int c = gbase + cl;
    const int b0 = P::idx(tl % N, 0, tl / N);
    const double cm = mc * INFO(c).detJ;
    double a[N], b[N], e[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      a[l] = fma(cm, CELL(c)[G::O_UX + b0 + l * P::PX], CELL(c)[G::O_SX + b0 + l * P::PX]);
      b[l] = CELL(c)[G::O_SZ + b0 + l * P::PX];
      e[l] = CELL(c)[G::O_SY + b0 + l * P::PX];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = e[j], t = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        s = fma(ta.M[j][l], a[l], s);
        t = fma(ta.M[j][l], b[l], t);
      }
      CELL(c)[G::O_SX + b0 + j * P::PX] = s;
      CELL(c)[G::O_SZ + b0 + j * P::PX] = t;
    }
  }
  SYNC_G();
  // D: z-lines: y = M_z SX + SZ   -> global
  double pq[1] = {0.0};
  for (int idx = it0; idx < gcnt * NF; idx += IST) {
    int cl, tl;
    split(idx, NF, cl, tl);
    const int c = gbase + cl;
    const int i = tl % N, j = tl / N;
    const int b0 = P::idx(i, j, 0);
    double a[N];
#pragma unroll
    for (int l = 0; l < N; ++l) a[l] = CELL(c)[G::O_SX + b0 + l * P::PY];
    double* yo = y + (size_t)(c0 + c) * NB + i + N * j;
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double s = CELL(c)[G::O_SZ + b0 + k * P::PY];
#pragma unroll
      for (int l = 0; l < N; ++l) s = fma(ta.M[k][l], a[l], s);
      yo[NF * k] = s;
      if (CGF) pq[0] = fma(CELL(c)[G::O_U + b0 + k * P::PY], s, pq[0]);
    }
  }
  if (CGF) {  // one deterministic partial per warp (shuffle tree), no CTA barrier at the tail
    double a = pq[0];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((tid & 31) == 0) cg.partial[blockIdx.x * (TT / 32) + (tid >> 5)] = a;
  }
#undef CELL
#undef INFO
#undef SYNC_G
}

// ===========================================================================
// Scalar SIP operator on UNIFORM Cartesian 3D grids, one THREAD per cell.
//
// With N = 2 or 3 nodes per direction a cell's values fit in registers, so the whole
// line split  y = sum_d (M (x) M (x) (S_d + mc detJ / 3 M_d)) u  runs thread-serially
// with compile-time indices: no per-stage shared-memory round trips (k_sip_axis moves
// ~88 shared wavefronts per Q2 cell, this kernel ~15) and no idle lanes.  A CTA owns a
// TX x TY x TZ tile of cells; the tile and its face-neighbour halo are staged once by
// row-wise coalesced cp.async copies (cells are x-fastest, so a box row is one
// contiguous range; cell stride odd: threads of a warp reading the same node of
// consecutive cells hit distinct banks), every thread reads its lines and its
// neighbours' lines from there, and the result goes back through the same buffer so the
// global stores are coalesced rows too.  CGF: <p, A p> per-warp partials as k_sip_axis.
// ===========================================================================
template <int KP>
struct SipCellCfg {
  static constexpr int N = KP + 1, NB = N * N * N, NF = N * N;
  // tile shape and register cap per degree (measured, profiles/experiments_r02.md): long x-rows
  // stage best; Q1: 80 registers (6 CTAs per SM), Q2: all 255 (2 CTAs per SM, shared-memory bound)
#ifndef DGB_SIPC_TX
#define DGB_SIPC_TX 16
#define DGB_SIPC_TY (KP == 1 ? 2 : 4)
#define DGB_SIPC_TZ (KP == 1 ? 4 : 2)
#endif
#ifndef DGB_SIPC_MINB1
#define DGB_SIPC_MINB1 6
#endif
#ifndef DGB_SIPC_MINB2
#define DGB_SIPC_MINB2 1
#endif
  static constexpr int TX = DGB_SIPC_TX, TY = DGB_SIPC_TY, TZ = DGB_SIPC_TZ, T = TX * TY * TZ;
  static constexpr int MINB = KP == 1 ? DGB_SIPC_MINB1 : DGB_SIPC_MINB2;
  static constexpr int BX = TX + 2, BY = TY + 2, BZ = TZ + 2, NBOX = BX * BY * BZ;
  static constexpr int CS = NB | 1;  // odd cell stride
  static constexpr size_t SMEM = (size_t)NBOX * CS * sizeof(double);
};

template <int KP, bool CGF = false>
__global__ void __launch_bounds__(SipCellCfg<KP>::T, SipCellCfg<KP>::MINB) k_sip_cell(MeshArgs m, UniformGrid ug, double mc, int dir_bdry,
                                                                 const double* __restrict__ x,
                                                                 double* __restrict__ y, SipCgArgs cg) {
  if (m.skip && *m.skip) return;
  using G = SipCellCfg<KP>;
  constexpr int N = G::N, NB = G::NB, NF = G::NF, CS = G::CS;
  constexpr int TX = G::TX, TY = G::TY, TZ = G::TZ, BX = G::BX, BY = G::BY, BZ = G::BZ;
  const FTab<N, N>& ta = c_ft<N, N>;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int n = ug.n;
  const int ntx = (n + TX - 1) / TX, nty = (n + TY - 1) / TY;
  const int bx = blockIdx.x % ntx, by = (blockIdx.x / ntx) % nty, bz = blockIdx.x / (ntx * nty);
  // owned z-layers [zlo, zhi): the whole mesh, or the layer range of dgb_set_cell_range
  // (z-slab applies; the layers next to the range are read as ghosts)
  const int zlo = m.cell0 / (n * n), zhi = m.cell1 < 0 ? n : m.cell1 / (n * n);
  const int x0 = bx * TX, y0 = by * TY, z0 = zlo + bz * TZ;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // ---- stage the box rows (tile + face halo; the box's edge rows are never read)
  {
    const int xa = max(x0 - 1, 0), xb = min(x0 + TX, n - 1);  // first / last cell of a row inside the domain
    const int e0 = (xa - (x0 - 1)) * NB, e1 = (xb - (x0 - 1) + 1) * NB;
    for (int r = warp; r < BY * BZ; r += G::T / 32) {
      const int rby = r % BY, rbz = r / BY;
      const bool hy = rby == 0 || rby == BY - 1, hz = rbz == 0 || rbz == BZ - 1;
      const int gy = y0 - 1 + rby, gz = z0 - 1 + rbz;
      if ((hy && hz) || gy < 0 || gy >= n || gz < 0 || gz >= n) continue;
      // tile rows beyond a partial tile's end are only needed as halo of the last row inside
      const double* src = x + ((size_t)((size_t)gz * n + gy) * n + (x0 - 1)) * NB;  // may point before x: only [e0, e1) is read
      double* dst = sm + (size_t)BX * (rby + BY * rbz) * CS;
      for (int e = e0 + lane; e < e1; e += 32) {
        const int so = CS == NB ? e : (e / NB) * CS + e % NB;
        cp_async8(dst + so, src + e);
      }
    }
  }
  cp_async_wait_all();
  __syncthreads();
  const int tx = tid % TX, ty = (tid / TX) % TY, tz = tid / (TX * TY);
  const int gx = x0 + tx, gy = y0 + ty, gz = z0 + tz;
  const bool live = gx < n && gy < n && gz < zhi;
  const int bc = (tx + 1) + BX * ((ty + 1) + BY * (tz + 1));
  const double* U = sm + (size_t)bc * CS;
  // uniform-grid cell record (the scalar operator treats every boundary face alike:
  // natural, or Dirichlet-type when dir_bdry; forms.cpp:218-242)
  CellInfo ci;
  const double sfac = (double)(N * N);
  ci.detJ = ug.detJ;
  const int co[3] = {gx, gy, gz};
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    ci.ih[d] = ug.ih;
    ci.A[d] = ug.detJ * ug.ih;
#pragma unroll
    for (int sd = 0; sd < 2; ++sd) {
      const bool bdry = sd ? co[d] == n - 1 : co[d] == 0;
      ci.type[2 * d + sd] = bdry ? 1 : 0;
      ci.pen[2 * d + sd] = sfac * (bdry ? ug.pen_bdry : ug.pen_int);
      ci.ihn[2 * d + sd] = bdry ? 0.0 : ug.ih;
    }
  }
  const double cm3 = mc * ug.detJ * (1.0 / 3.0);
  // line t of direction d (nodes base(t) + l * st of the cell array): o = (S_d + cm3 M_d) u
  auto line = [&](auto dtag, int p, int q, double* o) {
    constexpr int d = decltype(dtag)::value;
    constexpr int st = d == 0 ? 1 : (d == 1 ? N : NF);
    constexpr int bst = d == 0 ? 1 : (d == 1 ? BX : BX * BY);
    const double* UL = U - (size_t)bst * CS;
    const double* UR = U + (size_t)bst * CS;
    const int b0 = d == 0 ? N * (p + N * q) : (d == 1 ? p + NF * q : p + N * q);
    double u[N], uL[N], uR[N];
#pragma unroll
    for (int l = 0; l < N; ++l) {
      u[l] = U[b0 + l * st];
      uL[l] = UL[b0 + l * st];
      uR[l] = UR[b0 + l * st];
    }
    sip_line<N>(ta, ci, d, u, uL, uR, dir_bdry != 0, 1.0, o);
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double sacc = 0.0;
#pragma unroll
      for (int l = 0; l < N; ++l) sacc = fma(ta.M[i][l], u[l], sacc);
      o[i] = fma(cm3, sacc, o[i]);
    }
  };
  using D0 = std::integral_constant<int, 0>;
  using D1 = std::integral_constant<int, 1>;
  using D2 = std::integral_constant<int, 2>;
  // Y = M_y M_x A_z first (the only term whose lines cross the z-planes), then plane by plane
  // P_k = M_y A_x + M_x A_y (N^2 values) and Y[., ., k'] += M[k'][k] P_k: 1 + 1/N cell arrays live
  double Y[NB];
  double pq = 0.0;
  if (live) {
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double az[N][N];  // [i][k] of row j
#pragma unroll
      for (int i = 0; i < N; ++i) line(D2{}, i, j, az[i]);
#pragma unroll
      for (int k = 0; k < N; ++k)  // M_x along i
#pragma unroll
        for (int i2 = 0; i2 < N; ++i2) {
          double sacc = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) sacc = fma(ta.M[i2][i], az[i][k], sacc);
          Y[i2 + N * j + NF * k] = sacc;
        }
    }
#pragma unroll
    for (int k = 0; k < N; ++k)  // M_y along j, in place
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = Y[i + N * j + NF * k];
#pragma unroll
        for (int j2 = 0; j2 < N; ++j2) {
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) sacc = fma(ta.M[j2][j], v[j], sacc);
          Y[i + N * j2 + NF * k] = sacc;
        }
      }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      double ax[N][N], P[N][N];  // ax[j][i]; P[j][i]
#pragma unroll
      for (int j = 0; j < N; ++j) line(D0{}, j, k, ax[j]);
#pragma unroll
      for (int j2 = 0; j2 < N; ++j2)
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double sacc = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) sacc = fma(ta.M[j2][j], ax[j][i], sacc);
          P[j2][i] = sacc;
        }
#pragma unroll
      for (int i = 0; i < N; ++i) line(D1{}, i, k, ax[i]);  // ax[i][j] now holds A_y
#pragma unroll
      for (int j = 0; j < N; ++j)
#pragma unroll
        for (int i2 = 0; i2 < N; ++i2) {
          double sacc = P[j][i2];
#pragma unroll
          for (int i = 0; i < N; ++i) sacc = fma(ta.M[i2][i], ax[i][j], sacc);
          P[j][i2] = sacc;
        }
#pragma unroll
      for (int k2 = 0; k2 < N; ++k2)
#pragma unroll
        for (int j = 0; j < N; ++j)
#pragma unroll
          for (int i = 0; i < N; ++i) Y[i + N * j + NF * k2] = fma(ta.M[k2][k], P[j][i], Y[i + N * j + NF * k2]);
    }
    if (CGF) {
#pragma unroll
      for (int i = 0; i < NB; ++i) pq = fma(U[i], Y[i], pq);
    }
  }
  if (CGF) {  // one deterministic partial per warp (shuffle tree)
    double a = pq;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if (lane == 0) cg.partial[blockIdx.x * (G::T / 32) + warp] = a;
  }
  // ---- results back through the staging buffer: coalesced row stores
  __syncthreads();  // every neighbour has read this cell's values
  if (live) {
    double* O = sm + (size_t)bc * CS;
#pragma unroll
    for (int i = 0; i < NB; ++i) O[i] = Y[i];
  }
  __syncthreads();
  {
    const int xe = min(TX, n - x0) * NB;  // doubles of a tile row inside the domain
    for (int r = warp; r < TY * TZ; r += G::T / 32) {
      const int rty = r % TY, rtz = r / TY;
      const int gyr = y0 + rty, gzr = z0 + rtz;
      if (gyr >= n || gzr >= zhi) continue;
      double* dst = y + ((size_t)((size_t)gzr * n + gyr) * n + x0) * NB;
      const double* src = sm + (size_t)(1 + BX * ((rty + 1) + BY * (rtz + 1))) * CS;
      for (int e = lane; e < xe; e += 32) dst[e] = src[CS == NB ? e : (e / NB) * CS + e % NB];
    }
  }
}

// ===========================================================================
// Momentum operator, axis-aligned affine, 3D, skew = 0:
//   mass M x + visc A_sip x     (line-split, exact)
// + adv C_lf(w) x               (k+2 Gauss rule; sum factorisation)
// ===========================================================================
// MODE 0: fused operator; 1: mass + viscous only (writes y); 2: advection only (adds into y)
// (component, line) of pass-A item r for lines along direction d.  K = 2 orders the
// y- and z-line items component-fastest: their padded offsets then spread over the
// shared-memory banks (bank-conflict simulation: stages A_y / A_z / C / D drop from 57 to
// 21 excess wavefronts per cell); x-lines stay component-major (conflict-free that way).
template <int K, int NF>
__device__ __forceinline__ void line_item(int r, int d, int& comp, int& tl) {
  if (K == 2 && d != 0) {
    tl = r / 3;
    comp = r - 3 * tl;
  } else {
    comp = r / NF;
    tl = r - comp * NF;
  }
}

template <int K, int CC, int TH, int MODE = 0>
struct MomAxisCfg {
  static constexpr int N = K + 1, Q = K + 2, NB = N * N * N, NF = N * N, QN = Q * N, QQ = Q * Q;
#ifndef DGB_MOM_PX2
#define DGB_MOM_PX2 3
#endif
  using P = Pad<N, N == 3 ? DGB_MOM_PX2 : (N | 1)>;  // x-pitch of the staged cell tensors
  static constexpr int CT = P::CT | 1;  // odd component stride (bank-conflict-free field interleave)
  static constexpr int C = CC;   // cells per CTA
  static constexpr int T = TH;   // threads per CTA
  // persistent per-cell regions
  static constexpr int O_X = 0, O_W = 3 * CT, O_OUT = 6 * CT, O_INFO = 9 * CT;
  static constexpr int O_WORK = O_INFO + kInfoDoubles;
  // phase A: SX, SY, SZ, UX (3 comps each)
  static constexpr int A_SX = 0, A_SY = 3 * CT, A_SZ = 6 * CT, A_UX = 9 * CT, A_END = 12 * CT;
  // phase B (advection cell terms)
  // quadrature-plane stride of the YB / T tensors, odd so that per-layer items
  // (one plane each) start on different banks
  static constexpr int QQP = QQ | 1;
  // TZ/TY/TX [comp (stride BRC)][test][l][qxy]; K = 2 pads the component stride so S78's
  // (comp, l) items hit distinct banks (153 = 9 mod 16 collides comp 0 / 2; 154 does not)
  static constexpr int BRC = 3 * QQP * N + (K == 2 ? 1 : 0);
  static constexpr int B_R1 = 0;
  static constexpr int B_R2 = 3 * BRC;  // YB [field][k][qxy] (6 QQP N)
  static constexpr int B_END = B_R2 + 6 * QQP * N;
  // face phase (all 6 faces at once): V1 [8 fields][6][Q x N] -> FB [3][6][N x N];  FL [3][6][Q x N]
  // V1 [field][q][f][qp]: face-Gauss-point rows of all 6 faces contiguous (F2 reads them
  // conflict-free); the q-block stride VB is chosen so F1's (f, q) writes hit distinct banks
  // V1F: face stride inside a V1 row (K = 2: 5 instead of Q = 4 with VB = 39 takes F1's
  // store conflicts from 32 to 24 excess wavefronts per cell at the price of 8 in F2);
  // FLC: component stride of FL (K = 2: 6 QN + 1 takes F3's read conflicts from 36 to 12)
  static constexpr int VB = K == 3 ? 36 : (K == 2 ? 39 : 6 * Q), V1_SIZE = 8 * N * VB;
  static constexpr int V1F = K == 2 ? 5 : Q;
  static constexpr int FLC = 6 * QN + (K == 2 ? 1 : 0);
  static constexpr int F_V1 = 0, F_FL = V1_SIZE, F_END = F_FL + 2 * FLC + 6 * QN;
  // neighbour face traces [f (stride NBS)][x0, x1, x2, w_normal][p + N q], filled during S0 /
  // pass A and read by F1; disjoint from the pass-A regions and from V1
  static constexpr int NBS = 4 * NF + 1;
  static constexpr int F_NB = A_END > V1_SIZE ? A_END : V1_SIZE, F_NB_END = F_NB + 6 * NBS;
  static constexpr int BF0 = B_END > F_END ? B_END : F_END;
  static constexpr int BF = BF0 > F_NB_END ? BF0 : F_NB_END;
  static constexpr int WORK = MODE == 1 ? A_END : (MODE == 2 ? BF : (A_END > BF ? A_END : BF));
  static constexpr int PER = (O_WORK + WORK) | 1;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};
// default tuning per degree
// (SPLIT: launch mass+viscous and advection as two kernels with their own occupancy)
template <int K, int MODE> struct MomAxisTune { static constexpr int C = 6, T = 192; static constexpr bool SPLIT = false; };
template <int MODE> struct MomAxisTune<1, MODE> { static constexpr int C = 16, T = 128; static constexpr bool SPLIT = false; };
#ifndef DGB_MOM2_C
#define DGB_MOM2_C 6  // 6 cells / 192 threads: 3.63 -> 3.41 ms at cfg5 (after the unsplit S78)
#define DGB_MOM2_T 192
#endif
template <int MODE> struct MomAxisTune<2, MODE> { static constexpr int C = DGB_MOM2_C, T = DGB_MOM2_T; static constexpr bool SPLIT = false; };
#ifndef DGB_MOM3_C  // tuning overrides for experiments (tools/tune_mom.sh)
#define DGB_MOM3_C 6
#define DGB_MOM3_T 192
#endif
template <> struct MomAxisTune<3, 0> { static constexpr int C = DGB_MOM3_C, T = DGB_MOM3_T; static constexpr bool SPLIT = false; };
template <> struct MomAxisTune<3, 1> { static constexpr int C = 4, T = 128; static constexpr bool SPLIT = true; };
template <> struct MomAxisTune<3, 2> { static constexpr int C = 3, T = 96; static constexpr bool SPLIT = true; };

// RHS: the explicit stage right-hand side operator of momentum_rhs (forms.cpp:816-1084)
// instead: consistency-only viscous faces (no symmetry / penalty) and the central
// advective flux with w.n f on every boundary face; the caller passes the negated
// viscous / advective coefficients.  acc: y += result.
template <int K, int CC, int TH, int MODE, bool UNI, bool RHS = false>
#ifndef DGB_MOM_MINB  // minimum CTAs per SM promised to ptxas (0: no promise)
#define DGB_MOM_MINB 2
#endif
#ifndef DGB_MOM_MINB2  // the same for K = 2: shared memory allows 3 CTAs of 6 cells, 2 let ptxas take 123
#define DGB_MOM_MINB2 3  // registers and lose the third CTA (cfg5 3.59 ms; 3: 96 registers, 3.31 ms)
#endif
__global__ void __launch_bounds__(TH, K == 2 ? DGB_MOM_MINB2 : DGB_MOM_MINB) k_momentum_axis(MeshArgs m, UniformGrid ug, const double* __restrict__ aff, MomCoef co,
                                                      const double* __restrict__ x, const double* __restrict__ w,
                                                      double* __restrict__ y, int acc) {
  if (m.skip && *m.skip) return;
  using G = MomAxisCfg<K, CC, TH, MODE>;
  using P = typename G::P;
  constexpr int N = G::N, Q = G::Q, NB = G::NB, NF = G::NF, QN = G::QN, QQ = G::QQ, C = G::C, PER = G::PER;
  constexpr int TT = G::T, CT = G::CT;
  const FTab<N, Q>& tq = c_ft<N, Q>;  // k+2 rule: B, D, w (advection)
  const FTab<N, N>& ta = c_ft<N, N>;  // exact M, K, dE
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = m.cell0 + blockIdx.x * C;
  const int nc = min(C, (m.cell1 < 0 ? m.ncells : m.cell1) - c0);
  const int tid = threadIdx.x;
  const double sfac = (double)((K + 1) * (K + 1));
  const bool faces = MODE != 1 && co.adv != 0.0;
  // WPC: one warp per cell when the CTA has exactly 32 threads per cell.  After the
  // CTA-wide staging barrier every stage touches only its own cell (neighbour data is
  // read from the staged x or the trace stash), so stages sync with __syncwarp.
  constexpr bool WPC = TT == 32 * C;
  const int lane = tid & 31, wcell = tid >> 5;
  const int it0 = WPC ? lane : tid;
  constexpr int IST = WPC ? 32 : TT;
#define ITEMS(X) (WPC ? (wcell < nc ? (X) : 0) : nc * (X))
#define CELLOF(idx, X) (WPC ? wcell : (idx) / (X))
#define RESTOF(idx, c, X) (WPC ? (idx) : (idx) - (c) * (X))
#define SYNC_CELL()    \
  do {                 \
    if (WPC)           \
      __syncwarp();    \
    else               \
      __syncthreads(); \
  } while (0)
#define CELL(c) (sm + (c) * PER)
#define WK(c) (sm + (c) * PER + G::O_WORK)
#define INFO(c) (*reinterpret_cast<CellInfo*>(sm + (c) * PER + G::O_INFO))

  // ------------------------------------------------------------------ S0: x, w (padded), info
  // Pass-A neighbour lines: every thread issues the loads of ALL its stage-A items now
  // (registers), overlapping the cp.async staging and the info loads.  Neighbours
  // owned by this CTA are read from shared memory later instead.  Items of one
  // direction: (cell, comp, line) with the line index fastest.
  const bool passA = MODE != 2 && (co.mass != 0.0 || co.visc != 0.0);
  constexpr int NID = 3 * NF;                      // items per cell and direction
  constexpr int MAXJ = WPC ? (NID + 31) / 32 : (C * NID + TT - 1) / TT;  // items per thread and direction
  double nbL[3][MAXJ][N], nbR[3][MAXJ][N];
#ifndef DGB_WPC_S0
#define DGB_WPC_S0 1
#endif
#ifndef DGB_MOM_PF
#define DGB_MOM_PF 296  // 2 CTAs x 148 SMs ahead: cfg3 1.759 -> 1.749 ms (148 / 592: the same)
#endif
  if constexpr (DGB_MOM_PF > 0) {
    // pull the x / w blocks of the CTA that will run DGB_MOM_PF blocks later into L2, so
    // that its staging waits on L2 instead of HBM
    const long long pc0 = (long long)c0 + (long long)DGB_MOM_PF * C;
    constexpr int LINES = C * 3 * NB * 8 / 128;
    const long long lim = (m.cell1 < 0 ? m.ncells : m.cell1);
    if (pc0 + C <= lim && tid < 2 * LINES) {
      const double* src = (tid < LINES ? x : w) + pc0 * 3 * NB + (size_t)(tid % LINES) * 16;
      asm volatile("prefetch.global.L2 [%0];" ::"l"(src));
    }
  }
  if constexpr (WPC && DGB_WPC_S0) {
    // one warp stages its own cell: the six neighbours once per warp, element / item
    // indices from the lane and compile-time loop counters (the CTA-wide loops of the
    // generic staging spend most of their instructions on index divisions)
    const int c = wcell, cell = c0 + c;
    const bool live = c < nc;
    int nbf[6];
    cell_nbrs6<UNI>(m, ug, live ? cell : c0, nbf);
#ifndef DGB_MOM_S0V2
#define DGB_MOM_S0V2 1
#endif
    constexpr bool S0V2 = DGB_MOM_S0V2 && N == 4;
    if (S0V2 && live) {
      // N = 4: element e = lane + 32 k is node (lane & 3, (lane >> 2) & 3, (lane >> 4) + 2 (k & 1)) of
      // component k >> 1: one lane-dependent base, compile-time offsets per k
      const int lb = (lane & 3) + P::PX * ((lane >> 2) & 3) + P::PY * (lane >> 4);
      const unsigned sx = static_cast<unsigned>(__cvta_generic_to_shared(CELL(c) + G::O_X + lb));
      const double* xs = x + (size_t)cell * 3 * NB + lane;
      const double* ws = w + (size_t)cell * 3 * NB + lane;
#pragma unroll
      for (int k = 0; k < 6; ++k) {
        const unsigned off = ((k >> 1) * CT + 2 * P::PY * (k & 1)) * 8u;
        asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sx + off), "l"(xs + 32 * k) : "memory");
        if (MODE != 1)
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;\n" ::"r"(sx + (G::O_W - G::O_X) * 8u + off),
                       "l"(ws + 32 * k)
                       : "memory");
      }
    } else if (live) {
      const double* xs = x + (size_t)cell * 3 * NB;
      const double* ws = w + (size_t)cell * 3 * NB;
#pragma unroll
      for (int k = 0; k < (3 * NB + 31) / 32; ++k) {
        const int e = lane + 32 * k;
        if (e < 3 * NB) {
          const int comp = e / NB, i = e - comp * NB;
          const int pi = comp * CT + P::idx(i % N, (i / N) % N, i / NF);
          cp_async8(CELL(c) + G::O_X + pi, xs + e);
          if (MODE != 1) cp_async8(CELL(c) + G::O_W + pi, ws + e);
        }
      }
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int nl = nbf[2 * d], nr = nbf[2 * d + 1];
#ifndef DGB_NB_GLOBAL
#define DGB_NB_GLOBAL 1
#endif
      const bool extL = nl >= 0 && (DGB_NB_GLOBAL || nl < c0 || nl >= c0 + nc);
      const bool extR = nr >= 0 && (DGB_NB_GLOBAL || nr < c0 || nr >= c0 + nc);
      const int gst = d == 0 ? 1 : (d == 1 ? N : NF);
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        const int r = lane + 32 * j;
#pragma unroll
        for (int l = 0; l < N; ++l) nbL[d][j][l] = nbR[d][j][l] = 0.0;
        if (passA && live && r < NID) {
          int comp, tl;
          if (S0V2) {  // NF = 16: r = lane + 32 j -> component 2 j + (lane >> 4), line lane & 15
            comp = 2 * j + (lane >> 4);
            tl = lane & 15;
          } else {
            line_item<K, NF>(r, d, comp, tl);
          }
          const int p = tl % N, q = tl / N;
          const int g0 = comp * NB + (d == 0 ? N * (p + N * q) : (d == 1 ? p + NF * q : p + N * q));
#pragma unroll
          for (int l = 0; l < N; ++l) {
            if (extL) nbL[d][j][l] = __ldg(x + (size_t)nl * 3 * NB + g0 + l * gst);
            if (extR) nbR[d][j][l] = __ldg(x + (size_t)nr * 3 * NB + g0 + l * gst);
          }
        }
      }
    }
    if (faces && live) {  // neighbour w_a traces on each face (async; zeros on boundary faces)
#pragma unroll
      for (int k = 0; k < (6 * NF + 31) / 32; ++k) {
        const int r = lane + 32 * k;
        if (r < 6 * NF) {
          const int f = r / NF, t = r - f * NF;
          const int a = f >> 1, p = t % N, q = t / N;
          int nb = nbf[0];
#pragma unroll
          for (int ff = 1; ff < 6; ++ff) nb = f == ff ? nbf[ff] : nb;
          const int gst = a == 0 ? 1 : (a == 1 ? N : NF);
          const int go = (a == 0 ? N * (p + N * q) : (a == 1 ? p + NF * q : p + N * q)) + ((f & 1) ? 0 : N - 1) * gst;
          double* dst = WK(c) + G::F_NB + f * G::NBS + 3 * NF + t;
          if (nb >= 0)
            cp_async8(dst, w + (size_t)nb * 3 * NB + a * NB + go);
          else
            *dst = 0.0;
        }
      }
    }
  } else {
    for (int idx = tid; idx < nc * 3 * NB; idx += TT) {
      const int c = idx / (3 * NB), r = idx - c * 3 * NB;
      const int comp = r / NB, i = r - comp * NB;
      const int pi = comp * CT + P::idx(i % N, (i / N) % N, i / NF);
      cp_async8(CELL(c) + G::O_X + pi, x + (size_t)(c0 + c) * 3 * NB + r);
      if (MODE != 1) cp_async8(CELL(c) + G::O_W + pi, w + (size_t)(c0 + c) * 3 * NB + r);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
#pragma unroll
      for (int j = 0; j < MAXJ; ++j) {
        const int it = it0 + j * IST;
#pragma unroll
        for (int l = 0; l < N; ++l) nbL[d][j][l] = nbR[d][j][l] = 0.0;
        if (passA && it < ITEMS(NID)) {
          const int c = CELLOF(it, NID), r = RESTOF(it, c, NID);
          int comp, tl;
          line_item<K, NF>(r, d, comp, tl);
          const int p = tl % N, q = tl / N;
          const int nl = cell_nbr<UNI>(m, ug, c0 + c, 2 * d), nr = cell_nbr<UNI>(m, ug, c0 + c, 2 * d + 1);
          const int gst = d == 0 ? 1 : (d == 1 ? N : NF);
          const int g0 = comp * NB + (d == 0 ? N * (p + N * q) : (d == 1 ? p + NF * q : p + N * q));
          const bool extL = nl >= 0 && (nl < c0 || nl >= c0 + nc);
          const bool extR = nr >= 0 && (nr < c0 || nr >= c0 + nc);
#pragma unroll
          for (int l = 0; l < N; ++l) {
            if (extL) nbL[d][j][l] = __ldg(x + (size_t)nl * 3 * NB + g0 + l * gst);
            if (extR) nbR[d][j][l] = __ldg(x + (size_t)nr * 3 * NB + g0 + l * gst);
          }
        }
      }
    if (faces) {  // neighbour w_a traces on each face (async; zeros on boundary faces)
      for (int idx = tid; idx < nc * 6 * NF; idx += TT) {
        const int c = idx / (6 * NF), r = idx - c * 6 * NF;
        const int f = r / NF, t = r - f * NF;
        const int a = f >> 1, p = t % N, q = t / N;
        const int nb = cell_nbr<UNI>(m, ug, c0 + c, f);
        const int gst = a == 0 ? 1 : (a == 1 ? N : NF);
        const int go = (a == 0 ? N * (p + N * q) : (a == 1 ? p + NF * q : p + N * q)) + ((f & 1) ? 0 : N - 1) * gst;
        double* dst = WK(c) + G::F_NB + f * G::NBS + 3 * NF + t;
        if (nb >= 0)
          cp_async8(dst, w + (size_t)nb * 3 * NB + a * NB + go);
        else
          *dst = 0.0;
      }
    }
  }
  load_info_par<TT, UNI>(sm, PER, G::O_INFO, nc, m, ug, aff, c0, sfac);
  cp_async_wait_all();
  __syncthreads();
  for (int idx = it0; idx < ITEMS(6); idx += IST) {
    const int c = CELLOF(idx, 6);
    face_coefs(INFO(c), RESTOF(idx, c, 6), true, true, RHS);
  }
  SYNC_CELL();

  // ------------------------------------------------------------------ pass A: mass + viscous (line split)
  if (passA) {
  // A: lines of every direction: S_d (visc) on raw lines (+ neighbour lines), UX = M_x u
  auto stage_a = [&](auto dtag) {
    constexpr int d = decltype(dtag)::value;
    constexpr int st = d == 0 ? 1 : (d == 1 ? P::PX : P::PY);
    double* sdst = WK(0) + (d == 0 ? G::A_SX : (d == 1 ? G::A_SY : G::A_SZ));
#ifndef DGB_MOM_FCREG
#define DGB_MOM_FCREG 1
#endif
    // one warp per cell: the cell's line-operator coefficients are the same for every item of
    // the warp; read them once per direction (the stores of the item loop keep the compiler
    // from hoisting the shared-memory loads itself)
    CellInfo cir;
    if constexpr (WPC && DGB_MOM_FCREG && K == 3) {  // (K = 2: 3.36 vs 3.31 ms at cfg5, off)
      const CellInfo& c0i = INFO(wcell);
      cir.ih[d] = c0i.ih[d];
      cir.A[d] = c0i.A[d];
      cir.nb[2 * d] = c0i.nb[2 * d];
      cir.nb[2 * d + 1] = c0i.nb[2 * d + 1];
#pragma unroll
      for (int e = 0; e < 6; ++e) {
        cir.fc[2 * d][e] = c0i.fc[2 * d][e];
        cir.fc[2 * d + 1][e] = c0i.fc[2 * d + 1][e];
      }
    }
#pragma unroll
    for (int j = 0; j < MAXJ; ++j) {
      const int it = it0 + j * IST;
      if (it < ITEMS(NID)) {
        const int c = CELLOF(it, NID), r = RESTOF(it, c, NID);
        int comp, tl;
        line_item<K, NF>(r, d, comp, tl);
        const int p = tl % N, q = tl / N;
        const CellInfo& ci = (WPC && DGB_MOM_FCREG && K == 3) ? cir : INFO(c);
        const int b0 = comp * CT + (d == 0 ? P::idx(0, p, q) : (d == 1 ? P::idx(p, 0, q) : P::idx(p, q, 0)));
        double u[N], o[N], uL[N], uR[N];
        const double* us = CELL(c) + G::O_X + b0;
#pragma unroll
        for (int l = 0; l < N; ++l) u[l] = us[l * st];
        const int nl = ci.nb[2 * d], nr = ci.nb[2 * d + 1];
        const bool inL = !(WPC && DGB_WPC_S0 && DGB_NB_GLOBAL) && nl >= c0 && nl < c0 + nc;
        const bool inR = !(WPC && DGB_WPC_S0 && DGB_NB_GLOBAL) && nr >= c0 && nr < c0 + nc;
#pragma unroll
        for (int l = 0; l < N; ++l) {
          uL[l] = inL ? CELL(nl - c0)[G::O_X + b0 + l * st] : nbL[d][j][l];
          uR[l] = inR ? CELL(nr - c0)[G::O_X + b0 + l * st] : nbR[d][j][l];
        }
        if (faces) {  // neighbour x traces for the advective faces (F1)
          WK(c)[G::F_NB + (2 * d) * G::NBS + comp * NF + tl] = uL[N - 1];
          WK(c)[G::F_NB + (2 * d + 1) * G::NBS + comp * NF + tl] = uR[0];
        }
        sip_line_bf<N, d>(ta, ci, u, uL, uR, co.visc, o);
        double* so = sdst + c * PER + b0;
#pragma unroll
        for (int l = 0; l < N; ++l) so[l * st] = o[l];
        if (d == 0) {
#pragma unroll
          for (int i = 0; i < N; ++i) {
            double sacc = 0.0;
#pragma unroll
            for (int l = 0; l < N; ++l) sacc = fma(ta.M[i][l], u[l], sacc);
            WK(c)[G::A_UX + b0 + i] = sacc;
          }
        }
      }
    }
  };
  stage_a(std::integral_constant<int, 0>{});
  stage_a(std::integral_constant<int, 1>{});
  stage_a(std::integral_constant<int, 2>{});
  SYNC_CELL();
  // B, C, D work on independent output lines.  SPL = 2 splits each (comp, line) item in
  // two (the two fields of B / C, halves of the z-outputs of D) so 96 items fill three
  // full warp rounds instead of 48 filling two; measured slower at K = 3 (more shared
  // loads per FMA: 1.92 vs 1.81 ms), so it stays 1.
  constexpr int SPL = 1;
  // B: x-lines in place: SY <- M_x SY, SZ <- M_x SZ
  for (int idx = it0; idx < ITEMS(3 * NF * SPL); idx += IST) {
    const int c = CELLOF(idx, 3 * NF * SPL), r0 = RESTOF(idx, c, 3 * NF * SPL);
    const int r = r0 / SPL, part = r0 - r * SPL;
    const int comp = r / NF, tl = r - comp * NF;
    const int b0 = comp * CT + P::idx(0, tl % N, tl / N);
#pragma unroll
    for (int h = 0; h < 3 - SPL; ++h) {
      double* ln = WK(c) + ((SPL == 2 ? part : h) ? G::A_SZ : G::A_SY) + b0;
      double a[N];
#pragma unroll
      for (int l = 0; l < N; ++l) a[l] = ln[l];
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double sacc = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) sacc = fma(ta.M[i][l], a[l], sacc);
        ln[i] = sacc;
      }
    }
  }
  SYNC_CELL();
  // C: y-lines: SX <- M_y (SX + mass detJ UX) + SY ; SZ <- M_y SZ
  for (int idx = it0; idx < ITEMS(3 * NF * SPL); idx += IST) {
    const int c = CELLOF(idx, 3 * NF * SPL), r0 = RESTOF(idx, c, 3 * NF * SPL);
    const int r = r0 / SPL, part = r0 - r * SPL;
    int comp, tl;
    line_item<K, NF>(r, 1, comp, tl);
    const int b0 = comp * CT + P::idx(tl % N, 0, tl / N);
#pragma unroll
    for (int h = 0; h < 3 - SPL; ++h) {
      const bool zpart = SPL == 2 ? part != 0 : h != 0;
      double a[N], e[N];
      if (!zpart) {
        const double cm = co.mass * INFO(c).detJ;
#pragma unroll
        for (int l = 0; l < N; ++l) {
          a[l] = fma(cm, WK(c)[G::A_UX + b0 + l * P::PX], WK(c)[G::A_SX + b0 + l * P::PX]);
          e[l] = WK(c)[G::A_SY + b0 + l * P::PX];
        }
      } else {
#pragma unroll
        for (int l = 0; l < N; ++l) {
          a[l] = WK(c)[G::A_SZ + b0 + l * P::PX];
          e[l] = 0.0;
        }
      }
      double* dst = WK(c) + (zpart ? G::A_SZ : G::A_SX) + b0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double sacc = e[j];
#pragma unroll
        for (int l = 0; l < N; ++l) sacc = fma(ta.M[j][l], a[l], sacc);
        dst[j * P::PX] = sacc;
      }
    }
  }
  SYNC_CELL();
  // D: z-lines: OUT = M_z SX + SZ
  constexpr int NK = (N + SPL - 1) / SPL;
  for (int idx = it0; idx < ITEMS(3 * NF * SPL); idx += IST) {
    const int c = CELLOF(idx, 3 * NF * SPL), r0 = RESTOF(idx, c, 3 * NF * SPL);
    const int r = r0 / SPL, k0 = (r0 - r * SPL) * NK;
    int comp, tl;
    line_item<K, NF>(r, 2, comp, tl);
    const int b0 = comp * CT + P::idx(tl % N, tl / N, 0);
    double a[N];
#pragma unroll
    for (int l = 0; l < N; ++l) a[l] = WK(c)[G::A_SX + b0 + l * P::PY];
#pragma unroll
    for (int kk = 0; kk < NK; ++kk) {
      const int k = k0 + kk;
      if (k < N) {
        double sacc = WK(c)[G::A_SZ + b0 + k * P::PY];
#pragma unroll
        for (int l = 0; l < N; ++l) sacc = fma(ta.M[k][l], a[l], sacc);
        CELL(c)[G::O_OUT + b0 + k * P::PY] = sacc;
      }
    }
  }
  SYNC_CELL();

  } else {
    for (int idx = it0; idx < ITEMS(3 * CT); idx += IST) {
      const int c = CELLOF(idx, 3 * CT);
      CELL(c)[G::O_OUT + RESTOF(idx, c, 3 * CT)] = 0.0;
    }
    if (faces) {
      for (int idx = it0; idx < ITEMS(18 * NF); idx += IST) {
        const int c = CELLOF(idx, 18 * NF), r = RESTOF(idx, c, 18 * NF);
        const int f = r / (3 * NF), r2 = r - f * 3 * NF;
        const int comp = r2 / NF, t = r2 - comp * NF;
        const int a = f >> 1, p = t % N, q = t / N;
        const int nb = INFO(c).nb[f];
        const int gst = a == 0 ? 1 : (a == 1 ? N : NF);
        const int go = (a == 0 ? N * (p + N * q) : (a == 1 ? p + NF * q : p + N * q)) + ((f & 1) ? 0 : N - 1) * gst;
        WK(c)[G::F_NB + f * G::NBS + comp * NF + t] = nb >= 0 ? __ldg(x + (size_t)nb * 3 * NB + comp * NB + go) : 0.0;
      }
    }
    SYNC_CELL();
  }

  // ------------------------------------------------------------------ LF advective faces, all 6 at once
  if (faces) {
    // F1: traces of u (3 comps, own + neighbour) and w_a (own + neighbour) on face-node line q,
    //     contracted along p with B:  V1[field][f][qp + Q q]
    for (int idx = it0; idx < ITEMS(6 * N); idx += IST) {
      const int c = CELLOF(idx, 6 * N), r = RESTOF(idx, c, 6 * N);
      const int f = r / N, q = r - f * N;
      const int a = f >> 1, s = f & 1;
      const int Ls = s ? N - 1 : 0;
      double v[8][N];
      const double* nbt = WK(c) + G::F_NB + f * G::NBS + N * q;
#pragma unroll
      for (int p = 0; p < N; ++p) {
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) v[3 + comp][p] = nbt[comp * NF + p];
        v[7][p] = nbt[3 * NF + p];
      }
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const int li = a == 0 ? P::idx(Ls, p, q) : (a == 1 ? P::idx(p, Ls, q) : P::idx(p, q, Ls));
#pragma unroll
        for (int comp = 0; comp < 3; ++comp) v[comp][p] = CELL(c)[G::O_X + comp * CT + li];
        v[6][p] = CELL(c)[G::O_W + a * CT + li];
      }
      double* o = WK(c) + G::F_V1 + q * G::VB + f * G::V1F;
#pragma unroll
      for (int fl = 0; fl < 8; ++fl)
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(tq.B[qp][l], v[fl][l], acc);
          o[fl * N * G::VB + qp] = acc;
        }
    }
    SYNC_CELL();
    // F2: along q: values at the face Gauss points, LF flux, B^T back along q -> FL [comp][f][qp + Q l]
    for (int idx = it0; idx < ITEMS(6 * Q); idx += IST) {
      const int c = CELLOF(idx, 6 * Q), r = RESTOF(idx, c, 6 * Q);
      const int f = r / Q, qp = r - f * Q;
      const int a = f >> 1, s = f & 1;
      const CellInfo& ci = INFO(c);
      const double* in = WK(c) + G::F_V1 + f * G::V1F + qp;
      double v[8][N];
#pragma unroll
      for (int fl = 0; fl < 8; ++fl)
#pragma unroll
        for (int l = 0; l < N; ++l) v[fl][l] = in[fl * N * G::VB + l * G::VB];
      const double sgn = s ? 1.0 : -1.0;
      const double wbase = co.adv * ci.A[a] * tq.w[qp];
      const int ty = ci.type[f];
      double out[3][N];
#pragma unroll
      for (int comp = 0; comp < 3; ++comp)
#pragma unroll
        for (int l = 0; l < N; ++l) out[comp][l] = 0.0;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        double val[8];
#pragma unroll
        for (int fl = 0; fl < 8; ++fl) {
          double acc = 0.0;
#pragma unroll
          for (int l = 0; l < N; ++l) acc = fma(tq.B[qq][l], v[fl][l], acc);
          val[fl] = acc;
        }
        // hanging slot (mesh-table variant only: uniform grids have none; the select costs the
        // K = 2 uniform kernel 1.8 % at cfg5): zero surface weight
        const double wq = (!UNI && ty == 3) ? 0.0 : wbase * tq.w[qq];
        const double wns = sgn * val[6];
        double fl3[3];
        if (ty == 0) {  // forms.cpp:555-573
          const double wno = sgn * val[7];
          const double lam = RHS ? 0.0 : fmax(fabs(wns), fabs(wno));
#pragma unroll
          for (int comp = 0; comp < 3; ++comp)
            fl3[comp] = wq * (0.5 * (val[comp] * wns + val[3 + comp] * wno) + 0.5 * lam * (val[comp] - val[3 + comp]));
        } else {  // forms.cpp:592-599
          const double cf = (RHS || ty == 2) ? wns : fabs(wns);  // rhs: forms.cpp:1036-1048
#pragma unroll
          for (int comp = 0; comp < 3; ++comp) fl3[comp] = wq * cf * val[comp];
        }
#pragma unroll
        for (int comp = 0; comp < 3; ++comp)
#pragma unroll
          for (int l = 0; l < N; ++l) out[comp][l] = fma(tq.B[qq][l], fl3[comp], out[comp][l]);
      }
      double* o = WK(c) + G::F_FL + f * QN + qp;
#pragma unroll
      for (int comp = 0; comp < 3; ++comp)
#pragma unroll
        for (int l = 0; l < N; ++l) o[comp * G::FLC + Q * l] = out[comp][l];
    }
    SYNC_CELL();
    // F3: B^T along p, added straight into OUT at the face nodes; one axis at a time so
    //     edge / corner nodes shared by faces of different axes are never updated concurrently
#pragma unroll 1
    for (int a = 0; a < 3; ++a) {
      for (int idx = it0; idx < ITEMS(6 * N); idx += IST) {
        const int c = CELLOF(idx, 6 * N), r = RESTOF(idx, c, 6 * N);
        const int cs = r / N, q = r - cs * N;  // cs = comp * 2 + side
        const int comp = cs >> 1, f = 2 * a + (cs & 1);
        const double* in = WK(c) + G::F_FL + comp * G::FLC + f * QN + Q * q;
        double v[Q];
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) v[qp] = in[qp];
        const int L = (f & 1) ? N - 1 : 0;
        double* o = CELL(c) + G::O_OUT + comp * CT;
#pragma unroll
        for (int p = 0; p < N; ++p) {
          double acc = 0.0;
#pragma unroll
          for (int qp = 0; qp < Q; ++qp) acc = fma(tq.B[qp][p], v[qp], acc);
          o[a == 0 ? P::idx(L, p, q) : (a == 1 ? P::idx(p, L, q) : P::idx(p, q, L))] += acc;
        }
      }
      SYNC_CELL();
    }
  }

  // ------------------------------------------------------------------ pass B cell (advection, rule k+2)
  if (faces) {
  // S45: xy-planes of the 6 fields (u0..2, w0..2) at z-layer k: B along x then y, in
  //      registers  -> YB[f][k][qy][qx]
  for (int idx = it0; idx < ITEMS(6 * N); idx += IST) {
    const int c = CELLOF(idx, 6 * N), r = RESTOF(idx, c, 6 * N);
    const int f = r / N, k = r - f * N;
    const double* in = CELL(c) + (f < 3 ? G::O_X + f * CT : G::O_W + (f - 3) * CT) + P::idx(0, 0, k);
    double pl[N][N];  // [j][i]
#pragma unroll
    for (int j = 0; j < N; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) pl[j][i] = in[i + P::PX * j];
    double px[Q][N];  // [qx][j]
#pragma unroll
    for (int qx = 0; qx < Q; ++qx)
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double sacc = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) sacc = fma(tq.B[qx][i], pl[j][i], sacc);
        px[qx][j] = sacc;
      }
    double* o = WK(c) + G::B_R2 + (f * N + k) * G::QQP;
#pragma unroll
    for (int qy = 0; qy < Q; ++qy)
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        double sacc = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) sacc = fma(tq.B[qy][j], px[qx][j], sacc);
        o[qx + Q * qy] = sacc;
      }
  }
  SYNC_CELL();
  // S6: fused z: evaluate 6 columns, pointwise advective flux, z-integration of the 3x3 gradient tests
  for (int idx = it0; idx < ITEMS(QQ); idx += IST) {
    const int c = CELLOF(idx, QQ), qxy = RESTOF(idx, c, QQ);
    const CellInfo& ci = INFO(c);
    const double wxy = ci.detJ * tq.w[qxy % Q] * tq.w[qxy / Q];
    double col[6][Q];
#pragma unroll
    for (int f = 0; f < 6; ++f) {
      double v[N];
#pragma unroll
      for (int l = 0; l < N; ++l) v[l] = WK(c)[G::B_R2 + (f * N + l) * G::QQP + qxy];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        double s = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) s = fma(tq.B[qz][l], v[l], s);
        col[f][qz] = s;
      }
    }
    const double ih0 = -co.adv * ci.ih[0], ih1 = -co.adv * ci.ih[1], ih2 = -co.adv * ci.ih[2];
    // weighted advecting-field factors, shared by the three components
    double fx[Q], fy[Q], fz[Q];
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      const double wq = wxy * tq.w[qz];
      fx[qz] = col[3][qz] * (wq * ih0);
      fy[qz] = col[4][qz] * (wq * ih1);
      fz[qz] = col[5][qz] * (wq * ih2);
    }
#pragma unroll
    for (int comp = 0; comp < 3; ++comp) {
      double tz[N], ty[N], tx[N];
#pragma unroll
      for (int l = 0; l < N; ++l) tz[l] = ty[l] = tx[l] = 0.0;
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        const double uj = col[comp][qz];
        const double rx = uj * fx[qz];
        const double ry = uj * fy[qz];
        const double rz = uj * fz[qz];
#pragma unroll
        for (int l = 0; l < N; ++l) {
          tz[l] = fma(tq.D[qz][l], rz, tz[l]);
          ty[l] = fma(tq.B[qz][l], ry, ty[l]);
          tx[l] = fma(tq.B[qz][l], rx, tx[l]);
        }
      }
      double* o = WK(c) + G::B_R1 + comp * G::BRC + qxy;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        o[G::QQP * l] = tz[l];
        o[G::QQP * (N + l)] = ty[l];
        o[G::QQP * (2 * N + l)] = tx[l];
      }
    }
  }
  SYNC_CELL();
  // S78: per (component, z-layer l): y- then x-integration of the three gradient tests,
  //      qx by qx in registers, accumulated into OUT
  // (K = 3: items split over halves of the output y-rows so a warp-cell keeps more lanes
  // busy; K = 2: unsplit, measured 3% faster at cfg5.  DGB_MOM_JH overrides for tuning)
#ifdef DGB_MOM_JH
  constexpr int JH = WPC ? DGB_MOM_JH : 1, NJ = (N + JH - 1) / JH;
#else
  constexpr int JH = WPC && K != 2 ? 2 : 1, NJ = (N + JH - 1) / JH;
#endif
  for (int idx = it0; idx < ITEMS(3 * N * JH); idx += IST) {
    const int c = CELLOF(idx, 3 * N * JH), r = RESTOF(idx, c, 3 * N * JH);
    const int comp = r / (N * JH), r2 = r - comp * N * JH;
    const int l = r2 / JH, j0 = (r2 - l * JH) * NJ;
    const double* tp = WK(c) + G::B_R1 + comp * G::BRC + G::QQP * l;
    double acc[NJ][N];  // [j - j0][i]
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int i = 0; i < N; ++i) acc[j][i] = 0.0;
#ifndef DGB_S78_HOIST
#define DGB_S78_HOIST 0
#endif
#if DGB_S78_HOIST == 1
    // the y-test columns of this item's output rows, loaded once (j0 is a runtime index:
    // reading tq.B[qy][j] inside the qx loop re-issued a constant load per use)
    double By[NJ][Q], Dy[NJ][Q];
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        const bool ok = j0 + jj < N;
        By[jj][qy] = ok ? tq.B[qy][j0 + jj] : 0.0;
        Dy[jj][qy] = ok ? tq.D[qy][j0 + jj] : 0.0;
      }
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double vz[Q], vy[Q], vx[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        vz[qy] = tp[qx + Q * qy];
        vy[qy] = tp[G::QQP * N + qx + Q * qy];
        vx[qy] = tp[2 * G::QQP * N + qx + Q * qy];
      }
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        // three independent chains (B vz, D vy, B vx) instead of one of length 2Q
        double sa = 0.0, sd = 0.0, sb = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) {
          sa = fma(By[jj][qy], vz[qy], sa);
          sd = fma(Dy[jj][qy], vy[qy], sd);
          sb = fma(By[jj][qy], vx[qy], sb);
        }
        sa += sd;
#pragma unroll
        for (int i = 0; i < N; ++i) acc[jj][i] = fma(tq.B[qx][i], sa, fma(tq.D[qx][i], sb, acc[jj][i]));
      }
    }
#elif DGB_S78_HOIST == 2
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double vz[Q], vy[Q], vx[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        vz[qy] = tp[qx + Q * qy];
        vy[qy] = tp[G::QQP * N + qx + Q * qy];
        vx[qy] = tp[2 * G::QQP * N + qx + Q * qy];
      }
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        const int j = j0 + jj;
        if (j < N) {
          double sa = 0.0, sd = 0.0, sb = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) {
            sa = fma(tq.B[qy][j], vz[qy], sa);
            sd = fma(tq.D[qy][j], vy[qy], sd);
            sb = fma(tq.B[qy][j], vx[qy], sb);
          }
          sa += sd;
#pragma unroll
          for (int i = 0; i < N; ++i) acc[jj][i] = fma(tq.B[qx][i], sa, fma(tq.D[qx][i], sb, acc[jj][i]));
        }
      }
    }
#else
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double vz[Q], vy[Q], vx[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        vz[qy] = tp[qx + Q * qy];
        vy[qy] = tp[G::QQP * N + qx + Q * qy];
        vx[qy] = tp[2 * G::QQP * N + qx + Q * qy];
      }
#pragma unroll
      for (int jj = 0; jj < NJ; ++jj) {
        const int j = j0 + jj;
        if (j < N) {
          double sa = 0.0, sb = 0.0;
#pragma unroll
          for (int qy = 0; qy < Q; ++qy) {
            sa = fma(tq.B[qy][j], vz[qy], sa);
            sa = fma(tq.D[qy][j], vy[qy], sa);
            sb = fma(tq.B[qy][j], vx[qy], sb);
          }
#pragma unroll
          for (int i = 0; i < N; ++i) acc[jj][i] = fma(tq.B[qx][i], sa, fma(tq.D[qx][i], sb, acc[jj][i]));
        }
      }
    }
#endif
    double* o = CELL(c) + G::O_OUT + comp * CT + P::idx(0, 0, l);
#pragma unroll
    for (int jj = 0; jj < NJ; ++jj)
#pragma unroll
      for (int i = 0; i < N; ++i)
        if (j0 + jj < N) o[i + P::PX * (j0 + jj)] += acc[jj][i];
  }
  SYNC_CELL();
  }

  // ------------------------------------------------------------------ store
  for (int idx = it0; idx < ITEMS(3 * NB); idx += IST) {
    const int c = CELLOF(idx, 3 * NB), r = RESTOF(idx, c, 3 * NB);
    const int comp = r / NB, i = r - comp * NB;
    const int ii[3] = {i % N, (i / N) % N, i / NF};
    double v = CELL(c)[G::O_OUT + comp * CT + P::idx(ii[0], ii[1], ii[2])];
    if (MODE == 2 || acc) v += y[(size_t)(c0 + c) * 3 * NB + r];
    y[(size_t)(c0 + c) * 3 * NB + r] = v;
  }
#undef CELL
#undef WK
#undef INFO
#undef ITEMS
#undef CELLOF
#undef RESTOF
#undef SYNC_CELL
}

// ===========================================================================
// Weak pressure gradient of momentum_rhs (forms.cpp:850-855 cell, :895-912
// interior faces, :940-948 boundary faces), axis-aligned affine, 3D:
//   y_d += (G_d (x) Mvp (x) Mvp) p,
// G_d = 1D line operator along d (velocity test derivative x pressure value,
// exact for the k+1 rule) plus the {p} n_d v face terms at the two line ends;
// Mvp = mixed velocity/pressure 1D mass.  p already carries the coefficient.
// ===========================================================================
template <int K>
struct PTab {
  double Mvp[K + 1][K];  // sum_q w phi_i psi_j
  double G1[K + 1][K];   // sum_q w phi_i' psi_j
  double Dpv[K][K + 1];  // sum_q w psi_i' phi_j (divergence: pressure-test derivative x velocity)
};
template <int K>
__constant__ PTab<K> c_pt;

template <int K>
struct PGradCfg {
  static constexpr int N = K + 1, NP = K, NBP = NP * NP * NP, NB = N * N * N;
  static constexpr int C = 8, T = 128;
  static constexpr int L1 = 3 * N * NP * NP, L2 = 3 * N * N * NP;
  static constexpr int PER = (NBP + L1 + L2 + kInfoDoubles) | 1;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int K, bool UNI>
__global__ void __launch_bounds__(PGradCfg<K>::T) k_pgrad_axis(MeshArgs m, UniformGrid ug, const double* __restrict__ aff,
                                                               const double* __restrict__ p, double* __restrict__ y) {
  using G = PGradCfg<K>;
  constexpr int N = G::N, NP = G::NP, NBP = G::NBP, NB = G::NB, C = G::C, PER = G::PER, TT = G::T;
  const PTab<K>& pt = c_pt<K>;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x;
#define CELL(c) (sm + (c) * PER)
#define INFO(c) (*reinterpret_cast<const CellInfo*>(sm + (c) * PER + NBP + G::L1 + G::L2))
  for (int idx = tid; idx < nc * NBP; idx += TT) CELL(idx / NBP)[idx % NBP] = p[(size_t)c0 * NBP + idx];
  load_info_par<TT, UNI>(sm, PER, NBP + G::L1 + G::L2, nc, m, ug, aff, c0, 1.0);
  __syncthreads();
  // S1: line operator along d on the raw pressure lines (tangential (a, b), t1 < t2)
  for (int idx = tid; idx < nc * 3 * NP * NP; idx += TT) {
    const int c = idx / (3 * NP * NP), r = idx - c * 3 * NP * NP;
    const int d = r / (NP * NP), ab = r - d * NP * NP;
    const int a = ab % NP, b = ab / NP;
    const int st = d == 0 ? 1 : (d == 1 ? NP : NP * NP);
    const int b0 = d == 0 ? NP * a + NP * NP * b : (d == 1 ? a + NP * NP * b : a + NP * b);
    const CellInfo& ci = INFO(c);
    double pl[NP];
#pragma unroll
    for (int j = 0; j < NP; ++j) pl[j] = CELL(c)[b0 + j * st];
    const double cs = ci.detJ * ci.ih[d], A = ci.A[d];
    double o[N];
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < NP; ++j) acc = fma(pt.G1[i][j], pl[j], acc);
      o[i] = cs * acc;
    }
    // left face (n_d = -1): -{p} n_d -> +A pf at node 0; right face (n_d = +1): -A pf at node N-1
    {
      const int f = 2 * d, nb = ci.nb[f], ty = ci.type[f];
      const double own = pl[0];
      const double pf = ty == 0 ? 0.5 * (own + __ldg(p + (size_t)nb * NBP + b0 + (NP - 1) * st)) : (ty == 1 ? own : 0.0);
      o[0] = fma(A, pf, o[0]);
    }
    {
      const int f = 2 * d + 1, nb = ci.nb[f], ty = ci.type[f];
      const double own = pl[NP - 1];
      const double pf = ty == 0 ? 0.5 * (own + __ldg(p + (size_t)nb * NBP + b0)) : (ty == 1 ? own : 0.0);
      o[N - 1] = fma(-A, pf, o[N - 1]);
    }
    double* t1 = CELL(c) + NBP + d * N * NP * NP;
#pragma unroll
    for (int i = 0; i < N; ++i) t1[i + N * ab] = o[i];
  }
  __syncthreads();
  // S2: Mvp along t1:  t2[d][i + N (a' + N b)]
  for (int idx = tid; idx < nc * 3 * N * NP; idx += TT) {
    const int c = idx / (3 * N * NP), r = idx - c * 3 * N * NP;
    const int d = r / (N * NP), ib = r - d * N * NP;
    const int i = ib % N, b = ib / N;
    const double* t1 = CELL(c) + NBP + d * N * NP * NP;
    double v[NP];
#pragma unroll
    for (int a = 0; a < NP; ++a) v[a] = t1[i + N * (a + NP * b)];
    double* t2 = CELL(c) + NBP + G::L1 + d * N * N * NP;
#pragma unroll
    for (int a2 = 0; a2 < N; ++a2) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < NP; ++a) acc = fma(pt.Mvp[a2][a], v[a], acc);
      t2[i + N * (a2 + N * b)] = acc;
    }
  }
  __syncthreads();
  // S3: Mvp along t2, add into y
  for (int idx = tid; idx < nc * 3 * N * N; idx += TT) {
    const int c = idx / (3 * N * N), r = idx - c * 3 * N * N;
    const int d = r / (N * N), ia = r - d * N * N;
    const int i = ia % N, a2 = ia / N;
    const double* t2 = CELL(c) + NBP + G::L1 + d * N * N * NP;
    double v[NP];
#pragma unroll
    for (int b = 0; b < NP; ++b) v[b] = t2[i + N * (a2 + N * b)];
    double* yo = y + (size_t)(c0 + c) * 3 * NB + d * NB;
#pragma unroll
    for (int b2 = 0; b2 < N; ++b2) {
      double acc = 0.0;
#pragma unroll
      for (int b = 0; b < NP; ++b) acc = fma(pt.Mvp[b2][b], v[b], acc);
      const int node = d == 0 ? i + N * a2 + N * N * b2 : (d == 1 ? a2 + N * i + N * N * b2 : a2 + N * b2 + N * N * i);
      yo[node] += acc;
    }
  }
#undef CELL
#undef INFO
}

// ===========================================================================
// Exact diagonal of the momentum operator (momentum_diagonal, forms.cpp:606-810),
// axis-aligned affine, 3D, skew = 0.  One warp per cell.
//   mass + viscous: diag of sum_d (S_d (x) M (x) M) + mc detJ M (x) M (x) M, i.e. the 1D
//     line-operator diagonals (stiffness + the own-side face terms) times the mass
//     diagonals — exact, like the apply;
//   advection (k+2 rule): -adv detJ sum_d ih_d sum_q w_d(q) phi_b dphi_b/dxi_d, a
//     sum-factorised contraction of w_d at the Gauss points with w B^2 / w B D tables;
//   LF faces: adv sum_q (0.5 w.n + 0.5 lambda) phi_b^2 (|w.n| or w.n on boundaries) on
//     the face-layer nodes, w.n of both sides interpolated to the face Gauss points.
// The value is the same for the three components (forms.cpp:635).
// ===========================================================================
template <int K>
struct MomDiagCfg {
  static constexpr int N = K + 1, Q = K + 2, NB = N * N * N, NF = N * N, QN = Q * N, QQ = Q * Q;
  static constexpr int C = 4, T = 32 * C;
  // per cell: w (3 NB) | info | work: XW (3 Q N N), YW (3 Q Q N), WQ (3 Q^3), R (3 Q Q N / 3 Q N N), faces
  static constexpr int O_W = 0, O_INFO = 3 * NB;
  static constexpr int O_WK = O_INFO + kInfoDoubles;
  static constexpr int XW = 0, YW = XW + 3 * Q * NF, WQ = YW + 3 * QQ * N, R1 = WQ + 3 * QQ * Q,
                       R2 = R1 + 3 * QQ * N, R3 = R2 + 3 * Q * NF, FV = R3 + 3 * NB,
                       FG = FV + 6 * 2 * QN, FD = FG + 6 * QN, WEND = FD + 6 * NF;
  static constexpr int PER = (O_WK + WEND) | 1;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int K, bool UNI>
__global__ void __launch_bounds__(MomDiagCfg<K>::T) k_momentum_diag_axis(MeshArgs m, UniformGrid ug,
                                                                          const double* __restrict__ aff,
                                                                          MomCoef co, const double* __restrict__ w,
                                                                          double* __restrict__ y) {
  using G = MomDiagCfg<K>;
  constexpr int N = G::N, Q = G::Q, NB = G::NB, NF = G::NF, QN = G::QN, QQ = G::QQ, C = G::C, PER = G::PER;
  const FTab<N, Q>& tq = c_ft<N, Q>;
  const FTab<N, N>& ta = c_ft<N, N>;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const bool adv = co.adv != 0.0;
  double* cell = sm + wc * PER;
  double* wk = cell + G::O_WK;
  CellInfo& ci = *reinterpret_cast<CellInfo*>(cell + G::O_INFO);
  for (int idx = tid; idx < nc * 3 * NB; idx += G::T) {
    const int c = idx / (3 * NB), r = idx - c * 3 * NB;
    if (adv) cp_async8(sm + c * PER + G::O_W + r, w + (size_t)(c0 + c) * 3 * NB + r);
  }
  load_info_par<G::T, UNI>(sm, PER, G::O_INFO, nc, m, ug, aff, c0, (double)(N * N));
  cp_async_wait_all();
  __syncthreads();
  if (wc >= nc) return;
  const int cell_id = c0 + wc;
  if (lane < 6) face_coefs(ci, lane, true, true, false);
  __syncwarp();
  if (adv) {
    // w at the Gauss points: x, then y, then z (3 fields)
    for (int it = lane; it < 3 * NF; it += 32) {  // XW[f][qx][j][k]
      const int f = it / NF, jk = it - f * NF;
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = cell[G::O_W + f * NB + i + N * jk];
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        double a = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) a = fma(tq.B[qx][i], v[i], a);
        wk[G::XW + f * Q * NF + qx * NF + jk] = a;
      }
    }
    __syncwarp();
    for (int it = lane; it < 3 * Q * N; it += 32) {  // YW[f][qx][qy][k]
      const int f = it / (Q * N), r = it - f * Q * N, qx = r / N, k = r - qx * N;
      double v[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = wk[G::XW + f * Q * NF + qx * NF + j + N * k];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        double a = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) a = fma(tq.B[qy][j], v[j], a);
        wk[G::YW + f * QQ * N + (qx * Q + qy) * N + k] = a;
      }
    }
    __syncwarp();
    for (int it = lane; it < 3 * QQ; it += 32) {  // WQ[f][qx][qy][qz]
      const int f = it / QQ, r = it - f * QQ;
      double v[N];
#pragma unroll
      for (int k = 0; k < N; ++k) v[k] = wk[G::YW + f * QQ * N + r * N + k];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) {
        double a = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) a = fma(tq.B[qz][k], v[k], a);
        wk[G::WQ + f * QQ * Q + r * Q + qz] = a;
      }
    }
    __syncwarp();
    // T_d = sum_q w_d(q) prod_e tab_e[b_e][q_e], tab_d = w B D, tab_e = w B^2 (e != d)
    for (int it = lane; it < 3 * QQ; it += 32) {  // R1[d][qx][qy][bz]
      const int d = it / QQ, r = it - d * QQ;
      double v[Q];
#pragma unroll
      for (int qz = 0; qz < Q; ++qz) v[qz] = wk[G::WQ + d * QQ * Q + r * Q + qz];
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double a = 0.0;
#pragma unroll
        for (int qz = 0; qz < Q; ++qz)
          a = fma(tq.w[qz] * tq.B[qz][b] * (d == 2 ? tq.D[qz][b] : tq.B[qz][b]), v[qz], a);
        wk[G::R1 + d * QQ * N + r * N + b] = a;
      }
    }
    __syncwarp();
    for (int it = lane; it < 3 * Q * N; it += 32) {  // R2[d][qx][by][bz]
      const int d = it / (Q * N), r = it - d * Q * N, qx = r / N, bz = r - qx * N;
      double v[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) v[qy] = wk[G::R1 + d * QQ * N + (qx * Q + qy) * N + bz];
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double a = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy)
          a = fma(tq.w[qy] * tq.B[qy][b] * (d == 1 ? tq.D[qy][b] : tq.B[qy][b]), v[qy], a);
        wk[G::R2 + d * Q * NF + qx * NF + b * N + bz] = a;
      }
    }
    __syncwarp();
    for (int it = lane; it < 3 * NF; it += 32) {  // R3[d][bx][by][bz]
      const int d = it / NF, r = it - d * NF;  // r = by * N + bz
      double v[Q];
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) v[qx] = wk[G::R2 + d * Q * NF + qx * NF + r];
#pragma unroll
      for (int b = 0; b < N; ++b) {
        double a = 0.0;
#pragma unroll
        for (int qx = 0; qx < Q; ++qx)
          a = fma(tq.w[qx] * tq.B[qx][b] * (d == 0 ? tq.D[qx][b] : tq.B[qx][b]), v[qx], a);
        {
          const int by = r / N, bz = r - by * N;
          wk[G::R3 + d * NB + b + N * by + NF * bz] = a;
        }
      }
    }
    // LF face diagonals: w.n of both sides at the face Gauss points, then
    // adv * coef * (w B^2) (x) (w B^2) onto the face-layer nodes
    for (int it = lane; it < 6 * N; it += 32) {  // FV[f][side][q][qp]: B along p
      const int f = it / N, q = it - f * N, a = f >> 1, s = f & 1;
      const int Ls = s ? N - 1 : 0, Lo = s ? 0 : N - 1;
      const int nb = ci.nb[f];
      const int gst = a == 0 ? 1 : (a == 1 ? N : NF);
      double vs[N], vo[N];
#pragma unroll
      for (int p = 0; p < N; ++p) {
        const int base = a == 0 ? N * (p + N * q) : (a == 1 ? p + NF * q : p + N * q);
        vs[p] = cell[G::O_W + a * NB + base + Ls * gst];
        vo[p] = nb >= 0 ? __ldg(w + (size_t)nb * 3 * NB + a * NB + base + Lo * gst) : 0.0;
      }
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) {
        double as = 0.0, ao = 0.0;
#pragma unroll
        for (int p = 0; p < N; ++p) {
          as = fma(tq.B[qp][p], vs[p], as);
          ao = fma(tq.B[qp][p], vo[p], ao);
        }
        wk[G::FV + (f * 2 + 0) * QN + q * Q + qp] = as;
        wk[G::FV + (f * 2 + 1) * QN + q * Q + qp] = ao;
      }
    }
    __syncwarp();
    for (int it = lane; it < 6 * Q; it += 32) {  // FG[f][qp][q_]: B along q, coef, (w B^2) back along q
      const int f = it / Q, qp = it - f * Q, s = f & 1;
      const int ty = ci.type[f];
      const double sgn = s ? 1.0 : -1.0;
      double vs[N], vo[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        vs[q] = wk[G::FV + (f * 2 + 0) * QN + q * Q + qp];
        vo[q] = wk[G::FV + (f * 2 + 1) * QN + q * Q + qp];
      }
      double g[N];
#pragma unroll
      for (int b = 0; b < N; ++b) g[b] = 0.0;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        double ws = 0.0, wo = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          ws = fma(tq.B[qq][q], vs[q], ws);
          wo = fma(tq.B[qq][q], vo[q], wo);
        }
        const double wns = sgn * ws, wno = sgn * wo;
        const double cf = ty == 0 ? 0.5 * wns + 0.5 * fmax(fabs(wns), fabs(wno))
                                  : ((!UNI && ty == 3) ? 0.0 : (ty == 2 ? wns : fabs(wns)));  // 3: hanging slot
#pragma unroll
        for (int b = 0; b < N; ++b) g[b] = fma(tq.w[qq] * tq.B[qq][b] * tq.B[qq][b], cf, g[b]);
      }
#pragma unroll
      for (int b = 0; b < N; ++b) wk[G::FG + f * QN + qp * N + b] = g[b];
    }
    __syncwarp();
    for (int it = lane; it < 6 * N; it += 32) {  // FD[f][p_ + N q_]: (w B^2) along p
      const int f = it / N, bq = it - f * N;
      double v[Q];
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) v[qp] = wk[G::FG + f * QN + qp * N + bq];
      const double fa = co.adv * ci.A[f >> 1];
#pragma unroll
      for (int bp = 0; bp < N; ++bp) {
        double a = 0.0;
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) a = fma(tq.w[qp] * tq.B[qp][bp] * tq.B[qp][bp], v[qp], a);
        wk[G::FD + f * NF + bp + N * bq] = fa * a;
      }
    }
    __syncwarp();
  }
  // assemble: mass + viscous (line diagonals) + advection (cell + faces)
  const double cm = co.mass * ci.detJ;
  const double ca = -co.adv * ci.detJ;
  for (int b = lane; b < NB; b += 32) {
    const int bi[3] = {b % N, (b / N) % N, b / NF};
    double md[3], sd[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int i = bi[d];
      md[d] = ta.M[i][i];
      const double ih = ci.ih[d], sa = co.visc * ci.A[d], stiff = sa * ih;
      const double* cR = ci.fc[2 * d + 1];
      const double* cL = ci.fc[2 * d];
      double v = stiff * ta.K[i][i];
      if (i == N - 1) v += sa * (cR[0] * ta.dE[1][i] + cR[2]) + ta.dE[1][i] * stiff * cR[4];
      if (i == 0) v += sa * (cL[0] * ta.dE[0][i] + cL[2]) - ta.dE[0][i] * stiff * cL[4];
      sd[d] = v;
    }
    double v = sd[0] * md[1] * md[2] + md[0] * sd[1] * md[2] + md[0] * md[1] * sd[2] + cm * md[0] * md[1] * md[2];
    if (adv) {
      v += ca * (ci.ih[0] * wk[G::R3 + 0 * NB + b] + ci.ih[1] * wk[G::R3 + 1 * NB + b] +
                 ci.ih[2] * wk[G::R3 + 2 * NB + b]);
#pragma unroll
      for (int a = 0; a < 3; ++a) {
        const int t = (a == 0 ? bi[1] : bi[0]) + N * (a == 2 ? bi[1] : bi[2]);
        if (bi[a] == 0) v += wk[G::FD + (2 * a) * NF + t];
        if (bi[a] == N - 1) v += wk[G::FD + (2 * a + 1) * NF + t];
      }
    }
    double* yo = y + (size_t)cell_id * 3 * NB + b;
    yo[0] = v;
    yo[NB] = v;
    yo[2 * NB] = v;
  }
}

// ===========================================================================
// Divergence functional (divergence_functional, forms.cpp:1118-1197), axis-aligned
// affine, 3D:  y = sum_d (D_d (x) Mpv (x) Mpv) u_d,  D_d = 1D line operator along d
// (pressure-test derivative x velocity value, exact for the k+1 rule) plus the
// -{u_d} n_d q faces at the two line ends (own trace on non-outlet boundaries);
// Mpv = Mvp^T (pressure test x velocity value).
// ===========================================================================
template <int K>
struct DivCfg {
  static constexpr int N = K + 1, NP = K, NB = N * N * N, NBP = NP * NP * NP;
  static constexpr int C = 8, T = 128;
  static constexpr int L1 = 3 * NP * N * N, L2 = 3 * NP * NP * N;
  static constexpr int PER = (3 * NB + L1 + L2 + kInfoDoubles) | 1;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int K, bool UNI>
__global__ void __launch_bounds__(DivCfg<K>::T) k_div_axis(MeshArgs m, UniformGrid ug, const double* __restrict__ aff,
                                                           const double* __restrict__ u, double* __restrict__ y) {
  using G = DivCfg<K>;
  constexpr int N = G::N, NP = G::NP, NB = G::NB, NBP = G::NBP, C = G::C, PER = G::PER, TT = G::T;
  const PTab<K>& pt = c_pt<K>;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x;
#define CELL(c) (sm + (c) * PER)
#define INFO(c) (*reinterpret_cast<const CellInfo*>(sm + (c) * PER + 3 * NB + G::L1 + G::L2))
  for (int idx = tid; idx < nc * 3 * NB; idx += TT) cp_async8(CELL(idx / (3 * NB)) + idx % (3 * NB), u + (size_t)c0 * 3 * NB + idx);
  load_info_par<TT, UNI>(sm, PER, 3 * NB + G::L1 + G::L2, nc, m, ug, aff, c0, 1.0);
  cp_async_wait_all();
  __syncthreads();
  // S1: line operator along d on the u_d lines (tangential (a, b), t1 < t2) -> T1[d][i][a][b]
  for (int idx = tid; idx < nc * 3 * N * N; idx += TT) {
    const int c = idx / (3 * N * N), r = idx - c * 3 * N * N;
    const int d = r / (N * N), ab = r - d * N * N;
    const int a = ab % N, b = ab / N;
    const int st = d == 0 ? 1 : (d == 1 ? N : N * N);
    const int b0 = d * NB + (d == 0 ? N * a + N * N * b : (d == 1 ? a + N * N * b : a + N * b));
    const CellInfo& ci = INFO(c);
    double ul[N];
#pragma unroll
    for (int j = 0; j < N; ++j) ul[j] = CELL(c)[b0 + j * st];
    const double cs = ci.detJ * ci.ih[d], A = ci.A[d];
    double o[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      double acc = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) acc = fma(pt.Dpv[i][j], ul[j], acc);
      o[i] = cs * acc;
    }
    {  // left face, n_d = -1: -{u_d} n_d -> +A uf at pressure node 0
      const int f = 2 * d, nb = ci.nb[f], ty = ci.type[f];
      const double own = ul[0];
      const double uf = ty == 0 ? 0.5 * (own + __ldg(u + (size_t)nb * 3 * NB + b0 + (N - 1) * st)) : (ty == 1 ? own : 0.0);
      o[0] = fma(A, uf, o[0]);
    }
    {  // right face, n_d = +1: -A uf at pressure node NP-1
      const int f = 2 * d + 1, nb = ci.nb[f], ty = ci.type[f];
      const double own = ul[N - 1];
      const double uf = ty == 0 ? 0.5 * (own + __ldg(u + (size_t)nb * 3 * NB + b0)) : (ty == 1 ? own : 0.0);
      o[NP - 1] = fma(-A, uf, o[NP - 1]);
    }
    double* t1 = CELL(c) + 3 * NB + d * NP * N * N;
#pragma unroll
    for (int i = 0; i < NP; ++i) t1[i + NP * ab] = o[i];
  }
  __syncthreads();
  // S2: Mpv along t1 -> T2[d][i + NP (a' + NP b)]
  for (int idx = tid; idx < nc * 3 * NP * N; idx += TT) {
    const int c = idx / (3 * NP * N), r = idx - c * 3 * NP * N;
    const int d = r / (NP * N), ib = r - d * NP * N;
    const int i = ib % NP, b = ib / NP;
    const double* t1 = CELL(c) + 3 * NB + d * NP * N * N;
    double v[N];
#pragma unroll
    for (int a = 0; a < N; ++a) v[a] = t1[i + NP * (a + N * b)];
    double* t2 = CELL(c) + 3 * NB + G::L1 + d * NP * NP * N;
#pragma unroll
    for (int a2 = 0; a2 < NP; ++a2) {
      double acc = 0.0;
#pragma unroll
      for (int a = 0; a < N; ++a) acc = fma(pt.Mvp[a][a2], v[a], acc);
      t2[i + NP * (a2 + NP * b)] = acc;
    }
  }
  __syncthreads();
  // S3: Mpv along t2, summed over d, -> y
  for (int idx = tid; idx < nc * NBP; idx += TT) {
    const int c = idx / NBP, node = idx - c * NBP;
    const int ix = node % NP, iy = (node / NP) % NP, iz = node / (NP * NP);
    double sum = 0.0;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int i = d == 0 ? ix : (d == 1 ? iy : iz);
      const int a2 = d == 0 ? iy : ix, b2 = d == 2 ? iy : iz;
      const double* t2 = CELL(c) + 3 * NB + G::L1 + d * NP * NP * N;
#pragma unroll
      for (int b = 0; b < N; ++b) sum = fma(pt.Mvp[b][b2], t2[i + NP * (a2 + NP * b)], sum);
    }
    y[(size_t)(c0 + c) * NBP + node] = sum;
  }
#undef CELL
#undef INFO
}

// Exact diagonal of the scalar SIP operator (scalar_sip_diagonal, forms.cpp:246-329):
// diag(mc M (x) M (x) M + sum_d S_d (x) M (x) M).
template <int KP, bool UNI>
__global__ void __launch_bounds__(128) k_sip_diag_axis(MeshArgs m, UniformGrid ug, const double* __restrict__ aff,
                                                       double mc, int dir_bdry, double* __restrict__ y) {
  constexpr int N = KP + 1, NB = N * N * N, C = 16;
  const FTab<N, N>& ta = c_ft<N, N>;
  __shared__ double info[C][kInfoDoubles];
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  load_info_par<128, UNI>(&info[0][0], kInfoDoubles, 0, nc, m, ug, aff, c0, (double)(N * N));
  __syncthreads();
  for (int idx = threadIdx.x; idx < nc * 6; idx += 128)
    face_coefs(*reinterpret_cast<CellInfo*>(info[idx / 6]), idx % 6, dir_bdry != 0, false);
  __syncthreads();
  for (int idx = threadIdx.x; idx < nc * NB; idx += 128) {
    const int c = idx / NB, b = idx - c * NB;
    const CellInfo& ci = *reinterpret_cast<const CellInfo*>(info[c]);
    const int bi[3] = {b % N, (b / N) % N, b / (N * N)};
    double md[3], sd[3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const int i = bi[d];
      md[d] = ta.M[i][i];
      const double ih = ci.ih[d], sa = ci.A[d], stiff = sa * ih;
      const double* cR = ci.fc[2 * d + 1];
      const double* cL = ci.fc[2 * d];
      double v = stiff * ta.K[i][i];
      if (i == N - 1) v += sa * (cR[0] * ta.dE[1][i] + cR[2]) + ta.dE[1][i] * stiff * cR[4];
      if (i == 0) v += sa * (cL[0] * ta.dE[0][i] + cL[2]) - ta.dE[0][i] * stiff * cL[4];
      sd[d] = v;
    }
    y[(size_t)(c0 + c) * NB + b] = sd[0] * md[1] * md[2] + md[0] * sd[1] * md[2] + md[0] * md[1] * sd[2] +
                                   mc * ci.detJ * md[0] * md[1] * md[2];
  }
}

}  // namespace dgb
