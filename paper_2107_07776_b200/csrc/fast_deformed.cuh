// Fast path for deformed (non-affine) hexahedra: BASELINE cfg4.
//
// The scalar SIP operator (pressure Helmholtz / Laplacian, scalar_sip_apply,
// forms.cpp:148-243) with the per-quadrature-point geometry of the reference's
// GeometryCache (cell: Jinv + detJ w per Gauss point; faces: Jinv of both sides,
// unit normal, w ds per face point) streamed from HBM — SURVEY 8(d) counts this
// path HBM-bound.  The records are pre-contracted at setup to what the integrands
// consume: the cell metric detJw Jinv Jinv^T (6) + detJw, and per face point
// Jinv n, Jinv_nbr n (3 + 3) + w ds — 7 + 7 doubles instead of 10 + 22.
// Same quadrature sums as the reference (rule kp+2), sum-factorised:
//   cell: u and its reference gradient at the Q^3 points (x, y, z passes), the
//         pointwise metric Jinv^T (.) detJ w Jinv, the transposed passes back;
//   faces (element-centric, outward normal, all 6 at once): trace, tangential and
//         normal reference derivatives of both sides at the Q^2 face points, the SIP
//         flux / symmetry / penalty terms, the transposed face passes back onto the
//         face layer (value, tangential tests) and the normal line (normal test).
// One warp owns one cell after a CTA-wide staging barrier (stages sync with
// __syncwarp).  Geometry layout: host_setup.cpp build_qp_geometry.
#pragma once

#include "fast_axis.cuh"
#include "qp_layouts.hpp"

namespace dgb {

// work-area layout of one scalar SIP field on one cell (N nodes, Q Gauss points per direction).
// Stages overwrite inputs they no longer need: C3 writes PP/R0/R1 in place of the
// y-pass arrays it consumes (each lane owns its rows), C4 writes P2/R02 over the
// x-pass arrays; F3 writes FA over FL, F4 writes FON over FP.
template <int N, int Q>
struct QpSipWork {
  using L = QpLay<N, Q>;  // bank-conflict-optimal array layouts (qp_layouts.hpp)
  static constexpr int NF = N * N;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // cell phase
  static constexpr int XB = 0, XD = XB + L::X_SIZE, YBB = XD + L::X_SIZE, YDB = YBB + L::Y_SIZE,
                       YBD = YDB + L::Y_SIZE, PP = YBB, R0 = YDB, R1 = YBD, P2 = XB, R02 = XD,
                       CELL_END = YBD + L::Y_SIZE;
  // face phase: FL (F1 -> F2), FP (F2 -> F3), FA (F3 -> F4), FON (F4 -> F5); FA reuses FL and
  // FON reuses FP when they fit (their producers run after the last read of the old array)
  static constexpr int FL = 0, FP = FL + L::FL_SIZE;
  static constexpr int FON = L::FO_SIZE <= L::FP_SIZE ? FP : FP + L::FP_SIZE;
  static constexpr int FA = L::FA_SIZE <= L::FL_SIZE ? FL : mx(FP + L::FP_SIZE, FON + L::FO_SIZE);
  static constexpr int FACE_END = mx(mx(FP + L::FP_SIZE, FON + L::FO_SIZE), FA + L::FA_SIZE);
  // the six neighbour blocks (cp.async-staged by the caller during the cell phase, read in
  // F1): after the cell phase's arrays and after FL, which F1 writes while other lanes still
  // read the blocks (for N = 2 the round-1 layout let the two overlap), overwritten by F2 on
  static constexpr int NBR = mx(CELL_END, FL + L::FL_SIZE), NBR_END = NBR + 6 * N * N * N;
  static constexpr int SIZE = NBR_END > FACE_END ? NBR_END : FACE_END;
};

// strides of a face of axis a: node = l * sl + p * sp + q * sq (l along the normal,
// (p, q) the tangential axes in increasing order)
template <int N>
__device__ __forceinline__ void face_strides(int a, int& sl, int& sp, int& sq) {
  sl = a == 0 ? 1 : (a == 1 ? N : N * N);
  sp = a == 0 ? N : 1;
  sq = a == 2 ? N : N * N;
}
// linear node index of (normal-axis position l, tangential (p, q)) on a face of axis a
template <int N>
__device__ __forceinline__ int face_node(int a, int l, int p, int q) {
  return a == 0 ? l + N * (p + N * q) : (a == 1 ? p + N * (l + N * q) : p + N * (q + N * l));
}

// Bulk prefetch of a byte range into L2 (cp.async.bulk.prefetch.L2; 16-byte granular,
// clipped to [lo, hi) so it never reaches outside the array).  Issued for a cell's
// geometry records when the cell is staged, so the per-point loads of the later
// stages hit L2 instead of waiting on HBM.
__device__ __forceinline__ void prefetch_l2(const void* p, size_t bytes, const void* lo, const void* hi) {
  uintptr_t a = (uintptr_t)p, e = a + bytes;
  const uintptr_t l = ((uintptr_t)lo + 15) & ~(uintptr_t)15, h = (uintptr_t)hi & ~(uintptr_t)15;
  a = a & ~(uintptr_t)15;
  e = (e + 15) & ~(uintptr_t)15;
  if (a < l) a = l;
  if (e > h) e = h;
  if (e > a)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a), "r"((unsigned)(e - a)) : "memory");
}

// cp.async the six neighbour blocks of one field into NBR (warp-cooperative; faces
// without a neighbour are skipped, F1 never reads them).  Completed by the
// cp.async wait inside qp_sip_field, so the copies overlap its cell phase.
template <int N>
__device__ __forceinline__ void qp_stage_nbrs(double* NBR, const double* __restrict__ xg, int nstride, int noff,
                                              const double* nbv, int lane) {
  constexpr int NB = N * N * N;
#pragma unroll
  for (int f = 0; f < 6; ++f) {
    const int nb = (int)nbv[f];
    if (nb < 0) continue;
    const double* src = xg + (size_t)nb * nstride + noff;
    for (int n = lane; n < NB; n += 32) cp_async8(NBR + f * NB + n, src + n);
  }
}

// One scalar field through the SIP operator on one cell (warp-cooperative, lane loops +
// __syncwarp): OUT = mc M u + visc (K u + interior SIP faces + Dirichlet-type boundary
// faces where bit f of bdir is set).  U: the cell's nodal values in shared memory; the
// neighbours' values are read from xg[nb * nstride + noff + node].  Geometry: the
// compact records of this cell (7 doubles per cell point / per face point).
// RHS: the explicit viscous term of momentum_rhs instead (forms.cpp:839-857 cells,
// :863-889 interior faces, :919-931 boundary): consistency term only (no penalty, no
// symmetry term); the caller passes visc = -coef.
template <int N, int Q, bool RHS = false>
__device__ __forceinline__ void qp_sip_field(const double* U, double* NBF,
                                             const double* nbv, const double* penv, int bdir, double mc, double visc,
                                             const double* __restrict__ gcell, const double* __restrict__ gface,
                                             double* W, double* OUT, int lane) {
  using Wl = QpSipWork<N, Q>;
  using L = QpLay<N, Q>;
  constexpr int NF = N * N, NQF = Q * Q;
  const FTab<N, Q>& t = c_ft<N, Q>;
  // work-array element addresses (qp_layouts.hpp)
  auto xa = [](int qx, int j, int k) { return qx * L::X_qx + j * L::X_j + k * L::X_k; };
  auto ya = [](int qx, int qy, int k) { return qx * L::Y_qx + qy * L::Y_qy + k * L::Y_k; };
  auto fla = [](int f, int fld, int p, int q) { return f * L::FL_f + fld * L::FL_fld + p * L::FL_p + q * L::FL_q; };
  auto fpa = [](int f, int fld, int q, int qp) { return f * L::FP_f + fld * L::FP_fld + q * L::FP_q + qp * L::FP_qp; };
  auto faa = [](int f, int part, int qp, int b) { return f * L::FA_f + part * L::FA_part + qp * L::FA_qp + b * L::FA_b; };
  auto foa = [](int f, int h, int bp, int bq) { return f * L::FO_f + h * L::FO_h + bp * L::FO_bp + bq * L::FO_bq; };
  // ---- cell term
  for (int jk = lane; jk < NF; jk += 32) {  // C1: x pass (values, x-derivative)
    double u[N];
#pragma unroll
    for (int i = 0; i < N; ++i) u[i] = U[i + N * jk];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double b = 0.0, d = 0.0;
#pragma unroll
      for (int i = 0; i < N; ++i) {
        b = fma(t.B[qx][i], u[i], b);
        d = fma(t.D[qx][i], u[i], d);
      }
      W[Wl::XB + xa(qx, jk % N, jk / N)] = b;
      W[Wl::XD + xa(qx, jk % N, jk / N)] = d;
    }
  }
  __syncwarp();
  for (int it = lane; it < Q * N; it += 32) {  // C2: y pass
    const int qx = it / N, k = it - qx * N;
    double vb[N], vd[N];
#pragma unroll
    for (int j = 0; j < N; ++j) {
      vb[j] = W[Wl::XB + xa(qx, j, k)];
      vd[j] = W[Wl::XD + xa(qx, j, k)];
    }
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      double bb = 0.0, db = 0.0, bd = 0.0;
#pragma unroll
      for (int j = 0; j < N; ++j) {
        bb = fma(t.B[qy][j], vb[j], bb);
        db = fma(t.D[qy][j], vb[j], db);
        bd = fma(t.B[qy][j], vd[j], bd);
      }
      const int o = ya(qx, qy, k);
      W[Wl::YBB + o] = bb;
      W[Wl::YDB + o] = db;
      W[Wl::YBD + o] = bd;
    }
  }
  __syncwarp();
  for (int r = lane; r < Q * Q; r += 32) {  // C3: z pass, metric, z integration
    double vb[N], vy[N], vx[N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      vb[k] = W[Wl::YBB + ya(r / Q, r % Q, k)];
      vy[k] = W[Wl::YDB + ya(r / Q, r % Q, k)];
      vx[k] = W[Wl::YBD + ya(r / Q, r % Q, k)];
    }
    double pp[N], r0[N], r1[N];
#pragma unroll
    for (int k = 0; k < N; ++k) pp[k] = r0[k] = r1[k] = 0.0;
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      double val = 0.0, gr[3] = {0.0, 0.0, 0.0};
#pragma unroll
      for (int k = 0; k < N; ++k) {
        val = fma(t.B[qz][k], vb[k], val);
        gr[2] = fma(t.D[qz][k], vb[k], gr[2]);
        gr[1] = fma(t.B[qz][k], vy[k], gr[1]);
        gr[0] = fma(t.B[qz][k], vx[k], gr[0]);
      }
      constexpr int NQ = Q * Q * Q;  // records [7][qx][qy][qz]: lanes (qx, qy) read consecutive doubles
      const double* geo = gcell + r + Q * Q * qz;
      const double g00 = __ldg(geo), g01 = __ldg(geo + NQ), g02 = __ldg(geo + 2 * NQ), g11 = __ldg(geo + 3 * NQ),
                   g12 = __ldg(geo + 4 * NQ), g22 = __ldg(geo + 5 * NQ), jxw = __ldg(geo + 6 * NQ);
      double ra[3];  // detJw Jinv Jinv^T (reference gradient)
      ra[0] = g00 * gr[0] + g01 * gr[1] + g02 * gr[2];
      ra[1] = g01 * gr[0] + g11 * gr[1] + g12 * gr[2];
      ra[2] = g02 * gr[0] + g12 * gr[1] + g22 * gr[2];
      const double vi = mc * val * jxw;
      ra[0] *= visc;
      ra[1] *= visc;
      ra[2] *= visc;
#pragma unroll
      for (int k = 0; k < N; ++k) {
        pp[k] = fma(t.B[qz][k], vi, fma(t.D[qz][k], ra[2], pp[k]));
        r0[k] = fma(t.B[qz][k], ra[0], r0[k]);
        r1[k] = fma(t.B[qz][k], ra[1], r1[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < N; ++k) {
      W[Wl::PP + ya(r / Q, r % Q, k)] = pp[k];
      W[Wl::R0 + ya(r / Q, r % Q, k)] = r0[k];
      W[Wl::R1 + ya(r / Q, r % Q, k)] = r1[k];
    }
  }
  __syncwarp();
  for (int it = lane; it < Q * N; it += 32) {  // C4: y integration
    const int qx = it / N, k = it - qx * N;
    double p[Q], a0[Q], a1[Q];
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      const int o = ya(qx, qy, k);
      p[qy] = W[Wl::PP + o];
      a0[qy] = W[Wl::R0 + o];
      a1[qy] = W[Wl::R1 + o];
    }
#pragma unroll
    for (int j = 0; j < N; ++j) {
      double s = 0.0, u = 0.0;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        s = fma(t.B[qy][j], p[qy], fma(t.D[qy][j], a1[qy], s));
        u = fma(t.B[qy][j], a0[qy], u);
      }
      W[Wl::P2 + xa(qx, j, k)] = s;
      W[Wl::R02 + xa(qx, j, k)] = u;
    }
  }
  __syncwarp();
  for (int jk = lane; jk < NF; jk += 32) {  // C5: x integration -> OUT
    double p[Q], a0[Q];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      p[qx] = W[Wl::P2 + xa(qx, jk % N, jk / N)];
      a0[qx] = W[Wl::R02 + xa(qx, jk % N, jk / N)];
    }
#pragma unroll
    for (int i = 0; i < N; ++i) {
      double s = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) s = fma(t.B[qx][i], p[qx], fma(t.D[qx][i], a0[qx], s));
      OUT[i + N * jk] = s;
    }
  }
  __syncwarp();

  // ---- faces (all six at once)
  cp_async_wait_all();  // the neighbour blocks (qp_stage_nbrs)
  __syncwarp();
  for (int it = lane; it < 6 * NF; it += 32) {  // F1: traces and normal reference derivatives, both sides
    const int f = it / NF, tn = it - f * NF;
    const int a = f >> 1, s = f & 1, p = tn % N, q = tn / N;
    int sl, sp, sq;
    face_strides<N>(a, sl, sp, sq);
    const int base = p * sp + q * sq;
    const int nb = (int)nbv[f];
    double dns = 0.0, dno = 0.0, vo = 0.0, vs = 0.0;
#pragma unroll
    for (int l = 0; l < N; ++l) {
      const double v = U[base + l * sl];
      dns = fma(t.dE[s][l], v, dns);
      if (l == (s ? N - 1 : 0)) vs = v;
    }
    if (nb >= 0) {
      const double* xn = W + Wl::NBR + f * N * NF + base;
#pragma unroll
      for (int l = 0; l < N; ++l) {
        const double v = xn[l * sl];
        dno = fma(t.dE[1 - s][l], v, dno);
        if (l == (s ? 0 : N - 1)) vo = v;
      }
    }
    double* fl = W + Wl::FL;
    fl[fla(f, 0, p, q)] = vs;
    fl[fla(f, 1, p, q)] = dns;
    fl[fla(f, 2, p, q)] = vo;
    fl[fla(f, 3, p, q)] = dno;
    if (NBF) NBF[f * NF + tn] = vo;
  }
  __syncwarp();
  for (int it = lane; it < 6 * N; it += 32) {  // F2: along p (first tangential axis)
    const int f = it / N, q = it - f * N;
    const double* fl = W + Wl::FL;
    double v[4][N];
#pragma unroll
    for (int fld = 0; fld < 4; ++fld)
#pragma unroll
      for (int p = 0; p < N; ++p) v[fld][p] = fl[fla(f, fld, p, q)];
    double* fp = W + Wl::FP;
#pragma unroll
    for (int qp = 0; qp < Q; ++qp) {
      double o[6] = {0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int p = 0; p < N; ++p) {
        o[0] = fma(t.B[qp][p], v[0][p], o[0]);  // own value
        o[1] = fma(t.D[qp][p], v[0][p], o[1]);  // own d/dt1
        o[2] = fma(t.B[qp][p], v[1][p], o[2]);  // own d/dn
        o[3] = fma(t.B[qp][p], v[2][p], o[3]);  // nbr value
        o[4] = fma(t.D[qp][p], v[2][p], o[4]);  // nbr d/dt1
        o[5] = fma(t.B[qp][p], v[3][p], o[5]);  // nbr d/dn
      }
#pragma unroll
      for (int fld = 0; fld < 6; ++fld) fp[fpa(f, fld, q, qp)] = o[fld];
    }
  }
  __syncwarp();
  for (int it = lane; it < 6 * Q; it += 32) {  // F3: along q, SIP terms at the points, test integration along q
    const int f = it / Q, qp = it - f * Q;
    const int a = f >> 1;
    const int t1 = a == 0 ? 1 : 0, t2 = a == 2 ? 1 : 2;
    const int nb = (int)nbv[f];
    const double pen = penv[f];
    const bool act = nb >= 0 || ((bdir >> f) & 1);
    const double* fp = W + Wl::FP;
    double v[6][N];
#pragma unroll
    for (int fld = 0; fld < 6; ++fld)
#pragma unroll
      for (int q = 0; q < N; ++q) v[fld][q] = fp[fpa(f, fld, q, qp)];
    double A1[N], A2[N], A3[N];
#pragma unroll
    for (int b = 0; b < N; ++b) A1[b] = A2[b] = A3[b] = 0.0;
    if (act) {
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        double us = 0.0, d1s = 0.0, d2s = 0.0, dnr_s = 0.0, uo = 0.0, d1o = 0.0, d2o = 0.0, dnr_o = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) {
          us = fma(t.B[qq][q], v[0][q], us);
          d1s = fma(t.B[qq][q], v[1][q], d1s);
          d2s = fma(t.D[qq][q], v[0][q], d2s);
          dnr_s = fma(t.B[qq][q], v[2][q], dnr_s);
          uo = fma(t.B[qq][q], v[3][q], uo);
          d1o = fma(t.B[qq][q], v[4][q], d1o);
          d2o = fma(t.D[qq][q], v[3][q], d2o);
          dnr_o = fma(t.B[qq][q], v[5][q], dnr_o);
        }
        const double* geo = gface + (size_t)f * 7 * NQF + qp + Q * qq;  // records [f][7][qp + Q qq]
        double jn[3];  // Jinv n: physical normal derivative = reference gradient . (Jinv n)
#pragma unroll
        for (int d = 0; d < 3; ++d) jn[d] = __ldg(geo + d * NQF);
        const double wds = __ldg(geo + 6 * NQF);
        double grs[3];
        grs[a] = dnr_s;
        grs[t1] = d1s;
        grs[t2] = d2s;
        const double dns = jn[0] * grs[0] + jn[1] * grs[1] + jn[2] * grs[2];
        double F, ssym;
        if (nb >= 0) {
          double gro[3];
          gro[a] = dnr_o;
          gro[t1] = d1o;
          gro[t2] = d2o;
          const double dno = __ldg(geo + 3 * NQF) * gro[0] + __ldg(geo + 4 * NQF) * gro[1] + __ldg(geo + 5 * NQF) * gro[2];
          const double ju = us - uo;
          F = visc * (-0.5 * (dns + dno) + (RHS ? 0.0 : pen * ju)) * wds;  // forms.cpp:199-209 / 443-461
          ssym = RHS ? 0.0 : -0.5 * visc * ju * wds;
        } else {  // Dirichlet-type boundary, forms.cpp:232-240
          F = visc * (-dns + (RHS ? 0.0 : 2.0 * pen * us)) * wds;
          ssym = RHS ? 0.0 : -visc * us * wds;
        }
        double rr[3];
#pragma unroll
        for (int aa = 0; aa < 3; ++aa) rr[aa] = jn[aa] * ssym;
#pragma unroll
        for (int b = 0; b < N; ++b) {
          A1[b] = fma(t.B[qq][b], F, fma(t.D[qq][b], rr[t2], A1[b]));
          A2[b] = fma(t.B[qq][b], rr[t1], A2[b]);
          A3[b] = fma(t.B[qq][b], rr[a], A3[b]);
        }
      }
    }
    double* fa = W + Wl::FA;
#pragma unroll
    for (int b = 0; b < N; ++b) {
      fa[faa(f, 0, qp, b)] = A1[b];
      fa[faa(f, 1, qp, b)] = A2[b];
      fa[faa(f, 2, qp, b)] = A3[b];
    }
  }
  __syncwarp();
  for (int it = lane; it < 6 * N; it += 32) {  // F4: along p -> face-layer (value / tangential) and normal-test parts
    const int f = it / N, bq = it - f * N;
    const double* fa = W + Wl::FA;
    double a1[Q], a2[Q], a3[Q];
#pragma unroll
    for (int qp = 0; qp < Q; ++qp) {
      a1[qp] = fa[faa(f, 0, qp, bq)];
      a2[qp] = fa[faa(f, 1, qp, bq)];
      a3[qp] = fa[faa(f, 2, qp, bq)];
    }
    double* fo = W + Wl::FON;
#pragma unroll
    for (int bp = 0; bp < N; ++bp) {
      double lo = 0.0, ln = 0.0;
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) {
        lo = fma(t.B[qp][bp], a1[qp], fma(t.D[qp][bp], a2[qp], lo));
        ln = fma(t.B[qp][bp], a3[qp], ln);
      }
      fo[foa(f, 0, bp, bq)] = lo;
      fo[foa(f, 1, bp, bq)] = ln;
    }
  }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 3; ++a) {  // F5: per axis, the two faces' contributions along each normal line
    for (int tn = lane; tn < NF; tn += 32) {
      const int p = tn % N, q = tn / N;
      const double* fo = W + Wl::FON;
      const double n0 = fo[foa(2 * a, 1, p, q)], n1 = fo[foa(2 * a + 1, 1, p, q)];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double v = t.dE[0][l] * n0 + t.dE[1][l] * n1;
        if (l == 0) v += fo[foa(2 * a, 0, p, q)];
        if (l == N - 1) v += fo[foa(2 * a + 1, 0, p, q)];
        OUT[face_node<N>(a, l, p, q)] += v;
      }
    }
    __syncwarp();
  }
}

template <int KP>
struct SipQpCfg {
  static constexpr int N = KP + 1, Q = KP + 2, NB = N * N * N, NF = N * N, NQ = Q * Q * Q, NQF = Q * Q;
#ifndef DGB_SQP_C
#define DGB_SQP_C 4
#endif
  static constexpr int C = DGB_SQP_C, T = 32 * C;
  static constexpr int CS = 7, FS = 7;  // compact cell / face geometry records (DevCtx::qcm / qfn)
  // per cell: U | OUT | info (nb, type as doubles; pen) | work
  static constexpr int O_U = 0, O_OUT = NB, O_NB = 2 * NB, O_TY = O_NB + 6, O_PEN = O_TY + 6, O_WK = O_PEN + 6;
  static constexpr int WORK = QpSipWork<N, Q>::SIZE;
  static constexpr int PER = (O_WK + WORK) | 1;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

#ifndef DGB_SQP_MINB
#define DGB_SQP_MINB 4  // minimum CTAs per SM promised to ptxas: 128 registers, 16 warps per SM
                        // (cfg4 0.62 ms; MINB 1: 0.86, 5: 0.94; C = 2 / 6 / 8 cells per CTA: 0.82-1.15)
#endif
template <int KP>
__global__ void __launch_bounds__(SipQpCfg<KP>::T, DGB_SQP_MINB) k_sip_qp(MeshArgs m, const double* __restrict__ gc,
                                                             const double* __restrict__ gf, double mc, int dir_bdry,
                                                             const double* __restrict__ x, double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  using G = SipQpCfg<KP>;
  constexpr int N = G::N, Q = G::Q, NB = G::NB, NQ = G::NQ, NQF = G::NQF, C = G::C, PER = G::PER;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const double sfac = (double)(N * N);
  // ---- staging (CTA-wide): cell values, neighbours, face types, penalties
  for (int idx = tid; idx < nc * NB; idx += G::T) cp_async8(sm + (idx / NB) * PER + G::O_U + idx % NB, x + (size_t)c0 * NB + idx);
  for (int idx = tid; idx < nc * 6; idx += G::T) {
    const int c = idx / 6, f = idx - c * 6;
    double* cell = sm + c * PER;
    const int nb = m.nbr[(size_t)(c0 + c) * 6 + f];
    int ty = 0;
    if (nb < 0) {
      const int bid = -1 - nb;
      ty = (bid >= 0 && bid < 64 && m.bctype[bid] == 1) ? 2 : 1;  // the scalar operator treats outlets as walls
    }
    cell[G::O_NB + f] = (double)nb;
    cell[G::O_TY + f] = (double)ty;
    cell[G::O_PEN + f] = sfac * m.pen[(size_t)(c0 + c) * 6 + f];
  }
  if (tid < nc) {  // geometry of the CTA's cells -> L2
    const size_t cb = (size_t)NQ * G::CS * sizeof(double), fb = (size_t)6 * NQF * G::FS * sizeof(double);
    prefetch_l2(gc + (size_t)(c0 + tid) * NQ * G::CS, cb, gc, gc + (size_t)m.ncells * NQ * G::CS);
    prefetch_l2(gf + (size_t)(c0 + tid) * 6 * NQF * G::FS, fb, gf, gf + (size_t)m.ncells * 6 * NQF * G::FS);
  }
  cp_async_wait_all();
  __syncthreads();
  if (wc >= nc) return;
  const int cid = c0 + wc;
  double* cell = sm + wc * PER;
  double* U = cell + G::O_U;
  double* OUT = cell + G::O_OUT;
  double* W = cell + G::O_WK;
  const double* gcell = gc + (size_t)cid * NQ * G::CS;
  const double* gface = gf + (size_t)cid * 6 * NQF * G::FS;

  const int bdir = dir_bdry ? 0x3f : 0;  // the scalar operator: all boundary faces Dirichlet or all natural
  qp_stage_nbrs<N>(W + QpSipWork<N, Q>::NBR, x, NB, 0, cell + G::O_NB, lane);
  qp_sip_field<N, Q>(U, nullptr, cell + G::O_NB, cell + G::O_PEN, bdir, mc, 1.0, gcell, gface, W, OUT, lane);
  for (int i = lane; i < NB; i += 32) y[(size_t)cid * NB + i] = OUT[i];
}

// The advecting field's component-independent factors of the deformed momentum operator
// (apply and diagonal): W1 -> WT[a][q] = -adv (detJ w Jinv w)_a at the rule-B cell points,
// W2 -> FC = the Lax-Friedrichs weights a_s [6][Q^2] and a_o [6][Q^2] at the rule-B face
// points (forms.cpp:509-530, :555-573, :592-599).  WS: the cell's staged advecting field
// (3 components); W: work area (offsets BXO, BYO, FPWO, NWO); one warp per cell.
// RHS: the central advective flux of momentum_rhs (forms.cpp:1008-1048): no lambda term,
// w.n f on every boundary face
template <int N, int QB, int BXO, int BYO, int FPWO, int NWO, bool RHS = false>
__device__ __forceinline__ void qp_w_phase(const double* WS, double* W, double* WT, double* FC, const double* nbv,
                                           const double* tyv, const double* __restrict__ w,
                                           const double* __restrict__ gadv_c, const double* __restrict__ gfw_c,
                                           double adv, int lane) {
  constexpr int NB = N * N * N, NF = N * N, NQB = QB * QB * QB, NQFB = QB * QB;
  const FTab<N, QB>& tb = c_ft<N, QB>;
    // the neighbours' advecting-field face layers -> NW (waited for before W2)
    for (int i = lane; i < 6 * 3 * NF; i += 32) {
      const int f = i / (3 * NF), r = i - f * 3 * NF, d = r / NF, tn = r - d * NF;
      const int nb = (int)nbv[f];
      if (nb < 0) continue;
      int sl, sp, sq;
      face_strides<N>(f >> 1, sl, sp, sq);
      cp_async8(W + NWO + i, w + (size_t)nb * 3 * NB + d * NB + ((f & 1) ? 0 : N - 1) * sl + (tn % N) * sp + (tn / N) * sq);
    }
    // ---- W1: advecting field at the rule-B points -> Wt (component-independent)
#pragma unroll 1
    for (int d = 0; d < 3; ++d) {
      const double* Wd = WS + d * NB;
      for (int jk = lane; jk < NF; jk += 32) {
        double u[N];
#pragma unroll
        for (int i = 0; i < N; ++i) u[i] = Wd[i + N * jk];
#pragma unroll
        for (int qx = 0; qx < QB; ++qx) {
          double b = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) b = fma(tb.B[qx][i], u[i], b);
          W[BXO + qx * NF + jk] = b;
        }
      }
      __syncwarp();
      for (int it = lane; it < QB * N; it += 32) {
        const int qx = it / N, k = it - qx * N;
        double v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = W[BXO + qx * NF + j + N * k];
#pragma unroll
        for (int qy = 0; qy < QB; ++qy) {
          double b = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) b = fma(tb.B[qy][j], v[j], b);
          W[BYO + (qx * QB + qy) * N + k] = b;
        }
      }
      __syncwarp();
      for (int r = lane; r < QB * QB; r += 32) {
        const int qx = r / QB, qy = r - qx * QB;
        double v[N];
#pragma unroll
        for (int k = 0; k < N; ++k) v[k] = W[BYO + r * N + k];
#pragma unroll
        for (int qz = 0; qz < QB; ++qz) {
          double b = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) b = fma(tb.B[qz][k], v[k], b);
          WT[d * NQB + qx + QB * qy + QB * QB * qz] = b;
        }
      }
      __syncwarp();
    }
    {
      const double* g = gadv_c;
      for (int q = lane; q < NQB; q += 32) {
        const double w0 = WT[q], w1 = WT[NQB + q], w2 = WT[2 * NQB + q];
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const double t = __ldg(g + (a * 3 + 0) * NQB + q) * w0 + __ldg(g + (a * 3 + 1) * NQB + q) * w1 +
                           __ldg(g + (a * 3 + 2) * NQB + q) * w2;
          WT[a * NQB + q] = -adv * t;
        }
      }
    }
    // ---- W2: face factors a_s, a_o at the rule-B face points
    cp_async_wait_all();
    __syncwarp();
    for (int it = lane; it < 6 * 2 * N; it += 32) {
      const int f = it / (2 * N), rem = it - f * 2 * N, side = rem / N, q = rem - side * N;
      const int a = f >> 1, s = f & 1;
      const int nb = (int)nbv[f];
      int sl, sp, sq;
      face_strides<N>(a, sl, sp, sq);
      double* fp = W + FPWO + (f * 2 + side) * 3 * N * QB + q * QB;
#pragma unroll 1
      for (int d = 0; d < 3; ++d) {
        double v[N];
        if (side == 0) {
          const double* ws = WS + d * NB + (s ? N - 1 : 0) * sl + q * sq;
#pragma unroll
          for (int p = 0; p < N; ++p) v[p] = ws[p * sp];
        } else if (nb >= 0) {
          const double* wn = W + NWO + (f * 3 + d) * NF + N * q;
#pragma unroll
          for (int p = 0; p < N; ++p) v[p] = wn[p];
        } else {
#pragma unroll
          for (int p = 0; p < N; ++p) v[p] = 0.0;
        }
#pragma unroll
        for (int qp = 0; qp < QB; ++qp) {
          double b = 0.0;
#pragma unroll
          for (int p = 0; p < N; ++p) b = fma(tb.B[qp][p], v[p], b);
          fp[d * N * QB + qp] = b;
        }
      }
    }
    __syncwarp();
    for (int it = lane; it < 6 * QB; it += 32) {
      const int f = it / QB, qp = it - f * QB;
      const int ty = (int)tyv[f];
      const double* nw = gfw_c + (size_t)f * 3 * NQFB;
      double vs[3][N], vo[3][N];
#pragma unroll
      for (int d = 0; d < 3; ++d)
#pragma unroll
        for (int q = 0; q < N; ++q) {
          vs[d][q] = W[FPWO + (f * 2 + 0) * 3 * N * QB + d * N * QB + q * QB + qp];
          vo[d][q] = W[FPWO + (f * 2 + 1) * 3 * N * QB + d * N * QB + q * QB + qp];
        }
#pragma unroll
      for (int qq = 0; qq < QB; ++qq) {
        const int t = qp + QB * qq;
        double wns = 0.0, wno = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double ws = 0.0, wo = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            ws = fma(tb.B[qq][q], vs[d][q], ws);
            wo = fma(tb.B[qq][q], vo[d][q], wo);
          }
          const double nd = __ldg(nw + d * NQFB + t);
          wns = fma(ws, nd, wns);
          wno = fma(wo, nd, wno);
        }
        double as, ao;
        if (ty == 0) {
          const double lam = RHS ? 0.0 : fmax(fabs(wns), fabs(wno));
          as = 0.5 * adv * (wns + lam);
          ao = 0.5 * adv * (wno - lam);
        } else {
          as = adv * ((RHS || ty == 2) ? wns : fabs(wns));
          ao = 0.0;
        }
        FC[f * NQFB + t] = as;
        FC[6 * NQFB + f * NQFB + t] = ao;
      }
    }
    __syncwarp();
}

// ===========================================================================
// Momentum operator on deformed hexahedra (apply_momentum, forms.cpp:389-604)
// ===========================================================================
// Pass A (rule k+1, mass + SIP viscous) per component through qp_sip_field with the
// compact records of rule k+1.  Pass B (rule k+2, Lax-Friedrichs advection) needs the
// advecting field only through component-independent pointwise factors, computed once
// per cell before the component loop:
//   cell:  Wt_a(q) = -adv sum_d (detJ w Jinv)[a][d] w_d(q)   (the reference's
//          to_ref(Ji, -adv u w jxw) with u factored out, forms.cpp:509-530)
//   faces: flux = a_s u_s + a_o u_o with a_s = adv/2 (w_s.n + lam) ds w,
//          a_o = adv/2 (w_o.n - lam) ds w, lam = max(|w_s.n|, |w_o.n|) (forms.cpp:555-573);
//          boundary a_s = adv |w.n| ds w (outlet: adv w.n ds w), a_o = 0 (forms.cpp:592-599).
// Streamed pass-B geometry (DevCtx::qadv / qfw, rule k+2, per cell SoA): detJ w Jinv
// [9][Q^3] and n ds w [6][3][Q^2].
template <int K>
struct MomQpCfg {
  static constexpr int N = K + 1, QA = K + 1, QB = K + 2, NB = N * N * N, NF = N * N;
  static constexpr int NQB = QB * QB * QB, NQFB = QB * QB, NQA = QA * QA * QA, NQFA = QA * QA;
  static constexpr int WSIP = QpSipWork<N, QA>::SIZE;
  // pass-B work areas (offsets inside WORK): x / y passes, z-integrated A0 (over BY), A1, A2;
  // y-integrated X0 (over BX), X12
  static constexpr int BX = 0, BY = BX + QB * NF, BA0 = BY, BA1 = BY + QB * QB * N, BA2 = BA1 + QB * QB * N,
                       X0 = BX, X12 = BA2 + QB * QB * N, B_CELL_END = X12 + QB * NF;
  static constexpr int FPB = 0, FAB = FPB + 6 * 2 * N * QB, FOB = FAB + 6 * QB * N, B_FACE_END = FOB + 6 * NF;
  static constexpr int FPW = 0, W_END_F = FPW + 6 * 2 * 3 * N * QB, W_END_C = BY + QB * QB * N;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  static constexpr int NW = W_END_F;  // the neighbours' advecting-field face layers [6][3][NF] (cp.async)
  static constexpr int WORK = mx(mx(WSIP, B_CELL_END), mx(B_FACE_END, mx(NW + 6 * 3 * NF, W_END_C)));
  // per cell: X (3 comps) | OUT | nb | type | pen | WT | FC | WORK; the advecting field is
  // staged in FC (free until the face factors are written, after its last read)
  static constexpr int O_X = 0, O_OUT = 3 * NB, O_NB = O_OUT + NB, O_TY = O_NB + 6, O_PEN = O_TY + 6,
                       O_WT = O_PEN + 6, O_FC = O_WT + 3 * NQB, O_WS = O_FC, O_NBF = O_FC + 2 * 6 * NQFB,
                       O_WK = O_NBF + 6 * NF;
  static_assert(3 * NB <= 2 * 6 * NQFB, "advecting field must fit in FC");
  static constexpr int PER = (O_WK + WORK) | 1;
  static constexpr int C_FIT = (227 * 1024 / 8) / PER;
#ifndef DGB_MQP_CMAX
#define DGB_MQP_CMAX 8  // 8 warps: 2 per SM sub-partition at <= 256 registers
#endif
  static constexpr int C = C_FIT > DGB_MQP_CMAX ? DGB_MQP_CMAX : C_FIT, T = 32 * C;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

// RHS: the explicit stage operator of momentum_rhs (caller passes -visc / -adv
// coefficients), acc: y += result
template <int K, bool RHS = false>
__global__ void __launch_bounds__(MomQpCfg<K>::T) k_momentum_qp(MeshArgs m, const double* __restrict__ gcA,
                                                                const double* __restrict__ gfA,
                                                                const double* __restrict__ gadv,
                                                                const double* __restrict__ gfw, MomCoef co,
                                                                const double* __restrict__ x,
                                                                const double* __restrict__ w, double* __restrict__ y,
                                                                int acc = 0) {
  if (m.skip && *m.skip) return;
  using G = MomQpCfg<K>;
  constexpr int N = G::N, QA = G::QA, QB = G::QB, NB = G::NB, NF = G::NF, NQB = G::NQB, NQFB = G::NQFB;
  constexpr int C = G::C, PER = G::PER;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const bool passA = co.mass != 0.0 || co.visc != 0.0;
  const bool passB = co.adv != 0.0;
  const double sfac = (double)(N * N);  // sip_sigma (deg+1)^2, forms.hpp:175
  // ---- staging (CTA-wide): the cells' x (all components) and w, neighbours, face types, penalties
  for (int idx = tid; idx < nc * 3 * NB; idx += G::T) {
    const int c = idx / (3 * NB), i = idx - c * 3 * NB;
    cp_async8(sm + c * PER + G::O_X + i, x + (size_t)c0 * 3 * NB + idx);
    if (passB) cp_async8(sm + c * PER + G::O_WS + i, w + (size_t)c0 * 3 * NB + idx);
  }
  for (int idx = tid; idx < nc * 6; idx += G::T) {
    const int c = idx / 6, f = idx - c * 6;
    double* cell = sm + c * PER;
    const int nb = m.nbr[(size_t)(c0 + c) * 6 + f];
    int ty = 0;  // 0 interior, 1 Dirichlet wall, 2 outlet
    if (nb < 0) {
      const int bid = -1 - nb;
      ty = (bid >= 0 && bid < 64 && m.bctype[bid] == 1) ? 2 : 1;
    }
    cell[G::O_NB + f] = (double)nb;
    cell[G::O_TY + f] = (double)ty;
    cell[G::O_PEN + f] = sfac * m.pen[(size_t)(c0 + c) * 6 + f];
  }
  if (tid < nc) {  // geometry of the CTA's cells -> L2 (pass B records first: used first)
    const size_t n = m.ncells, c = c0 + tid;
    if (passB) {
      prefetch_l2(gadv + c * 9 * NQB, 9 * NQB * sizeof(double), gadv, gadv + n * 9 * NQB);
      prefetch_l2(gfw + c * 18 * NQFB, 18 * NQFB * sizeof(double), gfw, gfw + n * 18 * NQFB);
    }
    if (passA) {
      prefetch_l2(gcA + c * G::NQA * 7, G::NQA * 7 * sizeof(double), gcA, gcA + n * G::NQA * 7);
      prefetch_l2(gfA + c * 6 * G::NQFA * 7, 6 * G::NQFA * 7 * sizeof(double), gfA, gfA + n * 6 * G::NQFA * 7);
    }
  }
  cp_async_wait_all();
  __syncthreads();
  if (wc >= nc) return;
  const int cid = c0 + wc;
  double* cell = sm + wc * PER;
  double* OUT = cell + G::O_OUT;
  double* WT = cell + G::O_WT;
  double* FC = cell + G::O_FC;
  double* W = cell + G::O_WK;
  const double* nbv = cell + G::O_NB;
  const double* tyv = cell + G::O_TY;
  const FTab<N, QB>& tb = c_ft<N, QB>;
  int bdir = 0;  // viscous Dirichlet faces (outlets skip the viscous boundary terms, forms.cpp:469-493)
#pragma unroll
  for (int f = 0; f < 6; ++f) bdir |= ((int)tyv[f] == 1) << f;

  if (passB) {
    qp_w_phase<N, QB, G::BX, G::BY, G::FPW, G::NW, RHS>(cell + G::O_WS, W, WT, FC, nbv, tyv, w,
                                                   gadv + (size_t)cid * 9 * NQB, gfw + (size_t)cid * 18 * NQFB,
                                                   co.adv, lane);
  }

#pragma unroll 1
  for (int comp = 0; comp < 3; ++comp) {
    const double* U = cell + G::O_X + comp * NB;
    // ---- pass A: mass + SIP viscous at rule k+1
    if (passA) {
      qp_stage_nbrs<N>(W + QpSipWork<N, QA>::NBR, x, 3 * NB, comp * NB, nbv, lane);
      qp_sip_field<N, QA, RHS>(U, passB ? cell + G::O_NBF : nullptr, nbv, cell + G::O_PEN, bdir, co.mass, co.visc,
                          gcA + (size_t)cid * G::NQA * 7, gfA + (size_t)cid * 6 * G::NQFA * 7, W, OUT, lane);
    } else {
      for (int i = lane; i < NB; i += 32) OUT[i] = 0.0;
      __syncwarp();
    }
    if (passB) {
      // ---- pass B cell: u at the rule-B points, times Wt, integrated against the reference gradient tests
      for (int jk = lane; jk < NF; jk += 32) {
        double u[N];
#pragma unroll
        for (int i = 0; i < N; ++i) u[i] = U[i + N * jk];
#pragma unroll
        for (int qx = 0; qx < QB; ++qx) {
          double b = 0.0;
#pragma unroll
          for (int i = 0; i < N; ++i) b = fma(tb.B[qx][i], u[i], b);
          W[G::BX + qx * NF + jk] = b;
        }
      }
      __syncwarp();
      for (int it = lane; it < QB * N; it += 32) {
        const int qx = it / N, k = it - qx * N;
        double v[N];
#pragma unroll
        for (int j = 0; j < N; ++j) v[j] = W[G::BX + qx * NF + j + N * k];
#pragma unroll
        for (int qy = 0; qy < QB; ++qy) {
          double b = 0.0;
#pragma unroll
          for (int j = 0; j < N; ++j) b = fma(tb.B[qy][j], v[j], b);
          W[G::BY + (qx * QB + qy) * N + k] = b;
        }
      }
      __syncwarp();
      for (int r = lane; r < QB * QB; r += 32) {
        const int qx = r / QB, qy = r - qx * QB;
        double v[N], a0[N], a1[N], a2[N];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          v[k] = W[G::BY + r * N + k];
          a0[k] = a1[k] = a2[k] = 0.0;
        }
#pragma unroll
        for (int qz = 0; qz < QB; ++qz) {
          double val = 0.0;
#pragma unroll
          for (int k = 0; k < N; ++k) val = fma(tb.B[qz][k], v[k], val);
          const int pt = qx + QB * qy + QB * QB * qz;
          const double r0 = val * WT[pt], r1 = val * WT[NQB + pt], r2 = val * WT[2 * NQB + pt];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            a0[k] = fma(tb.B[qz][k], r0, a0[k]);
            a1[k] = fma(tb.B[qz][k], r1, a1[k]);
            a2[k] = fma(tb.D[qz][k], r2, a2[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          W[G::BA0 + r * N + k] = a0[k];
          W[G::BA1 + r * N + k] = a1[k];
          W[G::BA2 + r * N + k] = a2[k];
        }
      }
      __syncwarp();
      for (int it = lane; it < QB * N; it += 32) {
        const int qx = it / N, k = it - qx * N;
        double p0[QB], p1[QB], p2[QB];
#pragma unroll
        for (int qy = 0; qy < QB; ++qy) {
          const int o = (qx * QB + qy) * N + k;
          p0[qy] = W[G::BA0 + o];
          p1[qy] = W[G::BA1 + o];
          p2[qy] = W[G::BA2 + o];
        }
#pragma unroll
        for (int j = 0; j < N; ++j) {
          double s0 = 0.0, s12 = 0.0;
#pragma unroll
          for (int qy = 0; qy < QB; ++qy) {
            s0 = fma(tb.B[qy][j], p0[qy], s0);
            s12 = fma(tb.D[qy][j], p1[qy], fma(tb.B[qy][j], p2[qy], s12));
          }
          W[G::X0 + qx * NF + j + N * k] = s0;
          W[G::X12 + qx * NF + j + N * k] = s12;
        }
      }
      __syncwarp();
      for (int jk = lane; jk < NF; jk += 32) {
        double p0[QB], p12[QB];
#pragma unroll
        for (int qx = 0; qx < QB; ++qx) {
          p0[qx] = W[G::X0 + qx * NF + jk];
          p12[qx] = W[G::X12 + qx * NF + jk];
        }
#pragma unroll
        for (int i = 0; i < N; ++i) {
          double s = OUT[i + N * jk];
#pragma unroll
          for (int qx = 0; qx < QB; ++qx) s = fma(tb.D[qx][i], p0[qx], fma(tb.B[qx][i], p12[qx], s));
          OUT[i + N * jk] = s;
        }
      }
      __syncwarp();
      // ---- pass B faces: Lax-Friedrichs flux at the rule-B face points, tested with the face-layer traces
      for (int it = lane; it < 6 * 2 * N; it += 32) {
        const int f = it / (2 * N), rem = it - f * 2 * N, side = rem / N, q = rem - side * N;
        const int a = f >> 1, s = f & 1;
        const int nb = (int)nbv[f];
        int sl, sp, sq;
        face_strides<N>(a, sl, sp, sq);
        double v[N];
        if (side == 0) {
          const double* us = U + (s ? N - 1 : 0) * sl + q * sq;
#pragma unroll
          for (int p = 0; p < N; ++p) v[p] = us[p * sp];
        } else if (nb >= 0) {
          if (passA) {  // the neighbour face layer F1 left in NBF
            const double* xn = cell + G::O_NBF + f * NF + N * q;
#pragma unroll
            for (int p = 0; p < N; ++p) v[p] = xn[p];
          } else {
            const double* xn = x + (size_t)nb * 3 * NB + comp * NB + (s ? 0 : N - 1) * sl + q * sq;
#pragma unroll
            for (int p = 0; p < N; ++p) v[p] = __ldg(xn + p * sp);
          }
        } else {
#pragma unroll
          for (int p = 0; p < N; ++p) v[p] = 0.0;
        }
        double* fp = W + G::FPB + ((f * 2 + side) * N + q) * QB;
#pragma unroll
        for (int qp = 0; qp < QB; ++qp) {
          double b = 0.0;
#pragma unroll
          for (int p = 0; p < N; ++p) b = fma(tb.B[qp][p], v[p], b);
          fp[qp] = b;
        }
      }
      __syncwarp();
      for (int it = lane; it < 6 * QB; it += 32) {
        const int f = it / QB, qp = it - f * QB;
        double vs[N], vo[N], A[N];
#pragma unroll
        for (int q = 0; q < N; ++q) {
          vs[q] = W[G::FPB + ((f * 2 + 0) * N + q) * QB + qp];
          vo[q] = W[G::FPB + ((f * 2 + 1) * N + q) * QB + qp];
          A[q] = 0.0;
        }
#pragma unroll
        for (int qq = 0; qq < QB; ++qq) {
          double us = 0.0, uo = 0.0;
#pragma unroll
          for (int q = 0; q < N; ++q) {
            us = fma(tb.B[qq][q], vs[q], us);
            uo = fma(tb.B[qq][q], vo[q], uo);
          }
          const int t = qp + QB * qq;
          const double fl = FC[f * NQFB + t] * us + FC[6 * NQFB + f * NQFB + t] * uo;
#pragma unroll
          for (int b = 0; b < N; ++b) A[b] = fma(tb.B[qq][b], fl, A[b]);
        }
#pragma unroll
        for (int b = 0; b < N; ++b) W[G::FAB + (f * QB + qp) * N + b] = A[b];
      }
      __syncwarp();
      for (int it = lane; it < 6 * N; it += 32) {
        const int f = it / N, b = it - f * N;
        double av[QB];
#pragma unroll
        for (int qp = 0; qp < QB; ++qp) av[qp] = W[G::FAB + (f * QB + qp) * N + b];
#pragma unroll
        for (int bp = 0; bp < N; ++bp) {
          double s = 0.0;
#pragma unroll
          for (int qp = 0; qp < QB; ++qp) s = fma(tb.B[qp][bp], av[qp], s);
          W[G::FOB + f * NF + bp + N * b] = s;
        }
      }
      __syncwarp();
    }
    // ---- store (face-layer contributions of pass B added on the way out)
    double* yc = y + ((size_t)cid * 3 + comp) * NB;
    for (int n = lane; n < NB; n += 32) {
      double v = OUT[n];
      if (passB) {
        const int i = n % N, j = (n / N) % N, k = n / NF;
        const double* fo = W + G::FOB;
        if (i == 0) v += fo[0 * NF + j + N * k];
        if (i == N - 1) v += fo[1 * NF + j + N * k];
        if (j == 0) v += fo[2 * NF + i + N * k];
        if (j == N - 1) v += fo[3 * NF + i + N * k];
        if (k == 0) v += fo[4 * NF + i + N * j];
        if (k == N - 1) v += fo[5 * NF + i + N * j];
      }
      yc[n] = acc ? yc[n] + v : v;
    }
    __syncwarp();
  }
}


// ===========================================================================
// Weak pressure gradient of momentum_rhs and the divergence functional on deformed
// hexahedra (forms.cpp:850-855 / :895-912 / :940-948 and :1118-1197): the two mixed
// velocity-pressure forms, transposes of each other, both at the velocity rule k+1:
//   G(p)_{d,i} = (p, d_d phi_i) - <{p} n_d, phi_i>      (velocity tests, component d)
//   B(u)_i     = (u, grad psi_i) - <{u}.n, psi_i>       (pressure tests)
// element-centric (normal out of the working cell; {.} = mean on interior faces, the
// interior trace on walls, nothing on outlets).  One warp per cell, sum-factorised; the
// geometry enters through the streamed records detJ w Jinv [9][Q^3] and n ds w
// [6][3][Q^2] of rule k+1 (DevCtx::qadv / qfw, per cell SoA).  KP = K - 1.
// ===========================================================================
template <int K>
struct MixQpCfg {
  static constexpr int N = K + 1, NP = K, Q = K + 1, NB = N * N * N, NBP = NP * NP * NP, NF = N * N, NFP = NP * NP;
  static constexpr int NQ = Q * Q * Q, NQF = Q * Q;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // pressure gradient: P | PF (nbr layers -> face-node means) | OUT | cell work | face work
  static constexpr int G_P = 0, G_PF = G_P + NBP, G_OUT = G_PF + 6 * NFP, G_CW = G_OUT + NB;
  static constexpr int G_X = 0, G_Y = G_X + Q * NFP, G_A = 0, G_XI = G_A + 3 * NQF * N;  // offsets inside cell work
  static constexpr int G_CWS = mx(G_Y + NQF * NP, G_XI + 2 * Q * NF);
  static constexpr int G_FP = G_CW + G_CWS, G_FA = G_FP + 6 * NP * Q, G_FO = G_FA + 6 * Q * N, G_END = G_FO + 6 * NF;
  static constexpr int G_PER = G_END | 1;
  // divergence: U (3 comps) | UF (nbr layers -> face-node means, 3 comps) | OUT | cell work | face work
  static constexpr int D_U = 0, D_UF = D_U + 3 * NB, D_OUT = D_UF + 6 * 3 * NF, D_CW = D_OUT + NBP;
  static constexpr int D_X = 0, D_Y = D_X + Q * NF, D_YS = NQF * N;             // y-pass arrays of the 3 comps
  static constexpr int D_A = D_Y + 3 * D_YS, D_XI = D_A + 3 * NQF * NP;
  static constexpr int D_CWS = D_XI + 2 * Q * NFP;
  static constexpr int D_FP = D_CW + D_CWS, D_FA = D_FP + 6 * 3 * N * Q, D_FO = D_FA + 6 * Q * NP,
                       D_END = D_FO + 6 * NFP;
  static constexpr int D_PER = D_END | 1;
  static constexpr int C = 4, T = 32 * C;
  static constexpr size_t G_SMEM = (size_t)C * G_PER * sizeof(double);
  static constexpr size_t D_SMEM = (size_t)C * D_PER * sizeof(double);
};

struct PresTerms {
  int n = 0;
  double c[kMaxTerms];
  const double* f[kMaxTerms];
};

// y[cell][d][i] += sum_t c_t G(p_t)
template <int K>
__global__ void __launch_bounds__(MixQpCfg<K>::T) k_pgrad_qp(MeshArgs m, const double* __restrict__ gadv,
                                                              const double* __restrict__ gfw, PresTerms pt,
                                                              double* __restrict__ y) {
  using G = MixQpCfg<K>;
  constexpr int N = G::N, NP = G::NP, Q = G::Q, NB = G::NB, NBP = G::NBP, NF = G::NF, NFP = G::NFP, NQ = G::NQ,
                NQF = G::NQF;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
  const int cid = blockIdx.x * G::C + wc;
  if (cid >= m.ncells) return;
  double* cell = sm + wc * G::G_PER;
  double* P = cell + G::G_P;
  double* PF = cell + G::G_PF;
  double* OUT = cell + G::G_OUT;
  double* W = cell + G::G_CW;
  const FTab<N, Q>& tv = c_ft<N, Q>;    // velocity basis at the rule points (Q = N)
  const FTab<NP, Q>& tp = c_ft<NP, Q>;  // pressure basis at the rule points
  const double* ga = gadv + (size_t)cid * 9 * NQ;
  const double* gw = gfw + (size_t)cid * 18 * NQF;
  prefetch_l2(ga, 9 * NQ * sizeof(double), gadv, gadv + (size_t)m.ncells * 9 * NQ);
  prefetch_l2(gw, 18 * NQF * sizeof(double), gfw, gfw + (size_t)m.ncells * 18 * NQF);
  // ---- stage p = sum_t c_t p_t and the face-node means {p}
  for (int i = lane; i < NBP; i += 32) {
    double v = 0.0;
    for (int t = 0; t < pt.n; ++t) v = fma(pt.c[t], pt.f[t][(size_t)cid * NBP + i], v);
    P[i] = v;
  }
  __syncwarp();
  for (int it = lane; it < 6 * NFP; it += 32) {
    const int f = it / NFP, r = it - f * NFP, pp = r % NP, qq = r / NP;
    const int a = f >> 1, s = f & 1;
    const int nb = m.nbr[(size_t)cid * 6 + f];
    const double ps = P[face_node<NP>(a, s ? NP - 1 : 0, pp, qq)];
    double h;
    if (nb >= 0) {
      const int nn = face_node<NP>(a, s ? 0 : NP - 1, pp, qq);
      double po = 0.0;
      for (int t = 0; t < pt.n; ++t) po = fma(pt.c[t], __ldg(pt.f[t] + (size_t)nb * NBP + nn), po);
      h = 0.5 * (ps + po);
    } else {
      const int bid = -1 - nb;
      const bool outlet = bid >= 0 && bid < 64 && m.bctype[bid] == 1;
      h = outlet ? 0.0 : ps;
    }
    PF[it] = h;
  }
  // ---- p at the cell points: x and y passes (the z pass runs inside the pointwise stage)
  for (int jk = lane; jk < NFP; jk += 32) {
    double u[NP];
#pragma unroll
    for (int i = 0; i < NP; ++i) u[i] = P[i + NP * jk];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      double b = 0.0;
#pragma unroll
      for (int i = 0; i < NP; ++i) b = fma(tp.B[qx][i], u[i], b);
      W[G::G_X + qx * NFP + jk] = b;
    }
  }
  __syncwarp();
  // y pass through the work area; every lane then keeps its (qx, qy) columns in registers for
  // the three component passes below, which reuse the work area for their z-integrated arrays
  double vcol[(NQF + 31) / 32][NP];
  {
    for (int it = lane; it < Q * NP; it += 32) {
      const int qx = it / NP, k = it - qx * NP;
      double v[NP];
#pragma unroll
      for (int j = 0; j < NP; ++j) v[j] = W[G::G_X + qx * NFP + j + NP * k];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        double b = 0.0;
#pragma unroll
        for (int j = 0; j < NP; ++j) b = fma(tp.B[qy][j], v[j], b);
        W[G::G_Y + (qx * Q + qy) * NP + k] = b;
      }
    }
    __syncwarp();
#pragma unroll
    for (int rr = 0; rr < (NQF + 31) / 32; ++rr) {
      const int r = lane + 32 * rr;
#pragma unroll
      for (int k = 0; k < NP; ++k) vcol[rr][k] = r < NQF ? W[G::G_Y + r * NP + k] : 0.0;
    }
    __syncwarp();
  }
  // ---- face-point values of {p}: along p, then along q inside the flux stage
  for (int it = lane; it < 6 * NP; it += 32) {
    const int f = it / NP, q = it - f * NP;
    double v[NP];
#pragma unroll
    for (int pp = 0; pp < NP; ++pp) v[pp] = PF[f * NFP + pp + NP * q];
#pragma unroll
    for (int qp = 0; qp < Q; ++qp) {
      double b = 0.0;
#pragma unroll
      for (int pp = 0; pp < NP; ++pp) b = fma(tp.B[qp][pp], v[pp], b);
      cell[G::G_FP + (f * NP + q) * Q + qp] = b;
    }
  }
  __syncwarp();

#pragma unroll 1
  for (int d = 0; d < 3; ++d) {
    // ---- cell: p(q) (detJ w Jinv)[a][d] against the reference gradient tests
#pragma unroll
    for (int rr = 0; rr < (NQF + 31) / 32; ++rr) {
      const int r = lane + 32 * rr;
      if (r < NQF) {
        const int qx = r / Q, qy = r - qx * Q;
        double a0[N], a1[N], a2[N];
#pragma unroll
        for (int k = 0; k < N; ++k) a0[k] = a1[k] = a2[k] = 0.0;
#pragma unroll
        for (int qz = 0; qz < Q; ++qz) {
          double val = 0.0;
#pragma unroll
          for (int k = 0; k < NP; ++k) val = fma(tp.B[qz][k], vcol[rr][k], val);
          const int pnt = qx + Q * qy + Q * Q * qz;
          const double r0 = val * ga[(0 * 3 + d) * NQ + pnt], r1 = val * ga[(1 * 3 + d) * NQ + pnt],
                       r2 = val * ga[(2 * 3 + d) * NQ + pnt];
#pragma unroll
          for (int k = 0; k < N; ++k) {
            a0[k] = fma(tv.B[qz][k], r0, a0[k]);
            a1[k] = fma(tv.B[qz][k], r1, a1[k]);
            a2[k] = fma(tv.D[qz][k], r2, a2[k]);
          }
        }
#pragma unroll
        for (int k = 0; k < N; ++k) {
          W[G::G_A + r * N + k] = a0[k];
          W[G::G_A + NQF * N + r * N + k] = a1[k];
          W[G::G_A + 2 * NQF * N + r * N + k] = a2[k];
        }
      }
    }
    __syncwarp();
    for (int it = lane; it < Q * N; it += 32) {
      const int qx = it / N, k = it - qx * N;
      double p0[Q], p1[Q], p2[Q];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        const int o = (qx * Q + qy) * N + k;
        p0[qy] = W[G::G_A + o];
        p1[qy] = W[G::G_A + NQF * N + o];
        p2[qy] = W[G::G_A + 2 * NQF * N + o];
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        double s0 = 0.0, s12 = 0.0;
#pragma unroll
        for (int qy = 0; qy < Q; ++qy) {
          s0 = fma(tv.B[qy][j], p0[qy], s0);
          s12 = fma(tv.D[qy][j], p1[qy], fma(tv.B[qy][j], p2[qy], s12));
        }
        W[G::G_XI + qx * NF + j + N * k] = s0;
        W[G::G_XI + Q * NF + qx * NF + j + N * k] = s12;
      }
    }
    __syncwarp();
    for (int jk = lane; jk < NF; jk += 32) {
      double p0[Q], p12[Q];
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        p0[qx] = W[G::G_XI + qx * NF + jk];
        p12[qx] = W[G::G_XI + Q * NF + qx * NF + jk];
      }
#pragma unroll
      for (int i = 0; i < N; ++i) {
        double sacc = 0.0;
#pragma unroll
        for (int qx = 0; qx < Q; ++qx) sacc = fma(tv.D[qx][i], p0[qx], fma(tv.B[qx][i], p12[qx], sacc));
        OUT[i + N * jk] = sacc;
      }
    }
    // ---- faces: -{p} n_d ds w against the velocity traces
    for (int it = lane; it < 6 * Q; it += 32) {
      const int f = it / Q, qp = it - f * Q;
      double vs[NP], A[N];
#pragma unroll
      for (int q = 0; q < NP; ++q) vs[q] = cell[G::G_FP + (f * NP + q) * Q + qp];
#pragma unroll
      for (int b = 0; b < N; ++b) A[b] = 0.0;
#pragma unroll
      for (int qq = 0; qq < Q; ++qq) {
        double hv = 0.0;
#pragma unroll
        for (int q = 0; q < NP; ++q) hv = fma(tp.B[qq][q], vs[q], hv);
        const double fl = -hv * gw[(f * 3 + d) * NQF + qp + Q * qq];
#pragma unroll
        for (int b = 0; b < N; ++b) A[b] = fma(tv.B[qq][b], fl, A[b]);
      }
#pragma unroll
      for (int b = 0; b < N; ++b) cell[G::G_FA + (f * Q + qp) * N + b] = A[b];
    }
    __syncwarp();
    for (int it = lane; it < 6 * N; it += 32) {
      const int f = it / N, b = it - f * N;
      double av[Q];
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) av[qp] = cell[G::G_FA + (f * Q + qp) * N + b];
#pragma unroll
      for (int bp = 0; bp < N; ++bp) {
        double sacc = 0.0;
#pragma unroll
        for (int qp = 0; qp < Q; ++qp) sacc = fma(tv.B[qp][bp], av[qp], sacc);
        cell[G::G_FO + f * NF + bp + N * b] = sacc;
      }
    }
    __syncwarp();
    double* yc = y + ((size_t)cid * 3 + d) * NB;
    for (int n = lane; n < NB; n += 32) {
      double v = OUT[n];
      const int i = n % N, j = (n / N) % N, k = n / NF;
      const double* fo = cell + G::G_FO;
      if (i == 0) v += fo[0 * NF + j + N * k];
      if (i == N - 1) v += fo[1 * NF + j + N * k];
      if (j == 0) v += fo[2 * NF + i + N * k];
      if (j == N - 1) v += fo[3 * NF + i + N * k];
      if (k == 0) v += fo[4 * NF + i + N * j];
      if (k == N - 1) v += fo[5 * NF + i + N * j];
      yc[n] += v;
    }
    __syncwarp();
  }
}

// y[cell][i] = B(u)_i
template <int K>
__global__ void __launch_bounds__(MixQpCfg<K>::T) k_div_qp(MeshArgs m, const double* __restrict__ gadv,
                                                            const double* __restrict__ gfw,
                                                            const double* __restrict__ u, double* __restrict__ y) {
  using G = MixQpCfg<K>;
  constexpr int N = G::N, NP = G::NP, Q = G::Q, NB = G::NB, NBP = G::NBP, NF = G::NF, NFP = G::NFP, NQ = G::NQ,
                NQF = G::NQF;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
  const int cid = blockIdx.x * G::C + wc;
  if (cid >= m.ncells) return;
  double* cell = sm + wc * G::D_PER;
  double* U = cell + G::D_U;
  double* UF = cell + G::D_UF;
  double* OUT = cell + G::D_OUT;
  double* W = cell + G::D_CW;
  const FTab<N, Q>& tv = c_ft<N, Q>;
  const FTab<NP, Q>& tp = c_ft<NP, Q>;
  const double* ga = gadv + (size_t)cid * 9 * NQ;
  const double* gw = gfw + (size_t)cid * 18 * NQF;
  prefetch_l2(ga, 9 * NQ * sizeof(double), gadv, gadv + (size_t)m.ncells * 9 * NQ);
  prefetch_l2(gw, 18 * NQF * sizeof(double), gfw, gfw + (size_t)m.ncells * 18 * NQF);
  for (int i = lane; i < 3 * NB; i += 32) cp_async8(U + i, u + (size_t)cid * 3 * NB + i);
  cp_async_wait_all();
  __syncwarp();
  // ---- face-node means {u_d} (walls: the interior trace; outlets: none)
  for (int it = lane; it < 6 * 3 * NF; it += 32) {
    const int f = it / (3 * NF), r = it - f * 3 * NF, dd = r / NF, t = r - dd * NF, pp = t % N, qq = t / N;
    const int a = f >> 1, s = f & 1;
    const int nb = m.nbr[(size_t)cid * 6 + f];
    const double us = U[dd * NB + face_node<N>(a, s ? N - 1 : 0, pp, qq)];
    double h;
    if (nb >= 0) {
      h = 0.5 * (us + __ldg(u + (size_t)nb * 3 * NB + dd * NB + face_node<N>(a, s ? 0 : N - 1, pp, qq)));
    } else {
      const int bid = -1 - nb;
      const bool outlet = bid >= 0 && bid < 64 && m.bctype[bid] == 1;
      h = outlet ? 0.0 : us;
    }
    UF[it] = h;
  }
  // ---- u_d at the cell points: x / y passes per component
#pragma unroll 1
  for (int dd = 0; dd < 3; ++dd) {
    for (int jk = lane; jk < NF; jk += 32) {
      double v[N];
#pragma unroll
      for (int i = 0; i < N; ++i) v[i] = U[dd * NB + i + N * jk];
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) {
        double b = 0.0;
#pragma unroll
        for (int i = 0; i < N; ++i) b = fma(tv.B[qx][i], v[i], b);
        W[G::D_X + qx * NF + jk] = b;
      }
    }
    __syncwarp();
    for (int it = lane; it < Q * N; it += 32) {
      const int qx = it / N, k = it - qx * N;
      double v[N];
#pragma unroll
      for (int j = 0; j < N; ++j) v[j] = W[G::D_X + qx * NF + j + N * k];
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        double b = 0.0;
#pragma unroll
        for (int j = 0; j < N; ++j) b = fma(tv.B[qy][j], v[j], b);
        W[G::D_Y + dd * G::D_YS + (qx * Q + qy) * N + k] = b;
      }
    }
    __syncwarp();
  }
  // ---- pointwise: s_a = sum_d u_d (detJ w Jinv)[a][d], z-integrated against the pressure tests
  for (int r = lane; r < NQF; r += 32) {
    const int qx = r / Q, qy = r - qx * Q;
    double v[3][N], a0[NP], a1[NP], a2[NP];
#pragma unroll
    for (int dd = 0; dd < 3; ++dd)
#pragma unroll
      for (int k = 0; k < N; ++k) v[dd][k] = W[G::D_Y + dd * G::D_YS + r * N + k];
#pragma unroll
    for (int k = 0; k < NP; ++k) a0[k] = a1[k] = a2[k] = 0.0;
#pragma unroll
    for (int qz = 0; qz < Q; ++qz) {
      const int pnt = qx + Q * qy + Q * Q * qz;
      double r0 = 0.0, r1 = 0.0, r2 = 0.0;
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) {
        double val = 0.0;
#pragma unroll
        for (int k = 0; k < N; ++k) val = fma(tv.B[qz][k], v[dd][k], val);
        r0 = fma(val, ga[(0 * 3 + dd) * NQ + pnt], r0);
        r1 = fma(val, ga[(1 * 3 + dd) * NQ + pnt], r1);
        r2 = fma(val, ga[(2 * 3 + dd) * NQ + pnt], r2);
      }
#pragma unroll
      for (int k = 0; k < NP; ++k) {
        a0[k] = fma(tp.B[qz][k], r0, a0[k]);
        a1[k] = fma(tp.B[qz][k], r1, a1[k]);
        a2[k] = fma(tp.D[qz][k], r2, a2[k]);
      }
    }
#pragma unroll
    for (int k = 0; k < NP; ++k) {
      W[G::D_A + r * NP + k] = a0[k];
      W[G::D_A + NQF * NP + r * NP + k] = a1[k];
      W[G::D_A + 2 * NQF * NP + r * NP + k] = a2[k];
    }
  }
  __syncwarp();
  for (int it = lane; it < Q * NP; it += 32) {
    const int qx = it / NP, k = it - qx * NP;
    double p0[Q], p1[Q], p2[Q];
#pragma unroll
    for (int qy = 0; qy < Q; ++qy) {
      const int o = (qx * Q + qy) * NP + k;
      p0[qy] = W[G::D_A + o];
      p1[qy] = W[G::D_A + NQF * NP + o];
      p2[qy] = W[G::D_A + 2 * NQF * NP + o];
    }
#pragma unroll
    for (int j = 0; j < NP; ++j) {
      double s0 = 0.0, s12 = 0.0;
#pragma unroll
      for (int qy = 0; qy < Q; ++qy) {
        s0 = fma(tp.B[qy][j], p0[qy], s0);
        s12 = fma(tp.D[qy][j], p1[qy], fma(tp.B[qy][j], p2[qy], s12));
      }
      W[G::D_XI + qx * NFP + j + NP * k] = s0;
      W[G::D_XI + Q * NFP + qx * NFP + j + NP * k] = s12;
    }
  }
  __syncwarp();
  for (int jk = lane; jk < NFP; jk += 32) {
    double p0[Q], p12[Q];
#pragma unroll
    for (int qx = 0; qx < Q; ++qx) {
      p0[qx] = W[G::D_XI + qx * NFP + jk];
      p12[qx] = W[G::D_XI + Q * NFP + qx * NFP + jk];
    }
#pragma unroll
    for (int i = 0; i < NP; ++i) {
      double sacc = 0.0;
#pragma unroll
      for (int qx = 0; qx < Q; ++qx) sacc = fma(tp.D[qx][i], p0[qx], fma(tp.B[qx][i], p12[qx], sacc));
      OUT[i + NP * jk] = sacc;
    }
  }
  // ---- faces: -{u}.n ds w against the pressure traces
  for (int it = lane; it < 6 * 3 * N; it += 32) {
    const int f = it / (3 * N), r = it - f * 3 * N, dd = r / N, q = r - dd * N;
    double v[N];
#pragma unroll
    for (int pp = 0; pp < N; ++pp) v[pp] = UF[(f * 3 + dd) * NF + pp + N * q];
#pragma unroll
    for (int qp = 0; qp < Q; ++qp) {
      double b = 0.0;
#pragma unroll
      for (int pp = 0; pp < N; ++pp) b = fma(tv.B[qp][pp], v[pp], b);
      cell[G::D_FP + ((f * 3 + dd) * N + q) * Q + qp] = b;
    }
  }
  __syncwarp();
  for (int it = lane; it < 6 * Q; it += 32) {
    const int f = it / Q, qp = it - f * Q;
    double vs[3][N], A[NP];
#pragma unroll
    for (int dd = 0; dd < 3; ++dd)
#pragma unroll
      for (int q = 0; q < N; ++q) vs[dd][q] = cell[G::D_FP + ((f * 3 + dd) * N + q) * Q + qp];
#pragma unroll
    for (int b = 0; b < NP; ++b) A[b] = 0.0;
#pragma unroll
    for (int qq = 0; qq < Q; ++qq) {
      double un = 0.0;
#pragma unroll
      for (int dd = 0; dd < 3; ++dd) {
        double val = 0.0;
#pragma unroll
        for (int q = 0; q < N; ++q) val = fma(tv.B[qq][q], vs[dd][q], val);
        un = fma(val, gw[(f * 3 + dd) * NQF + qp + Q * qq], un);
      }
#pragma unroll
      for (int b = 0; b < NP; ++b) A[b] = fma(tp.B[qq][b], -un, A[b]);
    }
#pragma unroll
    for (int b = 0; b < NP; ++b) cell[G::D_FA + (f * Q + qp) * NP + b] = A[b];
  }
  __syncwarp();
  for (int it = lane; it < 6 * NP; it += 32) {
    const int f = it / NP, b = it - f * NP;
    double av[Q];
#pragma unroll
    for (int qp = 0; qp < Q; ++qp) av[qp] = cell[G::D_FA + (f * Q + qp) * NP + b];
#pragma unroll
    for (int bp = 0; bp < NP; ++bp) {
      double sacc = 0.0;
#pragma unroll
      for (int qp = 0; qp < Q; ++qp) sacc = fma(tp.B[qp][bp], av[qp], sacc);
      cell[G::D_FO + f * NFP + bp + NP * b] = sacc;
    }
  }
  __syncwarp();
  for (int n = lane; n < NBP; n += 32) {
    double v = OUT[n];
    const int i = n % NP, j = (n / NP) % NP, k = n / NFP;
    const double* fo = cell + G::D_FO;
    if (i == 0) v += fo[0 * NFP + j + NP * k];
    if (i == NP - 1) v += fo[1 * NFP + j + NP * k];
    if (j == 0) v += fo[2 * NFP + i + NP * k];
    if (j == NP - 1) v += fo[3 * NFP + i + NP * k];
    if (k == 0) v += fo[4 * NFP + i + NP * j];
    if (k == NP - 1) v += fo[5 * NFP + i + NP * j];
    y[(size_t)cid * NBP + n] = v;
  }
}

}  // namespace dgb

namespace dgb {

// ===========================================================================
// Momentum diagonal on deformed hexahedra (momentum_diagonal, forms.cpp:606-810)
// ===========================================================================
// Exact diagonal, sum-factorised: for basis function i = (ix, iy, iz) every integrand is a
// product of per-direction factors B^2, D^2 or B D at the quadrature points times a
// per-point weight, so each term is a tensor contraction of a Q^3 (cell) or Q^2 (face)
// weight field with those squared tables:
//   cell, rule k+1: mass detJw B^2B^2B^2 + visc sum_ab G_ab dphi_a dphi_b (G = the compact
//         metric detJw Jinv Jinv^T);
//   cell, rule k+2: sum_a Wt_a phi dphi_a (Wt from qp_w_phase: -adv detJw Jinv w);
//   faces (face-layer nodes only, outward normal, element-centric as in the apply):
//         rule k+1 visc (C' phi^2 - c1 phi (Jinv n . grad_ref phi)) w ds with C' = the
//         interior penalty / 2 sigma_K and c1 = 1 / 2 (interior / Dirichlet wall; outlets
//         none), rule k+2 a_s phi^2 (a_s from qp_w_phase).
// The value is the same for all three components (forms.cpp:635).  skew != 0: generic.
// SCALAR: the scalar SIP diagonal (pressure Helmholtz / Laplacian, helmholtz_diagonal
// forms.cpp:246-334) through the same stages: K = kp, rule kp+2, no advection, one
// component; boundary faces all Dirichlet (sdir = 1) or all natural (sdir = 0).
template <int K, bool SCALAR = false>
struct MomDiagQpCfg {
  static constexpr int N = K + 1, QA = SCALAR ? K + 2 : K + 1, QB = K + 2, NB = N * N * N, NF = N * N;
  static constexpr int NQA = QA * QA * QA, NQFA = QA * QA, NQB = QB * QB * QB, NQFB = QB * QB;
  // W phase (as MomQpCfg)
  static constexpr int BX = 0, BY = BX + QB * NF, FPW = 0, NW = FPW + 6 * 2 * 3 * N * QB;
  static constexpr int mx(int a, int b) { return a > b ? a : b; }
  // diagonal stages (after the W phase): cell z-stage [6][QA^2][N] -> y-stage [3][QA][N^2];
  // adv z-stage [3][QB^2][N] -> y-stage [2][QB][N^2]; faces: visc Y [6][3][QA][N], adv Y [6][QB][N]
  static constexpr int CZ = 0, CY = CZ + 6 * QA * QA * N, C_END = CY + 3 * QA * NF;
  static constexpr int AZ = 0, AY = AZ + 3 * QB * QB * N, A_END = AY + 2 * QB * NF;
  static constexpr int FV = 0, FA = FV + 6 * 3 * QA * N, FO = FA + 6 * QB * N, F_END = FO + 6 * NF;
  static constexpr int WORK = mx(mx(NW + 6 * 3 * NF, BY + QB * QB * N), mx(C_END, mx(A_END, F_END)));
  // per cell: nb | type | pen | WT | FC (advecting field staged here first) | D | WORK
  static constexpr int O_NB = 0, O_TY = 6, O_PEN = 12, O_WT = 18, O_FC = O_WT + 3 * NQB, O_WS = O_FC,
                       O_D = O_FC + 2 * 6 * NQFB, O_WK = O_D + NB;
  static_assert(3 * NB <= 2 * 6 * NQFB, "advecting field must fit in FC");
  static constexpr int PER = (O_WK + WORK) | 1;
  static constexpr int C_FIT = (227 * 1024 / 8) / PER;
  static constexpr int C = C_FIT > 8 ? 8 : C_FIT, T = 32 * C;
  static constexpr size_t SMEM = (size_t)C * PER * sizeof(double);
};

template <int K, bool SCALAR = false>
__global__ void __launch_bounds__(MomDiagQpCfg<K, SCALAR>::T) k_momentum_diag_qp(
    MeshArgs m, const double* __restrict__ gcA, const double* __restrict__ gfA, const double* __restrict__ gadv,
    const double* __restrict__ gfw, MomCoef co, const double* __restrict__ w, double* __restrict__ y,
    int sdir = 0) {
  using G = MomDiagQpCfg<K, SCALAR>;
  constexpr int N = G::N, QA = G::QA, QB = G::QB, NB = G::NB, NF = G::NF;
  constexpr int NQA = G::NQA, NQFA = G::NQFA, NQB = G::NQB, NQFB = G::NQFB, C = G::C, PER = G::PER;
  extern __shared__ double sm[];
  DGB_POISON_SMEM(m, sm);
  const int c0 = blockIdx.x * C;
  const int nc = min(C, m.ncells - c0);
  const int tid = threadIdx.x, lane = tid & 31, wc = tid >> 5;
  const bool adv = !SCALAR && co.adv != 0.0;
  const double sfac = (double)(N * N);
  for (int idx = tid; adv && idx < nc * 3 * NB; idx += G::T) {
    const int c = idx / (3 * NB), i = idx - c * 3 * NB;
    cp_async8(sm + c * PER + G::O_WS + i, w + (size_t)c0 * 3 * NB + idx);
  }
  for (int idx = tid; idx < nc * 6; idx += G::T) {
    const int c = idx / 6, f = idx - c * 6;
    double* cell = sm + c * PER;
    const int nb = m.nbr[(size_t)(c0 + c) * 6 + f];
    int ty = 0;
    if (nb < 0) {
      const int bid = -1 - nb;
      ty = SCALAR ? (sdir ? 1 : 2) : ((bid >= 0 && bid < 64 && m.bctype[bid] == 1) ? 2 : 1);
    }
    cell[G::O_NB + f] = (double)nb;
    cell[G::O_TY + f] = (double)ty;
    cell[G::O_PEN + f] = sfac * m.pen[(size_t)(c0 + c) * 6 + f];
  }
  cp_async_wait_all();
  __syncthreads();
  if (wc >= nc) return;
  const int cid = c0 + wc;
  double* cell = sm + wc * PER;
  double* WT = cell + G::O_WT;
  double* FC = cell + G::O_FC;
  double* D = cell + G::O_D;
  double* W = cell + G::O_WK;
  const double* nbv = cell + G::O_NB;
  const double* tyv = cell + G::O_TY;
  const FTab<N, QA>& ta = c_ft<N, QA>;
  const FTab<N, QB>& tb = c_ft<N, QB>;
  if (!SCALAR && adv)
    qp_w_phase<N, QB, G::BX, G::BY, G::FPW, G::NW>(cell + G::O_WS, W, WT, FC, nbv, tyv, w,
                                                   gadv + (size_t)cid * 9 * NQB, gfw + (size_t)cid * 18 * NQFB,
                                                   co.adv, lane);
  // ---- cell, rule k+1: z-contraction per (qx, qy) column of the six weight fields
  {
    const double* gc = gcA + (size_t)cid * NQA * 7;  // [7][qx][qy][qz] (see context.cu)
    for (int r = lane; r < QA * QA; r += 32) {
      double t[6][N];
#pragma unroll
      for (int j = 0; j < 6; ++j)
#pragma unroll
        for (int k = 0; k < N; ++k) t[j][k] = 0.0;
#pragma unroll
      for (int qz = 0; qz < QA; ++qz) {
        const double* g = gc + r + QA * QA * qz;
        const double g00 = __ldg(g), g01 = __ldg(g + NQA), g02 = __ldg(g + 2 * NQA), g11 = __ldg(g + 3 * NQA),
                     g12 = __ldg(g + 4 * NQA), g22 = __ldg(g + 5 * NQA), jxw = __ldg(g + 6 * NQA);
        const double vm = co.mass * jxw, v00 = co.visc * g00, v11 = co.visc * g11, v22 = co.visc * g22,
                     v01 = 2.0 * co.visc * g01, v02 = 2.0 * co.visc * g02, v12 = 2.0 * co.visc * g12;
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double b = ta.B[qz][k], d = ta.D[qz][k], b2 = b * b, d2 = d * d, bd = b * d;
          t[0][k] = fma(b2, vm, fma(d2, v22, t[0][k]));  // -> y B^2, x B^2 (mass + G22)
          t[1][k] = fma(b2, v00, t[1][k]);               // G00: y B^2, x D^2
          t[2][k] = fma(b2, v11, t[2][k]);               // G11: y D^2, x B^2
          t[3][k] = fma(b2, v01, t[3][k]);               // G01: y BD, x BD
          t[4][k] = fma(bd, v02, t[4][k]);               // G02: y B^2, x BD
          t[5][k] = fma(bd, v12, t[5][k]);               // G12: y BD, x B^2
        }
      }
#pragma unroll
      for (int j = 0; j < 6; ++j)
#pragma unroll
        for (int k = 0; k < N; ++k) W[G::CZ + (j * QA * QA + r) * N + k] = t[j][k];
    }
    __syncwarp();
    for (int it = lane; it < QA * N; it += 32) {  // y-contraction: items (qx, iz)
      const int qx = it / N, k = it - qx * N;
      double xb2[N], xd2[N], xbd[N];
#pragma unroll
      for (int j = 0; j < N; ++j) xb2[j] = xd2[j] = xbd[j] = 0.0;
#pragma unroll
      for (int qy = 0; qy < QA; ++qy) {
        const int o = (qx * QA + qy) * N + k;
        const double a0 = W[G::CZ + 0 * QA * QA * N + o], a1 = W[G::CZ + 1 * QA * QA * N + o],
                     a2 = W[G::CZ + 2 * QA * QA * N + o], a3 = W[G::CZ + 3 * QA * QA * N + o],
                     a4 = W[G::CZ + 4 * QA * QA * N + o], a5 = W[G::CZ + 5 * QA * QA * N + o];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double b = ta.B[qy][j], d = ta.D[qy][j], b2 = b * b, d2 = d * d, bd = b * d;
          xb2[j] = fma(b2, a0, fma(d2, a2, fma(bd, a5, xb2[j])));
          xd2[j] = fma(b2, a1, xd2[j]);
          xbd[j] = fma(bd, a3, fma(b2, a4, xbd[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        W[G::CY + 0 * QA * NF + qx * NF + j + N * k] = xb2[j];
        W[G::CY + 1 * QA * NF + qx * NF + j + N * k] = xd2[j];
        W[G::CY + 2 * QA * NF + qx * NF + j + N * k] = xbd[j];
      }
    }
    __syncwarp();
    for (int jk = lane; jk < NF; jk += 32) {  // x-contraction -> D
      double s[N];
#pragma unroll
      for (int i = 0; i < N; ++i) s[i] = 0.0;
#pragma unroll
      for (int qx = 0; qx < QA; ++qx) {
        const double xb2 = W[G::CY + qx * NF + jk], xd2 = W[G::CY + QA * NF + qx * NF + jk],
                     xbd = W[G::CY + 2 * QA * NF + qx * NF + jk];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double b = ta.B[qx][i], d = ta.D[qx][i];
          s[i] = fma(b * b, xb2, fma(d * d, xd2, fma(b * d, xbd, s[i])));
        }
      }
#pragma unroll
      for (int i = 0; i < N; ++i) D[i + N * jk] = s[i];
    }
    __syncwarp();
  }
  // ---- cell, rule k+2: advection sum_a Wt_a phi dphi_a
  if (adv) {
    for (int r = lane; r < QB * QB; r += 32) {
      const int qx = r / QB, qy = r - qx * QB;
      double u0[N], u1[N], u2[N];
#pragma unroll
      for (int k = 0; k < N; ++k) u0[k] = u1[k] = u2[k] = 0.0;
#pragma unroll
      for (int qz = 0; qz < QB; ++qz) {
        const int pt = qx + QB * qy + QB * QB * qz;
        const double w0 = WT[pt], w1 = WT[NQB + pt], w2 = WT[2 * NQB + pt];
#pragma unroll
        for (int k = 0; k < N; ++k) {
          const double b = tb.B[qz][k], d = tb.D[qz][k], b2 = b * b;
          u0[k] = fma(b2, w0, u0[k]);     // term 0: x BD, y B^2
          u1[k] = fma(b2, w1, u1[k]);     // term 1: x B^2, y BD
          u2[k] = fma(b * d, w2, u2[k]);  // term 2: x B^2, y B^2
        }
      }
#pragma unroll
      for (int k = 0; k < N; ++k) {
        W[G::AZ + (0 * QB * QB + r) * N + k] = u0[k];
        W[G::AZ + (1 * QB * QB + r) * N + k] = u1[k];
        W[G::AZ + (2 * QB * QB + r) * N + k] = u2[k];
      }
    }
    __syncwarp();
    for (int it = lane; it < QB * N; it += 32) {
      const int qx = it / N, k = it - qx * N;
      double xbd[N], xb2[N];
#pragma unroll
      for (int j = 0; j < N; ++j) xbd[j] = xb2[j] = 0.0;
#pragma unroll
      for (int qy = 0; qy < QB; ++qy) {
        const int o = (qx * QB + qy) * N + k;
        const double a0 = W[G::AZ + o], a1 = W[G::AZ + QB * QB * N + o], a2 = W[G::AZ + 2 * QB * QB * N + o];
#pragma unroll
        for (int j = 0; j < N; ++j) {
          const double b = tb.B[qy][j], d = tb.D[qy][j], b2 = b * b;
          xbd[j] = fma(b2, a0, xbd[j]);
          xb2[j] = fma(b * d, a1, fma(b2, a2, xb2[j]));
        }
      }
#pragma unroll
      for (int j = 0; j < N; ++j) {
        W[G::AY + qx * NF + j + N * k] = xbd[j];
        W[G::AY + QB * NF + qx * NF + j + N * k] = xb2[j];
      }
    }
    __syncwarp();
    for (int jk = lane; jk < NF; jk += 32) {
      double s[N];
#pragma unroll
      for (int i = 0; i < N; ++i) s[i] = D[i + N * jk];
#pragma unroll
      for (int qx = 0; qx < QB; ++qx) {
        const double xbd = W[G::AY + qx * NF + jk], xb2 = W[G::AY + QB * NF + qx * NF + jk];
#pragma unroll
        for (int i = 0; i < N; ++i) {
          const double b = tb.B[qx][i], d = tb.D[qx][i];
          s[i] = fma(b * d, xbd, fma(b * b, xb2, s[i]));
        }
      }
#pragma unroll
      for (int i = 0; i < N; ++i) D[i + N * jk] = s[i];
    }
    __syncwarp();
  }
  // ---- faces: face-layer nodes (p, q); viscous at rule k+1, Lax-Friedrichs at rule k+2
  {
    const double* gf = gfA + (size_t)cid * 6 * NQFA * 7;  // [f][7][qp + Q qq]
    for (int it = lane; it < 6 * QA; it += 32) {  // V1: along the second tangential axis
      const int f = it / QA, tp = it - f * QA;
      const int a = f >> 1, s = f & 1, ty = (int)tyv[f];
      const int t1 = a == 0 ? 1 : 0, t2 = a == 2 ? 1 : 2;
      const bool act = co.visc != 0.0 && ty != 2;
      const double c1 = ty == 0 ? 1.0 : 2.0, cp = (ty == 0 ? 1.0 : 2.0) * cell[G::O_PEN + f];
      const double dEL = ta.dE[s][s ? N - 1 : 0];
      double ya[N], yb[N], yc[N];
#pragma unroll
      for (int q = 0; q < N; ++q) ya[q] = yb[q] = yc[q] = 0.0;
      if (act) {
        const double* g = gf + (size_t)f * 7 * NQFA;
#pragma unroll
        for (int tq = 0; tq < QA; ++tq) {
          const int t = tp + QA * tq;
          double jn[3];
#pragma unroll
          for (int d = 0; d < 3; ++d) jn[d] = __ldg(g + d * NQFA + t);
          const double wds = __ldg(g + 6 * NQFA + t);
          const double wA = co.visc * wds * (cp - c1 * dEL * jn[a]);
          const double wB = -co.visc * c1 * wds * jn[t1];
          const double wC = -co.visc * c1 * wds * jn[t2];
#pragma unroll
          for (int q = 0; q < N; ++q) {
            const double b = ta.B[tq][q], d = ta.D[tq][q];
            ya[q] = fma(b * b, wA, ya[q]);
            yb[q] = fma(b * b, wB, yb[q]);
            yc[q] = fma(b * d, wC, yc[q]);
          }
        }
      }
#pragma unroll
      for (int q = 0; q < N; ++q) {
        W[G::FV + ((f * 3 + 0) * QA + tp) * N + q] = ya[q] + yc[q];
        W[G::FV + ((f * 3 + 1) * QA + tp) * N + q] = yb[q];
      }
    }
    for (int it = lane; adv && it < 6 * QB; it += 32) {  // A1
      const int f = it / QB, tp = it - f * QB;
      double ya[N];
#pragma unroll
      for (int q = 0; q < N; ++q) ya[q] = 0.0;
#pragma unroll
      for (int tq = 0; tq < QB; ++tq) {
        const double as = FC[f * NQFB + tp + QB * tq];
#pragma unroll
        for (int q = 0; q < N; ++q) ya[q] = fma(tb.B[tq][q] * tb.B[tq][q], as, ya[q]);
      }
#pragma unroll
      for (int q = 0; q < N; ++q) W[G::FA + (f * QB + tp) * N + q] = ya[q];
    }
    __syncwarp();
    for (int it = lane; it < 6 * N; it += 32) {  // V2 / A2: along the first tangential axis
      const int f = it / N, q = it - f * N;
      double o[N];
#pragma unroll
      for (int p = 0; p < N; ++p) o[p] = 0.0;
#pragma unroll
      for (int tp = 0; tp < QA; ++tp) {
        const double yac = W[G::FV + ((f * 3 + 0) * QA + tp) * N + q], yb = W[G::FV + ((f * 3 + 1) * QA + tp) * N + q];
#pragma unroll
        for (int p = 0; p < N; ++p) {
          const double b = ta.B[tp][p], d = ta.D[tp][p];
          o[p] = fma(b * b, yac, fma(b * d, yb, o[p]));
        }
      }
      if (adv) {
#pragma unroll
        for (int tp = 0; tp < QB; ++tp) {
          const double ya = W[G::FA + (f * QB + tp) * N + q];
#pragma unroll
          for (int p = 0; p < N; ++p) o[p] = fma(tb.B[tp][p] * tb.B[tp][p], ya, o[p]);
        }
      }
#pragma unroll
      for (int p = 0; p < N; ++p) W[G::FO + f * NF + p + N * q] = o[p];
    }
    __syncwarp();
  }
  // ---- store: cell + face-layer contributions, the same value for the three components
  double* yc = y + (size_t)cid * (SCALAR ? 1 : 3) * NB;
  for (int n = lane; n < NB; n += 32) {
    const int i = n % N, j = (n / N) % N, k = n / NF;
    const double* fo = W + G::FO;
    double v = D[n];
    if (i == 0) v += fo[0 * NF + j + N * k];
    if (i == N - 1) v += fo[1 * NF + j + N * k];
    if (j == 0) v += fo[2 * NF + i + N * k];
    if (j == N - 1) v += fo[3 * NF + i + N * k];
    if (k == 0) v += fo[4 * NF + i + N * j];
    if (k == N - 1) v += fo[5 * NF + i + N * j];
    yc[n] = v;
    if (!SCALAR) {
      yc[NB + n] = v;
      yc[2 * NB + n] = v;
    }
  }
}

// ===========================================================================
// Mass (apply_mass, forms.cpp:337-360) on deformed cells: y = B^T diag(detJ w) B x per
// component at rule Q, sum-factorised (three forward line passes N -> Q, the pointwise
// detJ w, three transposed passes Q -> N), detJ w read from the compact per-qp record
// (plane 6 of qcm[Q], [qx Q + qy + Q^2 qz]) — the generic kernel re-reads the full
// 10-double record per point and component.  One warp per cell, NC components at once;
// each line stage works in place on a Q^3 tile per component (a line is read whole
// into registers before its Q outputs are written).
// ===========================================================================
template <int N, int Q, int NC>
struct MassQpCfg {
  static constexpr int NB = N * N * N, NQ = Q * Q * Q, W = 4, T = 32 * W;
  static constexpr int S = NQ | 1;  // odd component stride
};
template <int N, int Q, int NC>
__global__ void __launch_bounds__(MassQpCfg<N, Q, NC>::T, 1) k_mass_qp(MeshArgs m, const double* __restrict__ gc,
                                                                     const double* __restrict__ x,
                                                                     double* __restrict__ y) {
  if (m.skip && *m.skip) return;
  using G = MassQpCfg<N, Q, NC>;
  constexpr int NB = G::NB, NQ = G::NQ, S = G::S, QQ = Q * Q;
  __shared__ double sm[G::W][NC * S];
  const FTab<N, Q>& tb = c_ft<N, Q>;
  const int lane = threadIdx.x & 31, wc = threadIdx.x >> 5;
  const int cell = blockIdx.x * G::W + wc;
  if (cell >= m.ncells) return;  // warp-uniform; no CTA barrier below
  double* t = sm[wc];
  const double* xc = x + (size_t)cell * NC * NB;
  constexpr int LX = (NC * NB + 31) / 32, LQ = (NQ + 31) / 32;
  double xv[LX], jv[LQ];  // every global load of the cell issued before the first use
  const double* jw = gc + (size_t)cell * 7 * NQ + 6 * NQ;
#pragma unroll
  for (int j = 0; j < LX; ++j) {
    const int i = lane + 32 * j;
    xv[j] = i < NC * NB ? __ldg(xc + i) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < LQ; ++j) {
    const int i = lane + 32 * j;
    const int qx = i % Q, qy = (i / Q) % Q, qz = i / QQ;
    jv[j] = i < NQ ? __ldg(jw + qx * Q + qy + QQ * qz) : 0.0;
  }
#pragma unroll
  for (int j = 0; j < LX; ++j) {
    const int i = lane + 32 * j;
    if (i < NC * NB) {
      const int comp = i / NB, r = i - comp * NB;
      t[comp * S + r % N + Q * ((r / N) % N) + QQ * (r / (N * N))] = xv[j];
    }
  }
  __syncwarp();
  // forward: lines (comp, a, b) along dir with stride st; a < A, b < Bn
  auto fwd = [&](int st, int sa, int A, int sb, int Bn) {
#pragma unroll 1
    for (int it = lane; it < NC * A * Bn; it += 32) {
      const int comp = it / (A * Bn), r = it - comp * A * Bn;
      double* ln = t + comp * S + (r % A) * sa + (r / A) * sb;
      double u[N];
#pragma unroll
      for (int l = 0; l < N; ++l) u[l] = ln[l * st];
#pragma unroll
      for (int q = 0; q < Q; ++q) {
        double v = 0.0;
#pragma unroll
        for (int l = 0; l < N; ++l) v = fma(tb.B[q][l], u[l], v);
        ln[q * st] = v;
      }
    }
    __syncwarp();
  };
  auto bwd = [&](int st, int sa, int A, int sb, int Bn) {
#pragma unroll 1
    for (int it = lane; it < NC * A * Bn; it += 32) {
      const int comp = it / (A * Bn), r = it - comp * A * Bn;
      double* ln = t + comp * S + (r % A) * sa + (r / A) * sb;
      double v[Q];
#pragma unroll
      for (int q = 0; q < Q; ++q) v[q] = ln[q * st];
#pragma unroll
      for (int l = 0; l < N; ++l) {
        double u = 0.0;
#pragma unroll
        for (int q = 0; q < Q; ++q) u = fma(tb.B[q][l], v[q], u);
        ln[l * st] = u;
      }
    }
    __syncwarp();
  };
  fwd(1, Q, N, QQ, N);   // x-lines (iy, iz)
  fwd(Q, 1, Q, QQ, N);   // y-lines (qx, iz)
  fwd(QQ, 1, Q, Q, Q);   // z-lines (qx, qy)
#pragma unroll
  for (int j = 0; j < LQ; ++j) {
    const int i = lane + 32 * j;
    if (i < NQ)
#pragma unroll
      for (int comp = 0; comp < NC; ++comp) t[comp * S + i] *= jv[j];
  }
  __syncwarp();
  bwd(QQ, 1, Q, Q, Q);   // z-lines (qx, qy)
  bwd(Q, 1, Q, QQ, N);   // y-lines (qx, iz)
  bwd(1, Q, N, QQ, N);   // x-lines (iy, iz)
  double* yc = y + (size_t)cell * NC * NB;
#pragma unroll
  for (int i = lane; i < NC * NB; i += 32) {
    const int comp = i / NB, r = i - comp * NB;
    yc[i] = t[comp * S + r % N + Q * ((r / N) % N) + QQ * (r / (N * N))];
  }
}

}  // namespace dgb
