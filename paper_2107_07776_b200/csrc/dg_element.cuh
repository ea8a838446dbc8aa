// Sum-factorised evaluate / integrate of one DG element (cell or face trace)
// for a batch of cells staged in shared memory.  Generic in DIM (2, 3) with
// 2D handled as 3D with a unit z extent.
//
// Cell:  values + reference gradients at the tensor Gauss rule (the work of
//        Eval::values/gradients, proj/src/forms.cpp:39-60) and the transposed
//        integration against values + reference gradients of the test basis
//        (TestAcc::flush, forms.cpp:90-108).
// Face:  the same through the face-embedded tables (space.cpp:216-237): with a
//        Gauss-Lobatto nodal basis the trace is the face layer and the normal
//        derivative is one 1xN contraction with phi'(0|1), then tangential
//        1D contractions.
#pragma once

#include "dg_common.cuh"

namespace dgb {

template <int DIM, int N, int Q>
struct Elem {
  static constexpr int ZN = DIM == 3 ? N : 1;
  static constexpr int ZQ = DIM == 3 ? Q : 1;
  static constexpr int NB = N * N * ZN;         // basis functions per component
  static constexpr int NQ = Q * Q * ZQ;         // cell quadrature points
  static constexpr int NQF = DIM == 3 ? Q * Q : Q;  // face quadrature points
  static constexpr int NBF = DIM == 3 ? N * N : N;  // face-layer nodes
  static constexpr int QB = (1 + DIM) * NQ;     // cell qp block: V, G_0..G_{DIM-1}
  static constexpr int FB = (1 + DIM) * NQF;    // face qp block
  // scratch (per cell) for the cell pass: X1, X2 [Q N ZN], Y1..Y3 [Q Q ZN]
  static constexpr int SX = Q * N * ZN;
  static constexpr int SY = Q * Q * ZN;
  static constexpr int SCR_CELL = 2 * SX + (DIM == 3 ? 3 * SY : 0);
  // scratch for a face: T0, T1 [NBF], P1..P3 [Q N] (3D)
  static constexpr int SCR_FACE = 2 * NBF + (DIM == 3 ? 3 * Q * N : 0);
  static constexpr int SCR = SCR_CELL > SCR_FACE ? SCR_CELL : SCR_FACE;

  // --------------------------------------------------------------- cell
  // u: [nc][cs_u] (NB used); scr: [nc][SCR]; qb: [nc][QB] -> V (+ G_a if GRAD)
  template <bool GRAD>
  __device__ static void eval_cell(const double* u, int cs_u, double* scr, double* qb, int nc) {
    double* X1 = scr;
    double* X2 = scr + SX;
    double* V = qb;
    double* G0 = qb + NQ;
    double* G1 = qb + 2 * NQ;
    contract<0, N, N, ZN, Q, false, MB<N, Q>>(u, cs_u, X1, SCR, nc);
    if (GRAD) contract<0, N, N, ZN, Q, false, MD<N, Q>>(u, cs_u, X2, SCR, nc);
    __syncthreads();
    if constexpr (DIM == 2) {
      contract<1, Q, N, 1, Q, false, MB<N, Q>>(X1, SCR, V, QB, nc);
      if (GRAD) {
        contract<1, Q, N, 1, Q, false, MD<N, Q>>(X1, SCR, G1, QB, nc);
        contract<1, Q, N, 1, Q, false, MB<N, Q>>(X2, SCR, G0, QB, nc);
      }
      __syncthreads();
    } else {
      double* Y1 = scr + 2 * SX;
      double* Y2 = Y1 + SY;
      double* Y3 = Y2 + SY;
      double* G2 = qb + 3 * NQ;
      contract<1, Q, N, N, Q, false, MB<N, Q>>(X1, SCR, Y1, SCR, nc);
      if (GRAD) {
        contract<1, Q, N, N, Q, false, MD<N, Q>>(X1, SCR, Y2, SCR, nc);
        contract<1, Q, N, N, Q, false, MB<N, Q>>(X2, SCR, Y3, SCR, nc);
      }
      __syncthreads();
      contract<2, Q, Q, N, Q, false, MB<N, Q>>(Y1, SCR, V, QB, nc);
      if (GRAD) {
        contract<2, Q, Q, N, Q, false, MD<N, Q>>(Y1, SCR, G2, QB, nc);
        contract<2, Q, Q, N, Q, false, MB<N, Q>>(Y2, SCR, G1, QB, nc);
        contract<2, Q, Q, N, Q, false, MB<N, Q>>(Y3, SCR, G0, QB, nc);
      }
      __syncthreads();
    }
  }

  // out[nc][cs_o] (+)= B^T V + sum_a D_a^T G_a  (qb holds the test integrands)
  template <bool GRAD, bool ACC>
  __device__ static void integrate_cell(const double* qb, double* scr, double* out, int cs_o, int nc) {
    double* X1 = scr;
    double* X2 = scr + SX;
    const double* V = qb;
    const double* G0 = qb + NQ;
    const double* G1 = qb + 2 * NQ;
    if constexpr (DIM == 2) {
      if (GRAD) {
        contract2<1, Q, Q, 1, N, false, MBt<N, Q>, MDt<N, Q>>(V, G1, QB, X1, SCR, nc);
        contract<1, Q, Q, 1, N, false, MBt<N, Q>>(G0, QB, X2, SCR, nc);
      } else {
        contract<1, Q, Q, 1, N, false, MBt<N, Q>>(V, QB, X1, SCR, nc);
      }
      __syncthreads();
    } else {
      double* Y1 = scr + 2 * SX;
      double* Y2 = Y1 + SY;
      double* Y3 = Y2 + SY;
      const double* G2 = qb + 3 * NQ;
      if (GRAD) {
        contract2<2, Q, Q, Q, N, false, MBt<N, Q>, MDt<N, Q>>(V, G2, QB, Y1, SCR, nc);
        contract<2, Q, Q, Q, N, false, MBt<N, Q>>(G1, QB, Y2, SCR, nc);
        contract<2, Q, Q, Q, N, false, MBt<N, Q>>(G0, QB, Y3, SCR, nc);
      } else {
        contract<2, Q, Q, Q, N, false, MBt<N, Q>>(V, QB, Y1, SCR, nc);
      }
      __syncthreads();
      if (GRAD) {
        contract2<1, Q, Q, N, N, false, MBt<N, Q>, MDt<N, Q>>(Y1, Y2, SCR, X1, SCR, nc);
        contract<1, Q, Q, N, N, false, MBt<N, Q>>(Y3, SCR, X2, SCR, nc);
      } else {
        contract<1, Q, Q, N, N, false, MBt<N, Q>>(Y1, SCR, X1, SCR, nc);
      }
      __syncthreads();
    }
    if (GRAD)
      contract2<0, Q, N, ZN, N, ACC, MBt<N, Q>, MDt<N, Q>>(X1, X2, SCR, out, cs_o, nc);
    else
      contract<0, Q, N, ZN, N, ACC, MBt<N, Q>>(X1, SCR, out, cs_o, nc);
    __syncthreads();
  }

  // --------------------------------------------------------------- face
  // Face F = 2*axis + side. Output face qp block fb: Vf, Gf_0..Gf_{DIM-1} (reference
  // gradient components, indexed by cell axis).
  __host__ __device__ static constexpr int ax(int F) { return F / 2; }
  __host__ __device__ static constexpr int t1(int F) { return DIM == 2 ? 1 - F / 2 : (F / 2 == 0 ? 1 : 0); }
  __host__ __device__ static constexpr int t2(int F) { return F / 2 == 2 ? 1 : 2; }
  __host__ __device__ static constexpr int ex(int a, int e) { return a == 0 ? e : N; }

  template <int F, bool GRAD>
  __device__ static void eval_face(const double* u, int cs_u, double* scr, double* fb, int nc) {
    constexpr int A = F / 2, S = F % 2;
    // extents after selecting along A
    constexpr int AX_ = A == 0 ? 1 : N, AY_ = A == 1 ? 1 : N, AZ_ = A == 2 ? 1 : ZN;
    double* T0 = scr;
    double* T1 = scr + NBF;
    contract<A, N, N, ZN, 1, false, MSel<N, S>>(u, cs_u, T0, SCR, nc);
    if (GRAD) contract<A, N, N, ZN, 1, false, MEd<N, Q, S>>(u, cs_u, T1, SCR, nc);
    __syncthreads();
    double* Vf = fb;
    if constexpr (DIM == 2) {
      constexpr int T = t1(F);
      contract<T, AX_, AY_, 1, Q, false, MB<N, Q>>(T0, SCR, Vf, FB, nc);
      if (GRAD) {
        contract<T, AX_, AY_, 1, Q, false, MD<N, Q>>(T0, SCR, fb + (1 + T) * NQF, FB, nc);
        contract<T, AX_, AY_, 1, Q, false, MB<N, Q>>(T1, SCR, fb + (1 + A) * NQF, FB, nc);
      }
      __syncthreads();
    } else {
      constexpr int U1 = t1(F), U2 = t2(F);
      double* P1 = scr + 2 * NBF;
      double* P2 = P1 + Q * N;
      double* P3 = P2 + Q * N;
      // along U1: N -> Q
      constexpr int BX = U1 == 0 ? Q : AX_, BY = U1 == 1 ? Q : AY_, BZ = U1 == 2 ? Q : AZ_;
      contract<U1, AX_, AY_, AZ_, Q, false, MB<N, Q>>(T0, SCR, P1, SCR, nc);
      if (GRAD) {
        contract<U1, AX_, AY_, AZ_, Q, false, MD<N, Q>>(T0, SCR, P2, SCR, nc);
        contract<U1, AX_, AY_, AZ_, Q, false, MB<N, Q>>(T1, SCR, P3, SCR, nc);
      }
      __syncthreads();
      contract<U2, BX, BY, BZ, Q, false, MB<N, Q>>(P1, SCR, Vf, FB, nc);
      if (GRAD) {
        contract<U2, BX, BY, BZ, Q, false, MD<N, Q>>(P1, SCR, fb + (1 + U2) * NQF, FB, nc);
        contract<U2, BX, BY, BZ, Q, false, MB<N, Q>>(P2, SCR, fb + (1 + U1) * NQF, FB, nc);
        contract<U2, BX, BY, BZ, Q, false, MB<N, Q>>(P3, SCR, fb + (1 + A) * NQF, FB, nc);
      }
      __syncthreads();
    }
  }

  // out[nc][cs_o] += trace-integration of the face qp block (value + reference-gradient tests)
  template <int F, bool GRAD>
  __device__ static void integrate_face(const double* fb, double* scr, double* out, int cs_o, int nc) {
    constexpr int A = F / 2, S = F % 2;
    constexpr int AX_ = A == 0 ? 1 : N, AY_ = A == 1 ? 1 : N, AZ_ = A == 2 ? 1 : ZN;
    double* T0 = scr;
    double* T1 = scr + NBF;
    const double* Vf = fb;
    if constexpr (DIM == 2) {
      constexpr int T = t1(F);
      constexpr int QX = T == 0 ? Q : AX_, QY = T == 1 ? Q : AY_;
      if (GRAD) {
        contract2<T, QX, QY, 1, N, false, MBt<N, Q>, MDt<N, Q>>(Vf, fb + (1 + T) * NQF, FB, T0, SCR, nc);
        contract<T, QX, QY, 1, N, false, MBt<N, Q>>(fb + (1 + A) * NQF, FB, T1, SCR, nc);
      } else {
        contract<T, QX, QY, 1, N, false, MBt<N, Q>>(Vf, FB, T0, SCR, nc);
      }
      __syncthreads();
    } else {
      constexpr int U1 = t1(F), U2 = t2(F);
      double* P1 = scr + 2 * NBF;
      double* P2 = P1 + Q * N;
      double* P3 = P2 + Q * N;
      // fully-Q face shape
      constexpr int QX = (U1 == 0 || U2 == 0) ? Q : AX_;
      constexpr int QY = (U1 == 1 || U2 == 1) ? Q : AY_;
      constexpr int QZ = (U1 == 2 || U2 == 2) ? Q : AZ_;
      if (GRAD) {
        contract2<U2, QX, QY, QZ, N, false, MBt<N, Q>, MDt<N, Q>>(Vf, fb + (1 + U2) * NQF, FB, P1, SCR, nc);
        contract<U2, QX, QY, QZ, N, false, MBt<N, Q>>(fb + (1 + U1) * NQF, FB, P2, SCR, nc);
        contract<U2, QX, QY, QZ, N, false, MBt<N, Q>>(fb + (1 + A) * NQF, FB, P3, SCR, nc);
      } else {
        contract<U2, QX, QY, QZ, N, false, MBt<N, Q>>(Vf, FB, P1, SCR, nc);
      }
      __syncthreads();
      // shape after U2: (U2 -> N)
      constexpr int RX = U2 == 0 ? N : QX, RY = U2 == 1 ? N : QY, RZ = U2 == 2 ? N : QZ;
      if (GRAD) {
        contract2<U1, RX, RY, RZ, N, false, MBt<N, Q>, MDt<N, Q>>(P1, P2, SCR, T0, SCR, nc);
        contract<U1, RX, RY, RZ, N, false, MBt<N, Q>>(P3, SCR, T1, SCR, nc);
      } else {
        contract<U1, RX, RY, RZ, N, false, MBt<N, Q>>(P1, SCR, T0, SCR, nc);
      }
      __syncthreads();
    }
    if (GRAD)
      contract2<A, AX_, AY_, AZ_, N, true, MSelt<N, S>, MEdt<N, Q, S>>(T0, T1, SCR, out, cs_o, nc);
    else
      contract<A, AX_, AY_, AZ_, N, true, MSelt<N, S>>(T0, SCR, out, cs_o, nc);
    __syncthreads();
  }

  // runtime face index -> template dispatch
  template <bool GRAD>
  __device__ static void eval_face_rt(int f, const double* u, int cs_u, double* scr, double* fb, int nc) {
    switch (f) {
      case 0: eval_face<0, GRAD>(u, cs_u, scr, fb, nc); break;
      case 1: eval_face<1, GRAD>(u, cs_u, scr, fb, nc); break;
      case 2: eval_face<2, GRAD>(u, cs_u, scr, fb, nc); break;
      case 3: eval_face<3, GRAD>(u, cs_u, scr, fb, nc); break;
      case 4: if constexpr (DIM == 3) eval_face<4, GRAD>(u, cs_u, scr, fb, nc); break;
      case 5: if constexpr (DIM == 3) eval_face<5, GRAD>(u, cs_u, scr, fb, nc); break;
    }
  }
  template <bool GRAD>
  __device__ static void integrate_face_rt(int f, const double* fb, double* scr, double* out, int cs_o, int nc) {
    switch (f) {
      case 0: integrate_face<0, GRAD>(fb, scr, out, cs_o, nc); break;
      case 1: integrate_face<1, GRAD>(fb, scr, out, cs_o, nc); break;
      case 2: integrate_face<2, GRAD>(fb, scr, out, cs_o, nc); break;
      case 3: integrate_face<3, GRAD>(fb, scr, out, cs_o, nc); break;
      case 4: if constexpr (DIM == 3) integrate_face<4, GRAD>(fb, scr, out, cs_o, nc); break;
      case 5: if constexpr (DIM == 3) integrate_face<5, GRAD>(fb, scr, out, cs_o, nc); break;
    }
  }
};

}  // namespace dgb
