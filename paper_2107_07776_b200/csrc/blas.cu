// Fused vector kernels (see blas.cuh).
#include "blas.cuh"

#include <cstdint>

namespace dgb {

static int g_sms = 148;

cudaError_t blas_init(int device) {
  int v = 0;
  cudaError_t e = cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, device);
  if (e == cudaSuccess && v > 0) g_sms = v;
  return e;
}

int blas_grid(size_t n) {
  const size_t per = (size_t)kBlasThreads * 4;
  size_t g = (n + per - 1) / per;
  const size_t cap = (size_t)g_sms * 4;  // 4 resident 512-thread blocks per SM
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}

#define GRID_STRIDE(i, n) \
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < (n); i += (size_t)gridDim.x * blockDim.x)

__global__ void k_axpby(size_t n, double a, const double* __restrict__ x, double b, double* __restrict__ y) {
  GRID_STRIDE(i, n) y[i] = fma(a, x[i], b * y[i]);  // the reference's AVX2 order (kernels_avx2.cpp:27-29)
}
__global__ void k_axpy(size_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  GRID_STRIDE(i, n) y[i] = fma(a, x[i], y[i]);
}
__global__ void k_scal(size_t n, double a, double* __restrict__ x) { GRID_STRIDE(i, n) x[i] *= a; }
__global__ void k_scale_copy(size_t n, double a, const double* __restrict__ x, double* __restrict__ y) {
  GRID_STRIDE(i, n) y[i] = a * x[i];
}
__global__ void k_mul(size_t n, const double* __restrict__ r, const double* __restrict__ d, double* __restrict__ z) {
  GRID_STRIDE(i, n) z[i] = r[i] * d[i];
}
__global__ void k_rsub(size_t n, const double* __restrict__ b, double* __restrict__ r) {
  GRID_STRIDE(i, n) r[i] = b[i] - r[i];
}
__global__ void k_addmul(size_t n, const double* __restrict__ d, const double* __restrict__ w, double* __restrict__ x) {
  GRID_STRIDE(i, n) x[i] += d[i] * w[i];
}
__global__ void k_fill(size_t n, double v, double* __restrict__ x) { GRID_STRIDE(i, n) x[i] = v; }

struct PtrPack {
  const double* v[64];
  double y[64];
};
__global__ void k_lincomb(size_t n, int k, PtrPack pp, double* __restrict__ w) {
  GRID_STRIDE(i, n) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s = fma(pp.y[j], pp.v[j][i], s);
    w[i] = s;
  }
}
__global__ void k_recip(size_t n, const double* __restrict__ d, double* __restrict__ inv,
                        unsigned long long* __restrict__ bad) {
  GRID_STRIDE(i, n) {
    const double v = d[i];
    if (v == 0.0) atomicMin(bad, (unsigned long long)i);
    inv[i] = 1.0 / v;
  }
}

// ---------------------------------------------------------------- reductions
__global__ void k_dot_part(size_t n, const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ partial) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) acc[0] = fma(x[i], y[i], acc[0]);
  block_reduce_store<1>(acc, partial);
}
__global__ void k_mad_part(size_t n, const double* __restrict__ x, const double* __restrict__ y,
                           double* __restrict__ partial) {
  double m = 0.0;
  GRID_STRIDE(i, n) m = fmax(m, fabs(x[i] - y[i]));
  __shared__ double red[kBlasThreads / 32];
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    double a = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) a = fmax(a, __shfl_xor_sync(0xffffffffu, a, o));
    if (threadIdx.x == 0) partial[blockIdx.x] = a;
  }
}
// one block: out[v] = sum_b partial[v*nparts + b]
__global__ void k_sum_parts(int nparts, int nv, const double* __restrict__ partial, double* __restrict__ out,
                            int is_max) {
  __shared__ double red[kBlasThreads / 32];
  for (int v = 0; v < nv; ++v) {
    double a = 0.0;
    for (int i = threadIdx.x; i < nparts; i += blockDim.x) {
      const double p = partial[v * nparts + i];
      a = is_max ? fmax(a, p) : a + p;
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double t = __shfl_xor_sync(0xffffffffu, a, o);
      a = is_max ? fmax(a, t) : a + t;
    }
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
    __syncthreads();
    if (threadIdx.x < 32) {
      double b = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) {
        const double t = __shfl_xor_sync(0xffffffffu, b, o);
        b = is_max ? fmax(b, t) : b + t;
      }
      if (threadIdx.x == 0) out[v] = b;
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------- device-resident CG
__global__ void k_cg_begin_part(size_t n, const double* __restrict__ r, const double* __restrict__ inv,
                                double* __restrict__ z, double* __restrict__ partial) {
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) {
    const double ri = r[i];
    const double zi = inv ? ri * inv[i] : ri;
    z[i] = zi;
    acc[0] = fma(ri, zi, acc[0]);
  }
  block_reduce_store<1>(acc, partial);
}
__device__ __forceinline__ double block_sum_parts(int nparts, const double* __restrict__ partial) {
  __shared__ double red[kBlasThreads / 32];
  double a = 0.0;
  for (int i = threadIdx.x; i < nparts; i += blockDim.x) a += partial[i];
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = a;
  __syncthreads();
  double b = 0.0;
  if (threadIdx.x < 32) {
    b = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  return b;  // valid in thread 0
}
__global__ void k_cg_begin_final(int nparts, const double* __restrict__ partial, CgState* st) {
  const double rho = block_sum_parts(nparts, partial);
  if (threadIdx.x == 0) {
    st->rho = rho;
    st->first = 1;
    st->done = 0;
    st->err = 0;
    if (rho == 0.0) {
      st->err = 3;  // DGB_E_BREAKDOWN
      st->done = 3;
    }
  }
}
__global__ void k_cg_dir(size_t n, const double* __restrict__ z, double* __restrict__ p, const CgState* st) {
  if (st->done) return;
  const int first = st->first;
  const double beta = first ? 0.0 : st->rho / st->rho_old;
  GRID_STRIDE(i, n) p[i] = first ? z[i] : fma(beta, p[i], z[i]);
}
// the same on pairs of elements (16-byte aligned vectors)
__global__ void __launch_bounds__(kBlasThreads) k_cg_dir2(size_t n, const double* __restrict__ z,
                                                          double* __restrict__ p, const CgState* st) {
  if (st->done) return;
  const int first = st->first;
  const double beta = first ? 0.0 : st->rho / st->rho_old;
  const double2* z2 = reinterpret_cast<const double2*>(z);
  double2* p2 = reinterpret_cast<double2*>(p);
  GRID_STRIDE(i, n >> 1) {
    const double2 zv = z2[i];
    double2 pv = p2[i];
    pv.x = first ? zv.x : fma(beta, pv.x, zv.x);
    pv.y = first ? zv.y : fma(beta, pv.y, zv.y);
    p2[i] = pv;
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) p[n - 1] = first ? z[n - 1] : fma(beta, p[n - 1], z[n - 1]);
}
__global__ void k_cg_pq_part(size_t n, const double* __restrict__ p, const double* __restrict__ q,
                             double* __restrict__ partial, CgState* st) {
  if (st->done) return;
  double acc[1] = {0.0};
  GRID_STRIDE(i, n) acc[0] = fma(p[i], q[i], acc[0]);
  block_reduce_store<1>(acc, partial);
  if (last_block_arrival(&st->cnt_pq)) cg_alpha_finish(gridDim.x, partial, st);
}
// two-level: each block sums a contiguous slice of the fused apply's partials into
// partial[nparts + block]; the last block to arrive sums those and forms alpha
constexpr int kAlphaBlocks = 64;
__global__ void __launch_bounds__(256) k_cg_alpha_final(int nparts, double* __restrict__ partial, CgState* st) {
  if (st->done) return;
  const int per = (nparts + gridDim.x - 1) / gridDim.x;
  const int b0 = blockIdx.x * per, n = max(0, min(per, nparts - b0));
  const double s = block_sum_l2(n, partial + b0);
  if (threadIdx.x == 0) partial[nparts + blockIdx.x] = s;
  if (last_block_arrival(&st->cnt_pq)) cg_alpha_finish(gridDim.x, partial + nparts, st);
}
__device__ __forceinline__ void cg_upd_finish(int nparts, const double* partial, CgState* st, double* hist);
__global__ void k_cg_upd_part(size_t n, const double* __restrict__ p, const double* __restrict__ q,
                              double* __restrict__ x, double* __restrict__ r, const double* __restrict__ inv,
                              double* __restrict__ z, double* __restrict__ partial, CgState* st,
                              double* __restrict__ hist) {
  if (st->done) return;
  const double a = st->alpha;
  double acc[2] = {0.0, 0.0};
  GRID_STRIDE(i, n) {
    x[i] = fma(a, p[i], x[i]);
    const double ri = fma(-a, q[i], r[i]);
    r[i] = ri;
    const double zi = inv ? ri * inv[i] : ri;
    z[i] = zi;
    acc[0] = fma(ri, ri, acc[0]);
    acc[1] = fma(ri, zi, acc[1]);
  }
  block_reduce_store<2>(acc, partial);
  if (last_block_arrival(&st->cnt_upd)) cg_upd_finish(gridDim.x, partial, st, hist);
}
// the same on pairs of elements (16-byte loads / stores; all vectors 16-byte aligned, an odd
// tail element is taken by thread 0 of block 0).  The per-element arithmetic and the
// order of the thread-local sums over a thread's own elements are those of the scalar
// kernel applied to elements 2i, 2i + 1.
#ifndef DGB_CG_UPD_VEC
#define DGB_CG_UPD_VEC 1
#endif
__global__ void __launch_bounds__(kBlasThreads) k_cg_upd_part2(size_t n, const double* __restrict__ p,
                                                               const double* __restrict__ q, double* __restrict__ x,
                                                               double* __restrict__ r, const double* __restrict__ inv,
                                                               double* __restrict__ z, double* __restrict__ partial,
                                                               CgState* st, double* __restrict__ hist) {
  if (st->done) return;
  const double a = st->alpha;
  double acc[2] = {0.0, 0.0};
  const size_t n2 = n >> 1;
  const double2* p2 = reinterpret_cast<const double2*>(p);
  const double2* q2 = reinterpret_cast<const double2*>(q);
  const double2* i2 = reinterpret_cast<const double2*>(inv);
  double2* x2 = reinterpret_cast<double2*>(x);
  double2* r2 = reinterpret_cast<double2*>(r);
  double2* z2 = reinterpret_cast<double2*>(z);
  GRID_STRIDE(i, n2) {
    const double2 pv = p2[i], qv = q2[i], iv = i2[i];
    double2 xv = x2[i], rv = r2[i], zv;
    xv.x = fma(a, pv.x, xv.x);
    xv.y = fma(a, pv.y, xv.y);
    rv.x = fma(-a, qv.x, rv.x);
    rv.y = fma(-a, qv.y, rv.y);
    zv.x = rv.x * iv.x;
    zv.y = rv.y * iv.y;
    x2[i] = xv;
    r2[i] = rv;
    z2[i] = zv;
    acc[0] = fma(rv.x, rv.x, acc[0]);
    acc[1] = fma(rv.x, zv.x, acc[1]);
    acc[0] = fma(rv.y, rv.y, acc[0]);
    acc[1] = fma(rv.y, zv.y, acc[1]);
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const size_t i = n - 1;
    x[i] = fma(a, p[i], x[i]);
    const double ri = fma(-a, q[i], r[i]);
    r[i] = ri;
    const double zi = ri * inv[i];
    z[i] = zi;
    acc[0] = fma(ri, ri, acc[0]);
    acc[1] = fma(ri, zi, acc[1]);
  }
  block_reduce_store<2>(acc, partial);
  if (last_block_arrival(&st->cnt_upd)) cg_upd_finish(gridDim.x, partial, st, hist);
}
// <r,r>, <r,z> from the partials; history, convergence / budget / breakdown flags
__device__ __forceinline__ void cg_upd_finish(int nparts, const double* partial, CgState* st, double* hist) {
  const double rr = block_sum_l2(nparts, partial);
  const double rz = block_sum_l2(nparts, partial + nparts);
  if (threadIdx.x == 0) {
    const int it = st->iter + 1;
    st->iter = it;
    const double rn = sqrt(rr);
    st->rnorm = rn;
    hist[it - 1] = rn;
    st->first = 0;
    st->rho_old = st->rho;
    st->rho = rz;
    if (rn <= st->tol) {
      st->done = 1;  // converged: back to the outer true-residual check
    } else if (it >= st->max_iter) {
      st->done = 2;  // budget exhausted
    } else if (rz == 0.0) {
      st->err = 3;  // next iteration's "<r,z> = 0" breakdown (krylov.cpp:77-78)
      st->done = 3;
    }
  }
}

// ---------------------------------------------------------------- one-reduce MGS
struct GsPack {
  const double* u[kGsChunk];
};
// NV basis vectors per pass, compile-time so that every load of an element
// iteration is issued before the first FMA (a runtime bound serialises them).
// Pairs of elements per thread (16-byte loads); the basis slots, w and uk are
// 16-byte aligned (pool allocations); an odd tail element is taken by thread 0.
constexpr int kGsThreads = 256;
#ifndef DGB_GSD_MINB  // tuning overrides (tools/tune_gs.sh)
#define DGB_GSD_MINB 1
#endif
#ifndef DGB_GS_CAP
#define DGB_GS_CAP 8
#endif
template <int NV>
__global__ void __launch_bounds__(kGsThreads, DGB_GSD_MINB) k_gs_dots_part(size_t n, GsPack P, const double* __restrict__ w,
                                                           const double* __restrict__ uk, int nl,
                                                           double* __restrict__ partial) {
  double acc[2 * NV];
#pragma unroll
  for (int j = 0; j < 2 * NV; ++j) acc[j] = 0.0;
  const double* ub = nl > 0 ? uk : w;  // harmless stand-in when there is no Gram row
  const size_t n2 = n >> 1;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  const double2* u2 = reinterpret_cast<const double2*>(ub);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    const double2 wi = w2[i];
    const double2 ui = u2[i];
    double2 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = reinterpret_cast<const double2*>(P.u[j])[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc[j] = fma(v[j].y, wi.y, fma(v[j].x, wi.x, acc[j]));
      acc[NV + j] = fma(v[j].y, ui.y, fma(v[j].x, ui.x, acc[NV + j]));
    }
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const size_t i = n - 1;
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      acc[j] = fma(P.u[j][i], w[i], acc[j]);
      acc[NV + j] = fma(P.u[j][i], ub[i], acc[NV + j]);
    }
  }
  block_reduce_store<2 * NV>(acc, partial);
}
// One warp: row k of the Gram matrix in parallel, then the unit lower-triangular solve
// h_j = s_j <w, U_j> - sum_{i<j} h_i L_ji with each row's sum split over the lanes
// (warp tree).  pre: the rows L_0..L_k are first copied into shared memory with all lanes
// (one round of independent loads instead of a dependent global load per row).
__global__ void __launch_bounds__(32) k_gs_solve(int k, const double* __restrict__ ab, double* __restrict__ L,
                                                 int ldl, double* __restrict__ sv, double sk, double* __restrict__ h,
                                                 double* __restrict__ g, int pre) {
  extern __shared__ double gsm[];
  const int lane = threadIdx.x, n = k + 1;
  double* hs = gsm;          // h_j
  double* ps = gsm + n;      // s_j <w, U_j>
  double* ss = gsm + 2 * n;  // s_j
  double* Ls = gsm + 3 * n;  // rows 0..k (pre)
  for (int j = lane; j < n; j += 32) {
    const double svj = j == k ? sk : sv[j];
    ss[j] = svj;
    ps[j] = svj * ab[(j / kGsChunk) * 2 * kGsChunk + (j % kGsChunk)];
    if (j < k) {
      const double v = sk * svj * ab[(j / kGsChunk) * 2 * kGsChunk + kGsChunk + (j % kGsChunk)];
      L[(size_t)k * ldl + j] = v;
      if (pre) Ls[k * n + j] = v;
    }
  }
  if (pre)
    for (int idx = lane; idx < k * k; idx += 32) {
      const int j = idx / k, i = idx - j * k;
      if (i < j) Ls[j * n + i] = L[(size_t)j * ldl + i];
    }
  __syncwarp();
  if (lane == 0) sv[k] = sk;
  for (int j = 0; j < n; ++j) {
    double part = 0.0;
    for (int i = lane; i < j; i += 32) part = fma(hs[i], pre ? Ls[j * n + i] : L[(size_t)j * ldl + i], part);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    const double t = ps[j] - part;
    if (lane == 0) {
      hs[j] = t;
      h[j] = t;
      g[j] = t * ss[j];
    }
    __syncwarp();
  }
}
// zout != nullptr: also zout = dinv (.) w_new (the next Arnoldi step's preconditioned
// input, unnormalised; the caller rescales the Hessenberg column)
template <int NV>
__global__ void __launch_bounds__(kGsThreads) k_gs_update_part(size_t n, GsPack P, const double* __restrict__ g,
                                                             double* __restrict__ w, int want_norm,
                                                             double* __restrict__ partial,
                                                             const double* __restrict__ dinv,
                                                             double* __restrict__ zout) {
  double c[NV];
#pragma unroll
  for (int j = 0; j < NV; ++j) c[j] = g[j];
  double acc[1] = {0.0};
  const size_t n2 = n >> 1;
  double2* w2 = reinterpret_cast<double2*>(w);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += (size_t)gridDim.x * blockDim.x) {
    double2 v[NV];
#pragma unroll
    for (int j = 0; j < NV; ++j) v[j] = reinterpret_cast<const double2*>(P.u[j])[i];
    double2 wi = w2[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) {
      wi.x = fma(-c[j], v[j].x, wi.x);
      wi.y = fma(-c[j], v[j].y, wi.y);
    }
    w2[i] = wi;
    if (zout) {
      double2 zi = wi;
      if (dinv) {
        const double2 di = reinterpret_cast<const double2*>(dinv)[i];
        zi.x *= di.x;
        zi.y *= di.y;
      }
      reinterpret_cast<double2*>(zout)[i] = zi;
    }
    acc[0] = fma(wi.y, wi.y, fma(wi.x, wi.x, acc[0]));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0) {
    const size_t i = n - 1;
    double wi = w[i];
#pragma unroll
    for (int j = 0; j < NV; ++j) wi = fma(-c[j], P.u[j][i], wi);
    w[i] = wi;
    if (zout) zout[i] = dinv ? wi * dinv[i] : wi;
    acc[0] = fma(wi, wi, acc[0]);
  }
  if (want_norm) block_reduce_store<1>(acc, partial);
}
__global__ void k_mul_scaled(size_t n, double a, const double* __restrict__ r, const double* __restrict__ d,
                             double* __restrict__ z) {
  GRID_STRIDE(i, n) z[i] = d ? a * r[i] * d[i] : a * r[i];
}

// ---------------------------------------------------------------- launchers
#define L1(kern, ...)                                              \
  do {                                                             \
    if (n == 0) return cudaSuccess;                                \
    kern<<<blas_grid(n), kBlasThreads, 0, s>>>(n, __VA_ARGS__);    \
    return cudaGetLastError();                                     \
  } while (0)

cudaError_t v_axpby(cudaStream_t s, size_t n, double a, const double* x, double b, double* y) { L1(k_axpby, a, x, b, y); }
cudaError_t v_axpy(cudaStream_t s, size_t n, double a, const double* x, double* y) { L1(k_axpy, a, x, y); }
cudaError_t v_scal(cudaStream_t s, size_t n, double a, double* x) { L1(k_scal, a, x); }
cudaError_t v_scale_copy(cudaStream_t s, size_t n, double a, const double* x, double* y) { L1(k_scale_copy, a, x, y); }
cudaError_t v_mul(cudaStream_t s, size_t n, const double* r, const double* d, double* z) { L1(k_mul, r, d, z); }
cudaError_t v_rsub(cudaStream_t s, size_t n, const double* b, double* r) { L1(k_rsub, b, r); }
cudaError_t v_addmul(cudaStream_t s, size_t n, const double* d, const double* w, double* x) { L1(k_addmul, d, w, x); }
cudaError_t v_fill(cudaStream_t s, size_t n, double v, double* x) { L1(k_fill, v, x); }
cudaError_t v_lincomb(cudaStream_t s, size_t n, int k, const double* const* V, const double* y, double* w) {
  if (k > 64) return cudaErrorInvalidValue;
  PtrPack pp;
  for (int j = 0; j < k; ++j) {
    pp.v[j] = V[j];
    pp.y[j] = y[j];
  }
  L1(k_lincomb, k, pp, w);
}
cudaError_t v_recip(cudaStream_t s, size_t n, const double* d, double* inv, long long* d_bad) {
  L1(k_recip, d, inv, reinterpret_cast<unsigned long long*>(d_bad));
}

cudaError_t r_sum(cudaStream_t s, int nparts, const double* partial, double* d_out) {
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(nparts, 1, partial, d_out, 0);
  return cudaGetLastError();
}
cudaError_t r_dot(cudaStream_t s, size_t n, const double* x, const double* y, double* scratch, double* d_out) {
  const int g = blas_grid(n);
  k_dot_part<<<g, kBlasThreads, 0, s>>>(n, x, y, scratch);
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, 1, scratch, d_out, 0);
  return cudaGetLastError();
}
cudaError_t r_maxabsdiff(cudaStream_t s, size_t n, const double* x, const double* y, double* scratch,
                         double* d_out) {
  const int g = blas_grid(n);
  k_mad_part<<<g, kBlasThreads, 0, s>>>(n, x, y, scratch);
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, 1, scratch, d_out, 1);
  return cudaGetLastError();
}
cudaError_t cg_begin(cudaStream_t s, size_t n, const double* r, const double* inv, double* z, double* scratch,
                     CgState* st) {
  const int g = blas_grid(n);
  k_cg_begin_part<<<g, kBlasThreads, 0, s>>>(n, r, inv, z, scratch);
  k_cg_begin_final<<<1, kBlasThreads, 0, s>>>(g, scratch, st);
  return cudaGetLastError();
}
cudaError_t cg_direction(cudaStream_t s, size_t n, const double* z, double* p, const CgState* st) {
  if ((((uintptr_t)z | (uintptr_t)p) & 15) == 0)
    k_cg_dir2<<<blas_grid(n), kBlasThreads, 0, s>>>(n, z, p, st);
  else
    k_cg_dir<<<blas_grid(n), kBlasThreads, 0, s>>>(n, z, p, st);
  return cudaGetLastError();
}
cudaError_t cg_alpha(cudaStream_t s, size_t n, const double* p, const double* q, double* scratch, CgState* st) {
  const int g = blas_grid(n);
  k_cg_pq_part<<<g, kBlasThreads, 0, s>>>(n, p, q, scratch, st);  // last block computes alpha
  return cudaGetLastError();
}
cudaError_t cg_alpha_from_partials(cudaStream_t s, int nparts, double* partial, CgState* st) {
  k_cg_alpha_final<<<kAlphaBlocks, 256, 0, s>>>(nparts, partial, st);
  return cudaGetLastError();
}
cudaError_t cg_update(cudaStream_t s, size_t n, const double* p, const double* q, double* x, double* r,
                      const double* inv, double* z, double* scratch, CgState* st, double* hist) {
  const int g = blas_grid(n);
  const uintptr_t al = (uintptr_t)p | (uintptr_t)q | (uintptr_t)x | (uintptr_t)r | (uintptr_t)inv | (uintptr_t)z;
  if (DGB_CG_UPD_VEC && inv && (al & 15) == 0)
    k_cg_upd_part2<<<g, kBlasThreads, 0, s>>>(n, p, q, x, r, inv, z, scratch, st, hist);
  else
    k_cg_upd_part<<<g, kBlasThreads, 0, s>>>(n, p, q, x, r, inv, z, scratch, st, hist);  // last block finishes
  return cudaGetLastError();
}
static int gs_grid(size_t n) {
  size_t g = ((n >> 1) + kGsThreads - 1) / kGsThreads;
  const size_t cap = (size_t)g_sms * DGB_GS_CAP;
  if (g > cap) g = cap;
  if (g < 1) g = 1;
  return (int)g;
}
cudaError_t gs_dots(cudaStream_t s, size_t n, int nv, const double* const* U, const double* w, const double* uk,
                    int nl, double* scratch, double* d_ab) {
  if (nv < 1 || nv > kGsChunk || nl > nv) return cudaErrorInvalidValue;
  GsPack P{};
  for (int j = 0; j < nv; ++j) P.u[j] = U[j];
  const int g = gs_grid(n);
  switch (nv) {
#define GS_CASE(NV)                                                               \
  case NV:                                                                        \
    k_gs_dots_part<NV><<<g, kGsThreads, 0, s>>>(n, P, w, uk, nl, scratch);        \
    k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, NV, scratch, d_ab, 0);              \
    if (nl > 0) k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, NV, scratch + (size_t)NV * g, d_ab + kGsChunk, 0); \
    break;
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
    GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12) GS_CASE(13) GS_CASE(14) GS_CASE(15) GS_CASE(16)
#if DGB_GS_CHUNK > 16
    GS_CASE(17) GS_CASE(18) GS_CASE(19) GS_CASE(20) GS_CASE(21) GS_CASE(22) GS_CASE(23) GS_CASE(24)
    GS_CASE(25) GS_CASE(26) GS_CASE(27) GS_CASE(28) GS_CASE(29) GS_CASE(30) GS_CASE(31) GS_CASE(32)
#endif
#undef GS_CASE
  }
  return cudaGetLastError();
}
cudaError_t gs_solve(cudaStream_t s, int k, const double* d_ab, double* L, int ldl, double* d_s, double sk,
                     double* d_h, double* d_g) {
  const size_t n = (size_t)k + 1;
  if (3 * n * sizeof(double) > 48 * 1024) return cudaErrorInvalidValue;  // restart > 2047
  const int pre = (3 * n + n * n) * sizeof(double) <= 48 * 1024;
  k_gs_solve<<<1, 32, (3 * n + (pre ? n * n : 0)) * sizeof(double), s>>>(k, d_ab, L, ldl, d_s, sk, d_h, d_g, pre);
  return cudaGetLastError();
}
cudaError_t gs_update(cudaStream_t s, size_t n, int nv, const double* const* U, const double* g, double* w,
                      double* scratch, double* norm_out, const double* dinv, double* zout) {
  if (nv < 1 || nv > kGsChunk) return cudaErrorInvalidValue;
  GsPack P{};
  for (int j = 0; j < nv; ++j) P.u[j] = U[j];
  const int gr = gs_grid(n);
  switch (nv) {
#define GS_CASE(NV)                                                                          \
  case NV: k_gs_update_part<NV><<<gr, kGsThreads, 0, s>>>(n, P, g, w, norm_out ? 1 : 0, scratch, dinv, zout); break;
    GS_CASE(1) GS_CASE(2) GS_CASE(3) GS_CASE(4) GS_CASE(5) GS_CASE(6) GS_CASE(7) GS_CASE(8)
    GS_CASE(9) GS_CASE(10) GS_CASE(11) GS_CASE(12) GS_CASE(13) GS_CASE(14) GS_CASE(15) GS_CASE(16)
#if DGB_GS_CHUNK > 16
    GS_CASE(17) GS_CASE(18) GS_CASE(19) GS_CASE(20) GS_CASE(21) GS_CASE(22) GS_CASE(23) GS_CASE(24)
    GS_CASE(25) GS_CASE(26) GS_CASE(27) GS_CASE(28) GS_CASE(29) GS_CASE(30) GS_CASE(31) GS_CASE(32)
#endif
#undef GS_CASE
  }
  if (norm_out) k_sum_parts<<<1, kBlasThreads, 0, s>>>(gr, 1, scratch, norm_out, 0);
  return cudaGetLastError();
}
cudaError_t v_mul_scaled(cudaStream_t s, size_t n, double a, const double* r, const double* d, double* z) {
  k_mul_scaled<<<blas_grid(n), kBlasThreads, 0, s>>>(n, a, r, d, z);
  return cudaGetLastError();
}

}  // namespace dgb
