// Fused vector kernels for the Krylov solvers (replacing kern::axpy / axpby /
// scal / dot, proj/src/kernels.cpp:17-39, and the scalar loops of
// JacobiPreconditioner / true_residual, krylov.cpp:18-41).  HBM-bound: grid
// = a multiple of the SM count, 128-bit vector loads where aligned, and
// single-pass two-level reductions with deterministic order (per-block
// partials in a fixed grid, summed by one block).
#pragma once

#include <cuda_runtime.h>

namespace dgb {

constexpr int kBlasThreads = 512;

#ifdef __CUDACC__
// per-block partial sums of NV accumulators -> partial[v * gridDim.x + blockIdx.x]
// (blockDim.x a multiple of 32, <= kBlasThreads)
template <int NV>
__device__ __forceinline__ void block_reduce_store(double (&acc)[NV], double* partial) {
  __shared__ double red[NV][kBlasThreads / 32];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    double a = acc[v];
    for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0) red[v][threadIdx.x >> 5] = a;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      double a = threadIdx.x < (blockDim.x >> 5) ? red[v][threadIdx.x] : 0.0;
      for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
      if (threadIdx.x == 0) partial[v * gridDim.x + blockIdx.x] = a;
    }
  }
}
#endif

cudaError_t blas_init(int device);  // caches the SM count
int blas_grid(size_t n);            // blocks for an n-element pass

// y = a x + b y
cudaError_t v_axpby(cudaStream_t s, size_t n, double a, const double* x, double b, double* y);
// y += a x
cudaError_t v_axpy(cudaStream_t s, size_t n, double a, const double* x, double* y);
// x *= a
cudaError_t v_scal(cudaStream_t s, size_t n, double a, double* x);
// y = a x
cudaError_t v_scale_copy(cudaStream_t s, size_t n, double a, const double* x, double* y);
// z = r * d (Jacobi apply)
cudaError_t v_mul(cudaStream_t s, size_t n, const double* r, const double* d, double* z);
// r = b - r  (true residual after r = A x)
cudaError_t v_rsub(cudaStream_t s, size_t n, const double* b, double* r);
// x += d * w  (GMRES update through the right preconditioner)
cudaError_t v_addmul(cudaStream_t s, size_t n, const double* d, const double* w, double* x);
// w = sum_j y_j V_j  (k <= 64 vectors)
cudaError_t v_lincomb(cudaStream_t s, size_t n, int k, const double* const* V, const double* y, double* w);
cudaError_t v_fill(cudaStream_t s, size_t n, double v, double* x);
// inv = 1 / d; *bad = first index with d == 0 (or -1)
cudaError_t v_recip(cudaStream_t s, size_t n, const double* d, double* inv, long long* d_bad);

// --- reductions: results land in d_out[0..] (device), partials scratch >= 2*grid doubles
cudaError_t r_dot(cudaStream_t s, size_t n, const double* x, const double* y, double* scratch, double* d_out);
cudaError_t r_maxabsdiff(cudaStream_t s, size_t n, const double* x, const double* y, double* scratch,
                         double* d_out);
// sum of nparts partials -> d_out
cudaError_t r_sum(cudaStream_t s, int nparts, const double* partial, double* d_out);

// ---- device-resident CG (krylov.cpp:69-98 inner loop without host round trips)
struct CgState {
  double rho, rho_old, alpha, rnorm, tol;
  int iter, max_iter, done, err, first;
  unsigned cnt_pq, cnt_upd;  // arrival counters of the last-block reductions (kept at 0 between launches)
};

#ifdef __CUDACC__
// true in the block that arrives last (after every block has published its partial);
// the counter is reset there, and that block then reads all partials
__device__ __forceinline__ bool last_block_arrival(unsigned* cnt) {
  __shared__ bool is_last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    const unsigned t = atomicAdd(cnt, 1u);
    is_last = t == gridDim.x - 1;
    if (is_last) *cnt = 0u;
  }
  __syncthreads();
  if (is_last) __threadfence();
  return is_last;
}
// sum of partial[0..nparts) by the whole block, fixed order; L2 loads (written by other SMs)
__device__ __forceinline__ double block_sum_l2(int nparts, const double* partial) {
  __shared__ double red2[32];
  // four independent accumulators: four loads in flight per thread per step (the partial
  // arrays of the fused CG apply hold ~10^5 entries)
  const int st = blockDim.x;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
  int i = threadIdx.x;
  for (; i + 3 * st < nparts; i += 4 * st) {
    a0 += __ldcg(partial + i);
    a1 += __ldcg(partial + i + st);
    a2 += __ldcg(partial + i + 2 * st);
    a3 += __ldcg(partial + i + 3 * st);
  }
  for (; i < nparts; i += st) a0 += __ldcg(partial + i);
  double a = (a0 + a1) + (a2 + a3);
  for (int o = 16; o > 0; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
  if ((threadIdx.x & 31) == 0) red2[threadIdx.x >> 5] = a;
  __syncthreads();
  double b = 0.0;
  if (threadIdx.x < 32) {
    b = threadIdx.x < (blockDim.x >> 5) ? red2[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) b += __shfl_xor_sync(0xffffffffu, b, o);
  }
  __syncthreads();
  return b;  // valid in thread 0
}
// alpha = rho / <p, q> from the partials (krylov.cpp:84-87); flags NOT_SPD
__device__ __forceinline__ void cg_alpha_finish(int nparts, const double* partial, CgState* st) {
  const double pq = block_sum_l2(nparts, partial);
  if (threadIdx.x == 0) {
    if (pq <= 0.0) {
      st->err = 4;  // DGB_E_NOT_SPD
      st->done = 3;
    } else {
      st->alpha = st->rho / pq;
    }
  }
}
#endif
// first iteration of an inner loop: z = M r, rho = <r,z>; sets first = 1, done = 0
cudaError_t cg_begin(cudaStream_t s, size_t n, const double* r, const double* inv, double* z, double* scratch,
                     CgState* st);
// p = z (first) or z + (rho/rho_old) p
cudaError_t cg_direction(cudaStream_t s, size_t n, const double* z, double* p, const CgState* st);
// alpha = rho / <p,q>  (flags NOT_SPD)
cudaError_t cg_alpha(cudaStream_t s, size_t n, const double* p, const double* q, double* scratch, CgState* st);
// x += alpha p, r -= alpha q, z = M r, rnorm -> history, convergence / breakdown flags
cudaError_t cg_update(cudaStream_t s, size_t n, const double* p, const double* q, double* x, double* r,
                      const double* inv, double* z, double* scratch, CgState* st, double* hist);
// MGS step with the projection read from device memory: w -= (*h) v_i ; *out = <w, v_next>
// alpha = rho / sum(partial[0..nparts))  (CG with the <p,q> partials from a fused apply)
cudaError_t cg_alpha_from_partials(cudaStream_t s, int nparts, double* partial, CgState* st);

// ---- one-reduce modified Gram-Schmidt for GMRES (krylov.cpp:140-160 restated).
// The basis is stored unnormalised, v_j = s_j U_j.  MGS's projections follow
// from one pass of dot products through the lower-triangular Gram correction
//   h_j = <w, v_j> - sum_{i<j} h_i <v_i, v_j>,
// which is MGS in exact arithmetic; the second pass applies w -= sum_j h_j v_j
// and yields |w|^2.  2k+5 vector passes per Arnoldi step instead of 4(k+1).
#ifndef DGB_GS_CHUNK  // basis vectors per Gram-Schmidt pass (16 or 32)
#define DGB_GS_CHUNK 32
#endif
constexpr int kGsChunk = DGB_GS_CHUNK;
// basis vectors per update pass: 16 (a 32-vector update pass measured slower at cfg3,
// 148 vs 142 ms per stage, while the 32-vector dot pass is faster, 120 vs 125 ms)
constexpr int kGsUpdChunk = 16;
// a_j = <w, U_j> (j < nv) and b_j = <uk, U_j> (j < nl) for one chunk of <= kGsChunk vectors
// -> d_ab[0..kGsChunk) = a, d_ab[kGsChunk..2 kGsChunk) = b
cudaError_t gs_dots(cudaStream_t s, size_t n, int nv, const double* const* U, const double* w, const double* uk,
                    int nl, double* scratch, double* d_ab);
// single-thread solve: row k of L from b, h (MGS projections) and g_j = h_j s_j
//   d_ab: per chunk 32 values (a, b); L: (ldl x ldl) device matrix; d_s[k] = sk
cudaError_t gs_solve(cudaStream_t s, int k, const double* d_ab, double* L, int ldl, double* d_s, double sk,
                     double* d_h, double* d_g);
// w -= sum_{j<nv} g_j U_j ; if norm_out: *norm_out = |w|^2
// zout (optional): also write zout = dinv (.) w_new (dinv == nullptr: w_new)
cudaError_t gs_update(cudaStream_t s, size_t n, int nv, const double* const* U, const double* g, double* w,
                      double* scratch, double* norm_out, const double* dinv = nullptr, double* zout = nullptr);
// z = a * r * d (d may be null: z = a r)
cudaError_t v_mul_scaled(cudaStream_t s, size_t n, double a, const double* r, const double* d, double* z);

}  // namespace dgb
