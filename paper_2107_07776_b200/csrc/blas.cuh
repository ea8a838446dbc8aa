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
// CG fused update: x += a p; r -= a q; z = r * inv (or r); out = {<r,r>, <r,z>}
cudaError_t r_cg_update(cudaStream_t s, size_t n, double a, const double* p, const double* q, double* x,
                        double* r, const double* inv, double* z, double* scratch, double* d_out);
// z = r * inv (or copy); out = {<r,z>}
cudaError_t r_precond_dot(cudaStream_t s, size_t n, const double* r, const double* inv, double* z,
                          double* scratch, double* d_out);
// MGS step: w -= h v_i ; out = <w, v_next> (v_next may equal w for the norm)
cudaError_t r_mgs_step(cudaStream_t s, size_t n, double h, const double* vi, double* w, const double* vnext,
                       double* scratch, double* d_out);
// sum of nparts partials -> d_out
cudaError_t r_sum(cudaStream_t s, int nparts, const double* partial, double* d_out);

}  // namespace dgb
