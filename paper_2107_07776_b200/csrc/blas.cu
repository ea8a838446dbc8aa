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
  GRID_STRIDE(i, n) y[i] = a * x[i] + b * y[i];
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
__global__ void k_cg_update_part(size_t n, double a, const double* __restrict__ p, const double* __restrict__ q,
                                 double* __restrict__ x, double* __restrict__ r, const double* __restrict__ inv,
                                 double* __restrict__ z, double* __restrict__ partial) {
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
}
__global__ void k_precond_dot_part(size_t n, const double* __restrict__ r, const double* __restrict__ inv,
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
__global__ void k_mgs_part(size_t n, double h, const double* __restrict__ vi, double* __restrict__ w,
                           const double* __restrict__ vnext, double* __restrict__ partial) {
  double acc[1] = {0.0};
  const bool self = (vnext == w);
  GRID_STRIDE(i, n) {
    const double wi = fma(-h, vi[i], w[i]);
    w[i] = wi;
    acc[0] = fma(wi, self ? wi : vnext[i], acc[0]);
  }
  block_reduce_store<1>(acc, partial);
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
cudaError_t r_cg_update(cudaStream_t s, size_t n, double a, const double* p, const double* q, double* x,
                        double* r, const double* inv, double* z, double* scratch, double* d_out) {
  const int g = blas_grid(n);
  k_cg_update_part<<<g, kBlasThreads, 0, s>>>(n, a, p, q, x, r, inv, z, scratch);
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, 2, scratch, d_out, 0);
  return cudaGetLastError();
}
cudaError_t r_precond_dot(cudaStream_t s, size_t n, const double* r, const double* inv, double* z,
                          double* scratch, double* d_out) {
  const int g = blas_grid(n);
  k_precond_dot_part<<<g, kBlasThreads, 0, s>>>(n, r, inv, z, scratch);
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, 1, scratch, d_out, 0);
  return cudaGetLastError();
}
cudaError_t r_mgs_step(cudaStream_t s, size_t n, double h, const double* vi, double* w, const double* vnext,
                       double* scratch, double* d_out) {
  const int g = blas_grid(n);
  k_mgs_part<<<g, kBlasThreads, 0, s>>>(n, h, vi, w, vnext, scratch);
  k_sum_parts<<<1, kBlasThreads, 0, s>>>(g, 1, scratch, d_out, 0);
  return cudaGetLastError();
}

}  // namespace dgb
