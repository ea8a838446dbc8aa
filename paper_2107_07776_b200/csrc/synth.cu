// Synthetic initial field on the device (BASELINE.json configs: curl of a
// random stream function / vector potential, nodal interpolation as in
// FunctionSpace::interpolate, space.cpp:239-253).  The host version
// (dgb_interpolate_synth) evaluates the same formula; this one exists so the
// 50 M-node configs do not spend minutes on host trigonometry.
#include <cuda_runtime.h>

#include <vector>

#include "../../include/dgb.h"
#include "context.hpp"

namespace {

struct SynthArgs {
  int dim, n1, nm;
  double scale;
  double nodes[8];
};

__global__ void k_interp_synth(SynthArgs a, int ncells, const double* __restrict__ cv,
                               const double* __restrict__ coef, double* __restrict__ u) {
  const int nb = a.dim == 2 ? a.n1 * a.n1 : a.n1 * a.n1 * a.n1;
  const int nv = 1 << a.dim;
  const double tp = 2.0 * 3.141592653589793238462643383279502884;
  for (size_t idx = (size_t)blockIdx.x * blockDim.x + threadIdx.x; idx < (size_t)ncells * nb;
       idx += (size_t)gridDim.x * blockDim.x) {
    const int cell = (int)(idx / nb), j = (int)(idx % nb);
    double ref[3] = {0, 0, 0}, x[3] = {0, 0, 0};
    int rem = j;
    for (int d = 0; d < a.dim; ++d) {
      ref[d] = a.nodes[rem % a.n1];
      rem /= a.n1;
    }
    for (int v = 0; v < nv; ++v) {  // multilinear map (mesh.cpp:44-53)
      double s = 1.0;
      for (int d = 0; d < a.dim; ++d) s *= ((v >> d) & 1) ? ref[d] : (1.0 - ref[d]);
      for (int d = 0; d < a.dim; ++d) x[d] += s * cv[((size_t)cell * nv + v) * a.dim + d];
    }
    double out[3];
    if (a.dim == 2) {
      double dx = 0.0, dy = 0.0;
      for (int m = 0; m < a.nm; ++m) {
        const int i0 = 1 + (m / 4), i1 = 1 + (m % 4);
        const double c = coef[2 * m] * tp * cos(tp * (i0 * x[0] + i1 * x[1]) + coef[2 * m + 1]);
        dx += i0 * c;
        dy += i1 * c;
      }
      out[0] = a.scale * dy;
      out[1] = -a.scale * dx;
    } else {
      double G[3][3] = {};
      for (int c = 0; c < 3; ++c)
        for (int m = 0; m < a.nm; ++m) {
          const int i0 = 1 + m / 16, i1 = 1 + (m / 4) % 4, i2 = 1 + m % 4;
          const double cc = coef[2 * (c * a.nm + m)] * tp *
                            cos(tp * (i0 * x[0] + i1 * x[1] + i2 * x[2]) + coef[2 * (c * a.nm + m) + 1]);
          G[c][0] += i0 * cc;
          G[c][1] += i1 * cc;
          G[c][2] += i2 * cc;
        }
      out[0] = a.scale * (G[2][1] - G[1][2]);
      out[1] = a.scale * (G[0][2] - G[2][0]);
      out[2] = a.scale * (G[1][0] - G[0][1]);
    }
    for (int comp = 0; comp < a.dim; ++comp) u[(size_t)cell * a.dim * nb + comp * nb + j] = out[comp];
  }
}

}  // namespace

extern "C" int dgb_interpolate_synth_device(dgb_ctx* h, const double* user, double* d_u) {
  if (!h || !user || !d_u) return DGB_E_ARG;
  DevGuard guard_(h);
  dgb::Context& c = h->c;
  SynthArgs a;
  a.dim = (int)user[0];
  a.scale = user[1];
  a.nm = (int)user[2];
  a.n1 = c.ku + 1;
  const std::vector<double> nodes = dgb::gauss_lobatto(a.n1);
  for (int i = 0; i < a.n1; ++i) a.nodes[i] = nodes[i];
  const int nv = 1 << c.dim;
  std::vector<double> cv((size_t)c.mesh.ncells * nv * c.dim);
  for (int cell = 0; cell < c.mesh.ncells; ++cell)
    for (int v = 0; v < nv; ++v)
      for (int d = 0; d < c.dim; ++d) cv[((size_t)cell * nv + v) * c.dim + d] = c.mesh.vert(cell, v)[d];
  const int ncoef = 2 * a.nm * (a.dim == 2 ? 1 : 3);
  double *d_cv = nullptr, *d_coef = nullptr;
  if (cudaMalloc(&d_cv, cv.size() * sizeof(double)) != cudaSuccess) return DGB_E_CUDA;
  if (cudaMalloc(&d_coef, ncoef * sizeof(double)) != cudaSuccess) {
    cudaFree(d_cv);
    return DGB_E_CUDA;
  }
  cudaMemcpy(d_cv, cv.data(), cv.size() * sizeof(double), cudaMemcpyHostToDevice);
  cudaMemcpy(d_coef, user + 3, ncoef * sizeof(double), cudaMemcpyHostToDevice);
  k_interp_synth<<<148 * 8, 256, 0, c.dc.stream>>>(a, c.mesh.ncells, d_cv, d_coef, d_u);
  ++c.launches;
  const cudaError_t e = cudaStreamSynchronize(c.dc.stream);
  cudaFree(d_cv);
  cudaFree(d_coef);
  return e == cudaSuccess ? DGB_OK : DGB_E_CUDA;
}
