// Hybrid multigrid preconditioner for the pressure Helmholtz operator (SURVEY 8(f) item 1:
// the paper preconditions the pressure Poisson solve with geometric multigrid,
// PAPER.md:505; the reference substitutes Jacobi).  Opt-in: the
// reference-parity path keeps Jacobi-CG (dgb_cg); this is dgb_pressure_cg_mg and
// dgb_step_params::pressure_precond = 1.
//
// 3D meshes with the lexicographic n x n x n topology of generate_cartesian on a cube
// (uniform, graded-free; deformed vertex positions allowed: cfg4).  Levels:
//   0      the DG Q_kp space itself, operator = the fast SIP apply (Context::sip),
//   1..L   continuous trilinear (Q1) finite elements on vertex grids of n, n/2, n/4, ...
//          cells per direction, operator = mc M + K assembled as a 27-point tensor
//          stencil (natural boundary conditions, like the pressure operator) of the
//          undeformed grid: exact Galerkin levels on Cartesian meshes, a spectrally
//          equivalent approximation on deformed ones (vertices moved by <= 10 % of h);
//   coarsest (n_c <= 4 or odd): exact solve with a dense inverse built on the host.
// Transfers: DG <- Q1 is the trilinear interpolation at the Gauss-Lobatto nodes of each
// cell; Q1 fine <- coarse the nested trilinear interpolation; restrictions are their
// transposes.  For continuous trilinear functions the SIP jump / penalty terms vanish,
// so P^T A_DG P equals the Q1 operator: the hierarchy is Galerkin-consistent.
// Smoother: Chebyshev polynomial of degree s in D^-1 A on every level (D = the exact
// diagonal; lambda_max from a power iteration at setup), the same polynomial before and
// after the coarse correction, so the V-cycle is symmetric positive definite and CG can
// use it as a fixed preconditioner.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "blas.cuh"
#include "context.hpp"
#include "host_setup.hpp"

namespace dgb {

#define CK(call)                                        \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(e_, #call); \
  } while (0)
#define OK(call)                 \
  do {                           \
    int s_ = (call);             \
    if (s_ != DGB_OK) return s_; \
  } while (0)

namespace {

constexpr int kT = 256;
inline int grid_for(size_t n) { return (int)std::min<size_t>((n + kT - 1) / kT, 148 * 32); }

struct GlNodes {
  double xi[8];
};

// 1D Q1 rows at vertex i of a grid with n cells, spacing h: offsets -1, 0, +1
__host__ __device__ inline void q1_rows(int i, int n, double h, double m[3], double k[3]) {
  const bool lo = i > 0, hi = i < n;
  m[0] = lo ? h / 6.0 : 0.0;
  m[2] = hi ? h / 6.0 : 0.0;
  m[1] = (lo ? h / 3.0 : 0.0) + (hi ? h / 3.0 : 0.0);
  k[0] = lo ? -1.0 / h : 0.0;
  k[2] = hi ? -1.0 / h : 0.0;
  k[1] = (lo ? 1.0 / h : 0.0) + (hi ? 1.0 / h : 0.0);
}

// y = (mc M + K) x on the (n+1)^3 vertex grid (27-point tensor stencil)
__global__ void k_q1_apply(int n, double h, double mc, const double* __restrict__ x, double* __restrict__ y) {
  const int nv = n + 1;
  const size_t tot = (size_t)nv * nv * nv;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < tot; v += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(v % nv), j = (int)((v / nv) % nv), k = (int)(v / ((size_t)nv * nv));
    double mx[3], kx[3], my[3], ky[3], mz[3], kz[3];
    q1_rows(i, n, h, mx, kx);
    q1_rows(j, n, h, my, ky);
    q1_rows(k, n, h, mz, kz);
    double s = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      const int kk = k + c - 1;
      if (kk < 0 || kk > n) continue;
#pragma unroll
      for (int b = 0; b < 3; ++b) {
        const int jj = j + b - 1;
        if (jj < 0 || jj > n) continue;
        const double myz = my[b] * mz[c], kyz = ky[b] * mz[c] + my[b] * kz[c];
        const double* xr = x + ((size_t)kk * nv + jj) * nv;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
          const int ii = i + a - 1;
          if (ii < 0 || ii > n) continue;
          s = fma((mc * mx[a] + kx[a]) * myz + mx[a] * kyz, xr[ii], s);
        }
      }
    }
    y[v] = s;
  }
}

__global__ void k_q1_diag_inv(int n, double h, double mc, double* __restrict__ inv) {
  const int nv = n + 1;
  const size_t tot = (size_t)nv * nv * nv;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < tot; v += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(v % nv), j = (int)((v / nv) % nv), k = (int)(v / ((size_t)nv * nv));
    double mx[3], kx[3], my[3], ky[3], mz[3], kz[3];
    q1_rows(i, n, h, mx, kx);
    q1_rows(j, n, h, my, ky);
    q1_rows(k, n, h, mz, kz);
    inv[v] = 1.0 / (mc * mx[1] * my[1] * mz[1] + kx[1] * my[1] * mz[1] + mx[1] * ky[1] * mz[1] +
                    mx[1] * my[1] * kz[1]);
  }
}

// DG Q_kp (cell-major, node lexicographic) <- Q1 vertex values: trilinear interpolation
template <int N>
__global__ void k_dg_from_q1(int n, GlNodes g, const double* __restrict__ xv, double* __restrict__ y) {
  constexpr int NB = N * N * N;
  const int nv = n + 1;
  const size_t tot = (size_t)n * n * n * NB;
  for (size_t t = blockIdx.x * (size_t)blockDim.x + threadIdx.x; t < tot; t += (size_t)gridDim.x * blockDim.x) {
    const size_t cell = t / NB;
    const int node = (int)(t - cell * NB);
    const int cx = (int)(cell % n), cy = (int)((cell / n) % n), cz = (int)(cell / ((size_t)n * n));
    const double ex = g.xi[node % N], ey = g.xi[(node / N) % N], ez = g.xi[node / (N * N)];
    const double* b = xv + ((size_t)cz * nv + cy) * nv + cx;
    const double v00 = (1.0 - ex) * b[0] + ex * b[1];
    const double v10 = (1.0 - ex) * b[nv] + ex * b[nv + 1];
    const double v01 = (1.0 - ex) * b[(size_t)nv * nv] + ex * b[(size_t)nv * nv + 1];
    const double v11 = (1.0 - ex) * b[(size_t)nv * nv + nv] + ex * b[(size_t)nv * nv + nv + 1];
    y[t] = (1.0 - ez) * ((1.0 - ey) * v00 + ey * v10) + ez * ((1.0 - ey) * v01 + ey * v11);
  }
}

// transpose of k_dg_from_q1: vertex sums over the (up to 8) cells around it
template <int N>
__global__ void k_q1_from_dg(int n, GlNodes g, const double* __restrict__ r, double* __restrict__ rv) {
  constexpr int NB = N * N * N;
  const int nv = n + 1;
  const size_t tot = (size_t)nv * nv * nv;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < tot; v += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(v % nv), j = (int)((v / nv) % nv), k = (int)(v / ((size_t)nv * nv));
    double s = 0.0;
    for (int dc = 0; dc < 8; ++dc) {
      const int cx = i - 1 + (dc & 1), cy = j - 1 + ((dc >> 1) & 1), cz = k - 1 + (dc >> 2);
      if (cx < 0 || cy < 0 || cz < 0 || cx >= n || cy >= n || cz >= n) continue;
      // the vertex is corner (a, b, c) of this cell: a = 1 when the cell lies below it
      const int a = (dc & 1) ? 0 : 1, b = ((dc >> 1) & 1) ? 0 : 1, c = (dc >> 2) ? 0 : 1;
      double lx[N], ly[N], lz[N];
#pragma unroll
      for (int q = 0; q < N; ++q) {
        lx[q] = a ? g.xi[q] : 1.0 - g.xi[q];
        ly[q] = b ? g.xi[q] : 1.0 - g.xi[q];
        lz[q] = c ? g.xi[q] : 1.0 - g.xi[q];
      }
      const double* rc = r + (((size_t)cz * n + cy) * n + cx) * NB;
#pragma unroll
      for (int kk = 0; kk < N; ++kk) {
        double sy = 0.0;
#pragma unroll
        for (int jj = 0; jj < N; ++jj) {
          double sx = 0.0;
#pragma unroll
          for (int ii = 0; ii < N; ++ii) sx = fma(lx[ii], rc[ii + N * (jj + N * kk)], sx);
          sy = fma(ly[jj], sx, sy);
        }
        s = fma(lz[kk], sy, s);
      }
    }
    rv[v] = s;
  }
}

// fine (2 nc cells) += P coarse (nc cells): nested trilinear interpolation
__global__ void k_q1_prolong_add(int nc, const double* __restrict__ xc, double* __restrict__ xf) {
  const int nf = 2 * nc, nvf = nf + 1, nvc = nc + 1;
  const size_t tot = (size_t)nvf * nvf * nvf;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < tot; v += (size_t)gridDim.x * blockDim.x) {
    const int I = (int)(v % nvf), J = (int)((v / nvf) % nvf), K = (int)(v / ((size_t)nvf * nvf));
    // per direction: even fine index -> one coarse vertex (weight 1), odd -> two (1/2 each)
    const int ia = I >> 1, ib = (I + 1) >> 1, ja = J >> 1, jb = (J + 1) >> 1, ka = K >> 1, kb = (K + 1) >> 1;
    const double wx = (I & 1) ? 0.5 : 1.0, wy = (J & 1) ? 0.5 : 1.0, wz = (K & 1) ? 0.5 : 1.0;
    double s = 0.0;
    for (int c = 0; c < ((K & 1) ? 2 : 1); ++c) {
      const int kk = c ? kb : ka;
      for (int b = 0; b < ((J & 1) ? 2 : 1); ++b) {
        const int jj = b ? jb : ja;
        const double* row = xc + ((size_t)kk * nvc + jj) * nvc;
        s += row[ia] + ((I & 1) ? row[ib] : 0.0);
      }
    }
    xf[v] += wx * wy * wz * s;
  }
}

// coarse = P^T fine (full weighting, unnormalised)
__global__ void k_q1_restrict(int nc, const double* __restrict__ rf, double* __restrict__ rc) {
  const int nf = 2 * nc, nvf = nf + 1, nvc = nc + 1;
  const size_t tot = (size_t)nvc * nvc * nvc;
  for (size_t v = blockIdx.x * (size_t)blockDim.x + threadIdx.x; v < tot; v += (size_t)gridDim.x * blockDim.x) {
    const int i = (int)(v % nvc), j = (int)((v / nvc) % nvc), k = (int)(v / ((size_t)nvc * nvc));
    double s = 0.0;
    for (int c = -1; c <= 1; ++c) {
      const int K = 2 * k + c;
      if (K < 0 || K > nf) continue;
      const double wz = c ? 0.5 : 1.0;
      for (int b = -1; b <= 1; ++b) {
        const int J = 2 * j + b;
        if (J < 0 || J > nf) continue;
        const double wyz = wz * (b ? 0.5 : 1.0);
        for (int a = -1; a <= 1; ++a) {
          const int I = 2 * i + a;
          if (I < 0 || I > nf) continue;
          s = fma(wyz * (a ? 0.5 : 1.0), rf[((size_t)K * nvf + J) * nvf + I], s);
        }
      }
    }
    rc[v] = s;
  }
}

// Chebyshev step: d = c1 d + c2 inv (b - Ax); x += d   (first step: c1 = 0, Ax unused when ax == nullptr)
__global__ void k_cheb(size_t n, double c1, double c2, const double* __restrict__ inv, const double* __restrict__ b,
                       const double* __restrict__ ax, double* __restrict__ d, double* __restrict__ x, int first) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    const double r = ax ? b[i] - ax[i] : b[i];
    const double di = (first ? 0.0 : c1 * d[i]) + c2 * inv[i] * r;
    d[i] = di;
    x[i] = first == 2 ? di : x[i] + di;  // first == 2: x starts at zero
  }
}

// r = b - Ax
__global__ void k_resid(size_t n, const double* __restrict__ b, const double* __restrict__ ax, double* __restrict__ r) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    r[i] = b[i] - ax[i];
}

// z = Ainv r (dense, coarsest level); one block
__global__ void k_dense_mv(int m, const double* __restrict__ A, const double* __restrict__ r, double* __restrict__ z) {
  for (int i = threadIdx.x; i < m; i += blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < m; ++j) s = fma(A[(size_t)i * m + j], r[j], s);
    z[i] = s;
  }
}

// y = x / inv  (D x from the inverse diagonal)
__global__ void k_div(size_t n, const double* __restrict__ x, const double* __restrict__ inv, double* __restrict__ y) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    y[i] = x[i] / inv[i];
}

// deterministic start vector of the power iteration
__global__ void k_pattern(size_t n, double* x) {
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    unsigned long long h = (i + 1) * 0x9E3779B97F4A7C15ull;
    h ^= h >> 29;
    h *= 0xBF58476D1CE4E5B9ull;
    h ^= h >> 32;
    x[i] = (double)(h >> 11) * (1.0 / 9007199254740992.0) - 0.5;
  }
}

// host: dense (mc M + K) on the (n+1)^3 grid, inverted by Gauss-Jordan (SPD, small)
bool dense_q1_inverse(int n, double side, double mc, std::vector<double>& inv) {
  const double h = side / n;
  const int nv = n + 1, m = nv * nv * nv;
  std::vector<double> A((size_t)m * m, 0.0);
  for (int k = 0; k < nv; ++k)
    for (int j = 0; j < nv; ++j)
      for (int i = 0; i < nv; ++i) {
        double mx[3], kx[3], my[3], ky[3], mz[3], kz[3];
        q1_rows(i, n, h, mx, kx);
        q1_rows(j, n, h, my, ky);
        q1_rows(k, n, h, mz, kz);
        const int row = i + nv * (j + nv * k);
        for (int c = 0; c < 3; ++c)
          for (int b = 0; b < 3; ++b)
            for (int a = 0; a < 3; ++a) {
              const int ii = i + a - 1, jj = j + b - 1, kk = k + c - 1;
              if (ii < 0 || jj < 0 || kk < 0 || ii > n || jj > n || kk > n) continue;
              A[(size_t)row * m + ii + nv * (jj + nv * kk)] =
                  mc * mx[a] * my[b] * mz[c] + kx[a] * my[b] * mz[c] + mx[a] * ky[b] * mz[c] + mx[a] * my[b] * kz[c];
            }
      }
  inv.assign((size_t)m * m, 0.0);
  for (int i = 0; i < m; ++i) inv[(size_t)i * m + i] = 1.0;
  for (int c = 0; c < m; ++c) {
    int piv = c;
    for (int r = c + 1; r < m; ++r)
      if (std::abs(A[(size_t)r * m + c]) > std::abs(A[(size_t)piv * m + c])) piv = r;
    if (A[(size_t)piv * m + c] == 0.0) return false;
    if (piv != c)
      for (int j = 0; j < m; ++j) {
        std::swap(A[(size_t)c * m + j], A[(size_t)piv * m + j]);
        std::swap(inv[(size_t)c * m + j], inv[(size_t)piv * m + j]);
      }
    const double d = 1.0 / A[(size_t)c * m + c];
    for (int j = 0; j < m; ++j) {
      A[(size_t)c * m + j] *= d;
      inv[(size_t)c * m + j] *= d;
    }
    for (int r = 0; r < m; ++r) {
      if (r == c) continue;
      const double f = A[(size_t)r * m + c];
      if (f == 0.0) continue;
      for (int j = 0; j < m; ++j) {
        A[(size_t)r * m + j] -= f * A[(size_t)c * m + j];
        inv[(size_t)r * m + j] -= f * inv[(size_t)c * m + j];
      }
    }
  }
  return true;
}

}  // namespace

// ------------------------------------------------------------------ hierarchy
struct MgLevel {
  int n = 0;  // cells per direction (Q1 levels); 0 for the DG level
  size_t size = 0;
  double h = 0.0, lmax = 1.0;
  double *inv = nullptr, *b = nullptr, *x = nullptr, *res = nullptr, *d = nullptr, *ax = nullptr;
};
struct MgHierarchy {
  double mc = -1.0;
  int degree = 4;      // Chebyshev degree (smoother)
  double range = 15.0;  // smoothing range lambda_max / lambda_min
  std::vector<MgLevel> lv;  // lv[0] = DG level
  double* coarse_inv = nullptr;  // dense inverse (coarsest Q1 level)
  int coarse_m = 0;
  GlNodes gl;
  std::vector<void*> allocs;
  ~MgHierarchy() {
    for (void* p : allocs) cudaFree(p);
  }
  double* alloc(size_t n) {
    void* p = nullptr;
    if (cudaMalloc(&p, std::max<size_t>(n, 1) * sizeof(double)) != cudaSuccess) return nullptr;
    allocs.push_back(p);
    return (double*)p;
  }
};

void mg_release(MgHierarchy* h) { delete h; }

// n if the mesh has generate_cartesian's lexicographic n^3 topology (neighbours and
// boundary ids by index) on a cube of side `side`, else 0
static int cartesian_topology(const HostMesh& m, double& side) {
  if (m.dim != 3) return 0;
  const int n = (int)std::lround(std::cbrt((double)m.ncells));
  if ((long long)n * n * n != m.ncells || n < 1) return 0;
  for (int c = 0; c < m.ncells; ++c)
    for (int f = 0; f < 6; ++f) {
      const int d = f >> 1, s = f & 1;
      const int co = d == 0 ? c % n : (d == 1 ? (c / n) % n : c / (n * n));
      const int stride = d == 0 ? 1 : (d == 1 ? n : n * n);
      const int want = s == 0 ? (co == 0 ? -1 - f : c - stride) : (co == n - 1 ? -1 - f : c + stride);
      if (m.nbr[(size_t)c * 6 + f] != want) return 0;
    }
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (size_t v = 0; v < m.vertices.size() / 3; ++v)
    for (int d = 0; d < 3; ++d) {
      lo[d] = std::min(lo[d], m.vertices[v * 3 + d]);
      hi[d] = std::max(hi[d], m.vertices[v * 3 + d]);
    }
  side = hi[0] - lo[0];
  for (int d = 1; d < 3; ++d)
    if (std::abs((hi[d] - lo[d]) - side) > 1e-12 * side) return 0;
  return side > 0.0 ? n : 0;
}

bool Context::mg_supported() const {
  if (dim != 3 || kp < 1 || kp > 3 || hang_) return false;
  if (mg_topo_n_ < 0) {
    double side = 0.0;
    mg_topo_n_ = cartesian_topology(mesh, side);
    mg_side_ = side;
  }
  int n = mg_topo_n_;
  if (n <= 0) return false;
  while (n % 2 == 0 && n > 4) n /= 2;
  return (size_t)(n + 1) * (n + 1) * (n + 1) <= 729;
}

int Context::mg_level_apply(int l, const double* x, double* y) {
  MgLevel& L = mg_->lv[l];
  if (l == 0) return sip(mg_->mc, 0, x, y);
  ++launches;
  k_q1_apply<<<grid_for(L.size), kT, 0, dc.stream>>>(L.n, L.h, mg_->mc, x, y);
  CK(cudaGetLastError());
  return DGB_OK;
}

// x = S(b) with zero start (first == true) or x += S(b - A x)
int Context::mg_smooth(int l, const double* b, double* x, bool zero_start) {
  MgLevel& L = mg_->lv[l];
  const int s = mg_->degree;
  const double bmax = 1.1 * L.lmax, amin = bmax / mg_->range;
  const double theta = 0.5 * (bmax + amin), delta = 0.5 * (bmax - amin), sigma = theta / delta;
  double rho = 1.0 / sigma;
  cudaStream_t st = dc.stream;
  const int g = grid_for(L.size);
  if (!zero_start) OK(mg_level_apply(l, x, L.ax));
  ++launches;
  k_cheb<<<g, kT, 0, st>>>(L.size, 0.0, 1.0 / theta, L.inv, b, zero_start ? nullptr : L.ax, L.d, x,
                           zero_start ? 2 : 1);
  CK(cudaGetLastError());
  for (int it = 1; it < s; ++it) {
    OK(mg_level_apply(l, x, L.ax));
    const double rn = 1.0 / (2.0 * sigma - rho);
    ++launches;
    k_cheb<<<g, kT, 0, st>>>(L.size, rn * rho, 2.0 * rn / delta, L.inv, b, L.ax, L.d, x, 0);
    CK(cudaGetLastError());
    rho = rn;
  }
  return DGB_OK;
}

int Context::mg_restrict(int l, const double* r_fine, double* r_coarse) {
  // level l -> l + 1
  MgLevel& C = mg_->lv[l + 1];
  cudaStream_t st = dc.stream;
  ++launches;
  if (l == 0) {
    switch (kp) {
      case 1: k_q1_from_dg<2><<<grid_for(C.size), kT, 0, st>>>(C.n, mg_->gl, r_fine, r_coarse); break;
      case 2: k_q1_from_dg<3><<<grid_for(C.size), kT, 0, st>>>(C.n, mg_->gl, r_fine, r_coarse); break;
      default: k_q1_from_dg<4><<<grid_for(C.size), kT, 0, st>>>(C.n, mg_->gl, r_fine, r_coarse); break;
    }
  } else {
    k_q1_restrict<<<grid_for(C.size), kT, 0, st>>>(C.n, r_fine, r_coarse);
  }
  CK(cudaGetLastError());
  return DGB_OK;
}

int Context::mg_prolong_add(int l, const double* x_coarse, double* x_fine) {
  // level l + 1 -> l, added
  MgLevel& F = mg_->lv[l];
  MgLevel& C = mg_->lv[l + 1];
  cudaStream_t st = dc.stream;
  launches += 1;
  if (l == 0) {
    double* t = F.ax;  // scratch: interpolated correction
    switch (kp) {
      case 1: k_dg_from_q1<2><<<grid_for(F.size), kT, 0, st>>>(C.n, mg_->gl, x_coarse, t); break;
      case 2: k_dg_from_q1<3><<<grid_for(F.size), kT, 0, st>>>(C.n, mg_->gl, x_coarse, t); break;
      default: k_dg_from_q1<4><<<grid_for(F.size), kT, 0, st>>>(C.n, mg_->gl, x_coarse, t); break;
    }
    CK(cudaGetLastError());
    ++launches;
    CK(v_axpy(st, F.size, 1.0, t, x_fine));
  } else {
    k_q1_prolong_add<<<grid_for(F.size), kT, 0, st>>>(C.n, x_coarse, x_fine);
    CK(cudaGetLastError());
  }
  return DGB_OK;
}

int Context::mg_vcycle(int l, const double* b, double* x) {
  const int nl = (int)mg_->lv.size();
  cudaStream_t st = dc.stream;
  if (l == nl - 1) {  // coarsest: exact
    ++launches;
    k_dense_mv<<<1, 512, 0, st>>>(mg_->coarse_m, mg_->coarse_inv, b, x);
    CK(cudaGetLastError());
    return DGB_OK;
  }
  MgLevel& L = mg_->lv[l];
  MgLevel& C = mg_->lv[l + 1];
  OK(mg_smooth(l, b, x, true));
  OK(mg_level_apply(l, x, L.ax));
  ++launches;
  k_resid<<<grid_for(L.size), kT, 0, st>>>(L.size, b, L.ax, L.res);
  CK(cudaGetLastError());
  OK(mg_restrict(l, L.res, C.b));
  OK(mg_vcycle(l + 1, C.b, C.x));
  OK(mg_prolong_add(l, C.x, x));
  OK(mg_smooth(l, b, x, false));
  return DGB_OK;
}

// lambda_max(D^-1 A) of level l: power iteration, then the generalised Rayleigh quotient
// (v, A v) / (v, D v) (a lower bound; the smoother interval takes 1.1 x it)
int Context::mg_lambda_max(int l, double& lmax) {
  MgLevel& L = mg_->lv[l];
  cudaStream_t st = dc.stream;
  double* v = L.x;
  double* w = L.res;
  ++launches;
  k_pattern<<<grid_for(L.size), kT, 0, st>>>(L.size, v);
  CK(cudaGetLastError());
  for (int it = 0; it < 12; ++it) {
    OK(mg_level_apply(l, v, L.ax));
    ++launches;
    CK(v_mul(st, L.size, L.ax, L.inv, w));  // D^-1 A v
    double ww;
    OK(dot(L.size, w, w, &ww));
    if (!(ww > 0.0)) break;
    ++launches;
    CK(v_scale_copy(st, L.size, 1.0 / std::sqrt(ww), w, v));
  }
  OK(mg_level_apply(l, v, L.ax));
  double vav, vdv;
  OK(dot(L.size, v, L.ax, &vav));
  ++launches;
  k_div<<<grid_for(L.size), kT, 0, st>>>(L.size, v, L.inv, w);  // D v
  CK(cudaGetLastError());
  OK(dot(L.size, v, w, &vdv));
  lmax = (vdv > 0.0 && vav > 0.0) ? vav / vdv : 2.0;
  return DGB_OK;
}

int Context::mg_setup(double mc) {
  if (!mg_supported())
    return fail(DGB_E_UNSUPPORTED, "pressure multigrid: needs a 3D mesh with Cartesian n^3 topology on a cube");
  if (mg_ && mg_->mc == mc) return DGB_OK;
  if (!mg_) {
    mg_ = new MgHierarchy();
    if (const char* e = std::getenv("DGB_MG_DEGREE")) mg_->degree = std::max(1, std::atoi(e));  // tuning
    if (const char* e = std::getenv("DGB_MG_RANGE")) mg_->range = std::max(1.5, std::atof(e));
    const std::vector<double> xi = gauss_lobatto(kp + 1);
    for (int i = 0; i <= kp; ++i) mg_->gl.xi[i] = xi[i];
    MgLevel L0;
    L0.size = np();
    mg_->lv.push_back(L0);
    int n = mg_topo_n_;
    mg_->lv.push_back(MgLevel{});
    mg_->lv.back().n = n;
    while (n % 2 == 0 && n > 4) {
      n /= 2;
      mg_->lv.push_back(MgLevel{});
      mg_->lv.back().n = n;
    }
    for (size_t l = 0; l < mg_->lv.size(); ++l) {
      MgLevel& L = mg_->lv[l];
      if (l > 0) {
        L.size = (size_t)(L.n + 1) * (L.n + 1) * (L.n + 1);
        L.h = mg_side_ / L.n;
      }
      L.inv = mg_->alloc(L.size);
      L.b = mg_->alloc(L.size);
      L.x = mg_->alloc(L.size);
      L.res = mg_->alloc(L.size);
      L.d = mg_->alloc(L.size);
      L.ax = mg_->alloc(L.size);
      if (!L.inv || !L.b || !L.x || !L.res || !L.d || !L.ax) return fail(DGB_E_CUDA, "pressure multigrid: out of device memory");
    }
    const MgLevel& Lc = mg_->lv.back();
    mg_->coarse_m = (int)Lc.size;
    mg_->coarse_inv = mg_->alloc(Lc.size * Lc.size);
    if (!mg_->coarse_inv) return fail(DGB_E_CUDA, "pressure multigrid: out of device memory");
  }
  mg_->mc = mc;
  cudaStream_t st = dc.stream;
  // diagonals
  OK(sip_diag(mc, 0, mg_->lv[0].inv));
  OK(jacobi_inverse(mg_->lv[0].size, mg_->lv[0].inv, mg_->lv[0].inv));
  for (size_t l = 1; l < mg_->lv.size(); ++l) {
    MgLevel& L = mg_->lv[l];
    ++launches;
    k_q1_diag_inv<<<grid_for(L.size), kT, 0, st>>>(L.n, L.h, mc, L.inv);
    CK(cudaGetLastError());
  }
  // smoother intervals (every level but the coarsest)
  for (size_t l = 0; l + 1 < mg_->lv.size(); ++l) OK(mg_lambda_max((int)l, mg_->lv[l].lmax));
  // coarsest: dense inverse
  std::vector<double> inv;
  if (!dense_q1_inverse(mg_->lv.back().n, mg_side_, mc, inv)) return fail(DGB_E_NOT_SPD, "pressure multigrid: singular coarse operator");
  CK(cudaMemcpyAsync(mg_->coarse_inv, inv.data(), inv.size() * sizeof(double), cudaMemcpyHostToDevice, st));
  CK(cudaStreamSynchronize(st));
  return DGB_OK;
}

int Context::mg_precondition(double mc, const double* r, double* z) {
  OK(mg_setup(mc));
  return mg_vcycle(0, r, z);
}

// CG with the multigrid V-cycle as preconditioner.  Same stopping rule and outer
// true-residual restarts as cg_solve (krylov.cpp:43-101); only z = B r differs.
int Context::cg_mg(double mc, const dgb_solver_settings& s, const double* b, double* x, SolveOut& out) {
  const size_t n = np();
  cudaStream_t st = dc.stream;
  out = SolveOut();
  OK(mg_setup(mc));
  double bb;
  OK(dot(n, b, b, &bb));
  const double bnorm = std::sqrt(bb);
  if (bnorm == 0.0) {
    ++launches;
    CK(v_fill(st, n, 0.0, x));
    return DGB_OK;
  }
  const double tol = std::max(s.rel_tol * bnorm, s.abs_tol);
  double* r = scratch_vec(20, n);
  double* z = scratch_vec(21, n);
  double* p = scratch_vec(22, n);
  double* q = scratch_vec(23, n);
  if (!r || !z || !p || !q) return fail(DGB_E_CUDA, "cg_mg: out of device memory");
  int iter = 0;
  while (true) {
    OK(sip(mc, 0, x, r));
    ++launches;
    CK(v_rsub(st, n, b, r));
    double rr;
    OK(dot(n, r, r, &rr));
    double rnorm = std::sqrt(rr);
    out.history.push_back(rnorm);
    if (rnorm <= tol) {
      out.iterations = iter;
      out.residual = rnorm;
      return DGB_OK;
    }
    if (iter >= s.max_iter)
      return fail(DGB_E_NO_CONVERGENCE, "cg_mg: no convergence in " + std::to_string(s.max_iter) +
                                            " iterations (residual " + std::to_string(rnorm) + ")");
    OK(mg_vcycle(0, r, z));
    double rz;
    OK(dot(n, r, z, &rz));
    CK(cudaMemcpyAsync(p, z, n * sizeof(double), cudaMemcpyDeviceToDevice, st));
    while (iter < s.max_iter) {
      OK(sip(mc, 0, p, q));
      double pq;
      OK(dot(n, p, q, &pq));
      if (!(pq > 0.0)) return fail(DGB_E_NOT_SPD, "cg_mg: operator or preconditioner not SPD");
      const double alpha = rz / pq;
      launches += 2;
      CK(v_axpy(st, n, alpha, p, x));
      CK(v_axpy(st, n, -alpha, q, r));
      ++iter;
      OK(dot(n, r, r, &rr));
      rnorm = std::sqrt(rr);
      out.history.push_back(rnorm);
      if (rnorm <= tol) break;
      OK(mg_vcycle(0, r, z));
      double rz_new;
      OK(dot(n, r, z, &rz_new));
      const double beta = rz_new / rz;
      rz = rz_new;
      ++launches;
      CK(v_axpby(st, n, 1.0, z, beta, p));
    }
  }
}

}  // namespace dgb
