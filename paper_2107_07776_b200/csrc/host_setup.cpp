// Host setup: tables, mesh, geometry.  See host_setup.hpp for the conventions
// and the reference lines each piece reproduces.
#include "host_setup.hpp"

#include <algorithm>
#include <cmath>
#include <map>
#include <random>
#include <thread>
#include <vector>

namespace dgb {

// ---------------------------------------------------------------------------
// 1D rules (algorithm of quadrature.cpp:11-69: Newton on P_n / P'_m)
// ---------------------------------------------------------------------------
static void legendre_pd(int n, double t, double& p, double& dp) {
  if (n == 0) {
    p = 1.0;
    dp = 0.0;
    return;
  }
  double pm1 = 1.0, pc = t;
  for (int k = 2; k <= n; ++k) {
    const double pk = ((2.0 * k - 1.0) * t * pc - (k - 1.0) * pm1) / k;
    pm1 = pc;
    pc = pk;
  }
  p = pc;
  dp = n * (t * pc - pm1) / (t * t - 1.0);
}

Rule1D gauss_legendre(int n) {
  Rule1D r;
  r.x.assign(n, 0.0);
  r.w.assign(n, 0.0);
  for (int i = 0; i < n; ++i) {
    double t = std::cos(M_PI * (i + 0.75) / (n + 0.5));
    double p, dp;
    for (int it = 0; it < 100; ++it) {
      legendre_pd(n, t, p, dp);
      const double step = p / dp;
      t -= step;
      if (std::abs(step) < 1e-16) break;
    }
    legendre_pd(n, t, p, dp);
    r.x[n - 1 - i] = 0.5 * (t + 1.0);
    r.w[n - 1 - i] = 1.0 / ((1.0 - t * t) * dp * dp);
  }
  return r;
}

std::vector<double> gauss_lobatto(int n) {
  std::vector<double> x(n, 0.0);
  x[n - 1] = 1.0;
  const int m = n - 1;
  for (int i = 1; i < m; ++i) {
    double t = std::cos(M_PI * (m - i) / m);
    for (int it = 0; it < 100; ++it) {
      double p, dp;
      legendre_pd(m, t, p, dp);
      const double d2p = (2.0 * t * dp - m * (m + 1.0) * p) / (1.0 - t * t);
      const double step = dp / d2p;
      t -= step;
      if (std::abs(step) < 1e-16) break;
    }
    x[i] = 0.5 * (t + 1.0);
  }
  return x;
}

void lagrange_tables(const std::vector<double>& nodes, const std::vector<double>& pts,
                     std::vector<double>& val, std::vector<double>& der) {
  const int m = static_cast<int>(nodes.size());
  const int np = static_cast<int>(pts.size());
  std::vector<double> bary(m, 1.0);
  for (int i = 0; i < m; ++i)
    for (int j = 0; j < m; ++j)
      if (j != i) bary[i] /= (nodes[i] - nodes[j]);
  val.assign(static_cast<size_t>(np) * m, 0.0);
  der.assign(static_cast<size_t>(np) * m, 0.0);
  for (int q = 0; q < np; ++q) {
    const double t = pts[q];
    double* v = &val[static_cast<size_t>(q) * m];
    double* g = &der[static_cast<size_t>(q) * m];
    int hit = -1;
    for (int i = 0; i < m; ++i)
      if (t == nodes[i]) hit = i;
    if (hit >= 0) {
      for (int j = 0; j < m; ++j) v[j] = (j == hit) ? 1.0 : 0.0;
    } else {
      double l = 1.0;
      for (int j = 0; j < m; ++j) l *= (t - nodes[j]);
      for (int i = 0; i < m; ++i) v[i] = l * bary[i] / (t - nodes[i]);
    }
    for (int i = 0; i < m; ++i) {
      double s = 0.0;
      for (int k = 0; k < m; ++k) {
        if (k == i) continue;
        double p = 1.0;
        for (int j = 0; j < m; ++j)
          if (j != i && j != k) p *= (t - nodes[j]);
        s += p;
      }
      g[i] = bary[i] * s;
    }
  }
}

// ---------------------------------------------------------------------------
// Mesh geometry primitives (mesh.cpp:20-72 conventions)
// ---------------------------------------------------------------------------
static int face_corner_vertex(int dim, int face, int corner) {
  const int a = face / 2, s = face % 2;
  int v = s << a;
  int t = 0;
  for (int d = 0; d < dim; ++d) {
    if (d == a) continue;
    v |= ((corner >> t) & 1) << d;
    ++t;
  }
  return v;
}

void map_point(const HostMesh& m, int c, const double* ref, double* x) {
  const int dim = m.dim;
  for (int d = 0; d < dim; ++d) x[d] = 0.0;
  for (int v = 0; v < m.nv_cell(); ++v) {
    double s = 1.0;
    for (int d = 0; d < dim; ++d) s *= ((v >> d) & 1) ? ref[d] : (1.0 - ref[d]);
    const double* X = m.vert(c, v);
    for (int d = 0; d < dim; ++d) x[d] += s * X[d];
  }
}

void jacobian(const HostMesh& m, int c, const double* ref, double* J) {
  const int dim = m.dim;
  for (int i = 0; i < dim * dim; ++i) J[i] = 0.0;
  for (int v = 0; v < m.nv_cell(); ++v) {
    const double* X = m.vert(c, v);
    for (int a = 0; a < dim; ++a) {
      double s = 1.0;
      for (int d = 0; d < dim; ++d) {
        if (d == a)
          s *= ((v >> d) & 1) ? 1.0 : -1.0;
        else
          s *= ((v >> d) & 1) ? ref[d] : (1.0 - ref[d]);
      }
      for (int d = 0; d < dim; ++d) J[d * dim + a] += s * X[d];
    }
  }
}

double invert(int dim, const double* J, double* inv) {
  if (dim == 2) {
    const double det = J[0] * J[3] - J[1] * J[2];
    const double id = 1.0 / det;
    inv[0] = J[3] * id;
    inv[1] = -J[1] * id;
    inv[2] = -J[2] * id;
    inv[3] = J[0] * id;
    return det;
  }
  auto j = [&](int r, int c) { return J[r * 3 + c]; };
  const double c00 = j(1, 1) * j(2, 2) - j(1, 2) * j(2, 1);
  const double c01 = j(1, 2) * j(2, 0) - j(1, 0) * j(2, 2);
  const double c02 = j(1, 0) * j(2, 1) - j(1, 1) * j(2, 0);
  const double det = j(0, 0) * c00 + j(0, 1) * c01 + j(0, 2) * c02;
  const double id = 1.0 / det;
  inv[0] = c00 * id;
  inv[1] = (j(0, 2) * j(2, 1) - j(0, 1) * j(2, 2)) * id;
  inv[2] = (j(0, 1) * j(1, 2) - j(0, 2) * j(1, 1)) * id;
  inv[3] = c01 * id;
  inv[4] = (j(0, 0) * j(2, 2) - j(0, 2) * j(2, 0)) * id;
  inv[5] = (j(0, 2) * j(1, 0) - j(0, 0) * j(1, 2)) * id;
  inv[6] = c02 * id;
  inv[7] = (j(0, 1) * j(2, 0) - j(0, 0) * j(2, 1)) * id;
  inv[8] = (j(0, 0) * j(1, 1) - j(0, 1) * j(1, 0)) * id;
  return det;
}

static double det_of(int dim, const double* J) {
  if (dim == 2) return J[0] * J[3] - J[1] * J[2];
  return J[0] * (J[4] * J[8] - J[5] * J[7]) - J[1] * (J[3] * J[8] - J[5] * J[6]) +
         J[2] * (J[3] * J[7] - J[4] * J[6]);
}

static bool check_jacobians(const HostMesh& m, std::string& err) {
  double ref[3], J[9];
  for (int c = 0; c < m.ncells; ++c) {
    for (int v = 0; v <= m.nv_cell(); ++v) {
      for (int d = 0; d < m.dim; ++d) ref[d] = v < m.nv_cell() ? ((v >> d) & 1) : 0.5;
      jacobian(m, c, ref, J);
      if (det_of(m.dim, J) <= 0.0) {
        err = "mesh: nonpositive Jacobian in cell " + std::to_string(c);
        return false;
      }
    }
  }
  return true;
}

bool finalize_mesh(HostMesh& m, std::string& err) {
  const int dim = m.dim, nf = m.nf_cell(), nv = m.nv_cell();
  if (!check_jacobians(m, err)) return false;
  // cell measure: 2-point tensor Gauss of det J (mesh.cpp:101-109)
  const Rule1D g2 = gauss_legendre(2);
  m.cell_measure.assign(m.ncells, 0.0);
  m.cell_diam.assign(m.ncells, 0.0);
  double ref[3], J[9];
  const int n2 = dim == 2 ? 4 : 8;
  m.affine = true;
  for (int c = 0; c < m.ncells; ++c) {
    double meas = 0.0;
    for (int i = 0; i < n2; ++i) {
      double w = 1.0;
      int rem = i;
      for (int d = 0; d < dim; ++d) {
        ref[d] = g2.x[rem % 2];
        w *= g2.w[rem % 2];
        rem /= 2;
      }
      jacobian(m, c, ref, J);
      meas += det_of(dim, J) * w;
    }
    m.cell_measure[c] = meas;
    double dmax = 0.0;
    for (int i = 0; i < nv; ++i)
      for (int j = i + 1; j < nv; ++j) {
        double s = 0.0;
        for (int d = 0; d < dim; ++d) {
          const double e = m.vert(c, i)[d] - m.vert(c, j)[d];
          s += e * e;
        }
        dmax = std::max(dmax, s);
      }
    m.cell_diam[c] = std::sqrt(dmax);
    // parallelepiped test: x_v = x_0 + sum_a bit_a(v) (x_{1<<a} - x_0)
    for (int v = 0; v < nv && m.affine; ++v)
      for (int d = 0; d < dim; ++d) {
        double pred = m.vert(c, 0)[d];
        for (int a = 0; a < dim; ++a)
          if ((v >> a) & 1) pred += m.vert(c, 1 << a)[d] - m.vert(c, 0)[d];
        if (std::abs(pred - m.vert(c, v)[d]) > 1e-13 * m.cell_diam[c]) {
          m.affine = false;
          break;
        }
      }
  }
  // face measures from this cell's corners (mesh.cpp:268-292)
  m.face_measure.assign(static_cast<size_t>(m.ncells) * nf, 0.0);
  for (int c = 0; c < m.ncells; ++c)
    for (int f = 0; f < nf; ++f) {
      const double* p[4];
      for (int j = 0; j < (1 << (dim - 1)); ++j) p[j] = m.vert(c, face_corner_vertex(dim, f, j));
      double meas;
      if (dim == 2) {
        double s = 0.0;
        for (int d = 0; d < 2; ++d) s += (p[1][d] - p[0][d]) * (p[1][d] - p[0][d]);
        meas = std::sqrt(s);
      } else {
        auto tri = [](const double* a, const double* b, const double* q) {
          const double u[3] = {b[0] - a[0], b[1] - a[1], b[2] - a[2]};
          const double v[3] = {q[0] - a[0], q[1] - a[1], q[2] - a[2]};
          const double x = u[1] * v[2] - u[2] * v[1];
          const double y = u[2] * v[0] - u[0] * v[2];
          const double z = u[0] * v[1] - u[1] * v[0];
          return 0.5 * std::sqrt(x * x + y * y + z * z);
        };
        meas = tri(p[0], p[1], p[3]) + tri(p[0], p[3], p[2]);
      }
      m.face_measure[static_cast<size_t>(c) * nf + f] = meas;
    }
  // reference face lists (mesh.cpp:316-377, conforming part)
  m.iface.clear();
  m.bface.clear();
  for (int c = 0; c < m.ncells; ++c)
    for (int f = 0; f < nf; ++f) {
      const int nb = m.nbr[static_cast<size_t>(c) * nf + f];
      if (m.hanging(c, f)) {  // recorded once per subface, from the fine side (mesh.cpp:344-375)
        const int h = m.hface[static_cast<size_t>(c) * nf + f];
        if (h >= 0) m.iface.insert(m.iface.end(), {c, f, m.hrec[4 * h + 2], m.hrec[4 * h + 3]});
      } else if (nb < 0) {
        m.bface.insert(m.bface.end(), {c, f, -1 - nb});
      } else if (c < nb) {
        m.iface.insert(m.iface.end(), {c, f, nb, f ^ 1});
      }
    }
  return true;
}

HostMesh make_cartesian(int dim, int n_el, double amp, unsigned seed, std::string& err) {
  HostMesh m;
  m.dim = dim;
  if (n_el < 1 || (dim != 2 && dim != 3)) {
    err = "make_cartesian: bad arguments";
    return m;
  }
  const int nv1 = n_el + 1;
  int nvert = 1, nc = 1;
  for (int d = 0; d < dim; ++d) {
    nvert *= nv1;
    nc *= n_el;
  }
  m.vertices.assign(static_cast<size_t>(nvert) * dim, 0.0);
  for (int i = 0; i < nvert; ++i) {
    int rem = i;
    for (int d = 0; d < dim; ++d) {
      const int id = rem % nv1;
      rem /= nv1;
      m.vertices[static_cast<size_t>(i) * dim + d] = 0.0 + (1.0 - 0.0) * id / n_el;
    }
  }
  m.ncells = nc;
  const int nv = 1 << dim, nf = 2 * dim;
  m.cell_v.assign(static_cast<size_t>(nc) * nv, 0);
  m.nbr.assign(static_cast<size_t>(nc) * nf, 0);
  for (int i = 0; i < nc; ++i) {
    int rem = i, ic[3] = {0, 0, 0};
    for (int d = 0; d < dim; ++d) {
      ic[d] = rem % n_el;
      rem /= n_el;
    }
    for (int b = 0; b < nv; ++b) {
      int vi = 0, stride = 1;
      for (int d = 0; d < dim; ++d) {
        vi += (ic[d] + ((b >> d) & 1)) * stride;
        stride *= nv1;
      }
      m.cell_v[static_cast<size_t>(i) * nv + b] = vi;
    }
    int cstride = 1;
    for (int d = 0; d < dim; ++d) {
      int* nb = &m.nbr[static_cast<size_t>(i) * nf];
      nb[2 * d] = ic[d] == 0 ? -1 - (2 * d) : i - cstride;
      nb[2 * d + 1] = ic[d] == n_el - 1 ? -1 - (2 * d + 1) : i + cstride;
      cstride *= n_el;
    }
  }
  if (amp != 0.0) {
    // distort (mesh.cpp:618-646): same engine, distribution and draw order
    std::vector<char> on_boundary(nvert, 0);
    for (int c = 0; c < nc; ++c)
      for (int f = 0; f < nf; ++f) {
        if (m.nbr[static_cast<size_t>(c) * nf + f] >= 0) continue;
        for (int j = 0; j < (1 << (dim - 1)); ++j)
          on_boundary[m.cell_v[static_cast<size_t>(c) * nv + face_corner_vertex(dim, f, j)]] = 1;
      }
    std::mt19937 rng(seed);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    for (int v = 0; v < nvert; ++v) {
      if (on_boundary[v]) continue;
      for (int d = 0; d < dim; ++d) m.vertices[static_cast<size_t>(v) * dim + d] += amp * uni(rng);
    }
  }
  if (!finalize_mesh(m, err)) m.ncells = 0;
  return m;
}

HostMesh make_from_arrays(int dim, int nverts, const double* verts, int ncells, const int* cell_v,
                          const int* boundary_ids, std::string& err, int n_hang, const int* hang_rec,
                          const double* hang_emb) {
  HostMesh m;
  m.dim = dim;
  m.ncells = ncells;
  const int nv = 1 << dim, nf = 2 * dim, nfc = 1 << (dim - 1);
  m.vertices.assign(verts, verts + static_cast<size_t>(nverts) * dim);
  m.cell_v.assign(cell_v, cell_v + static_cast<size_t>(ncells) * nv);
  m.nbr.assign(static_cast<size_t>(ncells) * nf, 0);
  // hanging subfaces (mesh.cpp:344-375): both sides' slots are taken out of the pairing
  if (n_hang > 0) {
    if (!hang_rec || !hang_emb) {
      err = "hanging faces: null record / embedding array";
      m.ncells = 0;
      return m;
    }
    m.hface.assign(static_cast<size_t>(ncells) * nf, -1);
    m.hrec.assign(hang_rec, hang_rec + static_cast<size_t>(n_hang) * 4);
    m.hemb.assign(hang_emb, hang_emb + static_cast<size_t>(n_hang) * dim * dim);
    for (int h = 0; h < n_hang; ++h) {
      const int K = hang_rec[4 * h], f = hang_rec[4 * h + 1], N = hang_rec[4 * h + 2], fN = hang_rec[4 * h + 3];
      if (K < 0 || K >= ncells || N < 0 || N >= ncells || K == N || f < 0 || f >= nf || fN < 0 || fN >= nf ||
          (boundary_ids && (boundary_ids[static_cast<size_t>(K) * nf + f] >= 0 ||
                            boundary_ids[static_cast<size_t>(N) * nf + fN] >= 0))) {
        err = "hanging face record " + std::to_string(h) + " is not an interior fine/coarse face pair";
        m.ncells = 0;
        return m;
      }
      int& sK = m.hface[static_cast<size_t>(K) * nf + f];
      int& sN = m.hface[static_cast<size_t>(N) * nf + fN];
      if (sK != -1 || sN >= 0) {
        err = "hanging face record " + std::to_string(h) + " reuses a face slot";
        m.ncells = 0;
        return m;
      }
      sK = h;
      sN = -2;
    }
  }
  std::map<std::array<int, 4>, std::pair<int, int>> open;
  for (int c = 0; c < ncells; ++c)
    for (int f = 0; f < nf; ++f) {
      const int bid = boundary_ids ? boundary_ids[static_cast<size_t>(c) * nf + f] : -1;
      if (bid >= 0) {
        m.nbr[static_cast<size_t>(c) * nf + f] = -1 - bid;
        continue;
      }
      if (m.hanging(c, f)) {
        m.nbr[static_cast<size_t>(c) * nf + f] = c;  // zero-weight self face (see HostMesh::hrec)
        continue;
      }
      std::array<int, 4> key{-1, -1, -1, -1};
      for (int j = 0; j < nfc; ++j) key[j] = cell_v[static_cast<size_t>(c) * nv + face_corner_vertex(dim, f, j)];
      std::sort(key.begin(), key.begin() + nfc);
      auto it = open.find(key);
      if (it == open.end()) {
        open.emplace(key, std::make_pair(c, f));
        continue;
      }
      const int N = it->second.first, fN = it->second.second;
      open.erase(it);
      // identity orientation: opposite side of the same axis, corners in the same order
      bool ok = (fN == (f ^ 1));
      for (int j = 0; j < nfc && ok; ++j)
        ok = cell_v[static_cast<size_t>(c) * nv + face_corner_vertex(dim, f, j)] ==
             cell_v[static_cast<size_t>(N) * nv + face_corner_vertex(dim, fN, j)];
      if (!ok) {
        err = "unsupported mesh: face between cells " + std::to_string(N) + " and " + std::to_string(c) +
              " is not identity-oriented (only Cartesian-topology meshes are supported)";
        m.ncells = 0;
        return m;
      }
      m.nbr[static_cast<size_t>(c) * nf + f] = N;
      m.nbr[static_cast<size_t>(N) * nf + fN] = c;
    }
  if (!open.empty()) {
    err = "mesh: interior face without neighbor or boundary id (hanging faces are not supported)";
    m.ncells = 0;
    return m;
  }
  if (!finalize_mesh(m, err)) m.ncells = 0;
  return m;
}

// ---------------------------------------------------------------------------
// Geometry tables
// ---------------------------------------------------------------------------
int cell_geo_stride(int dim) { return dim * dim + 1; }
int face_geo_stride(int dim) { return 2 * dim * dim + dim + 1; }
int affine_cell_stride(int dim) { return dim * dim + 1 + 2 * dim * (dim + 1); }

// reference point of face quadrature point t of local face f (canonical embedding,
// tangents = remaining axes in increasing order, x fastest in face coordinates)
static void face_ref_point(int dim, int f, int side_override, const Rule1D& r, int t, double* ref) {
  const int a = f / 2;
  ref[a] = side_override;
  int rem = t;
  for (int d = 0; d < dim; ++d) {
    if (d == a) continue;
    ref[d] = r.x[rem % r.x.size()];
    rem /= static_cast<int>(r.x.size());
  }
}

void embed_point(int dim, const double* emb, const Rule1D& r, int t, double* ref) {
  double xi[2] = {0.0, 0.0};
  int rem = t;
  for (int k = 0; k < dim - 1; ++k) {
    xi[k] = r.x[rem % r.x.size()];
    rem /= static_cast<int>(r.x.size());
  }
  for (int d = 0; d < dim; ++d) {
    double v = emb[d];
    for (int k = 0; k < dim - 1; ++k) v += xi[k] * emb[dim + k * dim + d];
    ref[d] = v;
  }
}

void canonical_embedding(int dim, int f, double* emb) {
  const int a = f / 2;
  for (int i = 0; i < dim * dim; ++i) emb[i] = 0.0;
  emb[a] = f % 2;
  int k = 0;
  for (int d = 0; d < dim; ++d)
    if (d != a) emb[dim + (k++) * dim + d] = 1.0;
}

static double face_weight(int dim, const Rule1D& r, int t) {
  double w = 1.0;
  int rem = t;
  for (int d = 0; d < dim - 1; ++d) {
    w *= r.w[rem % r.w.size()];
    rem /= static_cast<int>(r.w.size());
  }
  return w;
}

void face_frame(int dim, int f, const double* J, const double* Jinv, double* n, double& ds) {
  const int a = f / 2;
  const double sgn = (f % 2) == 1 ? 1.0 : -1.0;
  double tau[2][3];
  int t = 0;
  for (int d = 0; d < dim; ++d) {
    if (d == a) continue;
    for (int e = 0; e < dim; ++e) tau[t][e] = J[e * dim + d];
    ++t;
  }
  if (dim == 2) {
    ds = std::hypot(tau[0][0], tau[0][1]);
  } else {
    const double cr[3] = {tau[0][1] * tau[1][2] - tau[0][2] * tau[1][1],
                          tau[0][2] * tau[1][0] - tau[0][0] * tau[1][2],
                          tau[0][0] * tau[1][1] - tau[0][1] * tau[1][0]};
    ds = std::sqrt(cr[0] * cr[0] + cr[1] * cr[1] + cr[2] * cr[2]);
  }
  double nn = 0.0;
  for (int d = 0; d < dim; ++d) {
    n[d] = sgn * Jinv[a * dim + d];
    nn += n[d] * n[d];
  }
  nn = 1.0 / std::sqrt(nn);
  for (int d = 0; d < dim; ++d) n[d] *= nn;
}

void build_qp_geometry(const HostMesh& m, int Q, QpGeometry& g) {
  const int dim = m.dim, nf = m.nf_cell();
  const Rule1D r = gauss_legendre(Q);
  const int nq = dim == 2 ? Q * Q : Q * Q * Q;
  const int nqf = dim == 2 ? Q : Q * Q;
  const int cs = cell_geo_stride(dim), fs = face_geo_stride(dim);
  g.Q = Q;
  g.cell.assign(static_cast<size_t>(m.ncells) * nq * cs, 0.0);
  g.face.assign(static_cast<size_t>(m.ncells) * nf * nqf * fs, 0.0);
  // cells are independent: split them over the host threads (setup of the deformed
  // cfg4 mesh: ~30 s single-threaded)
  parallel_cells(m.ncells, [&](int c0, int c1) {
  double ref[3], J[9], Ji[9];
  for (int c = c0; c < c1; ++c) {
    for (int q = 0; q < nq; ++q) {
      int rem = q;
      double w = 1.0;
      for (int d = 0; d < dim; ++d) {
        ref[d] = r.x[rem % Q];
        w *= r.w[rem % Q];
        rem /= Q;
      }
      jacobian(m, c, ref, J);
      double* o = &g.cell[(static_cast<size_t>(c) * nq + q) * cs];
      const double det = invert(dim, J, o);
      o[dim * dim] = det * w;
    }
    for (int f = 0; f < nf; ++f) {
      const int nb = m.nbr[static_cast<size_t>(c) * nf + f];
      for (int t = 0; t < nqf; ++t) {
        double* o = &g.face[((static_cast<size_t>(c) * nf + f) * nqf + t) * fs];
        face_ref_point(dim, f, f % 2, r, t, ref);
        jacobian(m, c, ref, J);
        invert(dim, J, Ji);
        for (int i = 0; i < dim * dim; ++i) o[i] = Ji[i];
        double n[3], ds;
        face_frame(dim, f, J, Ji, n, ds);
        if (nb >= 0) {
          face_ref_point(dim, f, 1 - (f % 2), r, t, ref);
          double J2[9];
          jacobian(m, nb, ref, J2);
          invert(dim, J2, o + dim * dim);
        }
        for (int d = 0; d < dim; ++d) o[2 * dim * dim + d] = n[d];
        o[2 * dim * dim + dim] = m.hanging(c, f) ? 0.0 : ds * face_weight(dim, r, t);
      }
    }
  }
  });
}

void build_affine_geometry(const HostMesh& m, std::vector<double>& g) {
  const int dim = m.dim, nf = m.nf_cell(), st = affine_cell_stride(dim);
  g.assign(static_cast<size_t>(m.ncells) * st, 0.0);
  double ref[3] = {0.5, 0.5, 0.5}, J[9];
  for (int c = 0; c < m.ncells; ++c) {
    double* o = &g[static_cast<size_t>(c) * st];
    jacobian(m, c, ref, J);
    o[dim * dim] = invert(dim, J, o);
    for (int f = 0; f < nf; ++f) {
      double* of = o + dim * dim + 1 + f * (dim + 1);
      double ds;
      face_frame(dim, f, J, o, of, ds);
      of[dim] = m.hanging(c, f) ? 0.0 : ds;
    }
  }
}

void boundary_points(const HostMesh& m, int Q, std::vector<double>& xq) {
  const int dim = m.dim;
  const Rule1D r = gauss_legendre(Q);
  const int nqf = dim == 2 ? Q : Q * Q;
  const size_t nb = m.bface.size() / 3;
  xq.assign(nb * nqf * dim, 0.0);
  double ref[3];
  for (size_t b = 0; b < nb; ++b) {
    const int c = m.bface[3 * b], f = m.bface[3 * b + 1];
    for (int t = 0; t < nqf; ++t) {
      face_ref_point(dim, f, f % 2, r, t, ref);
      map_point(m, c, ref, &xq[(b * nqf + t) * dim]);
    }
  }
}

}  // namespace dgb

// ---------------------------------------------------------------------------
// Constant-table fillers used by dg_common.cuh (ensure_tab)
// ---------------------------------------------------------------------------
namespace dgb {
void host_tab(int N, int Q, double* B, double* D, double* dE) {
  const std::vector<double> nodes = gauss_lobatto(N);
  const Rule1D r = gauss_legendre(Q);
  std::vector<double> val, der;
  lagrange_tables(nodes, r.x, val, der);
  for (int i = 0; i < Q * N; ++i) {
    B[i] = val[i];
    D[i] = der[i];
  }
  lagrange_tables(nodes, {0.0, 1.0}, val, der);
  for (int i = 0; i < 2 * N; ++i) dE[i] = der[i];
}
void host_w(int Q, double* w) {
  const Rule1D r = gauss_legendre(Q);
  for (int i = 0; i < Q; ++i) w[i] = r.w[i];
}
}  // namespace dgb
