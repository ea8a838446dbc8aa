// Host-side setup for the device context: 1D shape tables, the conforming
// hexahedral / quadrilateral mesh in the reference's numbering, and the
// per-cell geometry the kernels consume.  Runs once per context.
//
// Conventions reproduced from the reference:
//  * Gauss-Legendre points ascending on [0,1], weights summing to 1
//    (proj/src/quadrature.cpp:25-46); Gauss-Lobatto nodal basis
//    (quadrature.cpp:48-69, space.cpp:189-203); barycentric Lagrange values /
//    product-rule derivatives (lagrange.cpp:10-50).
//  * vertices lexicographic v = ix + 2 iy + 4 iz, local face 2*axis+side
//    (mesh.hpp:5-15); Cartesian generator numbering and boundary ids
//    (mesh.cpp:571-616); seeded interior-vertex distortion (mesh.cpp:618-646).
//  * cell measure by 2-point Gauss of det J (mesh.cpp:101-109); face measure
//    from the corners (mesh.cpp:268-292); penalty sigma = (deg+1)^2 |F|/|K|
//    (forms.hpp:175-177), interior faces use the mean of both sides
//    (forms.cpp:111-121), boundary faces 2*sigma_K in the operators.
//  * Jinv stored row-major Jinv[a*dim+j] = d xi_a / d x_j (space.cpp:14-39,81);
//    face normal = Nanson direction from the owner side (space.cpp:133-142).
#pragma once

#include <array>
#include <cstdint>
#include <string>
#include <algorithm>
#include <thread>
#include <vector>

namespace dgb {

// ---------------------------------------------------------------------------
// 1D tables
// ---------------------------------------------------------------------------
struct Rule1D {
  std::vector<double> x, w;
};
Rule1D gauss_legendre(int n);
std::vector<double> gauss_lobatto(int n);

/// Lagrange basis on GL nodes evaluated at points: val[q][j], der[q][j].
void lagrange_tables(const std::vector<double>& nodes, const std::vector<double>& pts,
                     std::vector<double>& val, std::vector<double>& der);

// ---------------------------------------------------------------------------
// Mesh (conforming, every interior face with identity corner orientation)
// ---------------------------------------------------------------------------
struct HostMesh {
  int dim = 0;
  int ncells = 0;
  std::vector<double> vertices;      // nverts x dim
  std::vector<int> cell_v;           // ncells x 2^dim (vertex ids)
  std::vector<int> nbr;              // ncells x 2dim: neighbor cell, or -1 - boundary_id
  std::vector<double> face_measure;  // ncells x 2dim (from this cell's corners)
  std::vector<double> cell_measure;  // ncells
  std::vector<double> cell_diam;     // ncells
  // reference face lists (owner = lower index, cell-major order; mesh.cpp:316-377)
  std::vector<int> iface;  // n_interior x 4: cell_in, face_in, cell_out, face_out
  std::vector<int> bface;  // n_boundary x 3: cell, face, boundary_id
  bool affine = true;      // every cell a parallelepiped (constant Jacobian)
  // Hanging subfaces of a 1-irregular refined mesh (mesh.cpp:344-375), one record per
  // fine face: fine cell, fine face, coarse cell, coarse face, and the subface
  // embedding into the coarse cell's reference cell (FaceInfo::emb_out, mesh.hpp:28-36:
  // origin[dim], tangent[t][dim] for t < dim-1).  The element-centric kernels see a
  // hanging (cell, face) slot as an interior face to the cell itself with zero surface
  // weight (nbr = cell, ds = 0: every face integrand carries w_ds, so it contributes
  // nothing); hang.cu adds the two-sided subface terms.
  std::vector<int> hrec;     // n_hang x 4
  std::vector<double> hemb;  // n_hang x dim*dim
  std::vector<int> hface;    // ncells x 2dim: -1 conforming / boundary, h >= 0 fine side of record h, -2 coarse side
  int n_hang() const { return static_cast<int>(hrec.size() / 4); }
  bool hanging(int c, int f) const { return !hface.empty() && hface[static_cast<size_t>(c) * nf_cell() + f] != -1; }

  int nv_cell() const { return 1 << dim; }
  int nf_cell() const { return 2 * dim; }
  const double* vert(int c, int v) const { return &vertices[static_cast<size_t>(cell_v[c * nv_cell() + v]) * dim]; }
};

/// generate_cartesian on [0,1]^dim (mesh.cpp:571-616) + optional distort (mesh.cpp:618-646).
HostMesh make_cartesian(int dim, int n_el, double amp, unsigned seed, std::string& err);
/// From raw arrays (vertices, cell->vertex, boundary ids per cell face (-1 = none)).
HostMesh make_from_arrays(int dim, int nverts, const double* verts, int ncells, const int* cell_v,
                          const int* boundary_ids, std::string& err, int n_hang = 0, const int* hang_rec = nullptr,
                          const double* hang_emb = nullptr);
/// Recompute measures, diameters, face lists, affinity. Fills err on failure.
bool finalize_mesh(HostMesh& m, std::string& err);

// Multilinear map, Jacobian J[d][a] = dx_d/dxi_a, and inverse (space.cpp:14-39 convention).
void map_point(const HostMesh& m, int c, const double* ref, double* x);
void jacobian(const HostMesh& m, int c, const double* ref, double* J);
double invert(int dim, const double* J, double* Jinv);

// ---------------------------------------------------------------------------
// Geometry tables uploaded to the device
// ---------------------------------------------------------------------------
/// Per-quadrature-point geometry for rule Q (general / deformed cells):
///  cell[c][q] = {Jinv (dim^2), detJ*w}          (CellGeometry, space.hpp:27-32)
///  face[c][f][q] = {Jinv_self (dim^2), Jinv_nbr (dim^2), n_out (dim), w_ds}
/// seen from cell c (n points out of c; Jinv_nbr = 0 on boundary faces).
struct QpGeometry {
  int Q = 0;
  std::vector<double> cell, face;
};
int cell_geo_stride(int dim);
/// Reference point of face-quadrature point t (first face parameter fastest) under an
/// embedding {origin[dim], tangent[dim-1][dim]} (FaceEmbedding, mesh.hpp:28-36).
void embed_point(int dim, const double* emb, const Rule1D& r, int t, double* ref);
/// The canonical embedding of local face f (mesh.cpp:240-248).
void canonical_embedding(int dim, int f, double* emb);
/// Surface element of the canonical face-f parameterisation and the unit normal out of
/// the cell (Nanson, space.cpp:133-142) from J and Jinv at a face point.
void face_frame(int dim, int f, const double* J, const double* Jinv, double* n, double& ds);
int face_geo_stride(int dim);
void build_qp_geometry(const HostMesh& m, int Q, QpGeometry& g);
// fn(c0, c1) over [0, n) split into contiguous chunks, one per host thread (setup loops)
template <class Fn>
inline void parallel_cells(int n, Fn fn) {
  const int nt = std::max(1, std::min<int>((int)std::thread::hardware_concurrency(), 64));
  if (nt == 1 || n < 4096) {
    fn(0, n);
    return;
  }
  std::vector<std::thread> th;
  const int per = (n + nt - 1) / nt;
  for (int t = 0; t < nt; ++t) {
    const int c0 = t * per, c1 = std::min(n, c0 + per);
    if (c0 < c1) th.emplace_back(fn, c0, c1);
  }
  for (auto& x : th) x.join();
}


/// Per-cell geometry for affine cells: {Jinv (dim^2), detJ} + per face {n (dim), ds}
int affine_cell_stride(int dim);
void build_affine_geometry(const HostMesh& m, std::vector<double>& g);

/// Physical points of boundary-face quadrature points for rule Q, in the
/// reference boundary-face order (GeometryCache::boundary_faces xq).
void boundary_points(const HostMesh& m, int Q, std::vector<double>& xq);

/// Constant-table fillers (device tables are uploaded from these).
void host_tab(int N, int Q, double* B, double* D, double* dE);
void host_w(int Q, double* w);

}  // namespace dgb
