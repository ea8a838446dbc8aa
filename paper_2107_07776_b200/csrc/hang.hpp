// Hanging faces of 1-irregular refined meshes (Mesh::refine_and_coarsen,
// proj/src/mesh.hpp:125-128; subface records and embeddings mesh.cpp:344-375).
//
// The element-centric kernels (dg_ops.cuh, dg_ops_rhs.cuh) see every hanging
// (cell, face) slot as a zero-weight face (HostMesh::hrec).  This module adds
// the two-sided terms of each subface, the same interior-face integrands the
// reference evaluates through the subface embedding (forms.cpp:426-465,
// :537-576 momentum, :179-242 scalar SIP, :677-809 / :273-328 diagonals,
// :859-952 / :1010-1048 stage RHS, :1160-1190 divergence):
//   * one CTA per subface: both sides' traces (values + reference gradients) at
//     the subface Gauss points through dense tables of the basis at the embedded
//     points (GeometryCache / trace_table with a subface embedding,
//     space.cpp:60-162, :216-237), the per-side integrands of the
//     element-centric formulas (normal out of the side doing the work), and the
//     transposed tables back to both sides' coefficients -> a per-(subface,
//     side) contribution block;
//   * one CTA per touched cell adds its contribution blocks in a fixed order
//     (deterministic, no atomics).
// Hanging meshes are rare and small next to the uniform benchmark meshes, so
// this path favours generality (any dim / degree / embedding, runtime sizes).
#pragma once

#include <cuda_runtime.h>

#include <string>

#include "dispatch.hpp"
#include "host_setup.hpp"

namespace dgb {

struct HangState;

/// Build the subface tables / geometry / scatter lists of m and upload them.
/// Returns nullptr with err set on failure (m.n_hang() == 0: nullptr, err empty).
HangState* hang_setup(const HostMesh& m, int ku, int kp, std::string& err);
void hang_release(HangState* h);
/// 0: none, 1: dense-table subface kernels, 2: sum-factorised axis-aligned subface kernels
int hang_mode(const HangState* h);

// y += the hanging-subface terms (launched after the element-centric kernel of the op)
cudaError_t hang_momentum(cudaStream_t st, const HangState* h, MomCoef co, const double* w, const double* x,
                          double* y);
cudaError_t hang_momentum_diag(cudaStream_t st, const HangState* h, MomCoef co, const double* w, double* y);
cudaError_t hang_sip(cudaStream_t st, const HangState* h, const double* x, double* y);
cudaError_t hang_sip_diag(cudaStream_t st, const HangState* h, double* y);
cudaError_t hang_rhs(cudaStream_t st, const HangState* h, const RhsArgs& ra, double* y);
cudaError_t hang_divergence(cudaStream_t st, const HangState* h, const double* u, double* y);

}  // namespace dgb
