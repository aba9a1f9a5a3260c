// Non-moralising G-QSW operators (the demoralisation scheme).
//
// Mirrors proj/core/include/qsw/operators.hpp:16-83 (VertexSubspaces, nm_vsets,
// demoralised_weights, nm_H, nm_L, nm_H_rot, nm_rho_map, nm_measure).  These
// only build the small expanded-space operators; the walk then runs through
// build_global with the rotating Hamiltonian, on the same device kernels.
#pragma once

#include <cstdint>
#include <vector>

#include "sparse.hpp"

namespace qswg {

/// Original vertex i owns expanded indices [offsets[i], offsets[i] + dims[i]).
struct VertexSubspaces {
  std::vector<std::int64_t> offsets;  // vertex_count() + 1
  std::vector<std::int64_t> dims;
  std::int64_t vertex_count() const { return static_cast<std::int64_t>(dims.size()); }
  std::int64_t total_dim() const { return offsets.empty() ? 0 : offsets.back(); }
  static VertexSubspaces from_dims(const std::vector<std::int64_t>& dims);
};

enum class Dim2Rotation { Cancel, PauliY };

/// dims[i] = number of arcs into i in the symmetrized graph, at least 1
/// (operators.cpp nm_vsets).  Throws for a non-symmetric adjacency.
VertexSubspaces nm_vsets(const SparseMatrix& gu);
/// Arc k -> i of weight w spreads (dims_i dims_k w)^(-1/2) over every expanded arc.
SparseMatrix demoralised_weights(const SparseMatrix& g, const VertexSubspaces& v);
SparseMatrix nm_H(double gamma, const SparseMatrix& gu, const VertexSubspaces& v);
/// Demoralised Lindblad operator with Fourier phases of the destination subspace.
SparseMatrix nm_L(double gamma, const SparseMatrix& g, const VertexSubspaces& v);
/// Block-diagonal rotation: +i at (k+1 mod d, k), -i at (k-1 mod d, k).
SparseMatrix nm_H_rot(const VertexSubspaces& v, Dim2Rotation dim2 = Dim2Rotation::Cancel);
std::vector<double> nm_rho_map(const std::vector<double>& p, const VertexSubspaces& v);
std::vector<double> nm_measure(const std::vector<double>& diag, const VertexSubspaces& v);

}  // namespace qswg
