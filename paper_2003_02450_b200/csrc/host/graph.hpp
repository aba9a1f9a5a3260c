// Graph -> operator construction (host inputs of the hot path).
//
// Mirrors proj/core/include/qsw/graph.hpp:22-96 and operators.hpp:53-57.
// A graph is its adjacency matrix: column j holds the out-arcs of vertex j,
// so an arc j -> i is entry (i, j) (graph.hpp:32-41).  Every function that
// takes a graph validates it like WeightedDigraph::from_adjacency
// (graph.cpp:22-52): square, no self-loops, real strictly positive weights.
#pragma once

#include <vector>

#include "sparse.hpp"

namespace qswg {

struct SourceArc {
  std::int64_t target = 0;
  double rate = 0.0;
};

struct SinkArc {
  std::int64_t origin = 0;
  double rate = 0.0;
};

/// Throws std::invalid_argument when `adj` is not a valid weighted digraph.
void validate_adjacency(const SparseMatrix& adj);

/// w(i,j) = w(j,i) = max of the two (graph.cpp:152-173).
SparseMatrix symmetrize(const SparseMatrix& adj);
/// Column sums (graph.cpp:175-182).
std::vector<double> out_degrees(const SparseMatrix& adj);
/// Row sums (graph.cpp:184-191).
std::vector<double> in_degrees(const SparseMatrix& adj);
/// M_ij = -gamma G_ij, M_jj = gamma OutDeg(j) (graph.cpp:193-211).
SparseMatrix generator_matrix(double gamma, const SparseMatrix& adj);
/// C_ij = 1/OutDeg(j) where an arc exists (graph.cpp:217-228).
SparseMatrix markov_chain_matrix(const SparseMatrix& adj);
/// One new vertex per source (first) and sink (after) (graph.cpp:230-283).
SparseMatrix augment(const SparseMatrix& adj, const std::vector<SourceArc>& sources,
                     const std::vector<SinkArc>& sinks);
/// Entrywise sqrt|m| (operators.cpp:10-12).
SparseMatrix local_lindblad(const SparseMatrix& m);
/// The adjacency matrix itself (operators.cpp:14).
SparseMatrix global_lindblad(const SparseMatrix& adj);

}  // namespace qswg
