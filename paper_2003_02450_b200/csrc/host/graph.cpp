#include "graph.hpp"

#include <cmath>
#include <set>
#include <stdexcept>
#include <string>

namespace qswg {

void validate_adjacency(const SparseMatrix& a) {
  if (a.rows() != a.cols()) throw std::invalid_argument("adjacency matrix must be square");
  for (std::int64_t i = 0; i < a.rows(); ++i) {
    for (std::int64_t k = a.row_begin(i); k < a.row_end(i); ++k) {
      if (a.col_indices()[k] == i)
        throw std::invalid_argument("adjacency has a diagonal entry at vertex " + std::to_string(i) +
                                    " (self-loops are not allowed)");
      const Complex v = a.values()[k];
      if (v.imag() != 0.0) throw std::invalid_argument("adjacency weights must be real");
      if (!(v.real() > 0.0)) throw std::invalid_argument("adjacency weights must be strictly positive");
    }
  }
}

SparseMatrix symmetrize(const SparseMatrix& a) {
  validate_adjacency(a);
  const SparseMatrix t = a.transpose();
  std::vector<Triplet> e;
  e.reserve(static_cast<std::size_t>(2 * a.nnz()));
  for (std::int64_t i = 0; i < a.rows(); ++i) {
    std::int64_t p = a.row_begin(i), pe = a.row_end(i), q = t.row_begin(i), qe = t.row_end(i);
    while (p < pe || q < qe) {
      if (q == qe || (p < pe && a.col_indices()[p] < t.col_indices()[q])) {
        e.push_back({i, a.col_indices()[p], a.values()[p]});
        ++p;
      } else if (p == pe || t.col_indices()[q] < a.col_indices()[p]) {
        e.push_back({i, t.col_indices()[q], t.values()[q]});
        ++q;
      } else {
        e.push_back({i, a.col_indices()[p],
                     Complex{std::max(a.values()[p].real(), t.values()[q].real()), 0.0}});
        ++p;
        ++q;
      }
    }
  }
  SparseMatrix out = SparseMatrix::from_triplets(a.rows(), a.cols(), std::move(e));
  validate_adjacency(out);
  return out;
}

std::vector<double> out_degrees(const SparseMatrix& a) {
  std::vector<double> d(static_cast<std::size_t>(a.cols()), 0.0);
  for (std::int64_t k = 0; k < a.nnz(); ++k)
    d[static_cast<std::size_t>(a.col_indices()[k])] += a.values()[k].real();
  return d;
}

std::vector<double> in_degrees(const SparseMatrix& a) {
  std::vector<double> d(static_cast<std::size_t>(a.rows()), 0.0);
  for (std::int64_t i = 0; i < a.rows(); ++i)
    for (std::int64_t k = a.row_begin(i); k < a.row_end(i); ++k)
      d[static_cast<std::size_t>(i)] += a.values()[k].real();
  return d;
}

SparseMatrix generator_matrix(double gamma, const SparseMatrix& a) {
  if (!(gamma > 0.0)) throw std::invalid_argument("transition rate gamma must be positive");
  const std::vector<double> cs = out_degrees(a);
  std::vector<Triplet> e;
  e.reserve(static_cast<std::size_t>(a.nnz() + a.rows()));
  for (std::int64_t i = 0; i < a.rows(); ++i) {
    for (std::int64_t k = a.row_begin(i); k < a.row_end(i); ++k)
      e.push_back({i, a.col_indices()[k], Complex{-gamma * a.values()[k].real(), 0.0}});
    if (cs[static_cast<std::size_t>(i)] != 0.0)
      e.push_back({i, i, Complex{gamma * cs[static_cast<std::size_t>(i)], 0.0}});
  }
  return SparseMatrix::from_triplets(a.rows(), a.cols(), std::move(e));
}

SparseMatrix markov_chain_matrix(const SparseMatrix& a) {
  validate_adjacency(a);
  const std::vector<double> deg = out_degrees(a);
  std::vector<Triplet> e;
  e.reserve(static_cast<std::size_t>(a.nnz()));
  for (std::int64_t i = 0; i < a.rows(); ++i)
    for (std::int64_t k = a.row_begin(i); k < a.row_end(i); ++k) {
      const std::int64_t c = a.col_indices()[k];
      e.push_back({i, c, Complex{1.0 / deg[static_cast<std::size_t>(c)], 0.0}});
    }
  return SparseMatrix::from_triplets(a.rows(), a.cols(), std::move(e));
}

SparseMatrix augment(const SparseMatrix& a, const std::vector<SourceArc>& sources,
                     const std::vector<SinkArc>& sinks) {
  validate_adjacency(a);
  const std::int64_t n = a.rows();
  std::set<std::int64_t> st, so;
  for (const SourceArc& s : sources) {
    if (s.target < 0 || s.target >= n)
      throw std::out_of_range("source target vertex " + std::to_string(s.target) + " out of range");
    if (!(s.rate > 0.0)) throw std::invalid_argument("source rate must be strictly positive");
    if (!st.insert(s.target).second)
      throw std::invalid_argument("duplicate source attachment at vertex " + std::to_string(s.target));
  }
  for (const SinkArc& s : sinks) {
    if (s.origin < 0 || s.origin >= n)
      throw std::out_of_range("sink origin vertex " + std::to_string(s.origin) + " out of range");
    if (!(s.rate > 0.0)) throw std::invalid_argument("sink rate must be strictly positive");
    if (!so.insert(s.origin).second)
      throw std::invalid_argument("duplicate sink attachment at vertex " + std::to_string(s.origin));
  }
  const std::int64_t ns = static_cast<std::int64_t>(sources.size());
  const std::int64_t total = n + ns + static_cast<std::int64_t>(sinks.size());
  std::vector<Triplet> e;
  for (std::int64_t i = 0; i < n; ++i)
    for (std::int64_t k = a.row_begin(i); k < a.row_end(i); ++k)
      e.push_back({i, a.col_indices()[k], a.values()[k]});
  for (std::int64_t k = 0; k < ns; ++k)
    e.push_back({sources[static_cast<std::size_t>(k)].target, n + k,
                 Complex{sources[static_cast<std::size_t>(k)].rate, 0.0}});
  for (std::size_t k = 0; k < sinks.size(); ++k)
    e.push_back({n + ns + static_cast<std::int64_t>(k), sinks[k].origin, Complex{sinks[k].rate, 0.0}});
  return SparseMatrix::from_triplets(total, total, std::move(e));
}

SparseMatrix local_lindblad(const SparseMatrix& m) {
  return m.map_values([](Complex v) { return Complex{std::sqrt(std::abs(v)), 0.0}; });
}

SparseMatrix global_lindblad(const SparseMatrix& adj) {
  validate_adjacency(adj);
  return adj;
}

}  // namespace qswg
