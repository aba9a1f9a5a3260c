#include "nm.hpp"

#include <cmath>
#include <stdexcept>
#include <string>

#include "graph.hpp"

namespace qswg {

VertexSubspaces VertexSubspaces::from_dims(const std::vector<std::int64_t>& dims) {
  VertexSubspaces v;
  v.dims = dims;
  v.offsets.assign(dims.size() + 1, 0);
  for (std::size_t i = 0; i < dims.size(); ++i) {
    if (dims[i] < 1) throw std::invalid_argument("subspace dimensions must be >= 1");
    v.offsets[i + 1] = v.offsets[i] + dims[i];
  }
  return v;
}

VertexSubspaces nm_vsets(const SparseMatrix& gu) {
  validate_adjacency(gu);
  if (!(gu.transpose() == gu)) throw std::invalid_argument("nm_vsets requires a symmetric adjacency matrix");
  std::vector<std::int64_t> dims(static_cast<std::size_t>(gu.rows()));
  for (std::int64_t i = 0; i < gu.rows(); ++i)
    dims[static_cast<std::size_t>(i)] = std::max<std::int64_t>(gu.row_end(i) - gu.row_begin(i), 1);
  return VertexSubspaces::from_dims(dims);
}

namespace {

void same_size(const SparseMatrix& g, const VertexSubspaces& v) {
  if (v.vertex_count() != g.rows()) throw std::invalid_argument("vertex subspaces were built for a different graph size");
}

// e^{2 pi i k / n}; multiples of a quarter or a twelfth of a turn are exact,
// so Fourier-phase cancellations in small subspaces are exact too.
Complex unit_root(std::int64_t k, std::int64_t n) {
  const std::int64_t r = k % n;
  if ((12 * r) % n == 0) {
    const std::int64_t twelfth = 12 * r / n;  // 0..11, multiples of 30 degrees
    const double h = 0.5 * std::sqrt(3.0);
    switch (twelfth) {  // (cos, sin)
      case 0: return {1.0, 0.0};
      case 1: return {h, 0.5};
      case 2: return {0.5, h};
      case 3: return {0.0, 1.0};
      case 4: return {-0.5, h};
      case 5: return {-h, 0.5};
      case 6: return {-1.0, 0.0};
      case 7: return {-h, -0.5};
      case 8: return {-0.5, -h};
      case 9: return {0.0, -1.0};
      case 10: return {0.5, -h};
      default: return {h, -0.5};
    }
  }
  const double ang = 2.0 * M_PI * static_cast<double>(r) / static_cast<double>(n);
  return {std::cos(ang), std::sin(ang)};
}

}  // namespace

SparseMatrix demoralised_weights(const SparseMatrix& g, const VertexSubspaces& v) {
  same_size(g, v);
  std::vector<Triplet> e;
  for (std::int64_t i = 0; i < g.rows(); ++i) {
    for (std::int64_t k = g.row_begin(i); k < g.row_end(i); ++k) {
      const std::int64_t src = g.col_indices()[static_cast<std::size_t>(k)];
      const double deg = static_cast<double>(v.dims[static_cast<std::size_t>(i)] * v.dims[static_cast<std::size_t>(src)]);
      const double w = 1.0 / std::sqrt(deg * g.values()[static_cast<std::size_t>(k)].real());
      for (std::int64_t l = 0; l < v.dims[static_cast<std::size_t>(i)]; ++l)
        for (std::int64_t m = 0; m < v.dims[static_cast<std::size_t>(src)]; ++m)
          e.push_back({v.offsets[static_cast<std::size_t>(i)] + l, v.offsets[static_cast<std::size_t>(src)] + m, Complex{w, 0.0}});
    }
  }
  return SparseMatrix::from_triplets(v.total_dim(), v.total_dim(), std::move(e));
}

SparseMatrix nm_H(double gamma, const SparseMatrix& gu, const VertexSubspaces& v) {
  return generator_matrix(gamma, demoralised_weights(gu, v));
}

SparseMatrix nm_L(double gamma, const SparseMatrix& g, const VertexSubspaces& v) {
  if (!(gamma > 0.0)) throw std::invalid_argument("transition rate gamma must be positive");
  same_size(g, v);
  std::vector<Triplet> e;
  for (std::int64_t i = 0; i < g.rows(); ++i) {
    const std::int64_t d = v.dims[static_cast<std::size_t>(i)];
    std::int64_t arc = 0;  // index of the incoming arc (ascending source)
    for (std::int64_t k = g.row_begin(i); k < g.row_end(i); ++k, ++arc) {
      const std::int64_t src = g.col_indices()[static_cast<std::size_t>(k)];
      const double deg = static_cast<double>(d * v.dims[static_cast<std::size_t>(src)]);
      const double w = gamma / std::sqrt(deg * g.values()[static_cast<std::size_t>(k)].real());
      const std::int64_t fcol = (arc + 1) % d;  // Fourier column selected by this arc
      for (std::int64_t l = 0; l < d; ++l) {
        const Complex phase = unit_root(l * fcol, d);
        for (std::int64_t m = 0; m < v.dims[static_cast<std::size_t>(src)]; ++m)
          e.push_back({v.offsets[static_cast<std::size_t>(i)] + l, v.offsets[static_cast<std::size_t>(src)] + m, w * phase});
      }
    }
  }
  return SparseMatrix::from_triplets(v.total_dim(), v.total_dim(), std::move(e));
}

SparseMatrix nm_H_rot(const VertexSubspaces& v, Dim2Rotation dim2) {
  std::vector<Triplet> e;
  const Complex pi{0.0, 1.0};
  for (std::int64_t u = 0; u < v.vertex_count(); ++u) {
    const std::int64_t d = v.dims[static_cast<std::size_t>(u)], b = v.offsets[static_cast<std::size_t>(u)];
    if (d == 1) continue;
    if (d == 2) {  // (k+1) mod 2 == (k-1) mod 2: the two cases name the same entries
      if (dim2 == Dim2Rotation::PauliY) {
        e.push_back({b + 1, b, pi});
        e.push_back({b, b + 1, -pi});
      }
      continue;
    }
    for (std::int64_t k = 0; k < d; ++k) {
      e.push_back({b + (k + 1) % d, b + k, pi});
      e.push_back({b + (k + d - 1) % d, b + k, -pi});
    }
  }
  return SparseMatrix::from_triplets(v.total_dim(), v.total_dim(), std::move(e));
}

std::vector<double> nm_rho_map(const std::vector<double>& p, const VertexSubspaces& v) {
  if (static_cast<std::int64_t>(p.size()) != v.vertex_count())
    throw std::invalid_argument("probability vector length does not match the vertex count");
  double total = 0.0;
  for (double x : p) {
    if (x < 0.0) throw std::invalid_argument("probabilities must be non-negative");
    total += x;
  }
  if (std::abs(total - 1.0) > 1e-12)
    throw std::invalid_argument("probability vector is not normalized (sum = " + std::to_string(total) + ")");
  std::vector<double> out(static_cast<std::size_t>(v.total_dim()), 0.0);
  for (std::size_t i = 0; i < p.size(); ++i) {
    const double share = p[i] / static_cast<double>(v.dims[i]);
    for (std::int64_t l = 0; l < v.dims[i]; ++l) out[static_cast<std::size_t>(v.offsets[i] + l)] = share;
  }
  return out;
}

std::vector<double> nm_measure(const std::vector<double>& diag, const VertexSubspaces& v) {
  if (static_cast<std::int64_t>(diag.size()) != v.total_dim())
    throw std::invalid_argument("diagonal length does not match the expanded dimension");
  std::vector<double> p(static_cast<std::size_t>(v.vertex_count()), 0.0);
  for (std::size_t i = 0; i < p.size(); ++i)
    for (std::int64_t l = 0; l < v.dims[i]; ++l) p[i] += diag[static_cast<std::size_t>(v.offsets[i] + l)];
  return p;
}

}  // namespace qswg
