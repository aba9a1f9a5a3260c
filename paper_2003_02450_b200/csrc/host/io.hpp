// The data formats either side of the hot path:
// Matrix Market graph input and the "QSWBOX" result container.
//
// Mirrors WeightedDigraph::load_matrix_market / save_matrix_market
// (proj/core/src/graph.cpp:54-150, include/qsw/graph.hpp:11-15) and
// ResultContainer / write_container / read_container / emit_plot_data
// (proj/core/src/container.cpp:1-192, include/qsw/container.hpp:11-57),
// with the same byte layout, error classes and messages, so files written by
// either side are read by the other.
#pragma once

#include <cstdint>
#include <iosfwd>
#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "sparse.hpp"

namespace qswg {

/// A file that does not follow its declared format (graph.hpp:11-15).
class FileFormatError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

/// Filesystem-level failure: missing file, unwritable path (container.hpp:13-17).
class IoError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

/// Adjacency matrix of a `matrix coordinate real|integer general|symmetric`
/// stream: entry (i, j, w) is the arc j -> i.  Format problems throw
/// FileFormatError; a self-loop or a non-positive weight throws
/// std::invalid_argument (graph.cpp:54-136).
SparseMatrix load_matrix_market(std::istream& in);
/// The graph-file loader of run.cpp:14-25: IoError when the file cannot be
/// opened; every other failure becomes a FileFormatError naming the file.
SparseMatrix load_graph_file(const std::string& path);
/// `real general`, entries in column-major order, 17 significant digits
/// (graph.cpp:138-150).
void save_matrix_market(const SparseMatrix& adjacency, std::ostream& out);

/// One named float64 block, row-major with an explicit shape.
struct ArrayBlock {
  std::vector<std::uint64_t> shape;
  std::vector<double> data;
  std::uint64_t element_count() const;
};

/// "QSWBOX" v1: magic + u16 version, sections {u32 name length, name, u64
/// payload length, payload} ("meta" first, then the arrays by name), CRC-32
/// trailer over everything before it.  Array payload: u64 rank, u64 dims,
/// f64 data.  Little-endian.
struct ResultContainer {
  std::string metadata;
  std::map<std::string, ArrayBlock> arrays;

  std::string serialize() const;
  static ResultContainer parse(const std::string& bytes);
};

void write_container(const ResultContainer& c, const std::string& path);
ResultContainer read_container(const std::string& path);
/// One text row per time (the "times" array first when it has one entry per
/// row), the quantity's columns after it, 17 significant digits
/// (container.cpp:159-190).
std::string plot_data(const ResultContainer& c, const std::string& quantity);

std::uint32_t crc32(const void* data, std::size_t len);

}  // namespace qswg
