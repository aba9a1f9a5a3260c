// Matrix Market graphs and the QSWBOX result container (io.hpp).
#include "io.hpp"

#include <algorithm>
#include <array>
#include <bit>
#include <cctype>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <istream>
#include <ostream>
#include <sstream>

#include "graph.hpp"

namespace qswg {

static_assert(std::endian::native == std::endian::little, "QSWBOX is little-endian");

// ------------------------------------------------------------ Matrix Market
namespace {

bool is_blank(const std::string& s) {
  for (unsigned char c : s)
    if (!std::isspace(c)) return false;
  return true;
}

bool is_comment(const std::string& s) { return !s.empty() && s[0] == '%'; }

std::string lowercase(std::string s) {
  for (char& c : s) c = static_cast<char>(std::tolower(static_cast<unsigned char>(c)));
  return s;
}

std::string fmt17(double v) {
  char buf[64];
  std::snprintf(buf, sizeof buf, "%.17g", v);  // ostream precision(17), default floatfield
  return buf;
}

}  // namespace

SparseMatrix load_matrix_market(std::istream& in) {
  // graph.cpp:54-81: banner line
  std::string line;
  if (!std::getline(in, line)) throw FileFormatError("empty Matrix Market stream");
  std::string tok[5];
  {
    std::istringstream hs(line);
    for (auto& t : tok) hs >> t;
  }
  if (tok[0] != "%%MatrixMarket") throw FileFormatError("missing %%MatrixMarket banner");
  const std::string object = lowercase(tok[1]), format = lowercase(tok[2]), field = lowercase(tok[3]),
                    symmetry = lowercase(tok[4]);
  if (object != "matrix" || format != "coordinate")
    throw FileFormatError("only `matrix coordinate` Matrix Market data is supported");
  if (field != "real" && field != "integer")
    throw FileFormatError("adjacency input requires a real or integer field, got `" + field + "`");
  if (symmetry != "general" && symmetry != "symmetric")
    throw FileFormatError("unsupported symmetry `" + symmetry + "`");
  const bool mirror = symmetry == "symmetric";

  // graph.cpp:83-94: the size line is the first non-comment, non-blank line
  while (std::getline(in, line))
    if (!is_comment(line) && !is_blank(line)) break;
  long long n = -1, ncols = -1, declared = -1;
  {
    std::istringstream ss(line);
    if (!(ss >> n >> ncols >> declared) || n < 0 || ncols < 0 || declared < 0)
      throw FileFormatError("malformed Matrix Market size line: `" + line + "`");
  }
  if (n != ncols) throw FileFormatError("adjacency matrix must be square");

  // graph.cpp:96-127: exactly `declared` entries, 1-based, arcs j -> i
  std::vector<Triplet> arcs;
  arcs.reserve(static_cast<std::size_t>(declared) * (mirror ? 2 : 1));
  for (long long seen = 0; seen < declared;) {
    if (!std::getline(in, line)) throw FileFormatError("unexpected end of Matrix Market data");
    if (is_comment(line) || is_blank(line)) continue;
    std::istringstream es(line);
    long long i = 0, j = 0;
    double w = 0.0;
    if (!(es >> i >> j >> w)) throw FileFormatError("malformed Matrix Market entry: `" + line + "`");
    if (i < 1 || i > n || j < 1 || j > n)
      throw FileFormatError("Matrix Market index out of bounds: (" + std::to_string(i) + ", " + std::to_string(j) +
                            ")");
    if (i == j)
      throw std::invalid_argument("diagonal entry at vertex " + std::to_string(i) +
                                  " violates the simple-graph requirement");
    if (!(w > 0.0))
      throw std::invalid_argument("non-positive weight " + std::to_string(w) + " at (" + std::to_string(i) + ", " +
                                  std::to_string(j) + ")");
    arcs.push_back({i - 1, j - 1, Complex{w, 0.0}});
    if (mirror) arcs.push_back({j - 1, i - 1, Complex{w, 0.0}});
    ++seen;
  }

  // graph.cpp:129-135: a repeated coordinate is an error, not a sum
  std::vector<std::pair<std::int64_t, std::int64_t>> keys(arcs.size());
  for (std::size_t k = 0; k < arcs.size(); ++k) keys[k] = {arcs[k].row, arcs[k].col};
  std::sort(keys.begin(), keys.end());
  const auto dup = std::adjacent_find(keys.begin(), keys.end());
  if (dup != keys.end())
    throw FileFormatError("duplicate coordinate: duplicate sparse entry at (" + std::to_string(dup->first) + ", " +
                          std::to_string(dup->second) + ")");
  SparseMatrix adj = SparseMatrix::from_triplets(n, n, std::move(arcs));
  validate_adjacency(adj);
  return adj;
}

SparseMatrix load_graph_file(const std::string& path) {
  std::ifstream in(path);
  if (!in) throw IoError("cannot open graph file `" + path + "`");
  try {
    return load_matrix_market(in);
  } catch (const FileFormatError&) {
    throw;
  } catch (const std::exception& e) {
    throw FileFormatError("invalid graph file `" + path + "`: " + e.what());
  }
}

void save_matrix_market(const SparseMatrix& adjacency, std::ostream& out) {
  const SparseMatrix t = adjacency.transpose();  // row j of t = column j of the adjacency
  out << "%%MatrixMarket matrix coordinate real general\n";
  out << adjacency.rows() << " " << adjacency.cols() << " " << adjacency.nnz() << "\n";
  const auto& rp = t.row_starts();
  const auto& ci = t.col_indices();
  const auto& v = t.values();
  for (std::int64_t j = 0; j < t.rows(); ++j)
    for (std::int64_t k = rp[j]; k < rp[j + 1]; ++k) out << ci[k] + 1 << " " << j + 1 << " " << fmt17(v[k].real()) << "\n";
}

// ------------------------------------------------------------ QSWBOX
namespace {

constexpr char kMagic[6] = {'Q', 'S', 'W', 'B', 'O', 'X'};
constexpr std::uint16_t kVersion = 1;

constexpr std::array<std::uint32_t, 256> make_crc_table() {
  std::array<std::uint32_t, 256> t{};
  for (std::uint32_t b = 0; b < 256; ++b) {
    std::uint32_t r = b;
    for (int k = 0; k < 8; ++k) r = (r >> 1) ^ (0xEDB88320u & (0u - (r & 1u)));  // reflected IEEE 802.3
    t[b] = r;
  }
  return t;
}
constexpr auto kCrcTable = make_crc_table();

template <class T>
void emit(std::string& s, T v) {
  s.append(reinterpret_cast<const char*>(&v), sizeof v);
}

// Little-endian field reader over the whole file image (container.cpp:45-51
// bounds-checks against the image, trailer included).
struct Reader {
  const std::string& b;
  std::size_t pos;
  template <class T>
  T get() {
    if (pos + sizeof(T) > b.size()) throw FileFormatError("truncated container section");
    T v;
    std::memcpy(&v, b.data() + pos, sizeof v);
    pos += sizeof v;
    return v;
  }
};

}  // namespace

std::uint32_t crc32(const void* data, std::size_t len) {
  const auto* p = static_cast<const unsigned char*>(data);
  std::uint32_t c = 0xFFFFFFFFu;
  for (std::size_t k = 0; k < len; ++k) c = kCrcTable[(c ^ p[k]) & 0xFFu] ^ (c >> 8);
  return ~c;
}

std::uint64_t ArrayBlock::element_count() const {
  std::uint64_t n = 1;
  for (std::uint64_t d : shape) n *= d;
  return n;
}

std::string ResultContainer::serialize() const {
  std::string out(kMagic, sizeof kMagic);
  emit<std::uint16_t>(out, kVersion);
  const auto section = [&out](const std::string& name, std::uint64_t payload_len) {
    emit<std::uint32_t>(out, static_cast<std::uint32_t>(name.size()));
    out += name;
    emit<std::uint64_t>(out, payload_len);
  };
  section("meta", metadata.size());
  out += metadata;
  for (const auto& [name, a] : arrays) {
    if (a.data.size() != a.element_count())
      throw std::invalid_argument("array block `" + name + "` shape/data mismatch");
    section(name, 8 * (1 + a.shape.size()) + 8 * a.data.size());
    emit<std::uint64_t>(out, a.shape.size());
    for (std::uint64_t d : a.shape) emit<std::uint64_t>(out, d);
    out.append(reinterpret_cast<const char*>(a.data.data()), a.data.size() * sizeof(double));
  }
  emit<std::uint32_t>(out, crc32(out.data(), out.size()));
  return out;
}

ResultContainer ResultContainer::parse(const std::string& bytes) {
  if (bytes.size() < sizeof kMagic + sizeof(std::uint16_t) + sizeof(std::uint32_t))
    throw FileFormatError("container file too short");
  if (std::memcmp(bytes.data(), kMagic, sizeof kMagic) != 0)
    throw FileFormatError("not a qsw container (bad magic bytes)");
  Reader r{bytes, sizeof kMagic};
  const auto version = r.get<std::uint16_t>();
  if (version != kVersion) throw FileFormatError("unsupported container version " + std::to_string(version));
  const std::size_t body = bytes.size() - sizeof(std::uint32_t);
  std::uint32_t stored;
  std::memcpy(&stored, bytes.data() + body, sizeof stored);
  if (crc32(bytes.data(), body) != stored)
    throw FileFormatError("container checksum mismatch (truncated or corrupted file)");

  ResultContainer c;
  while (r.pos < body) {
    const auto name_len = r.get<std::uint32_t>();
    if (r.pos + name_len > body) throw FileFormatError("truncated container section name");
    std::string name = bytes.substr(r.pos, name_len);
    r.pos += name_len;
    const auto len = r.get<std::uint64_t>();
    if (r.pos + len > body) throw FileFormatError("truncated container payload");
    const std::size_t end = r.pos + len;
    if (name == "meta") {
      c.metadata = bytes.substr(r.pos, len);
      r.pos = end;
      continue;
    }
    ArrayBlock a;
    a.shape.resize(r.get<std::uint64_t>());
    for (auto& d : a.shape) d = r.get<std::uint64_t>();
    const std::uint64_t count = a.element_count();
    if (r.pos + count * sizeof(double) != end)
      throw FileFormatError("array section `" + name + "` has inconsistent dimensions");
    a.data.resize(count);
    std::memcpy(a.data.data(), bytes.data() + r.pos, count * sizeof(double));
    r.pos = end;
    c.arrays.emplace(std::move(name), std::move(a));  // first of a repeated name wins
  }
  return c;
}

void write_container(const ResultContainer& c, const std::string& path) {
  const std::string bytes = c.serialize();
  std::ofstream out(path, std::ios::binary);
  if (!out) throw IoError("cannot open `" + path + "` for writing");
  out.write(bytes.data(), static_cast<std::streamsize>(bytes.size()));
  if (!out) throw IoError("failed to write container stream");
}

ResultContainer read_container(const std::string& path) {
  std::ifstream in(path, std::ios::binary);
  if (!in) throw IoError("cannot open `" + path + "`");
  std::ostringstream buf;
  buf << in.rdbuf();
  return ResultContainer::parse(buf.str());
}

std::string plot_data(const ResultContainer& c, const std::string& quantity) {
  if (quantity.empty()) throw std::invalid_argument("no quantity requested");
  const auto it = c.arrays.find(quantity);
  if (it == c.arrays.end())
    throw std::invalid_argument("quantity `" + quantity + "` is not present in the container");
  const ArrayBlock& a = it->second;
  const std::uint64_t rows = a.shape.empty() ? 1 : a.shape.front();
  const std::uint64_t cols = a.element_count() / std::max<std::uint64_t>(rows, 1);
  const ArrayBlock* times = nullptr;
  if (const auto t = c.arrays.find("times"); t != c.arrays.end() && t->second.element_count() == rows)
    times = &t->second;
  std::string out;
  for (std::uint64_t r = 0; r < rows; ++r) {
    if (times) out += fmt17(times->data[r]) + " ";
    for (std::uint64_t k = 0; k < cols; ++k) {
      out += fmt17(a.data[r * cols + k]);
      if (k + 1 < cols) out += ' ';
    }
    out += '\n';
  }
  return out;
}

}  // namespace qswg
