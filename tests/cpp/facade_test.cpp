// Compiled C++ consumer of libqswg.so through the RAII facade
// include/qswg/qsw_gpu.hpp — the reference's own language calling the GPU
// library the way a maintainer's glue would.
//
//   facade_test cpu            host-only checks (no GPU needed): sparse
//                              round trip, graph -> operator helpers, the
//                              reference's exception types from the C codes
//   facade_test series <dir>   reads <dir>/input.txt (a walk: kind, omega, H,
//                              operators, rho(0) probabilities, times), runs
//                              WalkSystem::lqsw / gqsw -> series through the
//                              facade, writes <dir>/output.txt (populations of
//                              every output, the final state, SpMV count)
#include <qswg/qsw_gpu.hpp>

#include <cmath>
#include <cstdio>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <vector>

namespace g = qswg::gpu;

namespace {

int fails = 0;
#define EXPECT(cond)                                                  \
  do {                                                                \
    if (!(cond)) {                                                    \
      std::fprintf(stderr, "FAILED %s:%d: %s\n", __FILE__, __LINE__, #cond); \
      ++fails;                                                        \
    }                                                                 \
  } while (0)

template <class E, class F>
bool throws(F&& f) {
  try {
    f();
  } catch (const E&) {
    return true;
  } catch (...) {
    return false;
  }
  return false;
}

int cpu_checks() {
  // sparse round trip: duplicates summed, zeros dropped (sparse.hpp:35-37)
  const auto m = g::SparseMatrix::from_triplets(3, 3, {0, 2, 0, 1}, {1, 0, 1, 1}, {{1, 0}, {2, 0}, {0.5, 0}, {0, 0}});
  EXPECT(m.rows() == 3 && m.cols() == 3 && m.nnz() == 2);
  std::vector<int64_t> rp, ci;
  std::vector<g::Complex> v;
  m.export_csr(rp, ci, v);
  EXPECT(rp.size() == 4 && ci[0] == 1 && v[0] == g::Complex(1.5, 0) && ci[1] == 0 && v[1] == g::Complex(2, 0));
  // cycle graph of 4 vertices -> generator (Laplacian) and Markov matrix
  std::vector<int64_t> r, c;
  std::vector<g::Complex> w;
  for (int64_t i = 0; i < 4; ++i) {
    r.push_back((i + 1) % 4), c.push_back(i), w.push_back(1.0);
    r.push_back(i), c.push_back((i + 1) % 4), w.push_back(1.0);
  }
  const auto adj = g::SparseMatrix::from_triplets(4, 4, r, c, w);
  const auto lap = g::generator_matrix(1.0, adj);
  lap.export_csr(rp, ci, v);
  EXPECT(lap.nnz() == 12 && v[0] == g::Complex(2, 0));  // row 0: 2 on the diagonal, -1 at 1 and 3
  const auto mk = g::markov_chain_matrix(adj);
  mk.export_csr(rp, ci, v);
  EXPECT(mk.nnz() == 8 && v[0] == g::Complex(0.5, 0));
  // the reference's exception types (sparse.cpp, liouvillian.cpp validation)
  EXPECT(throws<std::out_of_range>([] { g::SparseMatrix::from_triplets(2, 2, {0, 5}, {0, 1}, {1.0, 2.0}); }));
  EXPECT(throws<std::invalid_argument>([] { g::SparseMatrix::from_triplets(2, 2, {0}, {0, 1}, {1.0}); }));
  const auto h2 = g::SparseMatrix::from_triplets(2, 3, {0}, {1}, {1.0});
  EXPECT(throws<std::invalid_argument>([&] { g::Liouvillian::build_local(0.5, h2, h2); }));   // not square
  EXPECT(throws<std::invalid_argument>([&] { g::Liouvillian::build_local(1.5, lap, mk); }));  // omega > 1
  const auto nh = g::SparseMatrix::from_triplets(2, 2, {0}, {1}, {{0, 1}});
  EXPECT(throws<std::invalid_argument>([&] { g::Liouvillian::build_global(0.5, nh, {}); }));  // not Hermitian
  std::fprintf(stderr, "cpu checks: %d failure(s)\n", fails);
  return fails ? 1 : 0;
}

g::SparseMatrix read_matrix(std::istream& in) {
  std::string tag, name;
  int64_t rows = 0, cols = 0, nnz = 0;
  in >> tag >> name >> rows >> cols >> nnz;
  std::vector<int64_t> r(static_cast<std::size_t>(nnz)), c(static_cast<std::size_t>(nnz));
  std::vector<g::Complex> v(static_cast<std::size_t>(nnz));
  for (int64_t k = 0; k < nnz; ++k) {
    double re = 0, im = 0;
    in >> r[static_cast<std::size_t>(k)] >> c[static_cast<std::size_t>(k)] >> re >> im;
    v[static_cast<std::size_t>(k)] = {re, im};
  }
  return g::SparseMatrix::from_triplets(rows, cols, r, c, v);
}

int series_case(const std::string& dir) {
  std::ifstream in(dir + "/input.txt");
  if (!in) {
    std::fprintf(stderr, "cannot open %s/input.txt\n", dir.c_str());
    return 2;
  }
  std::string key, kind;
  double omega = 0;
  int n_ops = 0, has_rot = 0;
  in >> key >> kind >> key >> omega >> key >> n_ops >> key >> has_rot;
  g::SparseMatrix h = read_matrix(in);
  std::vector<g::SparseMatrix> ops;
  for (int k = 0; k < n_ops; ++k) ops.push_back(read_matrix(in));
  std::optional<g::SparseMatrix> rot;
  if (has_rot) rot.emplace(read_matrix(in));
  int64_t n = 0;
  in >> key >> n;
  std::vector<double> p(static_cast<std::size_t>(n));
  for (auto& x : p) in >> x;
  double t1 = 0, tq = 0;
  int64_t steps = 0;
  in >> key >> t1 >> tq >> steps;

  g::WalkSystem walk = kind == "local" ? g::WalkSystem::lqsw(omega, std::move(h), std::move(ops[0]))
                                       : g::WalkSystem::gqsw(omega, std::move(h), ops, rot);
  EXPECT(throws<std::logic_error>([&] { walk.series(t1, tq, steps); }));  // no initial state (walk.cpp:154)
  walk.initial_state(p);
  const g::SeriesResult r = walk.series(t1, tq, steps);
  const std::vector<double> last = walk.gather_populations();
  std::ofstream out(dir + "/output.txt");
  out.precision(17);
  out << "spmvs " << r.info.spmvs << "\n";
  for (const auto& row : r.populations) {
    for (double x : row) out << x << " ";
    out << "\n";
  }
  out << "final";
  for (double x : last) out << " " << x;
  out << "\n";
  // the same final time through qsw::step from rho(0) (walk.step)
  walk.step(tq);
  out << "step";
  for (double x : walk.gather_populations()) out << " " << x;
  out << "\n";
  std::fprintf(stderr, "series: %d failure(s)\n", fails);
  return fails ? 1 : 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  try {
    if (mode == "cpu") return cpu_checks();
    if (mode == "series" && argc > 2) return series_case(argv[2]);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "uncaught: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "usage: facade_test cpu | series <dir>\n");
  return 2;
}
