// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-callable entry points into the UNMODIFIED reference's file formats and
// run() (proj/core/src/graph.cpp:54-150, container.cpp, run.cpp:88-171),
// compiled with ref_harness.cpp into oracle/_ref/libqswref*.so.  Used by
// oracle/make_golden.py to write the output-path golden fixtures
// (tests/golden/io/) and by tests/test_io.py to cross-check libqswg's
// Matrix Market parser and QSWBOX writer/reader against the reference.

#include <cstdint>
#include <cstring>
#include <exception>
#include <fstream>
#include <sstream>
#include <string>
#include <vector>

#include "qsw/config.hpp"
#include "qsw/container.hpp"
#include "qsw/graph.hpp"
#include "qsw/run.hpp"
#include "qsw/sparse.hpp"

namespace {

void put_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(len - 1));
    err[len - 1] = 0;
  }
}

// Codes of include/qswg.h: EINVAL 1, ERANGE 2, EFORMAT 10, EIO 11; ConfigError 12.
int io_code(const std::exception& e) {
  if (dynamic_cast<const qsw::FileFormatError*>(&e)) return 10;
  if (dynamic_cast<const qsw::IoError*>(&e)) return 11;
  if (dynamic_cast<const qsw::ConfigError*>(&e)) return 12;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  return 9;
}

template <class F>
int guard(char* err, int errlen, F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    put_err(err, errlen, e.what());
    return io_code(e);
  }
}

}  // namespace

extern "C" {

// WeightedDigraph::load_matrix_market on a memory stream; *out = new
// qsw::SparseMatrix (the adjacency), freed with ref_sparse_free.
int ref_mtx_parse(const char* text, std::int64_t len, void** out, char* err, int errlen) {
  return guard(err, errlen, [&] {
    std::istringstream in(std::string(text, static_cast<std::size_t>(len)));
    const qsw::WeightedDigraph g = qsw::WeightedDigraph::load_matrix_market(in);
    *out = new qsw::SparseMatrix(g.adjacency());
  });
}

// save_matrix_market of the graph with adjacency *sparse into path.
int ref_mtx_save(void* sparse, const char* path, char* err, int errlen) {
  return guard(err, errlen, [&] {
    const auto g = qsw::WeightedDigraph::from_adjacency(*static_cast<qsw::SparseMatrix*>(sparse));
    std::ofstream out(path);
    g.save_matrix_market(out);
  });
}

// write_container of {meta, arrays}: names[k] (NUL-terminated), ranks[k],
// shapes (concatenated), data (concatenated row-major blocks).
int ref_container_write(const char* path, const char* meta, std::int64_t meta_len, std::int64_t n_arrays,
                        const char* const* names, const std::int64_t* ranks, const std::int64_t* shapes,
                        const double* data, char* err, int errlen) {
  return guard(err, errlen, [&] {
    qsw::ResultContainer c;
    c.metadata.assign(meta, static_cast<std::size_t>(meta_len));
    for (std::int64_t k = 0; k < n_arrays; ++k) {
      qsw::ArrayBlock b;
      for (std::int64_t d = 0; d < ranks[k]; ++d) b.shape.push_back(static_cast<std::size_t>(*shapes++));
      const std::size_t count = b.element_count();
      b.data.assign(data, data + count);
      data += count;
      c.arrays.emplace(names[k], std::move(b));
    }
    qsw::write_container(c, path);
  });
}

// read_container + re-write (round trip through the reference's reader).
int ref_container_rewrite(const char* in_path, const char* out_path, char* err, int errlen) {
  return guard(err, errlen, [&] { qsw::write_container(qsw::read_container(in_path), out_path); });
}

// emit_plot_data(read_container(in_path), quantity, out_path).
int ref_plot_data(const char* in_path, const char* quantity, const char* out_path, char* err, int errlen) {
  return guard(err, errlen, [&] {
    qsw::emit_plot_data(qsw::read_container(in_path), std::string(quantity), std::filesystem::path(out_path));
  });
}

// qsw::run on a directly built RunConfig; the container goes to out_path.
// kind 0 local, 1 global, 2 nm_global; initial 0 mixed, 1 vertex, 2 file;
// series != 0: t1, tq, steps, else a single time t.
int ref_run(const char* graph, int kind, double omega, double gamma, int series, double t, double t1, double tq,
            std::int64_t steps, int initial, std::int64_t vertex, const char* initial_file, std::int64_t n_src,
            const std::int64_t* src_target, const double* src_rate, std::int64_t n_snk,
            const std::int64_t* snk_origin, const double* snk_rate, std::int64_t workers, int out_pops,
            int out_rho, int out_coh, const char* out_path, char* err, int errlen) {
  return guard(err, errlen, [&] {
    qsw::RunConfig c;
    c.walk_kind = kind == 0 ? qsw::WalkKind::Local
                            : (kind == 1 ? qsw::WalkKind::Global : qsw::WalkKind::NonMoralisingGlobal);
    c.graph_path = graph;
    c.omega = omega;
    c.gamma = gamma;
    c.time.is_series = series != 0;
    c.time.t = t;
    c.time.t1 = t1;
    c.time.tq = tq;
    c.time.steps = static_cast<std::size_t>(steps);
    c.initial_kind = initial == 0 ? qsw::InitialStateKind::Mixed
                                  : (initial == 1 ? qsw::InitialStateKind::Vertex : qsw::InitialStateKind::File);
    c.initial_vertex = static_cast<std::size_t>(vertex);
    if (initial_file) c.initial_file = initial_file;
    for (std::int64_t k = 0; k < n_src; ++k) c.sources.push_back({static_cast<std::size_t>(src_target[k]), src_rate[k]});
    for (std::int64_t k = 0; k < n_snk; ++k) c.sinks.push_back({static_cast<std::size_t>(snk_origin[k]), snk_rate[k]});
    c.workers = static_cast<std::size_t>(workers);
    c.out_populations = out_pops != 0;
    c.out_full_rho = out_rho != 0;
    c.out_coherence_norm = out_coh != 0;
    qsw::write_container(qsw::run(c), out_path);
  });
}

}  // extern "C"
