// extern "C" boundary (include/qswg.h).  Exceptions are mapped to codes
// exactly as the reference's exception classes:
//   std::invalid_argument -> QSWG_EINVAL, std::out_of_range -> QSWG_ERANGE,
//   NumericalError -> QSWG_ENUMERICAL, std::logic_error -> QSWG_ESTATE,
//   CUDA failures -> QSWG_ECUDA, allocation -> QSWG_ENOMEM.
#include "../../include/qswg.h"

#include <algorithm>
#include <cstring>
#include <fstream>
#include <iterator>
#include <memory>
#include <new>
#include <sstream>
#include <string>
#include <vector>

#include "host/comm.hpp"
#include "host/device.hpp"
#include "host/dist.hpp"
#include "host/expm.hpp"
#include "host/graph.hpp"
#include "host/io.hpp"
#include "host/liouvillian.hpp"
#include "host/nm.hpp"
#include "host/sparse.hpp"
#include "host/taylor.hpp"

struct qswg_sparse {
  qswg::SparseMatrix m;
};
struct qswg_liouvillian {
  std::unique_ptr<qswg::Liouvillian> l;
  qswg::DeviceBuffer<double> pops;  // (steps + 1) * n populations of the last series
  qswg::DeviceBuffer<unsigned long long> coh;  // steps + 1 coherence norms (bit patterns)
};
struct qswg_container {
  qswg::ResultContainer c;
};
struct qswg_state {
  const qswg_liouvillian* owner;
  qswg::DeviceBuffer<double2> v;  // local rows
  // exact Hermiticity of the matrix held (1 / 0), -1 unknown: checked once at
  // upload, known for states built from probabilities and for outputs of the
  // Hermitian kernels, so step/series need no check (and no synchronisation)
  int herm = -1;
};

namespace qswg {
Comm* comm_from_handle(qswg_comm* c);                       // comm_nccl.cpp
int comm_create(const uint8_t* id, int rank, int world, int device, qswg_comm** out);
void comm_destroy(qswg_comm* c);
int comm_unique_id_size();
int comm_get_unique_id(uint8_t* id);
}  // namespace qswg

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

template <class F>
int guarded(F&& f) {
  try {
    g_err.clear();
    f();
    return QSWG_OK;
  } catch (const qswg::NumericalError& e) {
    return fail(QSWG_ENUMERICAL, e.what());
  } catch (const qswg::FileFormatError& e) {
    return fail(QSWG_EFORMAT, e.what());
  } catch (const qswg::IoError& e) {
    return fail(QSWG_EIO, e.what());
  } catch (const std::out_of_range& e) {
    return fail(QSWG_ERANGE, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(QSWG_EINVAL, e.what());
  } catch (const std::logic_error& e) {
    return fail(QSWG_ESTATE, e.what());
  } catch (const qswg::CudaError& e) {
    return fail(QSWG_ECUDA, e.what());
  } catch (const std::bad_alloc&) {
    return fail(QSWG_ENOMEM, "out of memory");
  } catch (const std::exception& e) {
    return fail(QSWG_EINTERNAL, e.what());
  } catch (...) {
    return fail(QSWG_EINTERNAL, "unknown error");
  }
}

void need(const void* p, const char* what) {
  if (!p) throw std::invalid_argument(std::string(what) + " must not be NULL");
}

qswg::DeviceConfig device_config(const qswg_device_config* cfg) {
  qswg::DeviceConfig c;
  if (cfg) {
    c.device = cfg->device;
    c.group = cfg->group;
    if (cfg->format < 0 || cfg->format > 3) throw std::invalid_argument("unknown storage format");
    c.format = cfg->format;
    c.comm = cfg->comm ? qswg::comm_from_handle(cfg->comm) : nullptr;
  } else {
    int dev = 0;
    cudaGetDevice(&dev);
    c.device = dev;
  }
  // (the device itself is checked by the build, after the reference's argument validation)
  return c;
}

qswg_sparse* wrap(qswg::SparseMatrix m) { return new qswg_sparse{std::move(m)}; }

void check_state(const qswg_liouvillian* l, const qswg_state* s, const char* what) {
  need(s, what);
  if (s->owner != l) throw std::invalid_argument("state vector partition does not match the Liouvillian");
}

}  // namespace

extern "C" {

const char* qswg_last_error(void) { return g_err.c_str(); }

int qswg_version(int* major, int* minor) {
  return guarded([&] {
    need(major, "major");
    need(minor, "minor");
    *major = QSWG_VERSION_MAJOR;
    *minor = QSWG_VERSION_MINOR;
  });
}

int qswg_host_alloc(int64_t bytes, void** out) {
  return guarded([&] {
    need(out, "out");
    if (bytes < 0) throw std::invalid_argument("bytes must be non-negative");
    *out = nullptr;
    if (bytes > 0) QSWG_CHECK(cudaHostAlloc(out, static_cast<std::size_t>(bytes), cudaHostAllocPortable));
  });
}

void qswg_host_free(void* p) {
  if (p) cudaFreeHost(p);
}

int qswg_device_count(int* count) {
  return guarded([&] {
    need(count, "count");
    int c = 0;
    if (cudaGetDeviceCount(&c) != cudaSuccess) {
      cudaGetLastError();
      c = 0;
    }
    *count = c;
  });
}

// ---------------------------------------------------------------- sparse
int qswg_sparse_from_triplets(int64_t rows, int64_t cols, int64_t count, const int64_t* row,
                              const int64_t* col, const double* val, qswg_sparse** out) {
  return guarded([&] {
    need(out, "out");
    if (count < 0) throw std::invalid_argument("negative triplet count");
    std::vector<qswg::Triplet> t(static_cast<std::size_t>(count));
    for (int64_t k = 0; k < count; ++k)
      t[static_cast<std::size_t>(k)] = {row[k], col[k], qswg::Complex{val[2 * k], val[2 * k + 1]}};
    *out = wrap(qswg::SparseMatrix::from_triplets(rows, cols, std::move(t)));
  });
}

int qswg_sparse_from_csr(int64_t rows, int64_t cols, const int64_t* rowptr, const int64_t* col,
                         const double* val, qswg_sparse** out) {
  return guarded([&] {
    need(out, "out");
    need(rowptr, "rowptr");
    *out = wrap(qswg::SparseMatrix::from_csr(rows, cols, rowptr, col, val));
  });
}

int qswg_sparse_shape(const qswg_sparse* m, int64_t* rows, int64_t* cols, int64_t* nnz) {
  return guarded([&] {
    need(m, "matrix");
    if (rows) *rows = m->m.rows();
    if (cols) *cols = m->m.cols();
    if (nnz) *nnz = m->m.nnz();
  });
}

int qswg_sparse_export(const qswg_sparse* m, int64_t* rowptr, int64_t* col, double* val) {
  return guarded([&] {
    need(m, "matrix");
    const auto& rs = m->m.row_starts();
    if (rowptr) std::memcpy(rowptr, rs.data(), rs.size() * sizeof(int64_t));
    if (col) std::memcpy(col, m->m.col_indices().data(), m->m.col_indices().size() * sizeof(int64_t));
    if (val) std::memcpy(val, m->m.values().data(), m->m.values().size() * sizeof(qswg::Complex));
  });
}

void qswg_sparse_destroy(qswg_sparse* m) { delete m; }

// ---------------------------------------------------------------- graph
int qswg_symmetrize(const qswg_sparse* a, qswg_sparse** out) {
  return guarded([&] {
    need(a, "adjacency");
    need(out, "out");
    *out = wrap(qswg::symmetrize(a->m));
  });
}

int qswg_generator_matrix(double gamma, const qswg_sparse* a, qswg_sparse** out) {
  return guarded([&] {
    need(a, "adjacency");
    need(out, "out");
    *out = wrap(qswg::generator_matrix(gamma, a->m));
  });
}

int qswg_markov_chain_matrix(const qswg_sparse* a, qswg_sparse** out) {
  return guarded([&] {
    need(a, "adjacency");
    need(out, "out");
    *out = wrap(qswg::markov_chain_matrix(a->m));
  });
}

int qswg_local_lindblad(const qswg_sparse* m, qswg_sparse** out) {
  return guarded([&] {
    need(m, "matrix");
    need(out, "out");
    *out = wrap(qswg::local_lindblad(m->m));
  });
}

int qswg_augment(const qswg_sparse* a, const qswg_source_arc* sources, int64_t n_sources,
                 const qswg_sink_arc* sinks, int64_t n_sinks, qswg_sparse** out) {
  return guarded([&] {
    need(a, "adjacency");
    need(out, "out");
    std::vector<qswg::SourceArc> src;
    std::vector<qswg::SinkArc> snk;
    for (int64_t k = 0; k < n_sources; ++k) src.push_back({sources[k].target, sources[k].rate});
    for (int64_t k = 0; k < n_sinks; ++k) snk.push_back({sinks[k].origin, sinks[k].rate});
    *out = wrap(qswg::augment(a->m, src, snk));
  });
}

// ------------------------------------------------------- demoralisation
namespace {
qswg::VertexSubspaces vsets_of(const int64_t* dims, int64_t nv) {
  need(dims, "dims");
  if (nv < 0) throw std::invalid_argument("negative vertex count");
  return qswg::VertexSubspaces::from_dims(std::vector<std::int64_t>(dims, dims + nv));
}
}  // namespace

int qswg_nm_vsets(const qswg_sparse* gu, int64_t* dims) {
  return guarded([&] {
    need(gu, "gu");
    need(dims, "dims");
    const auto v = qswg::nm_vsets(gu->m);
    std::memcpy(dims, v.dims.data(), v.dims.size() * sizeof(int64_t));
  });
}

int qswg_nm_H(double gamma, const qswg_sparse* gu, const int64_t* dims, int64_t nv, qswg_sparse** out) {
  return guarded([&] {
    need(gu, "gu");
    need(out, "out");
    *out = wrap(qswg::nm_H(gamma, gu->m, vsets_of(dims, nv)));
  });
}

int qswg_nm_L(double gamma, const qswg_sparse* g, const int64_t* dims, int64_t nv, qswg_sparse** out) {
  return guarded([&] {
    need(g, "g");
    need(out, "out");
    *out = wrap(qswg::nm_L(gamma, g->m, vsets_of(dims, nv)));
  });
}

int qswg_nm_H_rot(const int64_t* dims, int64_t nv, int pauli_y, qswg_sparse** out) {
  return guarded([&] {
    need(out, "out");
    *out = wrap(qswg::nm_H_rot(vsets_of(dims, nv), pauli_y ? qswg::Dim2Rotation::PauliY : qswg::Dim2Rotation::Cancel));
  });
}

int qswg_nm_rho_map(const double* p, const int64_t* dims, int64_t nv, double* expanded) {
  return guarded([&] {
    need(p, "p");
    need(expanded, "expanded");
    const auto v = vsets_of(dims, nv);
    const auto e = qswg::nm_rho_map(std::vector<double>(p, p + nv), v);
    std::memcpy(expanded, e.data(), e.size() * sizeof(double));
  });
}

int qswg_nm_measure(const double* diag, const int64_t* dims, int64_t nv, double* p) {
  return guarded([&] {
    need(diag, "diag");
    need(p, "p");
    const auto v = vsets_of(dims, nv);
    const auto out = qswg::nm_measure(std::vector<double>(diag, diag + v.total_dim()), v);
    std::memcpy(p, out.data(), out.size() * sizeof(double));
  });
}

// ---------------------------------------------------------- liouvillian
int qswg_build_local(double omega, const qswg_sparse* h, const qswg_sparse* m_l,
                     const qswg_source_arc* sources, int64_t n_sources, const qswg_sink_arc* sinks,
                     int64_t n_sinks, const qswg_device_config* cfg, qswg_liouvillian** out) {
  return guarded([&] {
    need(h, "h");
    need(m_l, "m_l");
    need(out, "out");
    if (n_sources < 0 || n_sinks < 0) throw std::invalid_argument("negative source/sink count");
    std::vector<qswg::SourceArc> src;
    std::vector<qswg::SinkArc> snk;
    for (int64_t k = 0; k < n_sources; ++k) src.push_back({sources[k].target, sources[k].rate});
    for (int64_t k = 0; k < n_sinks; ++k) snk.push_back({sinks[k].origin, sinks[k].rate});
    const qswg::DeviceConfig c = device_config(cfg);
    auto l = std::make_unique<qswg_liouvillian>();
    l->l = qswg::build_local(omega, h->m, m_l->m, src, snk, c);
    *out = l.release();
  });
}

int qswg_build_global(double omega, const qswg_sparse* h, const qswg_sparse* const* lindblads,
                      int64_t n_lindblads, const qswg_sparse* h_rot, const qswg_device_config* cfg,
                      qswg_liouvillian** out) {
  return guarded([&] {
    need(h, "h");
    need(out, "out");
    if (n_lindblads < 0) throw std::invalid_argument("negative Lindblad count");
    std::vector<qswg::SparseMatrix> ls;
    for (int64_t k = 0; k < n_lindblads; ++k) {
      need(lindblads[k], "lindblad operator");
      ls.push_back(lindblads[k]->m);
    }
    std::optional<qswg::SparseMatrix> hr;
    if (h_rot) hr = h_rot->m;
    const qswg::DeviceConfig c = device_config(cfg);
    auto l = std::make_unique<qswg_liouvillian>();
    l->l = qswg::build_global(omega, h->m, ls, hr, c);
    *out = l.release();
  });
}

int qswg_liouvillian_query(const qswg_liouvillian* l, qswg_liouvillian_info* info) {
  return guarded([&] {
    need(l, "liouvillian");
    need(info, "info");
    const qswg::Liouvillian& L = *l->l;
    info->n = L.n();
    info->dim = L.dim();
    info->nnz = L.nnz_total();
    info->nnz_local = L.nnz_local();
    info->row0 = L.block().row0;
    info->rows = L.block().rows;
    info->omega = L.omega();
    for (int p = 0; p < 9; ++p) info->one_norms[p] = L.one_norms()[static_cast<std::size_t>(p)];
    info->group = L.group();
    info->device = L.device();
    info->rank = L.comm() ? L.comm()->rank() : 0;
    info->world = L.comm() ? L.comm()->world() : 1;
    info->format = L.format() == qswg::dev::Format::Sell   ? QSWG_FORMAT_SELL
                   : L.format() == qswg::dev::Format::Kron ? QSWG_FORMAT_KRON
                                                           : QSWG_FORMAT_CSR;
    info->padding = L.padding();
    info->kron_factored = L.kron_factored() ? 1 : 0;
    info->kron_ell = L.kron_ell() ? 1 : 0;
    info->kron_staged = L.kron_staged() ? 1 : 0;
    info->sell_fused = L.sell_fused() ? 1 : 0;
    info->kron_term_vectors = L.kron_term_vectors();
    info->sell_panels = L.format() == qswg::dev::Format::Sell ? L.sell_panels() : 0;
    info->kron_hermitian = L.matrix().kron.herm;
  });
}

int qswg_liouvillian_download(const qswg_liouvillian* l, int64_t* rowptr, int64_t* col, double* val) {
  return guarded([&] {
    need(l, "liouvillian");
    std::vector<int64_t> rp, c;
    std::vector<qswg::Complex> v;
    l->l->download(rp, c, v);
    if (rowptr) std::memcpy(rowptr, rp.data(), rp.size() * sizeof(int64_t));
    if (col) std::memcpy(col, c.data(), c.size() * sizeof(int64_t));
    if (val) std::memcpy(val, v.data(), v.size() * sizeof(qswg::Complex));
  });
}

void qswg_liouvillian_destroy(qswg_liouvillian* l) {
  if (!l) return;
  try {
    qswg::DeviceGuard g(l->l ? l->l->device() : 0);
    l->pops.reset();
    delete l;
  } catch (...) {
  }
}

int qswg_spmv(const qswg_liouvillian* l, const double* x, double* y) {
  return guarded([&] {
    need(l, "liouvillian");
    need(x, "x");
    need(y, "y");
    const qswg::Liouvillian& L = *l->l;
    if (L.comm() && L.comm()->world() > 1) throw std::logic_error("qswg_spmv is single-GPU");
    qswg::DeviceGuard g(L.device());
    qswg::DeviceBuffer<double2> dx(static_cast<std::size_t>(L.dim())), dy(static_cast<std::size_t>(L.block().rows));
    QSWG_CHECK(cudaMemcpyAsync(dx.get(), x, dx.bytes(), cudaMemcpyHostToDevice, L.stream()));
    L.multiply(dx.get(), dy.get(), 1.0);
    QSWG_CHECK(cudaMemcpyAsync(y, dy.get(), dy.bytes(), cudaMemcpyDeviceToHost, L.stream()));
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
  });
}

int qswg_time_spmv(const qswg_liouvillian* l, int iters, int group, double* ms) {
  return guarded([&] {
    need(l, "liouvillian");
    need(ms, "ms");
    if (iters < 1) throw std::invalid_argument("iters must be >= 1");
    const int g = group ? group : l->l->group();
    if (!qswg::dev::valid_group(g)) throw std::invalid_argument("group must be 1, 2, 4, 8, 16 or 32");
    *ms = l->l->time_spmv(iters, g);
  });
}

int qswg_time_series_term(const qswg_liouvillian* l, int iters, int count, double* ms) {
  return guarded([&] {
    need(l, "liouvillian");
    need(ms, "ms");
    *ms = qswg::time_series_term(*l->l, iters, count);
  });
}

int qswg_liouvillian_set_hermitian_mode(qswg_liouvillian* l, int mode) {
  return guarded([&] {
    need(l, "liouvillian");
    l->l->set_hermitian_mode(mode);
  });
}

int qswg_time_series_parts(const qswg_liouvillian* l, int iters, int count, double* ms4) {
  return guarded([&] {
    need(l, "liouvillian");
    need(ms4, "ms4");
    const auto t = qswg::time_series_parts(*l->l, iters, count);
    for (int k = 0; k < 4; ++k) ms4[k] = t[static_cast<std::size_t>(k)];
  });
}

int qswg_liouvillian_stream(const qswg_liouvillian* l, void** stream) {
  return guarded([&] {
    need(l, "liouvillian");
    need(stream, "stream");
    *stream = static_cast<void*>(l->l->stream());
  });
}

// ---------------------------------------------------------------- states
int qswg_state_create(const qswg_liouvillian* l, qswg_state** out) {
  return guarded([&] {
    need(l, "liouvillian");
    need(out, "out");
    qswg::DeviceGuard g(l->l->device());
    auto s = std::make_unique<qswg_state>();
    s->owner = l;
    s->v.resize(static_cast<std::size_t>(std::max<int64_t>(l->l->block().rows, 1)));
    QSWG_CHECK(cudaMemsetAsync(s->v.get(), 0, s->v.bytes(), l->l->stream()));
    QSWG_CHECK(cudaStreamSynchronize(l->l->stream()));
    *out = s.release();
  });
}

int qswg_state_upload(qswg_state* s, const double* vec) {
  return guarded([&] {
    need(s, "state");
    need(vec, "vec");
    const qswg::Liouvillian& L = *s->owner->l;
    qswg::DeviceGuard g(L.device());
    QSWG_CHECK(cudaMemcpyAsync(s->v.get(), vec + 2 * L.block().row0,
                               static_cast<std::size_t>(L.block().rows) * sizeof(double2),
                               cudaMemcpyHostToDevice, L.stream()));
    s->herm = L.hermitian_state(s->v.get());  // (synchronises; -1 where no kernel uses it)
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
  });
}

int qswg_state_from_probabilities(qswg_state* s, const double* p, int64_t n) {
  return guarded([&] {
    need(s, "state");
    need(p, "probabilities");
    const qswg::Liouvillian& L = *s->owner->l;
    // walk.cpp:120-125
    if (n != L.n()) throw std::invalid_argument("probability vector length " + std::to_string(n) +
                                                " does not match the walk dimension");
    double total = 0.0;
    for (int64_t i = 0; i < n; ++i) {
      if (p[i] < 0.0) throw std::invalid_argument("probabilities must be non-negative");
      total += p[i];
    }
    if (std::abs(total - 1.0) > 1e-12) throw std::invalid_argument("probability vector is not normalized");
    qswg::DeviceGuard g(L.device());
    qswg::DeviceBuffer<double> dp(static_cast<std::size_t>(n));
    QSWG_CHECK(cudaMemcpyAsync(dp.get(), p, dp.bytes(), cudaMemcpyHostToDevice, L.stream()));
    qswg::dev::state_from_probabilities(s->v.get(), L.block().row0, L.block().rows, L.n(), dp.get(), L.stream());
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
    s->herm = 1;  // a real diagonal matrix
  });
}

int qswg_state_download(const qswg_state* s, double* vec) {
  return guarded([&] {
    need(s, "state");
    need(vec, "vec");
    const qswg::Liouvillian& L = *s->owner->l;
    qswg::DeviceGuard g(L.device());
    QSWG_CHECK(cudaMemcpyAsync(vec, s->v.get(), static_cast<std::size_t>(L.block().rows) * sizeof(double2),
                               cudaMemcpyDeviceToHost, L.stream()));
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
  });
}

int qswg_state_populations(const qswg_state* s, double* out) {
  return guarded([&] {
    need(s, "state");
    need(out, "out");
    const qswg::Liouvillian& L = *s->owner->l;
    qswg::DeviceGuard g(L.device());
    qswg::DeviceBuffer<double> d(static_cast<std::size_t>(L.n()));
    QSWG_CHECK(cudaMemsetAsync(d.get(), 0, d.bytes(), L.stream()));
    qswg::dev::diag_real(s->v.get(), L.block().row0, L.block().rows, L.n(), d.get(), L.stream());
    if (L.comm() && L.comm()->world() > 1) L.comm()->allreduce_sum_f64(d.get(), static_cast<std::size_t>(L.n()), L.stream());
    QSWG_CHECK(cudaMemcpyAsync(out, d.get(), d.bytes(), cudaMemcpyDeviceToHost, L.stream()));
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
  });
}

int qswg_liouvillian_set_omega(qswg_liouvillian* l, double omega) {
  return guarded([&] {
    need(l, "liouvillian");
    l->l->set_omega(omega);
  });
}

int qswg_state_coherence(const qswg_state* s, double* out) {
  return guarded([&] {
    need(s, "state");
    need(out, "out");
    const qswg::Liouvillian& L = *s->owner->l;
    qswg::DeviceGuard g(L.device());
    qswg::DeviceBuffer<unsigned long long> d(1);
    QSWG_CHECK(cudaMemsetAsync(d.get(), 0, d.bytes(), L.stream()));
    qswg::dev::coherence_bits(s->v.get(), L.block().row0, L.block().rows, L.n(), d.get(), L.stream());
    if (L.comm() && L.comm()->world() > 1) L.comm()->allreduce_max_u64(d.get(), 1, L.stream());
    QSWG_CHECK(cudaMemcpyAsync(out, d.get(), d.bytes(), cudaMemcpyDeviceToHost, L.stream()));
    QSWG_CHECK(cudaStreamSynchronize(L.stream()));
  });
}

void qswg_state_destroy(qswg_state* s) {
  if (!s) return;
  try {
    qswg::DeviceGuard g(s->owner->l->device());
    delete s;
  } catch (...) {
  }
}

// ---------------------------------------------------------------- Taylor
int qswg_theta_table(double tolerance, double* theta55) {
  return guarded([&] {
    need(theta55, "theta");
    const auto& t = qswg::build_theta_table(tolerance);
    std::memcpy(theta55, t.theta.data(), sizeof(double) * 55);
  });
}

int qswg_select_parameters(const double* norms9, double t, double tolerance, int64_t* m_star, int64_t* s) {
  return guarded([&] {
    need(norms9, "one_norms");
    need(m_star, "m_star");
    need(s, "s");
    const auto sp = qswg::select_parameters(norms9, t, qswg::build_theta_table(tolerance));
    *m_star = sp.m_star;
    *s = sp.s;
  });
}

// ------------------------------------------------------------- evolution
int qswg_step(const qswg_liouvillian* l, const qswg_state* v, double t, double tolerance, qswg_state* out,
              qswg_step_info* info) {
  return guarded([&] {
    need(l, "liouvillian");
    check_state(l, v, "v");
    check_state(l, out, "out");
    if (out == v) throw std::invalid_argument("step output must not alias its input");
    const auto& params = qswg::build_theta_table(tolerance);
    const qswg::StepInfo si = qswg::step(*l->l, v->v.get(), t, params, out->v.get(), v->herm);
    const_cast<qswg_state*>(out)->herm = l->l->hermitian_mode() ? 1 : -1;  // mirrored tiles: exactly Hermitian
    if (info) *info = {si.m_star, si.s, si.spmvs, si.launches};
  });
}

int qswg_series(const qswg_liouvillian* l, const qswg_state* v, double t1, double tq, int64_t steps,
                double tolerance, double* pops_host, double* states_host, qswg_state* final_state,
                qswg_series_info* info) {
  return qswg_series_observe(l, v, t1, tq, steps, tolerance, pops_host, nullptr, states_host, final_state, info);
}

int qswg_series_observe(const qswg_liouvillian* l, const qswg_state* v, double t1, double tq, int64_t steps,
                        double tolerance, double* pops_host, double* coherence_host, double* states_host,
                        qswg_state* final_state, qswg_series_info* info) {
  return guarded([&] {
    need(l, "liouvillian");
    check_state(l, v, "v");
    if (final_state) check_state(l, final_state, "final_state");
    const auto& params = qswg::build_theta_table(tolerance);
    qswg_liouvillian* lm = const_cast<qswg_liouvillian*>(l);
    const qswg::Liouvillian& L = *l->l;
    qswg::DeviceGuard g(L.device());
    cudaStream_t s = L.stream();
    const int64_t n = L.n(), rows = L.block().rows;
    if (steps >= 1) {
      lm->pops.resize(static_cast<std::size_t>((steps + 1) * n));
      QSWG_CHECK(cudaMemsetAsync(lm->pops.get(), 0, lm->pops.bytes(), s));
      if (coherence_host) {
        lm->coh.resize(static_cast<std::size_t>(steps + 1));
        QSWG_CHECK(cudaMemsetAsync(lm->coh.get(), 0, lm->coh.bytes(), s));
      }
    }
    cudaEvent_t e0, e1;
    QSWG_CHECK(cudaEventCreate(&e0));
    QSWG_CHECK(cudaEventCreate(&e1));
    QSWG_CHECK(cudaEventRecord(e0, s));
    auto emit = [&](int64_t k, const double2* state) {
      qswg::dev::diag_real(state, L.block().row0, rows, n, lm->pops.get() + k * n, s);
      if (coherence_host) qswg::dev::coherence_bits(state, L.block().row0, rows, n, lm->coh.get() + k, s);
      if (states_host)
        QSWG_CHECK(cudaMemcpyAsync(states_host + 2 * rows * k, state, static_cast<std::size_t>(rows) * sizeof(double2),
                                   cudaMemcpyDeviceToHost, s));
      if (final_state && k == steps)
        QSWG_CHECK(cudaMemcpyAsync(final_state->v.get(), state, static_cast<std::size_t>(rows) * sizeof(double2),
                                   cudaMemcpyDeviceToDevice, s));
    };
    // populations only: every emit is a device kernel into lm->pops, so a
    // repeated identical call may replay a captured graph (expm.hpp: series)
    // (both targets are in the key: either buffer may be reallocated between calls)
    std::vector<const void*> graph_key;
    if (!states_host && !final_state) {
      graph_key.push_back(lm->pops.get());
      if (coherence_host) graph_key.push_back(lm->coh.get());
    }
    // the outputs' reads are enqueued before the call's one synchronisation
    const auto reads = [&] {
      if (L.comm() && L.comm()->world() > 1)  // every diagonal element has exactly one owner
        L.comm()->allreduce_sum_f64(lm->pops.get(), static_cast<std::size_t>((steps + 1) * n), s);
      if (coherence_host && L.comm() && L.comm()->world() > 1)
        L.comm()->allreduce_max_u64(lm->coh.get(), static_cast<std::size_t>(steps + 1), s);
      QSWG_CHECK(cudaEventRecord(e1, s));
      if (pops_host)
        QSWG_CHECK(cudaMemcpyAsync(pops_host, lm->pops.get(), lm->pops.bytes(), cudaMemcpyDeviceToHost, s));
      if (coherence_host)  // bit patterns of non-negative doubles are the doubles
        QSWG_CHECK(cudaMemcpyAsync(coherence_host, lm->coh.get(), lm->coh.bytes(), cudaMemcpyDeviceToHost, s));
    };
    const qswg::SeriesInfo si = qswg::series(L, v->v.get(), t1, tq, steps, params, emit, graph_key, v->herm, reads);
    if (final_state) final_state->herm = L.hermitian_mode() ? 1 : -1;
    float ms = 0.f;
    QSWG_CHECK(cudaEventElapsedTime(&ms, e0, e1));
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (info) {
      info->path = si.path;
      info->span_m_star = si.span_m_star;
      info->span_s = si.span_s;
      info->d = si.d;
      info->n_super = si.n_super;
      info->remainder = si.remainder;
      info->sub_m_star = si.sub_m_star;
      info->spmvs = si.spmvs;
      info->launches = si.launches + si.emits;
      info->device_ms = ms;
      info->host_waits = si.host_waits;
    }
  });
}

// ------------------------------------------------------------ planning
int qswg_plan_rows(int64_t n, const int64_t* colptr, int world, int64_t* starts) {
  return guarded([&] {
    need(colptr, "colptr");
    need(starts, "starts");
    const std::vector<int64_t> cp(colptr, colptr + n + 1);
    const std::vector<int64_t> st = qswg::partition_rows(cp, n, world);
    std::memcpy(starts, st.data(), st.size() * sizeof(int64_t));
  });
}

int qswg_plan_halo(const int64_t* cols, int64_t nnz, const int64_t* starts, int world, int rank, int64_t* lo,
                   int64_t* hi) {
  return guarded([&] {
    need(starts, "starts");
    need(lo, "lo");
    need(hi, "hi");
    if (rank < 0 || rank >= world) throw std::invalid_argument("rank out of range");
    const std::vector<int64_t> st(starts, starts + world + 1);
    const auto needs = qswg::halo_needs_host(cols, nnz, st, rank);
    for (int q = 0; q < world; ++q) {
      lo[q] = needs[static_cast<std::size_t>(q)].lo;
      hi[q] = needs[static_cast<std::size_t>(q)].hi;
    }
  });
}

int qswg_liouvillian_partition(const qswg_liouvillian* l, int64_t* starts, int64_t* halo_lo, int64_t* halo_hi) {
  return guarded([&] {
    need(l, "liouvillian");
    const auto& st = l->l->partition();
    const std::size_t w = st.size() - 1;
    if (starts) std::memcpy(starts, st.data(), st.size() * sizeof(int64_t));
    for (std::size_t r = 0; r < w; ++r)
      for (std::size_t q = 0; q < w; ++q) {
        if (halo_lo) halo_lo[r * w + q] = l->l->halo_lo()[r][q];
        if (halo_hi) halo_hi[r * w + q] = l->l->halo_hi()[r][q];
      }
  });
}

// ------------------------------------------------------------------ comm
int qswg_comm_unique_id_size(void) { return qswg::comm_unique_id_size(); }
int qswg_comm_get_unique_id(uint8_t* id) {
  return guarded([&] {
    need(id, "id");
    const int rc = qswg::comm_get_unique_id(id);
    if (rc) throw qswg::CudaError("ncclGetUniqueId failed");
  });
}
int qswg_comm_create(const uint8_t* id, int rank, int world, int device, qswg_comm** out) {
  int rc = QSWG_OK;
  const int g = guarded([&] {
    need(id, "id");
    need(out, "out");
    rc = qswg::comm_create(id, rank, world, device, out);
  });
  return g ? g : rc;
}
void qswg_comm_destroy(qswg_comm* c) { qswg::comm_destroy(c); }

int qswg_comm_create_local(int world, qswg_comm** outs) {
  return guarded([&] {
    need(outs, "outs");
    auto comms = qswg::make_local_comms(world);
    for (int r = 0; r < world; ++r) {
      auto h = std::make_unique<qswg_comm>();
      h->c = std::move(comms[static_cast<std::size_t>(r)]);
      outs[r] = h.release();
    }
  });
}


// ------------------------------------------------------------ file formats
int qswg_matrix_market_parse(const char* text, int64_t len, qswg_sparse** adjacency) {
  return guarded([&] {
    need(text, "text");
    need(adjacency, "adjacency");
    if (len < 0) throw std::invalid_argument("text length must be non-negative");
    std::istringstream in(std::string(text, static_cast<std::size_t>(len)));
    *adjacency = wrap(qswg::load_matrix_market(in));
  });
}

int qswg_matrix_market_load(const char* path, qswg_sparse** adjacency) {
  return guarded([&] {
    need(path, "path");
    need(adjacency, "adjacency");
    *adjacency = wrap(qswg::load_graph_file(path));
  });
}

int qswg_matrix_market_save(const qswg_sparse* adjacency, const char* path) {
  return guarded([&] {
    need(adjacency, "adjacency");
    need(path, "path");
    std::ofstream out(path);
    if (!out) throw qswg::IoError(std::string("cannot open `") + path + "` for writing");
    qswg::save_matrix_market(adjacency->m, out);
    if (!out) throw qswg::IoError(std::string("failed to write `") + path + "`");
  });
}

int qswg_container_create(qswg_container** out) {
  return guarded([&] {
    need(out, "out");
    *out = new qswg_container();
  });
}

void qswg_container_destroy(qswg_container* c) { delete c; }

int qswg_container_set_metadata(qswg_container* c, const char* text, int64_t len) {
  return guarded([&] {
    need(c, "container");
    need(text, "text");
    if (len < 0) throw std::invalid_argument("metadata length must be non-negative");
    c->c.metadata.assign(text, static_cast<std::size_t>(len));
  });
}

int qswg_container_get_metadata(const qswg_container* c, char* buf, int64_t cap, int64_t* len) {
  return guarded([&] {
    need(c, "container");
    if (len) *len = static_cast<int64_t>(c->c.metadata.size());
    if (buf && cap > 0)
      std::memcpy(buf, c->c.metadata.data(), std::min(static_cast<std::size_t>(cap), c->c.metadata.size()));
  });
}

int qswg_container_put_array(qswg_container* c, const char* name, int64_t rank, const int64_t* shape,
                             const double* data) {
  return guarded([&] {
    need(c, "container");
    need(name, "name");
    if (rank < 0) throw std::invalid_argument("array rank must be non-negative");
    if (rank > 0) need(shape, "shape");
    qswg::ArrayBlock a;
    for (int64_t k = 0; k < rank; ++k) {
      if (shape[k] < 0) throw std::invalid_argument("array dimensions must be non-negative");
      a.shape.push_back(static_cast<std::uint64_t>(shape[k]));
    }
    const std::uint64_t count = a.element_count();
    if (count) need(data, "data");
    a.data.assign(data, data + count);
    c->c.arrays[name] = std::move(a);
  });
}

int qswg_container_array_count(const qswg_container* c, int64_t* count) {
  return guarded([&] {
    need(c, "container");
    need(count, "count");
    *count = static_cast<int64_t>(c->c.arrays.size());
  });
}

namespace {
const std::pair<const std::string, qswg::ArrayBlock>& nth_array(const qswg_container* c, int64_t index) {
  if (index < 0 || index >= static_cast<int64_t>(c->c.arrays.size()))
    throw std::out_of_range("container array index out of range");
  return *std::next(c->c.arrays.begin(), index);
}
}  // namespace

int qswg_container_array_info(const qswg_container* c, int64_t index, char* name, int64_t name_cap,
                              int64_t* name_len, int64_t* rank, int64_t* shape, int64_t shape_cap) {
  return guarded([&] {
    need(c, "container");
    const auto& [nm, a] = nth_array(c, index);
    if (name_len) *name_len = static_cast<int64_t>(nm.size());
    if (name && name_cap > 0) std::memcpy(name, nm.data(), std::min(static_cast<std::size_t>(name_cap), nm.size()));
    if (rank) *rank = static_cast<int64_t>(a.shape.size());
    if (shape)
      for (std::size_t k = 0; k < a.shape.size() && static_cast<int64_t>(k) < shape_cap; ++k)
        shape[k] = static_cast<int64_t>(a.shape[k]);
  });
}

int qswg_container_array_data(const qswg_container* c, int64_t index, double* data) {
  return guarded([&] {
    need(c, "container");
    need(data, "data");
    const auto& a = nth_array(c, index).second;
    std::memcpy(data, a.data.data(), a.data.size() * sizeof(double));
  });
}

int qswg_container_write(const qswg_container* c, const char* path) {
  return guarded([&] {
    need(c, "container");
    need(path, "path");
    qswg::write_container(c->c, path);
  });
}

int qswg_container_read(const char* path, qswg_container** out) {
  return guarded([&] {
    need(path, "path");
    need(out, "out");
    auto h = std::make_unique<qswg_container>();
    h->c = qswg::read_container(path);
    *out = h.release();
  });
}

int qswg_container_plot_data(const qswg_container* c, const char* quantity, const char* path) {
  return guarded([&] {
    need(c, "container");
    need(quantity, "quantity");
    need(path, "path");
    const std::string text = qswg::plot_data(c->c, quantity);
    std::ofstream out(path);
    if (!out) throw qswg::IoError(std::string("cannot open `") + path + "` for writing");
    out << text;
    if (!out) throw qswg::IoError("failed to write plot data");
  });
}
}  // extern "C"
