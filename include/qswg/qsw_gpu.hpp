// qswg/qsw_gpu.hpp — header-only C++ RAII facade over the C ABI (qswg.h).
//
// The reference's hot path is a C++ library surface, not a plugin layer
// (SURVEY.md §8(b)); this header gives a C++ caller the same shape of API on
// the GPU library:
//
//   reference (proj/core/include/qsw/)          here (namespace qswg::gpu)
//   SparseMatrix::from_triplets (sparse.hpp)    SparseMatrix::from_triplets / from_csr
//   generator_matrix, markov_chain_matrix,      generator_matrix, markov_chain_matrix,
//     symmetrize (graph.hpp:78-88)                symmetrize, local_lindblad
//   build_local / build_global                  Liouvillian::build_local / build_global
//     (liouvillian.hpp:65-85)
//   DistributedLiouvillian::one_norms, dim,     Liouvillian::one_norms, dim, nnz, spmv
//     spmv (liouvillian.hpp:31, 93)
//   qsw::step, qsw::series (expm.hpp:51-63)     step(l, v, t), series(l, v, t1, tq, steps)
//   WalkSystem (walk.hpp:39-84)                 WalkSystem::lqsw / gqsw, initial_state,
//                                               set_omega, step, series, gather_populations
//
// Error behaviour is the reference's: std::invalid_argument,
// std::out_of_range, NumericalError, std::logic_error, FileFormatError and
// IoError are rethrown from the C codes (no exception crosses the C ABI);
// CUDA / NCCL failures become CudaError.  Every handle is move-only and frees
// its device memory in its destructor.  Complex values are std::complex<double>
// (layout-compatible with the ABI's interleaved doubles); vec(rho) is
// column-major, element n*j + i = rho(i, j) (state.hpp:10-12).
#pragma once

#include <qswg.h>

#include <array>
#include <complex>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

namespace qswg::gpu {

using Complex = std::complex<double>;
inline constexpr double kDoublePrecisionTol = 0x1p-53;  // expm.hpp: kDoublePrecisionTol

struct NumericalError : std::runtime_error {  // qsw::NumericalError (expm.hpp)
  using std::runtime_error::runtime_error;
};
struct FileFormatError : std::runtime_error {  // qsw::FileFormatError (graph.hpp:11-15)
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {  // qsw::IoError (container.hpp:13-17)
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {  // device / NCCL / internal failures
  using std::runtime_error::runtime_error;
};

/// Maps a qswg return code to the reference's exception types.
inline void check(int rc) {
  if (rc == QSWG_OK) return;
  const char* m = qswg_last_error();
  const std::string msg = m ? m : "";
  switch (rc) {
    case QSWG_EINVAL:
      throw std::invalid_argument(msg);
    case QSWG_ERANGE:
      throw std::out_of_range(msg);
    case QSWG_ENUMERICAL:
      throw NumericalError(msg);
    case QSWG_ESTATE:
      throw std::logic_error(msg);
    case QSWG_EFORMAT:
      throw FileFormatError(msg);
    case QSWG_EIO:
      throw IoError(msg);
    case QSWG_ENOMEM:
      throw std::bad_alloc();
    default:
      throw CudaError(msg.empty() ? "qswg error " + std::to_string(rc) : msg);
  }
}

namespace detail {
template <class T, void (*Destroy)(T*)>
class Handle {
 public:
  Handle() = default;
  explicit Handle(T* p) : p_(p) {}
  ~Handle() { reset(); }
  Handle(const Handle&) = delete;
  Handle& operator=(const Handle&) = delete;
  Handle(Handle&& o) noexcept : p_(std::exchange(o.p_, nullptr)) {}
  Handle& operator=(Handle&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = std::exchange(o.p_, nullptr);
    }
    return *this;
  }
  void reset() {
    if (p_) Destroy(p_);
    p_ = nullptr;
  }
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
};
inline const double* dp(const Complex* p) { return reinterpret_cast<const double*>(p); }
inline double* dp(Complex* p) { return reinterpret_cast<double*>(p); }
}  // namespace detail

/// Host canonical CSR, complex128 (sparse.hpp:29-84).
class SparseMatrix {
 public:
  /// SparseMatrix::from_triplets: sorts, sums duplicates, drops zeros.
  static SparseMatrix from_triplets(int64_t rows, int64_t cols, const std::vector<int64_t>& row,
                                    const std::vector<int64_t>& col, const std::vector<Complex>& val) {
    if (row.size() != col.size() || row.size() != val.size())
      throw std::invalid_argument("triplet arrays differ in length");
    qswg_sparse* h = nullptr;
    check(qswg_sparse_from_triplets(rows, cols, static_cast<int64_t>(row.size()), row.data(), col.data(),
                                    detail::dp(val.data()), &h));
    return SparseMatrix(h);
  }
  static SparseMatrix from_csr(int64_t rows, int64_t cols, const std::vector<int64_t>& rowptr,
                               const std::vector<int64_t>& col, const std::vector<Complex>& val) {
    qswg_sparse* h = nullptr;
    check(qswg_sparse_from_csr(rows, cols, rowptr.data(), col.data(), detail::dp(val.data()), &h));
    return SparseMatrix(h);
  }
  int64_t rows() const { return shape()[0]; }
  int64_t cols() const { return shape()[1]; }
  int64_t nnz() const { return shape()[2]; }
  /// (row_starts, col_indices, values) of the canonical CSR.
  void export_csr(std::vector<int64_t>& rowptr, std::vector<int64_t>& col, std::vector<Complex>& val) const {
    const auto s = shape();
    rowptr.resize(static_cast<std::size_t>(s[0]) + 1);
    col.resize(static_cast<std::size_t>(s[2]));
    val.resize(static_cast<std::size_t>(s[2]));
    check(qswg_sparse_export(h_.get(), rowptr.data(), col.data(), detail::dp(val.data())));
  }
  const qswg_sparse* handle() const { return h_.get(); }

 private:
  explicit SparseMatrix(qswg_sparse* h) : h_(h) {}
  std::array<int64_t, 3> shape() const {
    std::array<int64_t, 3> s{};
    check(qswg_sparse_shape(h_.get(), &s[0], &s[1], &s[2]));
    return s;
  }
  detail::Handle<qswg_sparse, qswg_sparse_destroy> h_;
  friend SparseMatrix symmetrize(const SparseMatrix&);
  friend SparseMatrix generator_matrix(double, const SparseMatrix&);
  friend SparseMatrix markov_chain_matrix(const SparseMatrix&);
  friend SparseMatrix local_lindblad(const SparseMatrix&);
};

/// graph.hpp:75-88, operators.hpp:53-54.
inline SparseMatrix symmetrize(const SparseMatrix& g) {
  qswg_sparse* o = nullptr;
  check(qswg_symmetrize(g.handle(), &o));
  return SparseMatrix(o);
}
inline SparseMatrix generator_matrix(double gamma, const SparseMatrix& g) {
  qswg_sparse* o = nullptr;
  check(qswg_generator_matrix(gamma, g.handle(), &o));
  return SparseMatrix(o);
}
inline SparseMatrix markov_chain_matrix(const SparseMatrix& g) {
  qswg_sparse* o = nullptr;
  check(qswg_markov_chain_matrix(g.handle(), &o));
  return SparseMatrix(o);
}
inline SparseMatrix local_lindblad(const SparseMatrix& m) {
  qswg_sparse* o = nullptr;
  check(qswg_local_lindblad(m.handle(), &o));
  return SparseMatrix(o);
}

/// Where and how the superoperator lives (the reference's n_workers).
struct DeviceConfig {
  int device = 0;
  int group = 0;                  // CSR lanes per row; 1 = bitwise reference order; 0 = autotune
  int format = QSWG_FORMAT_AUTO;  // QSWG_FORMAT_{AUTO,CSR,SELL,KRON}
  qswg_comm* comm = nullptr;      // multi-GPU communicator (borrowed), nullptr for one GPU
  qswg_device_config c() const { return qswg_device_config{device, group, format, comm}; }
};

/// The device superoperator (DistributedLiouvillian, liouvillian.hpp:21-63).
class Liouvillian {
 public:
  /// build_local (liouvillian.hpp:65-71).
  static Liouvillian build_local(double omega, const SparseMatrix& h, const SparseMatrix& m_l,
                                 const std::vector<qswg_source_arc>& sources = {},
                                 const std::vector<qswg_sink_arc>& sinks = {}, const DeviceConfig& cfg = {}) {
    const qswg_device_config c = cfg.c();
    qswg_liouvillian* l = nullptr;
    check(qswg_build_local(omega, h.handle(), m_l.handle(), sources.data(), static_cast<int64_t>(sources.size()),
                           sinks.data(), static_cast<int64_t>(sinks.size()), &c, &l));
    return Liouvillian(l);
  }
  /// build_global (liouvillian.hpp:73-85).
  static Liouvillian build_global(double omega, const SparseMatrix& h, const std::vector<const SparseMatrix*>& lindblads,
                                  const SparseMatrix* h_rot = nullptr, const DeviceConfig& cfg = {}) {
    std::vector<const qswg_sparse*> ls;
    for (const SparseMatrix* m : lindblads) ls.push_back(m->handle());
    const qswg_device_config c = cfg.c();
    qswg_liouvillian* l = nullptr;
    check(qswg_build_global(omega, h.handle(), ls.data(), static_cast<int64_t>(ls.size()),
                            h_rot ? h_rot->handle() : nullptr, &c, &l));
    return Liouvillian(l);
  }
  qswg_liouvillian_info info() const {
    qswg_liouvillian_info i{};
    check(qswg_liouvillian_query(h_.get(), &i));
    return i;
  }
  int64_t n() const { return info().n; }
  int64_t dim() const { return info().dim; }
  int64_t nnz() const { return info().nnz; }
  /// Upper bounds on ||L^p||_1, p = 1..9 (exact for dim <= 4096).
  std::array<double, 9> one_norms() const {
    const auto i = info();
    std::array<double, 9> a{};
    for (int k = 0; k < 9; ++k) a[static_cast<std::size_t>(k)] = i.one_norms[k];
    return a;
  }
  /// spmv(l, x) (liouvillian.hpp:93): y = L x.
  std::vector<Complex> spmv(const std::vector<Complex>& x) const {
    const auto i = info();
    if (static_cast<int64_t>(x.size()) != i.dim) throw std::invalid_argument("spmv: x must have dim entries");
    std::vector<Complex> y(static_cast<std::size_t>(i.rows));
    check(qswg_spmv(h_.get(), detail::dp(x.data()), detail::dp(y.data())));
    return y;
  }
  /// WalkSystem::set_omega: re-mixes in place; states of this handle stay valid.
  void set_omega(double omega) { check(qswg_liouvillian_set_omega(h_.get(), omega)); }
  const qswg_liouvillian* handle() const { return h_.get(); }

 private:
  explicit Liouvillian(qswg_liouvillian* l) : h_(l) {}
  detail::Handle<qswg_liouvillian, qswg_liouvillian_destroy> h_;
};

/// vec(rho) on the device (StateVector, state.hpp:13-27): this rank's rows.
class StateVector {
 public:
  explicit StateVector(const Liouvillian& l) {
    qswg_state* s = nullptr;
    check(qswg_state_create(l.handle(), &s));
    h_ = decltype(h_)(s);
  }
  /// StateVector::scatter(full): `vec` holds all dim entries of vec(rho).
  StateVector& upload(const std::vector<Complex>& vec) {
    check(qswg_state_upload(h_.get(), detail::dp(vec.data())));
    return *this;
  }
  /// WalkSystem::initial_state(probabilities) (walk.cpp:101-126).
  StateVector& from_probabilities(const std::vector<double>& p) {
    check(qswg_state_from_probabilities(h_.get(), p.data(), static_cast<int64_t>(p.size())));
    return *this;
  }
  std::vector<Complex> gather(int64_t rows) const {
    std::vector<Complex> v(static_cast<std::size_t>(rows));
    check(qswg_state_download(h_.get(), detail::dp(v.data())));
    return v;
  }
  /// populations_of(state) (walk.cpp:177-186).
  std::vector<double> populations(int64_t n) const {
    std::vector<double> p(static_cast<std::size_t>(n));
    check(qswg_state_populations(h_.get(), p.data()));
    return p;
  }
  qswg_state* handle() const { return h_.get(); }

 private:
  detail::Handle<qswg_state, qswg_state_destroy> h_;
};

/// w = exp(tL) v (qsw::step, expm.hpp:51-52).
inline StateVector step(const Liouvillian& l, const StateVector& v, double t, double tol = kDoublePrecisionTol,
                        qswg_step_info* info = nullptr) {
  StateVector out(l);
  check(qswg_step(l.handle(), v.handle(), t, tol, out.handle(), info));
  return out;
}

/// qsw::series (expm.hpp:55-63): outputs at t1 + k (tq - t1) / steps.
/// Populations of every output always; full states (this rank's rows) on
/// request — the reference returns every state, which for large walks is
/// most of the host memory traffic.
struct SeriesResult {
  std::vector<double> times;
  std::vector<std::vector<double>> populations;
  std::vector<std::vector<Complex>> states;  // empty unless requested
  qswg_series_info info{};
};

inline SeriesResult series(const Liouvillian& l, const StateVector& v, double t1, double tq, int64_t steps,
                           double tol = kDoublePrecisionTol, bool keep_states = false,
                           StateVector* final_state = nullptr) {
  const auto li = l.info();
  SeriesResult r;
  if (steps < 1) throw std::invalid_argument("series requires at least one step");
  std::vector<double> pops(static_cast<std::size_t>((steps + 1) * li.n));
  std::vector<Complex> states(keep_states ? static_cast<std::size_t>((steps + 1) * li.rows) : 0);
  check(qswg_series(l.handle(), v.handle(), t1, tq, steps, tol, pops.data(),
                    keep_states ? detail::dp(states.data()) : nullptr, final_state ? final_state->handle() : nullptr,
                    &r.info));
  const double h = (tq - t1) / static_cast<double>(steps);
  for (int64_t k = 0; k <= steps; ++k) {  // expm.cpp:222-223
    r.times.push_back(t1 + h * static_cast<double>(k));
    r.populations.emplace_back(pops.begin() + k * li.n, pops.begin() + (k + 1) * li.n);
    if (keep_states) r.states.emplace_back(states.begin() + k * li.rows, states.begin() + (k + 1) * li.rows);
  }
  return r;
}

/// One walk (WalkSystem, walk.hpp:39-84): operators, the device superoperator
/// and the evolution state; step / series always evolve from rho(0).
class WalkSystem {
 public:
  static WalkSystem lqsw(double omega, SparseMatrix h, SparseMatrix m_l, std::vector<qswg_source_arc> sources = {},
                         std::vector<qswg_sink_arc> sinks = {}, const DeviceConfig& cfg = {}) {
    return WalkSystem(Liouvillian::build_local(omega, h, m_l, sources, sinks, cfg));
  }
  static WalkSystem gqsw(double omega, SparseMatrix h, const std::vector<SparseMatrix>& lindblads,
                         const std::optional<SparseMatrix>& h_rot = std::nullopt, const DeviceConfig& cfg = {}) {
    std::vector<const SparseMatrix*> ls;
    for (const SparseMatrix& m : lindblads) ls.push_back(&m);
    return WalkSystem(Liouvillian::build_global(omega, h, ls, h_rot ? &*h_rot : nullptr, cfg));
  }
  int64_t dimension() const { return n_; }
  const Liouvillian& liouvillian() const { return l_; }
  /// Diagonal rho(0) from vertex probabilities (walk.cpp:101-126).
  void initial_state(const std::vector<double>& probabilities) {
    initial_.emplace(l_);
    initial_->from_probabilities(probabilities);
    result_.reset();
  }
  /// Full rho(0) as column-major vec(rho).
  void initial_state_vec(const std::vector<Complex>& vec) {
    initial_.emplace(l_);
    initial_->upload(vec);
    result_.reset();
  }
  bool has_state() const { return initial_.has_value(); }
  void set_omega(double omega) { l_.set_omega(omega); }
  /// Evolves rho(0) to t and stores the result (walk.cpp:147-151).
  void step(double t, double tol = kDoublePrecisionTol) {
    if (!initial_) throw std::logic_error("no initial state: call initial_state first");  // walk.cpp:148
    result_.emplace(gpu::step(l_, *initial_, t, tol));
  }
  /// Evolves rho(0) over [t1, tq]; the stored state ends at tq (walk.cpp:153-158).
  SeriesResult series(double t1, double tq, int64_t steps, double tol = kDoublePrecisionTol, bool keep_states = false) {
    if (!initial_) throw std::logic_error("no initial state: call initial_state first");  // walk.cpp:154
    StateVector fin(l_);
    SeriesResult r = gpu::series(l_, *initial_, t1, tq, steps, tol, keep_states, &fin);
    result_.emplace(std::move(fin));
    return r;
  }
  /// Vertex populations of the most recent state (rho(0) before any evolution).
  std::vector<double> gather_populations() const {
    if (result_) return result_->populations(n_);
    if (initial_) return initial_->populations(n_);
    throw std::logic_error("no state available: call initial_state first");
  }

 private:
  explicit WalkSystem(Liouvillian l) : l_(std::move(l)), n_(l_.n()) {}
  Liouvillian l_;
  int64_t n_ = 0;
  std::optional<StateVector> initial_, result_;
};

}  // namespace qswg::gpu
