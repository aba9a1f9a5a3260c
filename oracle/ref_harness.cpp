// TEST INFRASTRUCTURE ONLY — never linked into the product.
//
// C-callable harness around the UNMODIFIED reference library
// (/root/reference/proj/core), compiled from its own sources by
// oracle/Makefile into oracle/_ref/libqswref.so.  Used (a) to generate the
// golden fixtures under tests/golden/ (oracle/make_golden.py), (b) to pin the
// C restatement in oracle/qsw_oracle.c, and (c) as bench.py's CPU reference
// arm (cpu_baseline.kind = "reference").  It only calls the reference's public
// API: WalkSystem-free entry points build_local / build_global
// (liouvillian.hpp:73-85), step / series (expm.hpp:51-63), spmv
// (liouvillian.hpp:93), select_parameters / build_theta_table
// (expm.hpp:34-45) and the graph helpers (graph.hpp:78-96).
//
// Taylor-term counting: the link wraps
// DistributedLiouvillian::worker_multiply (-Wl,--wrap, see oracle/Makefile);
// __wrap_ counts calls for worker 0 (one per executed SpMV) and forwards.

#include <complex>
#include <cstdint>
#include <cstring>
#include <exception>
#include <optional>
#include <span>
#include <string>
#include <vector>

#include "qsw/expm.hpp"
#include "qsw/graph.hpp"
#include "qsw/liouvillian.hpp"
#include "qsw/operators.hpp"
#include "qsw/sparse.hpp"
#include "qsw/state.hpp"

using qsw::Complex;
using qsw::SparseMatrix;

// ---- SpMV counter (ld --wrap) -------------------------------------------
static std::uint64_t g_spmv_calls = 0;

#define WM_SYM \
  _ZNK3qsw22DistributedLiouvillian15worker_multiplyEmRKSt6vectorIS1_ISt7complexIdESaIS3_EESaIS5_EESt4spanIS3_Lm18446744073709551615EERS5_S3_
#define CAT2(a, b) a##b
#define CAT(a, b) CAT2(a, b)

extern "C" void CAT(__real_, WM_SYM)(const qsw::DistributedLiouvillian*, std::size_t,
                                     const std::vector<std::vector<Complex>>&,
                                     std::span<Complex>, std::vector<Complex>&, Complex);

extern "C" void CAT(__wrap_, WM_SYM)(const qsw::DistributedLiouvillian* self, std::size_t w,
                                     const std::vector<std::vector<Complex>>& x,
                                     std::span<Complex> y, std::vector<Complex>& ext,
                                     Complex scale) {
  if (w == 0) __atomic_add_fetch(&g_spmv_calls, 1, __ATOMIC_RELAXED);
  CAT(__real_, WM_SYM)(self, w, x, y, ext, scale);
}

namespace {

void set_err(char* err, int len, const char* msg) {
  if (err && len > 0) {
    std::strncpy(err, msg, static_cast<std::size_t>(len - 1));
    err[len - 1] = 0;
  }
}

// Exception class -> code, mirroring the product's C-ABI codes.
int code_of(const std::exception& e) {
  if (dynamic_cast<const qsw::NumericalError*>(&e)) return 3;
  if (dynamic_cast<const std::out_of_range*>(&e)) return 2;
  if (dynamic_cast<const std::invalid_argument*>(&e)) return 1;
  if (dynamic_cast<const std::logic_error*>(&e)) return 4;
  return 9;
}

SparseMatrix csr_in(std::int64_t rows, std::int64_t cols, const std::int64_t* rp,
                    const std::int64_t* ci, const double* v) {
  std::vector<qsw::Triplet> t;
  t.reserve(static_cast<std::size_t>(rp[rows]));
  for (std::int64_t i = 0; i < rows; ++i) {
    for (std::int64_t k = rp[i]; k < rp[i + 1]; ++k) {
      t.push_back({static_cast<std::size_t>(i), static_cast<std::size_t>(ci[k]),
                   Complex{v[2 * k], v[2 * k + 1]}});
    }
  }
  return SparseMatrix::from_triplets(static_cast<std::size_t>(rows),
                                     static_cast<std::size_t>(cols), std::move(t));
}

std::vector<Complex> vec_in(const double* v, std::size_t n) {
  std::vector<Complex> out(n);
  for (std::size_t i = 0; i < n; ++i) out[i] = Complex{v[2 * i], v[2 * i + 1]};
  return out;
}

void vec_out(const std::vector<Complex>& v, double* out) {
  for (std::size_t i = 0; i < v.size(); ++i) {
    out[2 * i] = v[i].real();
    out[2 * i + 1] = v[i].imag();
  }
}

struct Handle {
  qsw::DistributedLiouvillian l;
  std::size_t n = 0;  // operator (vertex) dimension
};

}  // namespace

extern "C" {

std::uint64_t ref_spmv_counter() { return g_spmv_calls; }
void ref_spmv_counter_reset() { g_spmv_calls = 0; }

// ---- sparse helpers -------------------------------------------------------
void* ref_sparse_new(std::int64_t rows, std::int64_t cols, const std::int64_t* rp,
                     const std::int64_t* ci, const double* v) {
  return new SparseMatrix(csr_in(rows, cols, rp, ci, v));
}
void ref_sparse_free(void* p) { delete static_cast<SparseMatrix*>(p); }
void ref_sparse_shape(void* p, std::int64_t* rows, std::int64_t* cols, std::int64_t* nnz) {
  auto* m = static_cast<SparseMatrix*>(p);
  *rows = static_cast<std::int64_t>(m->rows());
  *cols = static_cast<std::int64_t>(m->cols());
  *nnz = static_cast<std::int64_t>(m->nnz());
}
void ref_sparse_export(void* p, std::int64_t* rp, std::int64_t* ci, double* v) {
  auto* m = static_cast<SparseMatrix*>(p);
  auto s = m->row_starts();
  for (std::size_t i = 0; i < s.size(); ++i) rp[i] = static_cast<std::int64_t>(s[i]);
  auto c = m->col_indices();
  auto vals = m->values();
  for (std::size_t k = 0; k < c.size(); ++k) {
    ci[k] = static_cast<std::int64_t>(c[k]);
    v[2 * k] = vals[k].real();
    v[2 * k + 1] = vals[k].imag();
  }
}

// Graph -> operator helpers (graph.hpp:78-96, operators.hpp:53-57). `what`:
// 0 generator_matrix(gamma, G), 1 markov_chain_matrix(G),
// 2 symmetrize(G).adjacency(), 3 local_lindblad(m), 4 transpose,
// 5 conjugate_transpose.
void* ref_graph_op(int what, double gamma, void* adj, char* err, int errlen) {
  try {
    auto* a = static_cast<SparseMatrix*>(adj);
    switch (what) {
      case 0: return new SparseMatrix(qsw::generator_matrix(gamma, *a));
      case 1:
        return new SparseMatrix(
            qsw::markov_chain_matrix(qsw::WeightedDigraph::from_adjacency(*a)));
      case 2:
        return new SparseMatrix(
            qsw::symmetrize(qsw::WeightedDigraph::from_adjacency(*a)).adjacency());
      case 3: return new SparseMatrix(qsw::local_lindblad(*a));
      case 4: return new SparseMatrix(a->transpose());
      case 5: return new SparseMatrix(a->conjugate_transpose());
      default: set_err(err, errlen, "unknown op"); return nullptr;
    }
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

// Demoralisation operators (operators.hpp:59-83): what 0 nm_H(gamma, gu, V),
// 1 nm_L(gamma, g, V), 2 nm_H_rot(V, dim2), with V = nm_vsets(gu); dims_out
// (vertex count entries) receives V.dims.
void* ref_nm_op(int what, double gamma, void* g, void* gu, int pauli_y, std::int64_t* dims_out, char* err,
                int errlen) {
  try {
    const auto G = qsw::WeightedDigraph::from_adjacency(*static_cast<SparseMatrix*>(g));
    const auto GU = qsw::WeightedDigraph::from_adjacency(*static_cast<SparseMatrix*>(gu));
    const qsw::VertexSubspaces v = qsw::nm_vsets(GU);
    for (std::size_t i = 0; i < v.dims.size(); ++i) dims_out[i] = static_cast<std::int64_t>(v.dims[i]);
    switch (what) {
      case 0: return new SparseMatrix(qsw::nm_H(gamma, GU, v));
      case 1: return new SparseMatrix(qsw::nm_L(gamma, G, v));
      case 2:
        return new SparseMatrix(
            qsw::nm_H_rot(v, pauli_y ? qsw::Dim2Rotation::PauliY : qsw::Dim2Rotation::Cancel));
      default: set_err(err, errlen, "unknown op"); return nullptr;
    }
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

// ---- superoperator --------------------------------------------------------
void* ref_build_local(double omega, void* h, void* m_l, std::int64_t nsrc,
                      const std::int64_t* src_target, const double* src_rate,
                      std::int64_t nsnk, const std::int64_t* snk_origin,
                      const double* snk_rate, std::int64_t workers, int* code, char* err,
                      int errlen) {
  try {
    std::vector<qsw::SourceArc> src;
    for (std::int64_t k = 0; k < nsrc; ++k)
      src.push_back({static_cast<std::size_t>(src_target[k]), src_rate[k]});
    std::vector<qsw::SinkArc> snk;
    for (std::int64_t k = 0; k < nsnk; ++k)
      snk.push_back({static_cast<std::size_t>(snk_origin[k]), snk_rate[k]});
    auto* out = new Handle;
    out->l = qsw::build_local(omega, *static_cast<SparseMatrix*>(h),
                              *static_cast<SparseMatrix*>(m_l), src, snk,
                              static_cast<std::size_t>(workers));
    out->n = static_cast<SparseMatrix*>(h)->rows();
    *code = 0;
    return out;
  } catch (const std::exception& e) {
    *code = code_of(e);
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void* ref_build_global(double omega, void* h, std::int64_t k, void* const* lindblads,
                       void* h_rot, std::int64_t workers, int* code, char* err, int errlen) {
  try {
    std::vector<SparseMatrix> ls;
    for (std::int64_t i = 0; i < k; ++i) ls.push_back(*static_cast<SparseMatrix*>(lindblads[i]));
    std::optional<SparseMatrix> hr;
    if (h_rot) hr = *static_cast<SparseMatrix*>(h_rot);
    auto* out = new Handle;
    out->l = qsw::build_global(omega, *static_cast<SparseMatrix*>(h), ls, hr,
                               static_cast<std::size_t>(workers));
    out->n = static_cast<SparseMatrix*>(h)->rows();
    *code = 0;
    return out;
  } catch (const std::exception& e) {
    *code = code_of(e);
    set_err(err, errlen, e.what());
    return nullptr;
  }
}

void ref_free(void* p) { delete static_cast<Handle*>(p); }

void ref_info(void* p, std::int64_t* dim, std::int64_t* nnz, double* norms) {
  auto* hd = static_cast<Handle*>(p);
  *dim = static_cast<std::int64_t>(hd->l.dim());
  std::size_t total = 0;
  for (const auto& b : hd->l.local_blocks()) total += b.nnz();
  *nnz = static_cast<std::int64_t>(total);
  auto n = hd->l.one_norms();
  for (int i = 0; i < 9; ++i) norms[i] = n[i];
}

void ref_csr(void* p, std::int64_t* rp, std::int64_t* ci, double* v) {
  auto* hd = static_cast<Handle*>(p);
  SparseMatrix full = hd->l.gather_full();
  ref_sparse_export(&full, rp, ci, v);
}

int ref_spmv(void* p, const double* x, double* y) {
  auto* hd = static_cast<Handle*>(p);
  auto xs = qsw::StateVector::scatter(vec_in(x, hd->l.dim()), hd->l.partition());
  vec_out(qsw::spmv(hd->l, xs).gather(), y);
  return 0;
}

int ref_step(void* p, const double* v, double t, double* out, char* err, int errlen) {
  try {
    auto* hd = static_cast<Handle*>(p);
    auto vs = qsw::StateVector::scatter(vec_in(v, hd->l.dim()), hd->l.partition());
    vec_out(qsw::step(hd->l, vs, t).gather(), out);
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return code_of(e);
  }
}

// states_out: (steps+1) * dim complex, or null. pops_out: (steps+1) * n, or null.
int ref_series(void* p, const double* v, double t1, double tq, std::int64_t steps,
               double* states_out, double* pops_out, char* err, int errlen) {
  try {
    auto* hd = static_cast<Handle*>(p);
    const std::size_t dim = hd->l.dim();
    auto vs = qsw::StateVector::scatter(vec_in(v, dim), hd->l.partition());
    qsw::SeriesResult r = qsw::series(hd->l, vs, t1, tq, static_cast<std::size_t>(steps));
    for (std::size_t q = 0; q < r.states.size(); ++q) {
      std::vector<Complex> full = r.states[q].gather();
      if (states_out) vec_out(full, states_out + 2 * dim * q);
      if (pops_out) {
        for (std::size_t i = 0; i < hd->n; ++i) pops_out[hd->n * q + i] = full[i * hd->n + i].real();
      }
    }
    return 0;
  } catch (const std::exception& e) {
    set_err(err, errlen, e.what());
    return code_of(e);
  }
}

// ---- Taylor parameters ----------------------------------------------------
int ref_theta(double tol, double* out55) {
  try {
    const auto& t = qsw::build_theta_table(tol);
    for (int i = 0; i < 55; ++i) out55[i] = t.theta[i];
    return 0;
  } catch (const std::exception&) {
    return 1;
  }
}

void ref_select(const double* norms9, double t, double tol, std::int64_t* m, std::int64_t* s) {
  std::array<double, 9> n{};
  for (int i = 0; i < 9; ++i) n[i] = norms9[i];
  auto sp = qsw::select_parameters(n, t, qsw::build_theta_table(tol));
  *m = static_cast<std::int64_t>(sp.m_star);
  *s = static_cast<std::int64_t>(sp.s);
}

}  // extern "C"
