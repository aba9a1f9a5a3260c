// Superoperator construction: host operand preparation (small n x n
// operators) + device assembly and norms.  Validation and the emitted values
// follow proj/core/src/liouvillian.cpp (cited per block); the O(nnz) work
// runs on the GPU (cuda/assemble.cu, cuda/norms.cu).
#include "liouvillian.hpp"

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <numeric>
#include <type_traits>
#include <stdexcept>
#include <string>

#include "comm.hpp"
#include "dist.hpp"

namespace qswg {

namespace detail {

constexpr std::int64_t kExactNormDimLimit = 4096;  // liouvillian.cpp:13
constexpr std::int64_t kMaxVertices = 46340;       // n^2 must fit int32 columns
// Auto format: the matrix-free KRON action above this dimension; below it the
// stored superoperator (c1, dim 4096: SELL 1.57 ms vs KRON 2.55 ms per series —
// fewer launches per term for a launch-bound system).
constexpr std::int64_t kKronMinDim = 65536;
constexpr double kSellSortPadding = 1.02;  // sort rows (SELL-C-sigma) above this consecutive-row padding
// Sorting window of SELL-C-sigma (QSWG_SELL_SIGMA overrides; 32 disables).
int sell_sigma_setting() {
  static const int v = [] {
    const char* e = std::getenv("QSWG_SELL_SIGMA");
    // SELL term kernel vs sigma (profiles/r01_sell_sigma_sweep.jsonl): c3 (ER, dim 4.2M)
    // 32: 0.685 of HBM (padding 1.24), 256: 0.64, 4096: 0.71, 16384: 0.77, 65536: 0.76;
    // c4 in 6 column panels 16384: 0.63, 65536: 0.65, 262144: 0.66
    const int x = e ? std::atoi(e) : 65536;
    return x >= 32 ? x : 32;
  }();
  return v;
}
// Streamed SELL kernels (taylor.cu: slice_stream).  QSWG_SELL_STREAM: 0 = the
// register path everywhere, 1 = streamed everywhere; default: streamed for
// unsorted (regular) superoperators with short rows, whose register-path warps
// would drain at every slice boundary, and the register path (more resident
// warps) otherwise — long rows, or sigma-sorted (irregular) matrices whose
// scattered gathers need the latency hiding (measured).
constexpr double kStreamMaxRowLength = 24.0;
int sell_stream_setting() {
  static const int v = [] {
    const char* e = std::getenv("QSWG_SELL_STREAM");
    return e ? std::atoi(e) : -1;
  }();
  return v;
}
constexpr double kSellMaxPadding = 1.3;  // SELL if stored/nnz <= this (else CSR)
// Column panels of a SELL superoperator: when the gathered vector (the
// full-length x, also on every rank of a row-partitioned run) is larger than
// kPanelMinX and the rows are irregular (sorted: gathers go everywhere, c4),
// split the columns so each panel's slice of x (about kPanelX) stays in L2
// while the panel's entries stream.  QSWG_SELL_PANELS forces a count
// (tests); lattices and the bitwise mode keep one pass.
// With the fused natural-order B (x) I arrays (one GPU) a third to a half of
// the gathers are coalesced segments, the L2 carries less sector traffic, and
// larger panels win (c4: 4 panels of 67 MB 0.755 of HBM, 5: 0.747, 7: 0.727,
// 3: 0.745, 2: 0.71, 1: 0.62; without the fused arrays 6-7 panels of 40 MB).
constexpr double kPanelMinX = 96e6, kPanelX = 40e6, kPanelXFused = 70e6;
int sell_panel_count(int group, std::int64_t n, bool sorted, bool fused = false) {
  if (group == 1) return 1;
  int p = 1;
  if (const char* e = std::getenv("QSWG_SELL_PANELS")) {
    p = std::atoi(e);
  } else if (sorted) {
    const double xb = 16.0 * static_cast<double>(n) * static_cast<double>(n);
    if (xb > kPanelMinX) p = static_cast<int>(std::ceil(xb / (fused ? kPanelXFused : kPanelX)));
  }
  return static_cast<int>(std::clamp<std::int64_t>(p, 1, std::min<std::int64_t>(dev::kMaxSellPanels, n)));
}

// Fused B (x) I windows of the sorted SELL kernels (kernels.hpp: SellView::b_val).  A block
// takes a whole window of 64 slices, so small superoperators would leave SMs idle (c1,
// 128 slices: 2 blocks, 1.3 -> 3.6 ms per series): by default only from kFuseMinWindows
// windows (2 per SM of a B200) on.  QSWG_SELL_FUSE=0 keeps every entry in the sorted arrays,
// =1 fuses at any size (tests).
constexpr std::int64_t kFuseMinWindows = 296;
bool sell_fuse_setting(std::int64_t n_slices) {
  const char* e = std::getenv("QSWG_SELL_FUSE");
  if (e && e[0] == '0') return false;
  if (e && e[0] == '1') return true;
  return n_slices >= kFuseMinWindows * dev::kSellWindowSlices;
}

double hermiticity_tolerance(const SparseMatrix& m) { return 1e-15 * std::max(1.0, m.max_abs()); }

// Host-side multi-CSR (see dev::KronList): per-row entries in emission order,
// stably sorted by column.
struct MultiCsr {
  std::int64_t n = 0;
  std::vector<int> ptr, col;
  std::vector<double2> val;
  bool empty() const { return col.empty(); }
};

struct Entry {
  std::int64_t row, col;
  Complex v;
};

MultiCsr make_multi(std::int64_t n, const std::vector<Entry>& e) {
  MultiCsr m;
  m.n = n;
  m.ptr.assign(static_cast<std::size_t>(n) + 1, 0);
  for (const Entry& x : e) ++m.ptr[static_cast<std::size_t>(x.row) + 1];
  std::partial_sum(m.ptr.begin(), m.ptr.end(), m.ptr.begin());
  std::vector<std::size_t> order(e.size());
  {
    std::vector<int> cur(m.ptr.begin(), m.ptr.end() - 1);
    for (std::size_t k = 0; k < e.size(); ++k) order[static_cast<std::size_t>(cur[static_cast<std::size_t>(e[k].row)]++)] = k;
  }
  for (std::int64_t i = 0; i < n; ++i) {
    auto b = order.begin() + m.ptr[static_cast<std::size_t>(i)], en = order.begin() + m.ptr[static_cast<std::size_t>(i) + 1];
    std::stable_sort(b, en, [&](std::size_t x, std::size_t y) { return e[x].col < e[y].col; });
  }
  m.col.resize(e.size());
  m.val.resize(e.size());
  for (std::size_t k = 0; k < e.size(); ++k) {
    m.col[k] = static_cast<int>(e[order[k]].col);
    m.val[k] = make_double2(e[order[k]].v.real(), e[order[k]].v.imag());
  }
  return m;
}

// Stable transpose: duplicates of one (i, c) keep their emission order.
MultiCsr transpose_multi(const MultiCsr& a) {
  std::vector<Entry> e;
  e.reserve(a.col.size());
  for (std::int64_t i = 0; i < a.n; ++i)
    for (int k = a.ptr[static_cast<std::size_t>(i)]; k < a.ptr[static_cast<std::size_t>(i) + 1]; ++k)
      e.push_back({a.col[static_cast<std::size_t>(k)], i,
                   Complex{a.val[static_cast<std::size_t>(k)].x, a.val[static_cast<std::size_t>(k)].y}});
  return make_multi(a.n, e);
}

MultiCsr from_sparse(const SparseMatrix& s, const std::function<Complex(Complex)>& f) {
  std::vector<Entry> e;
  e.reserve(static_cast<std::size_t>(s.nnz()));
  for (std::int64_t i = 0; i < s.rows(); ++i)
    for (std::int64_t k = s.row_begin(i); k < s.row_end(i); ++k)
      e.push_back({i, s.col_indices()[static_cast<std::size_t>(k)], f(s.values()[static_cast<std::size_t>(k)])});
  return make_multi(s.rows(), e);
}

void append_entries(std::vector<Entry>& e, const SparseMatrix& s, const std::function<Complex(Complex)>& f) {
  for (std::int64_t i = 0; i < s.rows(); ++i)
    for (std::int64_t k = s.row_begin(i); k < s.row_end(i); ++k)
      e.push_back({i, s.col_indices()[static_cast<std::size_t>(k)], f(s.values()[static_cast<std::size_t>(k)])});
}

// Summed, zero-free copy of a multi-CSR (the matrix-free path needs each
// operand once, not its emission history).
MultiCsr canonical(const MultiCsr& m) {
  MultiCsr c;
  c.n = m.n;
  c.ptr.assign(m.ptr.size(), 0);
  for (std::int64_t i = 0; i < m.n; ++i) {
    for (int k = m.ptr[static_cast<std::size_t>(i)]; k < m.ptr[static_cast<std::size_t>(i) + 1];) {
      const int col = m.col[static_cast<std::size_t>(k)];
      double2 v = m.val[static_cast<std::size_t>(k++)];
      while (k < m.ptr[static_cast<std::size_t>(i) + 1] && m.col[static_cast<std::size_t>(k)] == col) {
        v.x += m.val[static_cast<std::size_t>(k)].x;
        v.y += m.val[static_cast<std::size_t>(k)].y;
        ++k;
      }
      if (v.x != 0.0 || v.y != 0.0) {
        c.col.push_back(col);
        c.val.push_back(v);
      }
    }
    c.ptr[static_cast<std::size_t>(i) + 1] = static_cast<int>(c.col.size());
  }
  return c;
}

}  // namespace detail

using namespace detail;

// The diagonal (diag = true) or off-diagonal entries of a multi-CSR, order kept.
MultiCsr filter_multi(const MultiCsr& m, bool diag) {
  MultiCsr f;
  f.n = m.n;
  f.ptr.assign(m.ptr.size(), 0);
  for (std::int64_t i = 0; i < m.n && !m.ptr.empty(); ++i) {
    for (int k = m.ptr[static_cast<std::size_t>(i)]; k < m.ptr[static_cast<std::size_t>(i) + 1]; ++k) {
      if ((m.col[static_cast<std::size_t>(k)] == i) != diag) continue;
      f.col.push_back(m.col[static_cast<std::size_t>(k)]);
      f.val.push_back(m.val[static_cast<std::size_t>(k)]);
    }
    f.ptr[static_cast<std::size_t>(i) + 1] = static_cast<int>(f.col.size());
  }
  return f;
}

// Operands of L = I(x)A + B(x)I + sum_k P_k(x)Q_k + T_diag + decay (kernels.hpp).
struct HostOperands {
  std::int64_t n = 0;
  MultiCsr a, b, t;
  std::vector<MultiCsr> p, q;
  std::vector<double> d_loc, d_ss;  // empty -> no decay term
  double omega = 0.0;
  // Every Hermitian X maps to a Hermitian L(X): true for the Lindblad form
  // whenever H (and H_rot) are exactly Hermitian.  The reference accepts H
  // within a tolerance and never checks H_rot (liouvillian.cpp:217-229), so
  // the Hermitian tile kernels are enabled only when this holds exactly.
  bool herm_preserving = true;
  // Factored dissipator of G-QSW for the matrix-free path: A = af, B = bf
  // (no L'L terms) and per Lindblad operator R_k = -w/2 L_k' (gathers in the
  // columns of W_k = L_k X), S_k = -w/2 L_k^T (streams the columns of
  // V_k = X L_k'), U_k = conj(L_k) (builds V_k from the columns of X).
  bool has_factored = false;
  MultiCsr af, bf;
  std::vector<MultiCsr> r, sfac, u;

  HostOperands transposed() const {
    HostOperands o;
    o.n = n;
    o.a = transpose_multi(a);
    o.b = transpose_multi(b);
    o.t = transpose_multi(t);
    for (const auto& x : p) o.p.push_back(transpose_multi(x));
    for (const auto& x : q) o.q.push_back(transpose_multi(x));
    o.d_loc = d_loc;
    o.d_ss = d_ss;
    o.omega = omega;
    o.herm_preserving = herm_preserving;
    return o;
  }

  HostOperands summed() const {
    HostOperands o = *this;
    o.a = canonical(a);
    o.b = canonical(b);
    o.t = canonical(t);
    if (has_factored) {
      o.af = canonical(af);
      o.bf = canonical(bf);
    }
    return o;
  }

  // Operand entries touched per output element (Kron kernels).
  // `herm`: one GPU, where Hermitian inputs read V_k as conj(W_k') from a
  // row-major copy of W_k instead of building it.
  double kron_cost(bool factored, bool herm = false) const {
    const double nn = static_cast<double>(n);
    auto e = [&](const MultiCsr& m) { return static_cast<double>(m.col.size()) / nn; };
    double c = 0.0;
    for (std::size_t k = 0; k < p.size(); ++k) c += e(p[k]) + e(q[k]);
    if (!factored) return c + e(a) + e(b);
    c += e(af) + e(bf);
    for (std::size_t k = 0; k < r.size(); ++k)
      c += e(r[k]) + e(sfac[k]) + (herm ? 1.0 : e(u[k]) + 2.0);  // + V_k pass, or the Wt_k store
    return c;
  }
};

// Device copy of HostOperands.
class DeviceOperands {
 public:
  DeviceOperands(const HostOperands& h, cudaStream_t s) {
    ops_.n = static_cast<int>(h.n);
    ops_.a = upload(h.a, s);
    ops_.b = upload(h.b, s);
    ops_.t = upload(h.t, s);
    ops_.nk = static_cast<int>(h.p.size());
    for (std::size_t k = 0; k < h.p.size(); ++k) {
      ops_.p[k] = upload(h.p[k], s, true);
      ops_.q[k] = upload(h.q[k], s, true);
    }
    if (!h.d_loc.empty()) {
      ops_.d_loc = upload_vec(h.d_loc, s);
      ops_.d_ss = upload_vec(h.d_ss, s);
    }
    ops_.omega = h.omega;
    QSWG_CHECK(cudaStreamSynchronize(s));
  }
  const dev::KronOperands& get() const { return ops_; }

 private:
  dev::KronList upload(const MultiCsr& m, cudaStream_t s, bool keep_empty = false) {
    if (m.empty() && !keep_empty) return {};
    dev::KronList l;
    l.ptr = upload_vec(m.ptr, s);
    l.col = m.col.empty() ? nullptr : upload_vec(m.col, s);
    l.val = m.val.empty() ? nullptr : upload_vec(m.val, s);
    return l;
  }
  template <class T>
  const T* upload_vec(const std::vector<T>& v, cudaStream_t s) {
    bufs_.emplace_back(v.size() * sizeof(T));
    QSWG_CHECK(cudaMemcpyAsync(bufs_.back().get(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return reinterpret_cast<const T*>(bufs_.back().get());
  }
  dev::KronOperands ops_;
  std::vector<DeviceBuffer<unsigned char>> bufs_;
};

// Sliced-ELL copy of a row-indexed operand (kernels.hpp: KronEll).
struct EllHost {
  std::vector<int> sptr, col;
  std::vector<double2> val;
};

// Every real row of every 32-row slice equally long: the sliced ELL holds no
// padding a kernel reads (the phantom lanes past n in the last slice are never
// addressed: columns are clamped to n - 1).
bool uniform_slices(const MultiCsr& m) {
  if (m.col.empty()) return false;
  for (std::int64_t s0 = 0; s0 < m.n; s0 += 32) {
    const int len0 = m.ptr[static_cast<std::size_t>(s0) + 1] - m.ptr[static_cast<std::size_t>(s0)];
    for (std::int64_t i = s0; i < std::min<std::int64_t>(m.n, s0 + 32); ++i)
      if (m.ptr[static_cast<std::size_t>(i) + 1] - m.ptr[static_cast<std::size_t>(i)] != len0) return false;
  }
  return true;
}

// The entry count every row of m has, or 0 when the rows differ (or m is
// empty).  The shuffled operand rows of the KRON kernels (KronView::a_len,
// q_len, r_len, s_len) take ONE length for the whole operand: slices that are
// uniform inside but differ from one another (a graph whose first 32 vertices
// have degree 2 and the next 32 degree 4) must not take that path.
int uniform_row_length(const MultiCsr& m) {
  if (m.col.empty() || m.ptr.size() < 2) return 0;
  const int len = m.ptr[1] - m.ptr[0];
  for (std::int64_t i = 0; i < m.n; ++i)
    if (m.ptr[static_cast<std::size_t>(i) + 1] - m.ptr[static_cast<std::size_t>(i)] != len) return 0;
  return len;
}

EllHost to_ell(const MultiCsr& m) {
  EllHost e;
  const std::int64_t ns = (m.n + 31) / 32;
  e.sptr.assign(static_cast<std::size_t>(ns) + 1, 0);
  for (std::int64_t sl = 0; sl < ns; ++sl) {
    int len = 0;
    for (std::int64_t i = sl * 32; i < std::min<std::int64_t>(m.n, sl * 32 + 32); ++i)
      len = std::max(len, m.ptr[static_cast<std::size_t>(i) + 1] - m.ptr[static_cast<std::size_t>(i)]);
    e.sptr[static_cast<std::size_t>(sl) + 1] = e.sptr[static_cast<std::size_t>(sl)] + 32 * len;
  }
  e.col.assign(static_cast<std::size_t>(e.sptr.back()), 0);
  e.val.assign(static_cast<std::size_t>(e.sptr.back()), make_double2(0.0, 0.0));
  for (std::int64_t sl = 0; sl < ns; ++sl) {
    const int len = (e.sptr[static_cast<std::size_t>(sl) + 1] - e.sptr[static_cast<std::size_t>(sl)]) / 32;
    for (int lane = 0; lane < 32; ++lane) {
      const std::int64_t i = sl * 32 + lane;
      const int b = i < m.n ? m.ptr[static_cast<std::size_t>(i)] : 0;
      const int cnt = i < m.n ? m.ptr[static_cast<std::size_t>(i) + 1] - b : 0;
      for (int k = 0; k < len; ++k) {
        const std::size_t at = static_cast<std::size_t>(e.sptr[static_cast<std::size_t>(sl)] + 32 * k + lane);
        if (k < cnt) {
          e.col[at] = m.col[static_cast<std::size_t>(b + k)];
          e.val[at] = m.val[static_cast<std::size_t>(b + k)];
        } else {
          e.col[at] = static_cast<int>(std::min<std::int64_t>(i, m.n - 1));  // padding: X(i, j) * 0
        }
      }
    }
  }
  return e;
}

// Device copy of the summed operands kept by a Kron-format Liouvillian.
// Splits the diagonal off a (summed) operand list: d[i] = m(i, i), 0 if absent.
MultiCsr strip_diagonal(const MultiCsr& m, std::vector<double2>& d) {
  MultiCsr o;
  o.n = m.n;
  d.assign(static_cast<std::size_t>(m.n), make_double2(0.0, 0.0));
  if (m.ptr.empty()) return o;
  o.ptr.assign(static_cast<std::size_t>(m.n) + 1, 0);
  for (std::int64_t i = 0; i < m.n; ++i) {
    for (int k = m.ptr[static_cast<std::size_t>(i)]; k < m.ptr[static_cast<std::size_t>(i) + 1]; ++k) {
      const auto uk = static_cast<std::size_t>(k);
      if (m.col[uk] == i) {
        d[static_cast<std::size_t>(i)].x += m.val[uk].x;
        d[static_cast<std::size_t>(i)].y += m.val[uk].y;
      } else {
        o.col.push_back(m.col[uk]);
        o.val.push_back(m.val[uk]);
      }
    }
    o.ptr[static_cast<std::size_t>(i) + 1] = static_cast<int>(o.col.size());
  }
  return o;
}

// Launch order of the upper tiles (I <= J) of the Hermitian KRON kernels.
// Concurrent blocks share L2: tile (I, J) gathers from row bands I and J of X
// and of the work vectors (and, on lattices, from bands a fixed offset away),
// so the order decides how much of x is re-read from HBM.
//   jmajor   J outer, I inner (columns J shared by blocks launched together)
//   blocked  B x B squares of tiles, J-major inside and between the squares:
//            the bands a wave touches shrink from all of them to ~2B
//   morton   Z-order of (I, J)
// QSWG_KRON_ORDER / QSWG_KRON_TILE_BLOCK override (experiments).
std::vector<int2> herm_tile_order(int nti) {
  std::string order = "jmajor";
  int bs = 16;
  if (const char* e = std::getenv("QSWG_KRON_ORDER")) order = e;
  if (const char* e = std::getenv("QSWG_KRON_TILE_BLOCK")) bs = std::max(1, std::atoi(e));
  std::vector<int2> tl;
  tl.reserve(static_cast<std::size_t>(nti) * (nti + 1) / 2);
  if (order == "blocked") {
    for (int J0 = 0; J0 < nti; J0 += bs)
      for (int I0 = 0; I0 <= J0; I0 += bs)
        for (int J = J0; J < std::min(nti, J0 + bs); ++J)
          for (int I = I0; I < std::min(J + 1, I0 + bs); ++I) tl.push_back(make_int2(I, J));
  } else if (order == "morton4") {  // tile index = q * D + r (lattice planes of D tiles): 4-D Z-order
    int D = 18;
    if (const char* e = std::getenv("QSWG_KRON_PERIOD")) D = std::max(1, std::atoi(e));
    std::vector<std::pair<std::uint64_t, int2>> keyed;
    for (int J = 0; J < nti; ++J)
      for (int I = 0; I <= J; ++I) {
        const unsigned c[4] = {static_cast<unsigned>(I % D), static_cast<unsigned>(I / D),
                               static_cast<unsigned>(J % D), static_cast<unsigned>(J / D)};
        std::uint64_t key = 0;
        for (int b = 0; b < 15; ++b)
          for (int d = 0; d < 4; ++d) key |= static_cast<std::uint64_t>((c[d] >> b) & 1u) << (4 * b + d);
        keyed.push_back({key, make_int2(I, J)});
      }
    std::sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& k : keyed) tl.push_back(k.second);
  } else if (order == "morton") {
    std::vector<std::pair<std::uint64_t, int2>> keyed;
    for (int J = 0; J < nti; ++J)
      for (int I = 0; I <= J; ++I) {
        std::uint64_t key = 0;
        for (int b = 0; b < 16; ++b)
          key |= (static_cast<std::uint64_t>((I >> b) & 1) << (2 * b)) |
                 (static_cast<std::uint64_t>((J >> b) & 1) << (2 * b + 1));
        keyed.push_back({key, make_int2(I, J)});
      }
    std::sort(keyed.begin(), keyed.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    for (const auto& k : keyed) tl.push_back(k.second);
  } else {
    for (int J = 0; J < nti; ++J)
      for (int I = 0; I <= J; ++I) tl.push_back(make_int2(I, J));
  }
  return tl;
}

// kernels.hpp: value classes.  A list with no entries is "real" (no term).
// With `cv`, kValConst is added when every entry equals one value (*cv).
int value_class(const std::vector<double2>& v, double2* cv = nullptr) {
  bool re = true, im = true, same = !v.empty();
  for (const double2& x : v) {
    re = re && x.y == 0.0;
    im = im && x.x == 0.0;
    same = same && x.x == v[0].x && x.y == v[0].y;
  }
  int k = re ? dev::kValReal : im ? dev::kValImag : dev::kValComplex;
  if (cv && same && k != dev::kValComplex) {
    *cv = v[0];
    k |= dev::kValConst;
  }
  return k;
}

// Whether b(j, c) = conj a(j, c) entry by entry (same pattern and order).
bool conj_pair(const MultiCsr& a, const MultiCsr& b) {
  if (a.ptr != b.ptr || a.col != b.col || a.val.size() != b.val.size() || a.col.empty()) return false;
  for (std::size_t k = 0; k < a.val.size(); ++k)
    if (!(b.val[k].x == a.val[k].x && b.val[k].y == -a.val[k].y)) return false;
  return true;
}

// Whether every entry of a lies on q's pattern (rows of both sorted by column).
bool pattern_within(const MultiCsr& a, const MultiCsr& q) {
  if (a.ptr.empty() || q.ptr.empty() || a.n != q.n) return false;
  for (std::int64_t i = 0; i < a.n; ++i) {
    int kq = q.ptr[static_cast<std::size_t>(i)];
    const int eq = q.ptr[static_cast<std::size_t>(i) + 1];
    for (int ka = a.ptr[static_cast<std::size_t>(i)]; ka < a.ptr[static_cast<std::size_t>(i) + 1]; ++ka) {
      while (kq < eq && q.col[static_cast<std::size_t>(kq)] < a.col[static_cast<std::size_t>(ka)]) ++kq;
      if (kq == eq || q.col[static_cast<std::size_t>(kq)] != a.col[static_cast<std::size_t>(ka)]) return false;
      ++kq;
    }
  }
  return true;
}

// q's pattern carrying a's values (0 where a has no entry); a within q.
MultiCsr aligned_values(const MultiCsr& a, const MultiCsr& q) {
  MultiCsr o = q;
  for (std::int64_t i = 0; i < q.n; ++i) {
    int ka = a.ptr[static_cast<std::size_t>(i)];
    const int ea = a.ptr[static_cast<std::size_t>(i) + 1];
    for (int kq = q.ptr[static_cast<std::size_t>(i)]; kq < q.ptr[static_cast<std::size_t>(i) + 1]; ++kq) {
      const bool hit = ka < ea && a.col[static_cast<std::size_t>(ka)] == q.col[static_cast<std::size_t>(kq)];
      o.val[static_cast<std::size_t>(kq)] = hit ? a.val[static_cast<std::size_t>(ka++)] : make_double2(0.0, 0.0);
    }
  }
  return o;
}

// Column offsets pre-multiplied by n (kernels.hpp: KronView), for the lists
// the kernels gather as base + c n: c n < n^2 = dim < 2^31.
MultiCsr scaled(const MultiCsr& m) {
  MultiCsr o = m;
  for (int& c : o.col) c *= static_cast<int>(m.n);
  return o;
}

// Staged tiles (kernels.hpp: KronView::staged).  For an operand m (rows r ->
// columns c) the column tiles c / 32 named by the rows of each 32-row tile T,
// in ascending order (nbr[T * kStageSlots + slot], -1 = none), and m with
// every column replaced by its element offset inside the staged region:
// (slot * 32 + c % 32) * 32 when the region holds rows c of the source
// (by_rows), slot * 1024 + c % 32 when it holds its columns c.
// false when some tile row names more than kStageSlots tiles.
bool localize(const MultiCsr& m, bool by_rows, std::vector<int>& nbr, MultiCsr& local, int& slots) {
  const std::int64_t nt = m.n / 32;
  if (m.ptr.empty() || m.col.empty()) return false;
  const int len = m.ptr[1] - m.ptr[0];  // one row length throughout (<= 8): slice s of the ELL copy starts at 32 s len
  if (len < 1 || len > 8) return false;
  for (std::int64_t r = 0; r < m.n; ++r)
    if (m.ptr[static_cast<std::size_t>(r) + 1] - m.ptr[static_cast<std::size_t>(r)] != len) return false;
  nbr.assign(static_cast<std::size_t>(nt) * dev::kStageSlots, -1);
  local = m;
  slots = 0;
  for (std::int64_t T = 0; T < nt; ++T) {
    std::vector<int> tiles;
    for (std::int64_t r = 32 * T; r < 32 * T + 32; ++r)
      for (int k = m.ptr[static_cast<std::size_t>(r)]; k < m.ptr[static_cast<std::size_t>(r) + 1]; ++k)
        tiles.push_back(m.col[static_cast<std::size_t>(k)] / 32);
    std::sort(tiles.begin(), tiles.end());
    tiles.erase(std::unique(tiles.begin(), tiles.end()), tiles.end());
    if (static_cast<int>(tiles.size()) > dev::kStageSlots) return false;
    slots = std::max(slots, static_cast<int>(tiles.size()));
    std::copy(tiles.begin(), tiles.end(), nbr.begin() + T * dev::kStageSlots);
    for (std::int64_t r = 32 * T; r < 32 * T + 32; ++r) {
      for (int k = m.ptr[static_cast<std::size_t>(r)]; k < m.ptr[static_cast<std::size_t>(r) + 1]; ++k) {
        const int c = m.col[static_cast<std::size_t>(k)];
        const int slot = static_cast<int>(std::lower_bound(tiles.begin(), tiles.end(), c / 32) - tiles.begin());
        local.col[static_cast<std::size_t>(k)] = by_rows ? (slot * 32 + c % 32) * 32 : slot * 1024 + c % 32;
      }
    }
  }
  return true;
}

struct KronStore {
  // Sliced ELL copies unless they store more than kEllMaxPadding x the
  // nonzeros; whether the kernels use them is autotuned per operator set at
  // build (ELL wins on lattices and on c3, CSR on c4's 2-hop rows).
  static constexpr double kEllMaxPadding = 2.0;
  KronStore(const HostOperands& h, bool single, cudaStream_t s) : host(h.summed()), ops(host, s) {
    // factor the L'L terms when that touches clearly fewer operand entries
    // (one GPU: c2 47.2 vs 47.8 ms per series factored, c4 factored either way)
    factored = host.has_factored && host.kron_cost(true, single) < (single ? 0.9 : 0.8) * host.kron_cost(false);
    if (const char* f = std::getenv("QSWG_KRON_FACTOR")) factored = host.has_factored && f[0] == '1';  // test knob
    // The diagonals of A and B both multiply X(i, j): the kernels apply them as
    // one coefficient (A_ii + B_jj) with one gather (c2: 22 -> 20 gathers per
    // element, exactly zero on regular graphs, then skipped; term 35.4 -> 33.9
    // us; with B transposed also c3 827 -> 812 ms, c5 term 2.93 -> 2.88 ms).
    // QSWG_KRON_DIAG=0 keeps them in the lists (experiment knob).
    const MultiCsr& a0 = factored ? host.af : host.a;
    const MultiCsr& b0 = factored ? host.bf : host.b;
    const char* dk = std::getenv("QSWG_KRON_DIAG");
    const bool split = !(dk && dk[0] == '0');
    if (!split) {
      a_list = upload_list(a0, s);
      a_sc = upload_list(scaled(a0), s);
      b_list = upload_list(scaled(b0), s);
      a = maybe_ell(a0, s);
      a_host = a0;
      b_host = b0;
    } else {
      std::vector<double2> dah, dbh;
      const MultiCsr a1 = strip_diagonal(a0, dah), b1 = strip_diagonal(b0, dbh);
      a_list = upload_list(a1, s);
      a_sc = upload_list(scaled(a1), s);
      b_list = upload_list(scaled(b1), s);
      a_host = a1;
      b_host = b1;
      a = maybe_ell(a1, s);
      // the merged coefficient A_ii + B_jj, as the kernels round it, vanishes for
      // every (i, j) exactly when diag(A) and diag(B) are constants a, b with
      // a + b == 0 (regular graphs: the coherent H_ii and -H_jj cancel); then
      // no term at all
      bool zero = true;
      for (std::size_t i = 0; i < dah.size() && zero; ++i)
        zero = dah[i].x + dbh[0].x == 0.0 && dah[i].y + dbh[0].y == 0.0 && dah[0].x + dbh[i].x == 0.0 &&
               dah[0].y + dbh[i].y == 0.0;
      if (!zero) {
        da = up(dah, s);
        db = up(dbh, s);
        std::vector<double2> both(dah);
        both.insert(both.end(), dbh.begin(), dbh.end());
        vk_d = value_class(both);
      }
    }
    for (const MultiCsr& qk : host.q) q.push_back(maybe_ell(qk, s));
    // P_k as padding-free sliced ELL (every row of a slice equally long, e.g. a
    // regular lattice): then the Hermitian tile kernels apply P_k in the
    // transposed section from the row-major W_k copy and the column-major copy
    // is not written at all (c2: W kernel 17.0 -> 14.9 us).
    p_rows = factored && single && !host.p.empty();
    for (const MultiCsr& pk : host.p) {
      const bool exact = uniform_slices(pk);
      p_rows = p_rows && exact;
      p_ell.push_back(exact ? upload_ell(to_ell(pk), s) : dev::KronEll{});
    }
    if (const char* pr = std::getenv("QSWG_KRON_PROWS")) p_rows = p_rows && pr[0] == '1';  // experiment knob
    // B likewise (lane = j, X(i, c) read as conj X(c, i) = conj x[n i + c]):
    // one operand load feeds the four rows of a thread.
    // (only after P in the per-element order A, R, P, B: B joins the transposed
    // section when P is there too or there is no P)
    // A (transposed, rows i warp-uniform): with uniform ELL slices of at most 8
    // entries, the four rows of a thread are consecutive lanes of one slice,
    // so a warp fetches all their column indices in one load and hands them
    // out by shuffle (the index -> gather chain starts without an L1 round trip).
    const char* ash = std::getenv("QSWG_KRON_ASHFL");  // experiment knob: 0 = no shuffled operand rows
    if (const int al = uniform_row_length(a_host); single && !(ash && ash[0] == '0') && al > 0 && al <= 8) {
      a_ellu = upload_ell(to_ell(scaled(a_host)), s);
      a_len = al;
    }
    for (std::size_t k = 0; k < host.q.size(); ++k) {  // Q_k, and R_k / S_k when factored
      const auto shfl = [&](const MultiCsr& m, dev::KronEll& e, int& len) {
        const int ul = uniform_row_length(m);
        if (!single || (ash && ash[0] == '0') || ul < 1 || ul > 8) return;
        e = upload_ell(to_ell(scaled(m)), s);
        len = ul;
      };
      dev::KronEll e;
      int len = 0;
      shfl(host.q[k], e, len);
      q_ellu.push_back(e);
      q_len.push_back(len);
      dev::KronEll er, es;
      int lr = 0, ls = 0;
      if (factored) {
        shfl(host.r[k], er, lr);
        shfl(host.sfac[k], es, ls);
      }
      r_ellu.push_back(er);
      r_len.push_back(lr);
      s_ellu.push_back(es);
      s_len.push_back(ls);
    }
    if (single && (p_rows || host.p.empty()) && uniform_slices(b_host)) {
      b_ell = upload_ell(to_ell(b_host), s);
      b_rows = true;
    }
    if (const char* br = std::getenv("QSWG_KRON_BROWS")) b_rows = b_rows && br[0] == '1';  // experiment knob
    vk_a = value_class(a_host.val, &cv_a);
    vk_b = value_class(b_host.val, &cv_b);
    vk_t = value_class(host.t.val);
    for (std::size_t k = 0; k < host.p.size(); ++k) {
      double2 c{};
      vk_p.push_back(value_class(host.p[k].val, &c));
      cv_p.push_back(c);
      vk_q.push_back(value_class(host.q[k].val, &c));
      cv_q.push_back(c);
      vk_r.push_back(factored ? value_class(host.r[k].val, &c) : dev::kValComplex);
      cv_r.push_back(c);
      vk_s.push_back(factored ? value_class(host.sfac[k].val, &c) : dev::kValComplex);
      cv_s.push_back(c);
      vk_u.push_back(factored ? value_class(host.u[k].val) : dev::kValComplex);
      p_sc.push_back(upload_list(scaled(host.p[k]), s));
      q_sc.push_back(upload_list(scaled(host.q[k]), s));
    }
    // AX from the gathers of W_0 (kernels.hpp: KronView::ax)
    ax = factored && single && host.q.size() == 1 && (vk_q[0] & 3) == dev::kValReal &&
         (vk_a & 3) == dev::kValImag && conj_pair(a_host, b_host) && pattern_within(a_host, host.q[0]);
    if (const char* e = std::getenv("QSWG_KRON_AX"); e && e[0] == '0') ax = false;  // experiment knob
    if (ax) {
      const MultiCsr aq = aligned_values(a_host, host.q[0]);  // Q_0's pattern, A's values (0 elsewhere)
      vk_aq = value_class(aq.val, &cv_aq);
      aq_sc_val = up(aq.val, s);
      if (q_len[0] > 0) aq_ellu_val = up(to_ell(aq).val, s);  // the layout of q_ellu[0]
    }
    // Staged Hermitian tiles (kernels.hpp: KronView::staged): a lattice-like
    // operand set on one GPU.  Factored G-QSW with one Lindblad operator and
    // the AX path (c2): R_0, P_0 and S_0 gather from Wt_0; L-QSW (c5): A and B
    // gather from x.  Opt-in (QSWG_KRON_STAGED=1): bit-identical to the global
    // gathers but measured slower — c2 term 27.7 us against 23.6 us, c5 2.92 ms
    // against 2.23 ms: with the one block per SM its 176 - 192 KB allow, a
    // tile costs ~340 KB of shared-memory reads and ~190 KB of copy writes
    // through the same 128 B/clk port.
    {
      const char* sk = std::getenv("QSWG_KRON_STAGED");
      const bool want = single && host.n % 32 == 0 && host.n >= 64 && sk && sk[0] == '1';
      std::vector<int> nb[3];
      MultiCsr lc[3];
      int sl[3] = {0, 0, 0};
      bool ok = false;
      if (want && factored && host.q.size() == 1 && ax && p_rows && r_len[0] > 0 && s_len[0] > 0) {
        ok = localize(host.r[0], true, nb[0], lc[0], sl[0]) && localize(host.p[0], false, nb[1], lc[1], sl[1]) &&
             localize(host.sfac[0], true, nb[2], lc[2], sl[2]);
      } else if (want && !factored && host.p.empty() && a_len > 0 && b_rows) {
        ok = localize(a_host, true, nb[0], lc[0], sl[0]) && localize(b_host, false, nb[1], lc[1], sl[1]);
      }
      // 16 KB per tile — the patterns' and AXt(I, J), AXt(J, I), x(I, J) — next to the kernel's static 18 KB
      if (ok && sl[0] + sl[1] + sl[2] + (factored ? 3 : 1) <= 12) {
        staged = true;
        for (int p3 = 0; p3 < 3; ++p3) {
          st_slots[p3] = sl[p3];
          if (sl[p3] == 0) continue;
          st_len[p3] = lc[p3].ptr[1] - lc[p3].ptr[0];
          st_nbr[p3] = up(nb[p3], s);
          st_col[p3] = up(to_ell(lc[p3]).col, s);
        }
      }
    }
    // a constant decay coefficient, as the kernels round it (kernels.hpp: d_const)
    if (!host.d_loc.empty()) {
      bool same = true;
      for (std::size_t i = 0; i < host.d_loc.size() && same; ++i)
        same = host.d_loc[i] == host.d_loc[0] && host.d_ss[i] == 0.0;
      if (same) {
        d_const = true;
        d_val = 0.5 * ((host.omega * (host.d_loc[0] + host.d_loc[0]) + 0.0) + 0.0);
      }
    }
    if (const char* vk = std::getenv("QSWG_KRON_VALCLASS"); vk && vk[0] == '0') {  // experiment knob: all complex
      vk_a = vk_b = vk_t = vk_d = dev::kValComplex;
      for (auto* v : {&vk_p, &vk_q, &vk_r, &vk_s, &vk_u}) std::fill(v->begin(), v->end(), dev::kValComplex);
      ax = false;
    } else if (vk && vk[0] == '1') {  // experiment knob: classes without the constant-value loads
      vk_a &= 3;
      vk_b &= 3;
      for (auto* v : {&vk_p, &vk_q, &vk_r, &vk_s, &vk_u})
        for (int& x : *v) x &= 3;
    }
    if (single) {  // the upper 32 x 32 tiles in launch order (kernels.hpp: KronTiles)
      const std::vector<int2> tl = herm_tile_order(static_cast<int>((host.n + 31) / 32));
      herm_tiles.resize(tl.size());
      QSWG_CHECK(cudaMemcpyAsync(herm_tiles.get(), tl.data(), tl.size() * sizeof(int2), cudaMemcpyHostToDevice, s));
    }
    if (factored) {
      af = upload_list(host.af, s);
      bf = upload_list(host.bf, s);
      for (std::size_t k = 0; k < host.r.size(); ++k) {
        r.push_back(upload_list(host.r[k], s));
        r_sc.push_back(upload_list(scaled(host.r[k]), s));
        sfac.push_back(upload_list(scaled(host.sfac[k]), s));
        u.push_back(upload_list(scaled(host.u[k]), s));
      }
    }
    QSWG_CHECK(cudaStreamSynchronize(s));
  }
  HostOperands host;
  DeviceOperands ops;  // CSR lists (B, P, T; and A, Q for on-demand assembly)
  dev::KronEll a;               // A without its diagonal, sliced ELL (or empty)
  dev::KronList a_list, b_list;  // A and B without their diagonals, CSR
  const double2* da = nullptr;   // diag(A), diag(B) (nullptr when both vanish)
  const double2* db = nullptr;
  std::vector<dev::KronEll> q;
  std::vector<dev::KronEll> p_ell;  // padding-free ELL copies of P_k (or empty)
  bool p_rows = false;              // Hermitian tiles apply P_k transposed (from Wt_k)
  MultiCsr a_host, b_host;          // A and B as the kernels apply them
  dev::KronEll a_ellu;              // uniform-slice ELL copy of A (or empty)
  int a_len = 0;                    // its row length (<= 8) when the shuffle path is on
  std::vector<dev::KronEll> q_ellu, r_ellu, s_ellu;  // the same for Q_k, R_k, S_k
  std::vector<int> q_len, r_len, s_len;
  dev::KronEll b_ell;               // padding-free ELL copy of B (or empty)
  bool b_rows = false;              // Hermitian tiles apply B transposed
  bool factored = false;
  int vk_a = dev::kValComplex, vk_b = dev::kValComplex, vk_t = dev::kValComplex, vk_d = dev::kValComplex;
  std::vector<int> vk_p, vk_q, vk_r, vk_s, vk_u;  // kernels.hpp: value classes
  double2 cv_a{}, cv_b{};
  std::vector<double2> cv_p, cv_q, cv_r, cv_s;
  DeviceBuffer<int2> herm_tiles;               // one GPU: upper tiles in launch order
  bool staged = false;                         // kernels.hpp: KronView::staged
  int st_slots[3] = {0, 0, 0};
  int st_len[3] = {0, 0, 0};
  const int* st_nbr[3] = {nullptr, nullptr, nullptr};
  const int* st_col[3] = {nullptr, nullptr, nullptr};
  bool ax = false;                             // kernels.hpp: KronView::ax
  bool d_const = false;                        // kernels.hpp: KronView::d_const
  double d_val = 0.0;
  int vk_aq = dev::kValComplex;
  double2 cv_aq{};
  const double2* aq_sc_val = nullptr;
  const double2* aq_ellu_val = nullptr;
  dev::KronList a_sc;                          // A (as a_list) with columns scaled by n
  std::vector<dev::KronList> p_sc, q_sc, r_sc;  // P_k, Q_k, R_k with columns scaled by n
  dev::KronList af, bf;
  std::vector<dev::KronList> r, sfac, u;

 private:
  dev::KronEll maybe_ell(const MultiCsr& m, cudaStream_t s) {
    if (m.col.empty()) return {};
    EllHost e = to_ell(m);
    if (static_cast<double>(e.col.size()) > kEllMaxPadding * static_cast<double>(m.col.size())) return {};
    return upload_ell(e, s);
  }
  dev::KronList upload_list(const MultiCsr& m, cudaStream_t s) {
    dev::KronList l;
    if (m.col.empty()) return l;
    l.ptr = up(m.ptr, s);
    l.col = up(m.col, s);
    l.val = up(m.val, s);
    return l;
  }
  dev::KronEll upload_ell(const EllHost& e, cudaStream_t s) {
    dev::KronEll d;
    if (e.col.empty()) return d;  // empty operand: no term
    d.sptr = up(e.sptr, s);
    d.col = up(e.col, s);
    d.val = up(e.val, s);
    return d;
  }
  template <class T>
  const T* up(const std::vector<T>& v, cudaStream_t s) {
    bufs_.emplace_back(v.size() * sizeof(T));
    QSWG_CHECK(cudaMemcpyAsync(bufs_.back().get(), v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return reinterpret_cast<const T*>(bufs_.back().get());
  }
  std::vector<DeviceBuffer<unsigned char>> bufs_;
};

namespace {

void validate_common(double omega, const SparseMatrix& h) {
  if (h.cols() != h.rows()) throw std::invalid_argument("Hamiltonian must be square");
  if (!(omega >= 0.0 && omega <= 1.0)) throw std::invalid_argument("omega must be in [0, 1]");
  if (!h.is_hermitian(hermiticity_tolerance(h))) throw std::invalid_argument("Hamiltonian must be Hermitian");
  if (h.rows() > kMaxVertices)
    throw std::invalid_argument("operator dimension " + std::to_string(h.rows()) +
                                " exceeds the int32 column range of the device CSR");
}

}  // namespace

// ------------------------------------------------------------------ builder
class LiouvillianBuilder {
 public:
  static std::unique_ptr<Liouvillian> build(double omega, std::int64_t n, const HostOperands& ops,
                                            const DeviceConfig& cfg,
                                            const std::vector<std::int64_t>* fixed_starts = nullptr);
  // Builds from operands(omega) and keeps the recipe for set_omega.
  template <class Ops>
  static std::unique_ptr<Liouvillian> with_rebuild(double omega, std::int64_t n, Ops operands, const DeviceConfig& cfg) {
    std::unique_ptr<Liouvillian> l = build(omega, n, operands(omega), cfg);
    l->rebuild_ = [n, operands = std::move(operands), cfg](double w, const std::vector<std::int64_t>* starts) {
      return build(w, n, operands(w), cfg, starts);
    };
    return l;
  }
};

void Liouvillian::adopt(Liouvillian& o) {
  DeviceGuard g(device_);
  QSWG_CHECK(cudaStreamSynchronize(stream_));
  std::swap(omega_, o.omega_);
  std::swap(group_, o.group_);
  std::swap(block_, o.block_);
  std::swap(starts_, o.starts_);
  std::swap(nnz_local_, o.nnz_local_);
  std::swap(nnz_total_, o.nnz_total_);
  std::swap(norms_, o.norms_);
  std::swap(format_, o.format_);
  std::swap(padding_, o.padding_);
  std::swap(n_slices_, o.n_slices_);
  std::swap(slice_ptr_, o.slice_ptr_);
  std::swap(perm_, o.perm_);
  std::swap(sigma_, o.sigma_);
  std::swap(pre_, o.pre_);
  std::swap(part_, o.part_);
  std::swap(sell_work_, o.sell_work_);
  std::swap(fused_, o.fused_);
  std::swap(main_c_lo_, o.main_c_lo_);
  std::swap(local_first_, o.local_first_);
  std::swap(rowptr_, o.rowptr_);
  std::swap(col_, o.col_);
  std::swap(val_, o.val_);
  std::swap(halo_lo_, o.halo_lo_);
  std::swap(halo_hi_, o.halo_hi_);
  std::swap(whalo_lo_, o.whalo_lo_);
  std::swap(whalo_hi_, o.whalo_hi_);
  std::swap(vhalo_lo_, o.vhalo_lo_);
  std::swap(vhalo_hi_, o.vhalo_hi_);
  std::swap(kron_, o.kron_);
  std::swap(kron_ell_, o.kron_ell_);
  std::swap(kron_w_, o.kron_w_);
  std::swap(kron_v_, o.kron_v_);
  std::swap(herm_flag_, o.herm_flag_);
  std::swap(kron_wt_, o.kron_wt_);
  std::swap(kron_axt_, o.kron_axt_);
  std::swap(ws_, o.ws_);  // drops captured series graphs and control blocks of the old operator
  herm_ = 0;
}

void Liouvillian::set_omega(double omega) {
  if (!(omega >= 0.0 && omega <= 1.0)) throw std::invalid_argument("omega must be in [0, 1]");
  if (!rebuild_) throw std::logic_error("this superoperator has no build inputs to re-mix");
  std::unique_ptr<Liouvillian> fresh = rebuild_(omega, &starts_);
  adopt(*fresh);
}

Liouvillian::~Liouvillian() {
  if (stream_) {
    DeviceGuard g(device_);
    cudaStreamSynchronize(stream_);
    rowptr_.reset();
    col_.reset();
    val_.reset();
    ws_ = Workspace{};
    if (side_) {
      cudaStreamSynchronize(side_);
      cudaStreamDestroy(side_);
      cudaEventDestroy(ev_[0]);
      cudaEventDestroy(ev_[1]);
    }
    cudaStreamDestroy(stream_);
  }
}

cudaStream_t Liouvillian::side_stream(cudaEvent_t* ev) const {
  if (!side_) {
    DeviceGuard g(device_);
    QSWG_CHECK(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
    QSWG_CHECK(cudaEventCreateWithFlags(&ev_[0], cudaEventDisableTiming));
    QSWG_CHECK(cudaEventCreateWithFlags(&ev_[1], cudaEventDisableTiming));
  }
  ev[0] = ev_[0];
  ev[1] = ev_[1];
  return side_;
}

dev::CsrView Liouvillian::view() const {
  dev::CsrView v;
  v.rowptr = rowptr_.get();
  v.col = col_.get();
  v.val = val_.get();
  v.rows = block_.rows;
  v.row0 = block_.row0;
  return v;
}

namespace {
std::vector<std::int64_t> count_scan(const dev::KronOperands& ops, std::int64_t n,
                                     DeviceBuffer<std::int64_t>& grp, cudaStream_t s);
template <class V>
void fill_block(const dev::KronOperands& ops, const DeviceBuffer<std::int64_t>& grp,
                const std::vector<std::int64_t>& colptr, std::int64_t n, const RowBlock& blk,
                DeviceBuffer<std::int64_t>& rowptr, DeviceBuffer<int>& col, DeviceBuffer<V>& val,
                std::int64_t& nnz, cudaStream_t s);
}  // namespace

bool Liouvillian::kron_factored() const { return kron_ != nullptr && kron_->factored; }
bool Liouvillian::kron_staged() const {
  return kron_ != nullptr && kron_->staged && herm_flag_.size() > 0 && (!kron_->factored || (kron_->ax && kron_axt_.get()));
}
// Factored: Wt_k only when P_k is applied transposed (one GPU), else W_k and
// Wt_k (one GPU) or W_k and V_k (row-partitioned); unfactored: W_k.
int Liouvillian::kron_term_vectors() const {
  if (!kron_) return 0;
  if (!kron_->factored) return 1;
  return kron_->p_rows && (comm_ == nullptr || comm_->world() == 1) ? 1 : 2;
}
int Liouvillian::kron_prepare_vectors() const { return kron_term_vectors(); }

dev::DevMatrix Liouvillian::matrix(int group_override) const {
  dev::DevMatrix m;
  m.format = format_;
  m.group = group_override ? group_override : group_;
  m.csr = view();
  m.sell.slice_ptr = slice_ptr_.get();
  m.sell.col = col_.get();
  m.sell.val = val_.get();
  m.sell.rows = block_.rows;
  m.sell.row0 = block_.row0;
  m.sell.n_slices = n_slices_;
  m.sell.perm = perm_.size() ? perm_.get() : nullptr;
  // Per panel: streamed (a scheduling counter in SellView::work) for unsorted panels with
  // short rows — a register-path warp drains its loads at every slice boundary (c5, 13 entries
  // per row: 0.84 of HBM against 0.96-0.99 streamed) — and the register path otherwise: long
  // rows keep it busy (c2, 41 per row: 0.94 at 3 blocks against 0.91 streamed), and sorted
  // (irregular) panels need its resident warps for their scattered gathers.
  const int stream = sell_stream_setting();
  const bool may_stream = format_ == dev::Format::Sell && sell_work_.size() && m.group != 1 && stream != 0;
  const auto wants_stream = [&](bool sorted, std::int64_t entries) {
    const double row_len = static_cast<double>(entries) / static_cast<double>(std::max<std::int64_t>(block_.rows, 1));
    return may_stream && (stream == 1 || (!sorted && row_len <= kStreamMaxRowLength));
  };
  std::int64_t pre_entries = 0;
  for (const SellPanel& pn : pre_) pre_entries += pn.entries;
  // (a panel with fused B (x) I arrays always takes the window path: they hold part of its entries)
  if (!fused_.b_val.size() &&
      wants_stream(perm_.size() > 0, static_cast<std::int64_t>(static_cast<double>(nnz_local_) * padding_) - pre_entries))
    m.sell.work = sell_work_.get() + pre_.size();
  if (fused_.b_val.size() && !m.sell.work) {  // fused B (x) I windows (one GPU, sorted rows)
    m.sell.b_slice_ptr = fused_.b_slice_ptr.get();
    m.sell.b_col = fused_.b_col.get();
    m.sell.b_val = fused_.b_val.get();
    m.sell.win_slices = dev::kSellWindowSlices;
    m.sell.win_work = sell_work_.get() + pre_.size();
  }
  if (!pre_.empty()) {  // column panels
    m.n_pre = static_cast<int>(pre_.size());
    for (std::size_t q = 0; q < pre_.size(); ++q) {
      dev::SellView& v = m.sell_pre[q];
      v = m.sell;
      v.work = !pre_[q].b_val.size() && wants_stream(pre_[q].perm.size() > 0, pre_[q].entries) ? sell_work_.get() + q
                                                                                                    : nullptr;
      v.slice_ptr = pre_[q].slice_ptr.get();
      v.col = pre_[q].col.get();
      v.val = pre_[q].val.get();
      v.perm = pre_[q].perm.size() ? pre_[q].perm.get() : nullptr;
      v.b_slice_ptr = pre_[q].b_val.size() && !v.work ? pre_[q].b_slice_ptr.get() : nullptr;
      v.b_col = v.b_slice_ptr ? pre_[q].b_col.get() : nullptr;
      v.b_val = v.b_slice_ptr ? pre_[q].b_val.get() : nullptr;
      v.win_slices = v.b_slice_ptr ? dev::kSellWindowSlices : 0;
      v.win_work = v.b_slice_ptr ? sell_work_.get() + q : nullptr;
    }
    m.part = part_.get();
    m.sell.part_in = part_.get();
    m.local_first = local_first_;
  }
  if (kron_) {
    const dev::KronOperands& o = kron_->ops.get();
    m.kron.n = static_cast<int>(n_);
    m.kron.rows = block_.rows;
    m.kron.row0 = block_.row0;
    m.kron.a_ell = kron_ell_ ? kron_->a : dev::KronEll{};
    m.kron.a = kron_->a_list;
    m.kron.b = kron_->b_list;
    m.kron.da = kron_->da;
    m.kron.db = kron_->db;
    m.kron.factored = kron_->factored ? 1 : 0;
    m.kron.t = o.t;
    m.kron.nk = o.nk;
    for (int k = 0; k < o.nk; ++k) {
      m.kron.q_ell[k] = kron_ell_ ? kron_->q[static_cast<std::size_t>(k)] : dev::KronEll{};
      m.kron.q[k] = o.q[k];
      if (kron_->factored) {
        m.kron.r[k] = kron_->r[static_cast<std::size_t>(k)];
        m.kron.s[k] = kron_->sfac[static_cast<std::size_t>(k)];
        m.kron.u[k] = kron_->u[static_cast<std::size_t>(k)];
        m.kron.v[k] = kron_v_[static_cast<std::size_t>(k)].get();
      }
      m.kron.w[k] = kron_w_[static_cast<std::size_t>(k)].get();
      if (kron_->p_rows) m.kron.p_ell[k] = kron_->p_ell[static_cast<std::size_t>(k)];
    }
    m.kron.cv_a = kron_->cv_a;
    m.kron.cv_b = kron_->cv_b;
    m.kron.a_sc = kron_->a_sc;
    for (std::size_t k = 0; k < kron_->cv_p.size(); ++k) {
      m.kron.cv_p[k] = kron_->cv_p[k];
      m.kron.cv_q[k] = kron_->cv_q[k];
      m.kron.cv_r[k] = kron_->cv_r[k];
      m.kron.cv_s[k] = kron_->cv_s[k];
      m.kron.p[k] = kron_->p_sc[k];
      m.kron.q_sc[k] = kron_->q_sc[k];
      if (kron_->factored) m.kron.r_sc[k] = kron_->r_sc[k];
    }
    {
      dev::KronTiles& tg = m.kron.tg;
      tg.nc = static_cast<int>(block_.rows / n_);
      tg.c0 = static_cast<int>(block_.row0 / n_);
      tg.nti = static_cast<int>((n_ + 31) / 32);
      tg.ntj = (tg.nc + 31) / 32;
      tg.ntiles = static_cast<long long>(tg.nti) * tg.ntj;
      tg.ntiles_herm = static_cast<long long>(tg.nti) * (tg.nti + 1) / 2;
      tg.herm_tiles = kron_->herm_tiles.get();
    }
    m.kron.vk_a = kron_->vk_a;
    m.kron.vk_b = kron_->vk_b;
    m.kron.vk_t = kron_->vk_t;
    m.kron.vk_d = kron_->vk_d;
    for (std::size_t k = 0; k < kron_->vk_p.size(); ++k) {
      m.kron.vk_p[k] = kron_->vk_p[k];
      m.kron.vk_q[k] = kron_->vk_q[k];
      m.kron.vk_r[k] = kron_->vk_r[k];
      m.kron.vk_s[k] = kron_->vk_s[k];
      m.kron.vk_u[k] = kron_->vk_u[k];
    }
    m.kron.p_rows = kron_->p_rows ? 1 : 0;
    m.kron.b_rows = kron_->b_rows ? 1 : 0;
    m.kron.a_len = kron_->a_len;
    m.kron.a_ellu = kron_->a_ellu;
    for (std::size_t k = 0; k < kron_->q_len.size(); ++k) {
      m.kron.q_len[k] = kron_->q_len[k];
      m.kron.q_ellu[k] = kron_->q_ellu[k];
      m.kron.r_len[k] = kron_->r_len[k];
      m.kron.r_ellu[k] = kron_->r_ellu[k];
      m.kron.s_len[k] = kron_->s_len[k];
      m.kron.s_ellu[k] = kron_->s_ellu[k];
    }
    m.kron.b_ell = kron_->b_rows ? kron_->b_ell : dev::KronEll{};
    m.kron.d_loc = o.d_loc;
    m.kron.d_ss = o.d_ss;
    m.kron.d_const = kron_->d_const ? 1 : 0;
    m.kron.d_val = kron_->d_val;
    m.kron.omega = o.omega;
    m.kron.herm_flag = herm_flag_.get();
    m.kron.herm = herm_;
    for (std::size_t k = 0; k < kron_wt_.size(); ++k) m.kron.wt[k] = kron_wt_[k].get();
    if (kron_->ax && kron_axt_.get()) {
      m.kron.ax = 1;
      m.kron.b_sep = 1;
      m.kron.axt = kron_axt_.get();
      m.kron.aq_ellu_val = kron_->aq_ellu_val;
      m.kron.aq_sc_val = kron_->aq_sc_val;
      m.kron.vk_aq = kron_->vk_aq;
      m.kron.cv_aq = kron_->cv_aq;
    }
    if (kron_->staged && (!kron_->factored || m.kron.ax)) {
      m.kron.staged = 1;
      for (int p = 0; p < 3; ++p) {
        m.kron.st_slots[p] = kron_->st_slots[p];
        m.kron.st_len[p] = kron_->st_len[p];
        m.kron.st_nbr[p] = kron_->st_nbr[p];
        m.kron.st_col[p] = kron_->st_col[p];
      }
    }
  }
  return m;
}

void Liouvillian::download(std::vector<std::int64_t>& rowptr, std::vector<std::int64_t>& col,
                           std::vector<Complex>& val) const {
  DeviceGuard g(device_);
  if (format_ == dev::Format::Kron) {
    // no superoperator is stored: assemble the block's CSR from the operands
    DeviceBuffer<std::int64_t> grp, rp;
    DeviceBuffer<int> cc;
    DeviceBuffer<double2> vv;
    std::int64_t nz = 0;
    const std::vector<std::int64_t> colptr = count_scan(kron_->ops.get(), n_, grp, stream_);
    fill_block(kron_->ops.get(), grp, colptr, n_, block_, rp, cc, vv, nz, stream_);
    rowptr.resize(static_cast<std::size_t>(block_.rows) + 1);
    std::vector<int> c32(static_cast<std::size_t>(nz));
    val.resize(static_cast<std::size_t>(nz));
    QSWG_CHECK(cudaMemcpy(rowptr.data(), rp.get(), rowptr.size() * sizeof(std::int64_t), cudaMemcpyDeviceToHost));
    if (nz) {
      QSWG_CHECK(cudaMemcpy(c32.data(), cc.get(), c32.size() * sizeof(int), cudaMemcpyDeviceToHost));
      QSWG_CHECK(cudaMemcpy(val.data(), vv.get(), val.size() * sizeof(double2), cudaMemcpyDeviceToHost));
    }
    col.assign(c32.begin(), c32.end());
    return;
  }
  if (format_ == dev::Format::Sell) {
    // de-pad: a row's genuine entries precede its padding (val == 0 exactly;
    // canonical entries are never zero); column panels hold increasing
    // column ranges, so a row is its panels' pieces in panel order
    struct View {
      const std::int64_t* sp;
      const int* perm;
      const int* col;
      const double2* val;
    };
    std::vector<std::pair<std::int64_t, View>> pv;  // (first column, panel), walked in column order
    for (const SellPanel& pn : pre_) {
      pv.push_back({pn.c_lo, {pn.slice_ptr.get(), pn.perm.size() ? pn.perm.get() : nullptr, pn.col.get(), pn.val.get()}});
      if (pn.b_val.size()) pv.push_back({pn.c_lo, {pn.b_slice_ptr.get(), nullptr, pn.b_col.get(), pn.b_val.get()}});
    }
    pv.push_back({main_c_lo_, {slice_ptr_.get(), perm_.size() ? perm_.get() : nullptr, col_.get(), val_.get()}});
    if (fused_.b_val.size())
      pv.push_back({main_c_lo_, {fused_.b_slice_ptr.get(), nullptr, fused_.b_col.get(), fused_.b_val.get()}});
    std::stable_sort(pv.begin(), pv.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
    std::vector<View> views;
    for (const auto& e : pv) views.push_back(e.second);
    const std::size_t rows = static_cast<std::size_t>(block_.rows);
    std::vector<std::vector<int>> rc(rows);
    std::vector<std::vector<Complex>> rv(rows);
    for (const View& w : views) {
      std::vector<std::int64_t> sp(static_cast<std::size_t>(n_slices_) + 1);
      QSWG_CHECK(cudaMemcpy(sp.data(), w.sp, sp.size() * sizeof(std::int64_t), cudaMemcpyDeviceToHost));
      const std::size_t total = static_cast<std::size_t>(sp.back());
      std::vector<int> c32(total);
      std::vector<Complex> v(total);
      if (total) {
        QSWG_CHECK(cudaMemcpy(c32.data(), w.col, total * sizeof(int), cudaMemcpyDeviceToHost));
        QSWG_CHECK(cudaMemcpy(v.data(), w.val, total * sizeof(double2), cudaMemcpyDeviceToHost));
      }
      std::vector<int> perm(rows);
      if (w.perm) {
        QSWG_CHECK(cudaMemcpy(perm.data(), w.perm, rows * sizeof(int), cudaMemcpyDeviceToHost));
      } else {
        for (std::size_t t = 0; t < rows; ++t) perm[t] = static_cast<int>(t);
      }
      for (std::size_t t = 0; t < rows; ++t) {  // slot t holds row perm[t]
        const std::size_t r = static_cast<std::size_t>(perm[t]);
        const std::size_t sl = t / dev::kSlice, lane = t % dev::kSlice;
        const std::int64_t len = (sp[sl + 1] - sp[sl]) / dev::kSlice;
        for (std::int64_t k = 0; k < len; ++k) {
          const std::size_t e = static_cast<std::size_t>(sp[sl] + k * dev::kSlice) + lane;
          if (v[e] == Complex{}) break;
          rc[r].push_back(c32[e]);
          rv[r].push_back(v[e]);
        }
      }
    }
    if (fused_.b_val.size()) {  // a row's B (x) I entries and its other entries are stored apart: back to column order
      for (std::size_t r = 0; r < rows; ++r) {
        std::vector<std::size_t> o(rc[r].size());
        std::iota(o.begin(), o.end(), std::size_t{0});
        std::stable_sort(o.begin(), o.end(), [&](std::size_t a, std::size_t b) { return rc[r][a] < rc[r][b]; });
        std::vector<int> c2(o.size());
        std::vector<Complex> v2(o.size());
        for (std::size_t k = 0; k < o.size(); ++k) {
          c2[k] = rc[r][o[k]];
          v2[k] = rv[r][o[k]];
        }
        rc[r].swap(c2);
        rv[r].swap(v2);
      }
    }
    rowptr.assign(rows + 1, 0);
    col.clear();
    val.clear();
    col.reserve(static_cast<std::size_t>(nnz_local_));
    val.reserve(static_cast<std::size_t>(nnz_local_));
    for (std::size_t r = 0; r < rows; ++r) {
      col.insert(col.end(), rc[r].begin(), rc[r].end());
      val.insert(val.end(), rv[r].begin(), rv[r].end());
      rowptr[r + 1] = static_cast<std::int64_t>(col.size());
    }
    return;
  }
  rowptr.resize(static_cast<std::size_t>(block_.rows) + 1);
  std::vector<int> c32(static_cast<std::size_t>(nnz_local_));
  val.resize(static_cast<std::size_t>(nnz_local_));
  QSWG_CHECK(cudaMemcpyAsync(rowptr.data(), rowptr_.get(), rowptr.size() * sizeof(std::int64_t),
                             cudaMemcpyDeviceToHost, stream_));
  if (nnz_local_) {
    QSWG_CHECK(cudaMemcpyAsync(c32.data(), col_.get(), c32.size() * sizeof(int), cudaMemcpyDeviceToHost, stream_));
    QSWG_CHECK(cudaMemcpyAsync(val.data(), val_.get(), val.size() * sizeof(double2), cudaMemcpyDeviceToHost, stream_));
  }
  QSWG_CHECK(cudaStreamSynchronize(stream_));
  col.assign(c32.begin(), c32.end());
}

void Liouvillian::multiply(const double2* x, double2* y, double scale) const {
  DeviceGuard g(device_);
  set_hermitian_input(x);
  dev::spmv(matrix(), x, y, scale, stream_);
}

int Liouvillian::hermitian_state(const double2* x) const {
  if (format_ != dev::Format::Kron || !herm_flag_.get()) return -1;
  DeviceGuard g(device_);
  return dev::kron_hermitian_check(matrix(), x, stream_) ? 1 : 0;
}

void Liouvillian::set_hermitian_input(const double2* x, int known) const {
  DeviceGuard g(device_);
  static const bool off = [] {
    const char* e = std::getenv("QSWG_KRON_HERM");  // experiment knob: 0 = always the general kernels
    return e != nullptr && e[0] == '0';
  }();
  if (off || !herm_mode_ || format_ != dev::Format::Kron || !herm_flag_.get()) {
    herm_ = 0;
    return;
  }
  herm_ = (known >= 0 ? known != 0 : dev::kron_hermitian_check(matrix(), x, stream_)) ? 1 : 0;
}

double Liouvillian::time_spmv(int iters, int group) const {
  DeviceGuard g(device_);
  DeviceBuffer<double2> x(static_cast<std::size_t>(dim())), y(static_cast<std::size_t>(std::max<std::int64_t>(block_.rows, 1)));
  if (std::getenv("QSWG_TIME_PATTERN") && format_ == dev::Format::Kron && herm_flag_.get())
    dev::fill_pattern_hermitian(x.get(), n_, stream_);  // experiment knob: density-matrix-like input
  else
    QSWG_CHECK(cudaMemsetAsync(x.get(), 0, x.bytes(), stream_));
  cudaEvent_t e0, e1;
  QSWG_CHECK(cudaEventCreate(&e0));
  QSWG_CHECK(cudaEventCreate(&e1));
  set_hermitian_input(x.get());  // x = 0 is Hermitian: the one-GPU Kron product runs in that mode
  const dev::DevMatrix m = matrix(group);
  dev::spmv(m, x.get(), y.get(), 1.0, stream_);  // warm-up
  QSWG_CHECK(cudaEventRecord(e0, stream_));
  for (int i = 0; i < iters; ++i) dev::spmv(m, x.get(), y.get(), 1.0, stream_);
  QSWG_CHECK(cudaEventRecord(e1, stream_));
  QSWG_CHECK(cudaEventSynchronize(e1));
  float ms = 0.f;
  QSWG_CHECK(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  return static_cast<double>(ms) / iters;
}

namespace {

// Counts every row of the operator described by `ops` and scans them into a
// global int64 row pointer on the device (all ranks do this, so they agree on
// the partition without communication).  Returns colptr[j] = rowptr[j*n],
// the nnz prefix at every rho-column boundary.
std::vector<std::int64_t> count_scan(const dev::KronOperands& ops, std::int64_t n,
                                     DeviceBuffer<std::int64_t>& grp, cudaStream_t s) {
  const std::int64_t dim = n * n;
  DeviceBuffer<std::int64_t> counts(static_cast<std::size_t>(dim) + 1);
  QSWG_CHECK(cudaMemsetAsync(counts.get(), 0, counts.bytes(), s));
  dev::assemble_count(ops, 0, dim, counts.get(), s);
  grp.resize(static_cast<std::size_t>(dim) + 1);
  std::size_t tmp_bytes = 0;
  dev::exclusive_scan(counts.get(), grp.get(), dim + 1, nullptr, tmp_bytes, s);
  DeviceBuffer<unsigned char> tmp(tmp_bytes);
  dev::exclusive_scan(counts.get(), grp.get(), dim + 1, tmp.get(), tmp_bytes, s);
  std::vector<std::int64_t> colptr(static_cast<std::size_t>(n) + 1);
  QSWG_CHECK(cudaMemcpy2DAsync(colptr.data(), sizeof(std::int64_t), grp.get(),
                               static_cast<std::size_t>(n) * sizeof(std::int64_t), sizeof(std::int64_t),
                               static_cast<std::size_t>(n) + 1, cudaMemcpyDeviceToHost, s));
  QSWG_CHECK(cudaStreamSynchronize(s));
  return colptr;
}

template <class V>
void fill_block(const dev::KronOperands& ops, const DeviceBuffer<std::int64_t>& grp,
                const std::vector<std::int64_t>& colptr, std::int64_t n, const RowBlock& blk,
                DeviceBuffer<std::int64_t>& rowptr, DeviceBuffer<int>& col, DeviceBuffer<V>& val,
                std::int64_t& nnz, cudaStream_t s) {
  const std::int64_t j0 = blk.row0 / n, j1 = (blk.row0 + blk.rows) / n;
  const std::int64_t base = colptr[static_cast<std::size_t>(j0)];
  nnz = colptr[static_cast<std::size_t>(j1)] - base;
  rowptr.resize(static_cast<std::size_t>(blk.rows) + 1);
  dev::rebase_rowptr(grp.get() + blk.row0, base, rowptr.get(), blk.rows + 1, s);
  col.resize(static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
  val.resize(static_cast<std::size_t>(std::max<std::int64_t>(nnz, 1)));
  if constexpr (std::is_same_v<V, double2>) {
    dev::assemble_fill(ops, blk.row0, blk.rows, rowptr.get(), col.get(), val.get(), s);
  } else {
    dev::assemble_fill_abs(ops, blk.row0, blk.rows, rowptr.get(), col.get(), val.get(), s);
  }
  QSWG_CHECK(cudaStreamSynchronize(s));
}

int heuristic_group(double mean_row) {
  if (mean_row <= 6) return 4;
  if (mean_row <= 20) return 8;
  if (mean_row <= 48) return 16;
  return 32;
}

}  // namespace

namespace {

// Halo tables of the Kron format, replicated on every rank from the (small,
// identical) operands: rank r reads X columns B(j, .) and T(j, .) and W_k
// columns P_k(j, .) for its own rho columns j; each peer's share is sent as
// the hull of whole columns.
void kron_halos(const HostOperands& h, bool factored, std::int64_t n, const std::vector<std::int64_t>& starts,
                std::vector<std::vector<std::int64_t>>& lo, std::vector<std::vector<std::int64_t>>& hi,
                std::vector<std::vector<std::int64_t>>& wlo, std::vector<std::vector<std::int64_t>>& whi,
                std::vector<std::vector<std::int64_t>>& vlo, std::vector<std::vector<std::int64_t>>& vhi) {
  const int world = static_cast<int>(starts.size()) - 1;
  const auto W = static_cast<std::size_t>(world);
  lo.assign(W, std::vector<std::int64_t>(W, 0));
  hi = lo;
  wlo = lo;
  whi = lo;
  vlo = lo;
  vhi = lo;
  if (world == 1) return;
  auto owner = [&](std::int64_t col) {
    int q = 0;
    while (q + 1 < world && starts[static_cast<std::size_t>(q) + 1] <= col * n) ++q;
    return q;
  };
  auto add = [&](std::vector<std::vector<std::int64_t>>& L, std::vector<std::vector<std::int64_t>>& H, int r,
                 std::int64_t col) {
    const int q = owner(col);
    if (q == r) return;
    auto& a = L[static_cast<std::size_t>(r)][static_cast<std::size_t>(q)];
    auto& b = H[static_cast<std::size_t>(r)][static_cast<std::size_t>(q)];
    if (a == b) {
      a = col * n;
      b = (col + 1) * n;
    } else {
      a = std::min(a, col * n);
      b = std::max(b, (col + 1) * n);
    }
  };
  auto row_cols = [](const MultiCsr& m, std::int64_t row, const std::function<void(std::int64_t)>& f) {
    if (m.ptr.empty()) return;
    for (int k = m.ptr[static_cast<std::size_t>(row)]; k < m.ptr[static_cast<std::size_t>(row) + 1]; ++k)
      f(m.col[static_cast<std::size_t>(k)]);
  };
  for (int r = 0; r < world; ++r) {
    for (std::int64_t j = starts[static_cast<std::size_t>(r)] / n; j < starts[static_cast<std::size_t>(r) + 1] / n; ++j) {
      row_cols(factored ? h.bf : h.b, j, [&](std::int64_t c) { add(lo, hi, r, c); });
      row_cols(h.t, j, [&](std::int64_t c) { add(lo, hi, r, c); });
      for (const MultiCsr& p : h.p) row_cols(p, j, [&](std::int64_t c) { add(wlo, whi, r, c); });
      if (factored) {
        for (const MultiCsr& u : h.u) row_cols(u, j, [&](std::int64_t c) { add(lo, hi, r, c); });  // V_k(:, j)
        for (const MultiCsr& sk : h.sfac) row_cols(sk, j, [&](std::int64_t c) { add(vlo, vhi, r, c); });
      }
    }
  }
}

}  // namespace

// Several GPUs, format "auto".  Row-partitioned, the
// matrix-free action loses the Hermitian halving and exchanges x plus the
// W_k (V_k) work vectors every term; the stored superoperator streams
// 20 B/nnz of its own rows and exchanges x only.  Per rank and term, from the
// one-GPU measurements:
//   KRON  operand entries per element (+ W's) * 16 B * rows / 7 TB/s (the L2
//         gather rate the KRON kernels reach on c2-c5), at least 1.5 us per
//         entry (the dependent gather chain of one tile), + (x, W_k, V_k halos) / 900 GB/s
//   SELL  (20 nnz + 48 rows) / (0.75 * 6.5 TB/s) (stored SpMV at 0.66-0.85 of
//         HBM), at least 60 us, + its x halo (the hull of x and W's) / 900 GB/s
// Every input is rank-independent (totals / world, the halo tables of all
// ranks), so every rank picks the same format; the stored copy must also fit
// (20 B/nnz per rank within 40% of the device memory).  QSWG_MULTI_FORMAT=kron /
// sell overrides.
bool stored_beats_kron(const HostOperands& hops, std::int64_t n, std::int64_t nnz_total,
                       const std::vector<std::int64_t>& starts) {
  const int world = static_cast<int>(starts.size()) - 1;
  if (const char* e = std::getenv("QSWG_MULTI_FORMAT")) return std::string(e) == "sell";
  const HostOperands h = hops.summed();
  const bool factored = h.has_factored && h.kron_cost(true, false) < 0.8 * h.kron_cost(false);
  std::vector<std::vector<std::int64_t>> lo, hi, wlo, whi, vlo, vhi;
  kron_halos(h, factored, n, starts, lo, hi, wlo, whi, vlo, vhi);
  double kron_halo = 0.0, sell_halo = 0.0;
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) {
      const auto R = static_cast<std::size_t>(r), Q = static_cast<std::size_t>(q);
      const double x = static_cast<double>(hi[R][Q] - lo[R][Q]), wv = static_cast<double>(whi[R][Q] - wlo[R][Q]);
      kron_halo += x + wv + static_cast<double>(vhi[R][Q] - vlo[R][Q]);
      const std::int64_t slo = std::min(lo[R][Q] == hi[R][Q] ? wlo[R][Q] : lo[R][Q], wlo[R][Q] == whi[R][Q] ? lo[R][Q] : wlo[R][Q]);
      const std::int64_t shi = std::max(hi[R][Q], whi[R][Q]);
      sell_halo += static_cast<double>(shi - slo);
    }
  const double w = static_cast<double>(world), rows = static_cast<double>(n) * static_cast<double>(n) / w;
  const double entries = h.kron_cost(factored, false);  // operand entries per output element
  // (a latency floor: a KRON term is at least one tile's dependent gather
  // chain, ~1.5 us per operand entry per element — c2 on one GPU, one wave)
  const double t_kron = std::max(entries * 16.0 * rows / 7e12, 1.5e-6 * entries) + 16.0 * kron_halo / w / 9e11;
  // (a floor as well: a sharded stored term with its panel and flush launches
  // took 62 us per rank on c2 at N = 8, profiles/r02_scaling_sell.jsonl)
  const double t_sell = std::max((20.0 * static_cast<double>(nnz_total) / w + 48.0 * rows) / (0.75 * 6.5e12), 60e-6) +
                        16.0 * sell_halo / w / 9e11;
  std::size_t free_b = 0, total_b = 0;
  cudaMemGetInfo(&free_b, &total_b);  // (the total: the same on every rank)
  const bool fits = 20.0 * static_cast<double>(nnz_total) / w < 0.4 * static_cast<double>(total_b);
  if (std::getenv("QSWG_DEBUG_FORMAT"))
    std::fprintf(stderr, "qswg: world %d: modelled term KRON %.1f us, stored %.1f us%s\n", world, 1e6 * t_kron,
                 1e6 * t_sell, fits ? "" : " (stored does not fit)");
  return fits && t_sell < t_kron;
}

std::unique_ptr<Liouvillian> LiouvillianBuilder::build(double omega, std::int64_t n, const HostOperands& hops,
                                                       const DeviceConfig& cfg,
                                                       const std::vector<std::int64_t>* fixed_starts) {
  {  // after the reference's argument validation (build_local / build_global), before any device work
    int count = 0;
    if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0) {
      cudaGetLastError();
      throw CudaError("no CUDA device available (qswg has no CPU fallback)");
    }
    if (cfg.device < 0 || cfg.device >= count) throw std::invalid_argument("CUDA device ordinal out of range");
  }
  std::unique_ptr<Liouvillian> l(new Liouvillian);
  l->n_ = n;
  l->omega_ = omega;
  l->device_ = cfg.device;
  l->comm_ = cfg.comm;
  DeviceGuard guard(cfg.device);
  QSWG_CHECK(cudaStreamCreateWithFlags(&l->stream_, cudaStreamNonBlocking));
  cudaStream_t s = l->stream_;
  const std::int64_t dim = n * n;
  const int world = cfg.comm ? cfg.comm->world() : 1;
  const int rank = cfg.comm ? cfg.comm->rank() : 0;

  DeviceOperands ops(hops, s);
  DeviceBuffer<std::int64_t> grp;
  const std::vector<std::int64_t> colptr = count_scan(ops.get(), n, grp, s);
  l->nnz_total_ = colptr.back();
  l->starts_ = fixed_starts ? *fixed_starts : partition_rows(colptr, n, world);
  l->block_ = {l->starts_[static_cast<std::size_t>(rank)],
               l->starts_[static_cast<std::size_t>(rank) + 1] - l->starts_[static_cast<std::size_t>(rank)]};

  // ---- 1-norm power series (liouvillian.cpp:309-344) ----
  if (dim <= kExactNormDimLimit) {
    // exact: every rank assembles the (small) full matrix
    DeviceBuffer<std::int64_t> rp;
    DeviceBuffer<int> cc;
    DeviceBuffer<double2> vv;
    std::int64_t nz = 0;
    fill_block(ops.get(), grp, colptr, n, RowBlock{0, dim}, rp, cc, vv, nz, s);
    dev::CsrView full{rp.get(), cc.get(), vv.get(), dim, 0};
    DeviceBuffer<double2> w0(static_cast<std::size_t>(dim * dim)), w1(static_cast<std::size_t>(dim * dim));
    DeviceBuffer<double> colsum(static_cast<std::size_t>(dim));
    dev::exact_norms(full, dim, w0.get(), w1.get(), colsum.get(), l->norms_.data(), s);
  } else {
    // bound: v <- |L|^T v from v = 1, over |L^T| assembled from transposed operands
    const HostOperands th = hops.transposed();
    DeviceOperands tops(th, s);
    DeviceBuffer<std::int64_t> tgrp;
    const std::vector<std::int64_t> tcolptr = count_scan(tops.get(), n, tgrp, s);
    DeviceBuffer<std::int64_t> rp;
    DeviceBuffer<int> cc;
    DeviceBuffer<double> vv;
    std::int64_t nz = 0;
    fill_block(tops.get(), tgrp, tcolptr, n, l->block_, rp, cc, vv, nz, s);
    tgrp.reset();
    dev::RealCsrView lt{rp.get(), cc.get(), vv.get(), l->block_.rows, l->block_.row0};
    DeviceBuffer<double> v(static_cast<std::size_t>(dim)), next(static_cast<std::size_t>(dim));
    DeviceBuffer<unsigned long long> mx(9);
    QSWG_CHECK(cudaMemsetAsync(mx.get(), 0, mx.bytes(), s));
    {
      std::vector<double> ones(static_cast<std::size_t>(dim), 1.0);
      QSWG_CHECK(cudaMemcpyAsync(v.get(), ones.data(), v.bytes(), cudaMemcpyHostToDevice, s));
      QSWG_CHECK(cudaStreamSynchronize(s));
    }
    for (int p = 0; p < 9; ++p) {
      dev::abs_transpose_product(lt, v.get(), next.get() + l->block_.row0, s);
      if (cfg.comm) cfg.comm->allgather_rows(next.get(), l->starts_, sizeof(double), s);
      dev::max_reduce(next.get(), dim, mx.get() + p, s);
      std::swap(v, next);
    }
    unsigned long long bits[9];
    QSWG_CHECK(cudaMemcpyAsync(bits, mx.get(), sizeof(bits), cudaMemcpyDeviceToHost, s));
    QSWG_CHECK(cudaStreamSynchronize(s));
    for (int p = 0; p < 9; ++p) std::memcpy(&l->norms_[static_cast<std::size_t>(p)], &bits[p], sizeof(double));
  }

  // ---- matrix-free Kronecker action: no superoperator stored ----
  // (the default: fewest bytes and fastest on every BASELINE config on one
  // GPU; the bitwise reference-order mode needs a stored superoperator; on
  // several GPUs a cost model may pick the stored one)
  if ((cfg.format == 3 || (cfg.format == 0 && dim > kKronMinDim && !(world > 1 && stored_beats_kron(hops, n, l->nnz_total_, l->starts_)))) &&
      cfg.group != 1) {
    const std::int64_t j0 = l->block_.row0 / n, j1 = (l->block_.row0 + l->block_.rows) / n;
    l->nnz_local_ = colptr[static_cast<std::size_t>(j1)] - colptr[static_cast<std::size_t>(j0)];
    l->format_ = dev::Format::Kron;
    l->kron_ = std::make_shared<KronStore>(hops, world == 1, s);
    for (std::size_t k = 0; k < hops.p.size(); ++k) {
      l->kron_w_.emplace_back(static_cast<std::size_t>(dim));
      QSWG_CHECK(cudaMemsetAsync(l->kron_w_.back().get(), 0, l->kron_w_.back().bytes(), s));
      if (l->kron_->factored) {
        l->kron_v_.emplace_back(static_cast<std::size_t>(dim));
        QSWG_CHECK(cudaMemsetAsync(l->kron_v_.back().get(), 0, l->kron_v_.back().bytes(), s));
      }
    }
    if (world == 1 && hops.herm_preserving) {
      l->herm_flag_.resize(1);
      QSWG_CHECK(cudaMemsetAsync(l->herm_flag_.get(), 0, sizeof(int), s));
      if (l->kron_->factored)
        for (std::size_t k = 0; k < hops.p.size(); ++k) l->kron_wt_.emplace_back(static_cast<std::size_t>(dim));
      if (l->kron_->ax) l->kron_axt_.resize(static_cast<std::size_t>(dim));
    }
    QSWG_CHECK(cudaStreamSynchronize(s));
    grp.reset();
    kron_halos(l->kron_->host, l->kron_->factored, n, l->starts_, l->halo_lo_, l->halo_hi_, l->whalo_lo_,
               l->whalo_hi_, l->vhalo_lo_, l->vhalo_hi_);
    l->group_ = 32;
    // sliced-ELL vs CSR row-indexed operands: time both (local products only)
    bool has_ell = l->kron_->a.sptr != nullptr;
    for (const auto& q : l->kron_->q) has_ell = has_ell || q.sptr != nullptr;
    l->kron_ell_ = has_ell;
    if (has_ell && dim >= (1 << 16)) {
      double t_ell = 1e300, t_csr = 1e300;
      for (int rep = 0; rep < 2; ++rep) {  // interleaved, best of two
        l->kron_ell_ = true;
        t_ell = std::min(t_ell, l->time_spmv(4, 32));
        l->kron_ell_ = false;
        t_csr = std::min(t_csr, l->time_spmv(4, 32));
      }
      l->kron_ell_ = t_ell <= t_csr;
    }
    return l;
  }

  // ---- the superoperator row block: SELL-32 when its padding is small ----
  {
    const std::int64_t j0 = l->block_.row0 / n, j1 = (l->block_.row0 + l->block_.rows) / n;
    l->nnz_local_ = colptr[static_cast<std::size_t>(j1)] - colptr[static_cast<std::size_t>(j0)];
  }
  l->n_slices_ = (l->block_.rows + dev::kSlice - 1) / dev::kSlice;
  std::int64_t sell_entries = 0;
  if (l->n_slices_ > 0) {
    DeviceBuffer<std::int64_t> se(static_cast<std::size_t>(l->n_slices_) + 1);
    l->slice_ptr_.resize(static_cast<std::size_t>(l->n_slices_) + 1);
    std::size_t tmp_bytes = 0;
    dev::exclusive_scan(se.get(), l->slice_ptr_.get(), l->n_slices_ + 1, nullptr, tmp_bytes, s);
    DeviceBuffer<unsigned char> tmp(tmp_bytes);
    const auto entries_for = [&](const int* perm) {
      QSWG_CHECK(cudaMemsetAsync(se.get(), 0, se.bytes(), s));
      dev::sell_slice_entries(grp.get() + l->block_.row0, l->block_.rows, perm, se.get(), s);
      dev::exclusive_scan(se.get(), l->slice_ptr_.get(), l->n_slices_ + 1, tmp.get(), tmp_bytes, s);
      std::int64_t e = 0;
      QSWG_CHECK(cudaMemcpyAsync(&e, l->slice_ptr_.get() + l->n_slices_, sizeof(std::int64_t),
                                 cudaMemcpyDeviceToHost, s));
      QSWG_CHECK(cudaStreamSynchronize(s));
      return e;
    };
    sell_entries = entries_for(nullptr);
    // SELL-C-sigma: sort rows by length inside windows of sigma rows when the
    // consecutive-row slices pad by more than kSellSortPadding
    const int sigma = sell_sigma_setting();
    if (sigma > dev::kSlice && l->nnz_local_ > 0 &&
        static_cast<double>(sell_entries) > kSellSortPadding * static_cast<double>(l->nnz_local_)) {
      l->perm_.resize(static_cast<std::size_t>(l->block_.rows));
      dev::sell_sort_rows(grp.get() + l->block_.row0, l->block_.rows, sigma, l->perm_.get(), s);
      const std::int64_t sorted = entries_for(l->perm_.get());
      if (sorted < sell_entries) {
        sell_entries = sorted;
        l->sigma_ = sigma;
      } else {
        l->perm_.reset();
        sell_entries = entries_for(nullptr);
      }
    }
  }
  const double pad = l->nnz_local_ ? static_cast<double>(sell_entries) / static_cast<double>(l->nnz_local_) : 1.0;
  const bool use_sell = l->nnz_local_ > 0 && (cfg.format == 2 || (cfg.format == 0 && pad <= kSellMaxPadding));
  if (cfg.format == 3) throw std::invalid_argument("the Kron format has no bitwise (group = 1) mode");
  // Column ranges of the panels.  One GPU: equal ranges when x outgrows L2
  // (sell_panel_count).  Row-partitioned (stored, non-bitwise): this rank's own
  // columns first — that panel needs no halo, so its partial sums run while the
  // halo of the next input is exchanged (Exec::exchange_overlap) — then the
  // columns before and after, in chunks of about kPanelX when x is large.
  std::vector<std::pair<std::int64_t, std::int64_t>> ranges;
  int local_first = 0;  // leading panels that cover this rank's own columns
  if (use_sell && world > 1 && cfg.group != 1) {
    const std::int64_t lo = l->block_.row0, hi = l->block_.row0 + l->block_.rows;
    const int per = std::max(1, sell_panel_count(cfg.group, n, l->perm_.size() > 0));
    std::int64_t chunk = std::max<std::int64_t>(n, (dim + per - 1) / per / n * n);  // whole rho columns
    do {  // (coarser chunks if the three runs would exceed the panel limit)
      ranges.clear();
      for (std::int64_t c = lo; c < hi; c += chunk) ranges.push_back({c, std::min(hi, c + chunk)});
      local_first = static_cast<int>(ranges.size());
      for (std::int64_t c = 0; c < lo; c += chunk) ranges.push_back({c, std::min(lo, c + chunk)});
      for (std::int64_t c = hi; c < dim; c += chunk) ranges.push_back({c, std::min(dim, c + chunk)});
      chunk *= 2;
    } while (static_cast<int>(ranges.size()) > dev::kMaxSellPanels);
  } else if (use_sell) {
    bool fuse_ok = world == 1 && cfg.group != 1 && l->perm_.size() > 0 && !hops.b.empty() && sell_fuse_setting(l->n_slices_);
    for (const MultiCsr& qk : hops.q)  // (the conditions of the fused B (x) I arrays below)
      for (std::int64_t i = 0; fuse_ok && i < qk.n; ++i)
        for (int k = qk.ptr[static_cast<std::size_t>(i)]; k < qk.ptr[static_cast<std::size_t>(i) + 1]; ++k)
          if (qk.col[static_cast<std::size_t>(k)] == i) fuse_ok = false;
    const int panels = sell_panel_count(cfg.group, n, l->perm_.size() > 0, fuse_ok);
    for (int q = 0; panels > 1 && q < panels; ++q)
      ranges.push_back({n * (static_cast<std::int64_t>(q) * n / panels), n * (static_cast<std::int64_t>(q + 1) * n / panels)});
  }
  // Fused B (x) I windows (one GPU, sigma-sorted rows; kernels.hpp: SellView::b_val).  The
  // B (x) I entries of row (i, j) sit at columns n c + i, c in row j of B: for the 32
  // consecutive rows of a natural-order slice they are the same list and their gathers one
  // coalesced 512-byte segment (4 L1 wavefronts) — until the sigma sort scatters the rows of a
  // slice, after which every lane's gather is its own 32-byte sector and wavefront, the bound
  // of the irregular configs (about one sector per clock and SM).  So every panel keeps those
  // entries in a second, natural-order sliced ELL (no padding inside a rho column: every row
  // has row j's count) and sorts only the rest, inside windows of kSellWindowSlices slices
  // whose natural-order sums a block holds in shared memory.  B's diagonal stays with the
  // rest (it shares its position with A's diagonal), and every Q_k must be diagonal-free so
  // that no position is stored twice.
  bool fuse = use_sell && world == 1 && cfg.group != 1 && l->perm_.size() > 0 && !hops.b.empty() && sell_fuse_setting(l->n_slices_);
  for (const MultiCsr& qk : hops.q)
    for (std::int64_t i = 0; fuse && i < qk.n; ++i)
      for (int k = qk.ptr[static_cast<std::size_t>(i)]; k < qk.ptr[static_cast<std::size_t>(i) + 1]; ++k)
        if (qk.col[static_cast<std::size_t>(k)] == i) fuse = false;
  std::unique_ptr<DeviceOperands> ops_boff, ops_rest;
  if (fuse) {
    HostOperands hb;
    hb.n = hops.n;
    hb.omega = hops.omega;
    hb.b = filter_multi(hops.b, false);
    HostOperands hr = hops;
    hr.b = filter_multi(hops.b, true);
    fuse = !hb.b.col.empty();
    if (fuse) {
      ops_boff = std::make_unique<DeviceOperands>(hb, s);
      ops_rest = std::make_unique<DeviceOperands>(hr, s);
      if (ranges.size() < 2) ranges.assign(1, {0, dim});
      l->sigma_ = dev::kSellWindowSlices * dev::kSlice;
    }
  }
  const int panels = ranges.size() > 1 ? static_cast<int>(ranges.size()) : 1;
  std::int64_t main_entries = 0;
  l->local_first_ = panels > 1 ? std::min(local_first, panels - 1) : 0;
  if (use_sell && (panels > 1 || fuse)) {
    // ---- column panels: x slices that stay in L2 while their entries stream ----
    l->format_ = dev::Format::Sell;
    const std::int64_t rows = l->block_.rows;
    DeviceBuffer<std::int64_t> cnt(static_cast<std::size_t>(rows) + 1), g(static_cast<std::size_t>(rows) + 1);
    DeviceBuffer<std::int64_t> se(static_cast<std::size_t>(l->n_slices_) + 1);
    std::size_t tmp_bytes = 0;
    dev::exclusive_scan(cnt.get(), g.get(), std::max(rows + 1, l->n_slices_ + 1), nullptr, tmp_bytes, s);
    DeviceBuffer<unsigned char> tmp(tmp_bytes);
    std::int64_t stored = 0;
    l->pre_.clear();
    for (int q = 0; q < panels; ++q) {
      SellPanel pn;
      pn.c_lo = ranges[static_cast<std::size_t>(q)].first;
      pn.c_hi = ranges[static_cast<std::size_t>(q)].second;
      const dev::KronOperands& po = fuse ? ops_rest->get() : ops.get();
      if (fuse) {  // the B (x) I entries of this column range: natural row order, no permutation
        QSWG_CHECK(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
        dev::assemble_count(ops_boff->get(), l->block_.row0, rows, cnt.get(), s, pn.c_lo, pn.c_hi);
        dev::exclusive_scan(cnt.get(), g.get(), rows + 1, tmp.get(), tmp_bytes, s);
        QSWG_CHECK(cudaMemsetAsync(se.get(), 0, se.bytes(), s));
        dev::sell_slice_entries(g.get(), rows, nullptr, se.get(), s);
        pn.b_slice_ptr.resize(static_cast<std::size_t>(l->n_slices_) + 1);
        dev::exclusive_scan(se.get(), pn.b_slice_ptr.get(), l->n_slices_ + 1, tmp.get(), tmp_bytes, s);
        std::int64_t eb = 0;
        QSWG_CHECK(cudaMemcpyAsync(&eb, pn.b_slice_ptr.get() + l->n_slices_, sizeof(std::int64_t), cudaMemcpyDeviceToHost, s));
        QSWG_CHECK(cudaStreamSynchronize(s));
        stored += eb;
        pn.b_col.resize(static_cast<std::size_t>(std::max<std::int64_t>(eb, 1)));
        pn.b_val.resize(static_cast<std::size_t>(std::max<std::int64_t>(eb, 1)));
        dev::assemble_fill_sell(ops_boff->get(), l->block_.row0, rows, pn.b_slice_ptr.get(), nullptr, pn.b_col.get(),
                                pn.b_val.get(), s, pn.c_lo, pn.c_hi);
      }
      QSWG_CHECK(cudaMemsetAsync(cnt.get(), 0, cnt.bytes(), s));
      dev::assemble_count(po, l->block_.row0, rows, cnt.get(), s, pn.c_lo, pn.c_hi);
      dev::exclusive_scan(cnt.get(), g.get(), rows + 1, tmp.get(), tmp_bytes, s);
      if (l->sigma_ > dev::kSlice) {
        pn.perm.resize(static_cast<std::size_t>(rows));
        dev::sell_sort_rows(g.get(), rows, l->sigma_, pn.perm.get(), s);
      }
      QSWG_CHECK(cudaMemsetAsync(se.get(), 0, se.bytes(), s));
      dev::sell_slice_entries(g.get(), rows, pn.perm.size() ? pn.perm.get() : nullptr, se.get(), s);
      pn.slice_ptr.resize(static_cast<std::size_t>(l->n_slices_) + 1);
      dev::exclusive_scan(se.get(), pn.slice_ptr.get(), l->n_slices_ + 1, tmp.get(), tmp_bytes, s);
      std::int64_t e = 0;
      QSWG_CHECK(cudaMemcpyAsync(&e, pn.slice_ptr.get() + l->n_slices_, sizeof(std::int64_t), cudaMemcpyDeviceToHost, s));
      QSWG_CHECK(cudaStreamSynchronize(s));
      stored += e;
      pn.entries = e;
      pn.col.resize(static_cast<std::size_t>(std::max<std::int64_t>(e, 1)));
      pn.val.resize(static_cast<std::size_t>(std::max<std::int64_t>(e, 1)));
      dev::assemble_fill_sell(po, l->block_.row0, rows, pn.slice_ptr.get(),
                              pn.perm.size() ? pn.perm.get() : nullptr, pn.col.get(), pn.val.get(), s, pn.c_lo,
                              pn.c_hi);
      QSWG_CHECK(cudaStreamSynchronize(s));
      if (q + 1 < panels) {
        l->pre_.push_back(std::move(pn));
      } else {  // the last panel lives in the main arrays (its kernel runs the epilogue)
        l->slice_ptr_ = std::move(pn.slice_ptr);
        l->perm_ = std::move(pn.perm);
        l->col_ = std::move(pn.col);
        l->val_ = std::move(pn.val);
        l->main_c_lo_ = pn.c_lo;
        main_entries = e;
        l->fused_.b_slice_ptr = std::move(pn.b_slice_ptr);
        l->fused_.b_col = std::move(pn.b_col);
        l->fused_.b_val = std::move(pn.b_val);
      }
    }
    l->part_.resize(static_cast<std::size_t>(std::max<std::int64_t>(rows, 1)));
    l->sell_work_.resize(dev::kMaxSellPanels);  // scheduling counters of the streamed kernels, one per panel
    QSWG_CHECK(cudaMemsetAsync(l->sell_work_.get(), 0, l->sell_work_.bytes(), s));
    QSWG_CHECK(cudaStreamSynchronize(s));
    l->padding_ = static_cast<double>(stored) / static_cast<double>(l->nnz_local_);
    sell_entries = main_entries;  // the halo hull below walks the earlier panels separately
  } else if (use_sell) {
    l->format_ = dev::Format::Sell;
    l->padding_ = pad;
    l->sell_work_.resize(dev::kMaxSellPanels);
    QSWG_CHECK(cudaMemsetAsync(l->sell_work_.get(), 0, l->sell_work_.bytes(), s));
    l->col_.resize(static_cast<std::size_t>(std::max<std::int64_t>(sell_entries, 1)));
    l->val_.resize(static_cast<std::size_t>(std::max<std::int64_t>(sell_entries, 1)));
    dev::assemble_fill_sell(ops.get(), l->block_.row0, l->block_.rows, l->slice_ptr_.get(),
                            l->perm_.size() ? l->perm_.get() : nullptr, l->col_.get(), l->val_.get(), s);
    QSWG_CHECK(cudaStreamSynchronize(s));
  } else {
    l->slice_ptr_.reset();
    l->perm_.reset();
    l->sigma_ = dev::kSlice;
    l->format_ = dev::Format::Csr;
    fill_block(ops.get(), grp, colptr, n, l->block_, l->rowptr_, l->col_, l->val_, l->nnz_local_, s);
  }
  grp.reset();

  // ---- halo plan: hull of every peer's columns this block references ----
  l->halo_lo_.assign(static_cast<std::size_t>(world), std::vector<std::int64_t>(static_cast<std::size_t>(world), 0));
  l->halo_hi_ = l->halo_lo_;
  if (world > 1) {
    const std::int64_t stored = l->format_ == dev::Format::Sell ? sell_entries : l->nnz_local_;
    DeviceBuffer<std::int64_t> dstarts(static_cast<std::size_t>(world) + 1);
    DeviceBuffer<std::int64_t> table(static_cast<std::size_t>(2 * world * world));  // [rank][lo.., hi..]
    QSWG_CHECK(cudaMemcpyAsync(dstarts.get(), l->starts_.data(), dstarts.bytes(), cudaMemcpyHostToDevice, s));
    std::vector<std::int64_t> init(static_cast<std::size_t>(2 * world));
    for (int q = 0; q < world; ++q) {
      init[static_cast<std::size_t>(q)] = INT64_MAX;
      init[static_cast<std::size_t>(world + q)] = INT64_MIN;
    }
    std::int64_t* mine = table.get() + 2 * world * rank;
    QSWG_CHECK(cudaMemcpyAsync(mine, init.data(), init.size() * sizeof(std::int64_t), cudaMemcpyHostToDevice, s));
    dev::halo_hulls(l->col_.get(), stored, dstarts.get(), world, rank, mine, mine + world, s);
    for (const SellPanel& pn : l->pre_)  // column panels: every panel's columns
      dev::halo_hulls(pn.col.get(), pn.entries, dstarts.get(), world, rank, mine, mine + world, s);
    std::vector<std::int64_t> tstarts(static_cast<std::size_t>(world) + 1);
    for (int w = 0; w <= world; ++w) tstarts[static_cast<std::size_t>(w)] = 2 * world * w;
    cfg.comm->allgather_rows(table.get(), tstarts, sizeof(std::int64_t), s);
    std::vector<std::int64_t> h(table.size());
    QSWG_CHECK(cudaMemcpyAsync(h.data(), table.get(), table.bytes(), cudaMemcpyDeviceToHost, s));
    QSWG_CHECK(cudaStreamSynchronize(s));
    for (int r = 0; r < world; ++r)
      for (int q = 0; q < world; ++q) {
        const std::int64_t lo = h[static_cast<std::size_t>(2 * world * r + q)];
        const std::int64_t hi = h[static_cast<std::size_t>(2 * world * r + world + q)];
        if (lo < hi) {
          l->halo_lo_[static_cast<std::size_t>(r)][static_cast<std::size_t>(q)] = lo;
          l->halo_hi_[static_cast<std::size_t>(r)][static_cast<std::size_t>(q)] = hi;
        }
      }
  }

  // ---- SpMV lanes per row ----
  const double mean_row = l->block_.rows ? static_cast<double>(l->nnz_local_) / l->block_.rows : 1.0;
  if (cfg.group) {
    if (!dev::valid_group(cfg.group)) throw std::invalid_argument("group must be 1, 2, 4, 8, 16 or 32");
    l->group_ = cfg.group;
  } else if (l->format_ == dev::Format::Sell) {
    l->group_ = 32;  // lane per row; `group` only distinguishes the bitwise mode (1)
  } else if (l->nnz_local_ < (1 << 22)) {
    l->group_ = heuristic_group(mean_row);
  } else {
    double best = 1e300;
    for (int g : {4, 8, 16, 32}) {
      if (g > 4 * mean_row + 4) continue;
      const double t = l->time_spmv(3, g);
      if (t < best) {
        best = t;
        l->group_ = g;
      }
    }
  }
  return l;
}

// ------------------------------------------------------------ build_local
std::unique_ptr<Liouvillian> build_local(double omega, const SparseMatrix& h, const SparseMatrix& m_l,
                                         const std::vector<SourceArc>& sources,
                                         const std::vector<SinkArc>& sinks, const DeviceConfig& cfg) {
  // validation: liouvillian.cpp:133-151
  const std::int64_t n = h.rows();
  if (h.cols() != n) throw std::invalid_argument("Hamiltonian must be square");
  if (m_l.rows() != n || m_l.cols() != n)
    throw std::invalid_argument("condensed Lindblad matrix dimension mismatch");
  validate_common(omega, h);
  const std::int64_t nsrc = static_cast<std::int64_t>(sources.size());
  const std::int64_t nsnk = static_cast<std::int64_t>(sinks.size());
  if (n < nsrc + nsnk) throw std::invalid_argument("operator dimension smaller than the augmentation");
  const std::int64_t n_base = n - nsrc - nsnk;
  for (const SourceArc& s : sources)
    if (s.target < 0 || s.target >= n_base) throw std::out_of_range("source target out of range");
  for (const SinkArc& s : sinks)
    if (s.origin < 0 || s.origin >= n_base) throw std::out_of_range("sink origin out of range");

  const bool exact_herm = h.is_hermitian(0.0);
  auto operands = [n, n_base, nsrc, nsnk, h, m_l, sources, sinks, exact_herm](double omega) {
  HostOperands o;
  o.n = n;
  o.herm_preserving = exact_herm;
  o.omega = omega;
  const Complex coh{0.0, -(1.0 - omega)};
  const SparseMatrix ht = h.transpose();
  if (coh != Complex{}) {
    o.a = from_sparse(h, [&](Complex v) { return coh * v; });    // -i(1-w) I(x)H
    o.b = from_sparse(ht, [&](Complex v) { return -coh * v; });  // +i(1-w) H^T(x)I
  } else {
    o.a = make_multi(n, {});
    o.b = make_multi(n, {});
  }
  // decay: d = column sums of |m_l|^2 (liouvillian.cpp:19-26), d_ss from rates
  o.d_loc.assign(static_cast<std::size_t>(n), 0.0);
  for (std::int64_t k = 0; k < m_l.nnz(); ++k)
    o.d_loc[static_cast<std::size_t>(m_l.col_indices()[static_cast<std::size_t>(k)])] += std::norm(m_l.values()[static_cast<std::size_t>(k)]);
  o.d_ss.assign(static_cast<std::size_t>(n), 0.0);
  for (std::int64_t k = 0; k < nsrc; ++k) o.d_ss[static_cast<std::size_t>(n_base + k)] += sources[static_cast<std::size_t>(k)].rate;
  for (const SinkArc& s : sinks) o.d_ss[static_cast<std::size_t>(s.origin)] += s.rate;
  // transfer onto the vec diagonal (liouvillian.cpp:185-206), emission order
  std::vector<Entry> te;
  if (omega != 0.0) append_entries(te, m_l, [&](Complex v) { return Complex{omega * std::norm(v), 0.0}; });
  for (std::int64_t k = 0; k < nsrc; ++k) {
    const std::int64_t u = n_base + k;
    te.push_back({sources[static_cast<std::size_t>(k)].target, u, Complex{sources[static_cast<std::size_t>(k)].rate, 0.0}});
  }
  for (std::int64_t k = 0; k < nsnk; ++k)
    te.push_back({n_base + nsrc + k, sinks[static_cast<std::size_t>(k)].origin, Complex{sinks[static_cast<std::size_t>(k)].rate, 0.0}});
  o.t = make_multi(n, te);
  return o;
  };
  return LiouvillianBuilder::with_rebuild(omega, n, std::move(operands), cfg);
}

// ----------------------------------------------------------- build_global
std::unique_ptr<Liouvillian> build_global(double omega, const SparseMatrix& h,
                                          const std::vector<SparseMatrix>& lindblads,
                                          const std::optional<SparseMatrix>& h_rot,
                                          const DeviceConfig& cfg) {
  // validation: liouvillian.cpp:216-229
  const std::int64_t n = h.rows();
  validate_common(omega, h);
  for (const SparseMatrix& l : lindblads)
    if (l.rows() != n || l.cols() != n) throw std::invalid_argument("Lindblad operator dimension mismatch");
  if (h_rot && (h_rot->rows() != n || h_rot->cols() != n))
    throw std::invalid_argument("rotating Hamiltonian dimension mismatch");
  if (static_cast<int>(lindblads.size()) > dev::kMaxKron)
    throw std::invalid_argument("at most " + std::to_string(dev::kMaxKron) + " Lindblad operators are supported");

  const bool exact_herm = h.is_hermitian(0.0) && (!h_rot || h_rot->is_hermitian(0.0));
  auto operands = [n, h, lindblads, h_rot, exact_herm](double omega) {
  HostOperands o;
  o.n = n;
  o.omega = omega;
  o.herm_preserving = exact_herm;
  const Complex coh{0.0, -(1.0 - omega)};
  const Complex rot{0.0, omega};
  const SparseMatrix ht = h.transpose();
  std::vector<Entry> ae, be;
  if (coh != Complex{}) {
    append_entries(ae, h, [&](Complex v) { return coh * v; });
    append_entries(be, ht, [&](Complex v) { return -coh * v; });
  }
  if (h_rot && rot != Complex{}) {
    append_entries(ae, *h_rot, [&](Complex v) { return rot * v; });
    append_entries(be, h_rot->transpose(), [&](Complex v) { return -rot * v; });
  }
  o.af = make_multi(n, ae);  // coherent parts only (before the L'L terms)
  o.bf = make_multi(n, be);
  o.has_factored = omega != 0.0 && !lindblads.empty();
  if (o.has_factored) {
    for (const SparseMatrix& l : lindblads) {
      o.r.push_back(from_sparse(l.conjugate_transpose(), [&](Complex v) { return -0.5 * omega * v; }));
      o.sfac.push_back(from_sparse(l.transpose(), [&](Complex v) { return -0.5 * omega * v; }));
      o.u.push_back(from_sparse(l, [](Complex v) { return std::conj(v); }));
    }
  }
  if (omega != 0.0) {
    for (const SparseMatrix& l : lindblads) {
      const SparseMatrix ll = l.conjugate_transpose() * l;  // liouvillian.cpp:236-242
      append_entries(ae, ll, [&](Complex v) { return -0.5 * omega * v; });
      append_entries(be, ll.transpose(), [&](Complex v) { return -0.5 * omega * v; });
      o.p.push_back(from_sparse(l, [&](Complex v) { return omega * std::conj(v); }));  // w L*
      o.q.push_back(from_sparse(l, [](Complex v) { return v; }));                      // L
    }
  }
  o.a = make_multi(n, ae);
  o.b = make_multi(n, be);
  o.t = make_multi(n, {});
  return o;
  };
  return LiouvillianBuilder::with_rebuild(omega, n, std::move(operands), cfg);
}

}  // namespace qswg
