// The device-resident superoperator: the B200 counterpart of
// qsw::DistributedLiouvillian (proj/core/include/qsw/liouvillian.hpp:21-93).
//
// One Liouvillian lives on one GPU and owns a contiguous row block of L
// (the whole matrix when world == 1) in CSR with int64 row pointers, int32
// global columns and complex128 values.  Rows are split on rho-column
// boundaries (r = n*j + i, so block = a range of rho columns j) balanced by
// nnz.  Construction assembles the rows on the device (cuda/assemble.cu) and
// computes the 1-norm power series (cuda/norms.cu).
#pragma once

#include <array>
#include <functional>
#include <memory>
#include <optional>
#include <vector>

#include "../kernels.hpp"
#include "device.hpp"
#include "graph.hpp"
#include "sparse.hpp"

namespace qswg {

class Comm;         // multi-GPU exchange (comm.hpp); nullptr when world == 1
struct KronStore;   // operands of the matrix-free (Kron) format (liouvillian.cpp)

struct DeviceConfig {
  int device = 0;       // CUDA ordinal
  int group = 0;        // lanes per row for the SpMV kernels; 0 = autotune
  int format = 0;       // 0 auto, 1 CSR, 2 SELL-32, 3 matrix-free Kronecker action
  Comm* comm = nullptr; // borrowed; shared by every handle on this rank
};

// Lazily grown scratch vectors and device control blocks reused by every
// step/series call on one Liouvillian (not thread-safe per handle, like the
// reference's per-object use).
struct Workspace {
  std::vector<DeviceBuffer<double2>> vec;
  DeviceBuffer<dev::StepCtl> step_ctl;
  DeviceBuffer<dev::SeriesCtl> series_ctl;
  std::shared_ptr<void> series_graph;  // expm.cpp: captured launch sequence of a repeated series call
  std::shared_ptr<PinnedBuffer<int>> flags;  // expm.cpp: error / SpMV counters read back once per call
  double2* get(std::size_t idx, std::size_t len) {
    if (vec.size() <= idx) vec.resize(idx + 1);
    if (vec[idx].size() < len) vec[idx].resize(len);
    return vec[idx].get();
  }
};

// One SELL column panel (liouvillian.cpp: column panels).
struct SellPanel {
  DeviceBuffer<std::int64_t> slice_ptr;
  DeviceBuffer<int> perm;  // empty: identity
  DeviceBuffer<int> col;
  DeviceBuffer<double2> val;
  std::int64_t c_lo = 0, c_hi = 0;  // global column range
  std::int64_t entries = 0;          // stored entries (padding included)
  // fused B (x) I part in natural row order (dev::SellView::b_val); empty: none
  DeviceBuffer<std::int64_t> b_slice_ptr;
  DeviceBuffer<int> b_col;
  DeviceBuffer<double2> b_val;
};

struct RowBlock {
  std::int64_t row0 = 0;  // first global row owned
  std::int64_t rows = 0;  // rows owned
};

class Liouvillian {
 public:
  ~Liouvillian();
  Liouvillian(const Liouvillian&) = delete;
  Liouvillian& operator=(const Liouvillian&) = delete;

  std::int64_t n() const { return n_; }             // operator (vertex) dimension
  std::int64_t dim() const { return n_ * n_; }
  double omega() const { return omega_; }
  std::int64_t nnz_local() const { return nnz_local_; }
  std::int64_t nnz_total() const { return nnz_total_; }
  const RowBlock& block() const { return block_; }
  const std::vector<std::int64_t>& partition() const { return starts_; }  // world + 1 row starts
  /// Upper bounds on ||L^p||_1, p = 1..9 (exact when dim <= 4096).
  const std::array<double, 9>& one_norms() const { return norms_; }
  int group() const { return group_; }
  int device() const { return device_; }
  cudaStream_t stream() const { return stream_; }
  Comm* comm() const { return comm_; }
  dev::CsrView view() const;
  /// The local block as the Taylor kernels see it (format + lanes per row).
  dev::DevMatrix matrix(int group_override = 0) const;
  dev::Format format() const { return format_; }
  /// Stored entries / nnz (SELL padding; 1.0 for CSR).
  double padding() const { return padding_; }
  /// SELL sorting window (32: slices of consecutive rows).
  int sell_sigma() const { return sigma_; }
  /// SELL column panels (1: the whole row in one pass).
  int sell_panels() const { return static_cast<int>(pre_.size()) + 1; }
  /// Second stream (and two events) for halo exchanges overlapped with the
  /// own-column panel of a row-partitioned stored superoperator.
  cudaStream_t side_stream(cudaEvent_t* ev) const;
  bool kron_factored() const;
  /// Per Lindblad term, the n^2-vectors the Hermitian-path (one GPU) Kron
  /// kernels touch: read by the term kernel (W_k, Wt_k) and written by the
  /// prepare kernel (roofline byte counts).
  int kron_term_vectors() const;
  int kron_prepare_vectors() const;
  bool kron_ell() const { return kron_ != nullptr && kron_ell_; }
  /// The Hermitian series term runs on staged tiles (kernels.hpp: KronView::staged).
  bool kron_staged() const;
  /// SELL with the fused natural-order B (x) I arrays (kernels.hpp: SellView::b_val).
  bool sell_fused() const { return format_ == dev::Format::Sell && fused_.b_val.size() > 0; }

  /// Local row block downloaded as CSR with global columns (parity / debug).
  void download(std::vector<std::int64_t>& rowptr, std::vector<std::int64_t>& col,
                std::vector<Complex>& val) const;
  /// Kron on one GPU: selects the Hermitian kernels for the products that
  /// follow when x (full-length) is exactly Hermitian.  known >= 0: the
  /// caller already knows (a state checked at upload, built from
  /// probabilities, or produced by the Hermitian kernels): no check, no
  /// synchronisation; -1: check on the device (synchronises).
  void set_hermitian_input(const double2* x, int known = -1) const;
  /// 1 if x is exactly Hermitian, 0 if not, -1 when no kernel here uses it
  /// (not the one-GPU Kron format); synchronises when it checks.
  int hermitian_state(const double2* x) const;
  /// Whether the products since the last set_hermitian_input ran the
  /// Hermitian kernels (their outputs are then exactly Hermitian).
  bool hermitian_mode() const { return herm_ != 0; }
  /// 0: never take the Hermitian kernels; 1 (default): when the input is Hermitian.
  void set_hermitian_mode(int mode) { herm_mode_ = mode ? 1 : 0; }
  /// Re-mixes the superoperator for a new omega in place (SURVEY.md §8(f)
  /// item 1; WalkSystem::set_omega, walk.cpp:141-145): the n x n operands
  /// are re-derived on the host from the inputs kept at build, the device
  /// reassembles the same handle (format choice, norms, halos) on the same
  /// row partition, so every state of this handle stays valid.
  void set_omega(double omega);
  /// y = scale * L x for device vectors: x full-length (dim), y local (rows).
  void multiply(const double2* x, double2* y, double scale) const;
  /// Mean device time (ms) of one term kernel launch over `iters` launches.
  double time_spmv(int iters, int group) const;
  Workspace& workspace() const { return ws_; }
  /// halo_lo()[r][q], halo_hi()[r][q]: global rows of rank q's segment that
  /// rank r gathers before every SpMV (empty when lo == hi).
  const std::vector<std::vector<std::int64_t>>& halo_lo() const { return halo_lo_; }
  const std::vector<std::vector<std::int64_t>>& halo_hi() const { return halo_hi_; }
  /// Kron format: halos of the W_k = Q_k X work vectors (same layout).
  const std::vector<std::vector<std::int64_t>>& w_halo_lo() const { return whalo_lo_; }
  const std::vector<std::vector<std::int64_t>>& w_halo_hi() const { return whalo_hi_; }
  const std::vector<std::vector<std::int64_t>>& v_halo_lo() const { return vhalo_lo_; }
  const std::vector<std::vector<std::int64_t>>& v_halo_hi() const { return vhalo_hi_; }

 private:
  Liouvillian() = default;
  friend class LiouvillianBuilder;

  std::int64_t n_ = 0;
  double omega_ = 0.0;
  int device_ = 0;
  int group_ = 8;
  cudaStream_t stream_ = nullptr;
  Comm* comm_ = nullptr;
  RowBlock block_;
  std::vector<std::int64_t> starts_;
  std::int64_t nnz_local_ = 0, nnz_total_ = 0;
  std::array<double, 9> norms_{};
  dev::Format format_ = dev::Format::Csr;
  double padding_ = 1.0;
  std::int64_t n_slices_ = 0;
  DeviceBuffer<std::int64_t> slice_ptr_;  // SELL
  DeviceBuffer<int> perm_;                // SELL-C-sigma slot -> row (empty: identity)
  int sigma_ = dev::kSlice;
  std::vector<SellPanel> pre_;            // SELL column panels before the main arrays (one GPU)
  DeviceBuffer<double2> part_;            // their row sums
  SellPanel fused_;                       // the main panel's fused B (x) I arrays (b_* only)
  DeviceBuffer<unsigned> sell_work_;          // one scheduling counter per panel (dev::SellView::work)
  std::int64_t main_c_lo_ = 0;            // column range of the main SELL arrays
  int local_first_ = 0;                   // leading panels = this rank's own columns (overlap the halo exchange)
  mutable cudaStream_t side_ = nullptr;   // halo exchanges overlapped with the local panel
  mutable cudaEvent_t ev_[2] = {nullptr, nullptr};
  DeviceBuffer<std::int64_t> rowptr_;     // CSR
  DeviceBuffer<int> col_;
  DeviceBuffer<double2> val_;
  std::vector<std::vector<std::int64_t>> halo_lo_, halo_hi_;
  std::vector<std::vector<std::int64_t>> whalo_lo_, whalo_hi_, vhalo_lo_, vhalo_hi_;
  std::shared_ptr<KronStore> kron_;
  mutable bool kron_ell_ = false;  // use the sliced-ELL copies of A / Q_k
  std::vector<DeviceBuffer<double2>> kron_w_, kron_v_;
  DeviceBuffer<int> herm_flag_;  // Kron on one GPU: device flag of the Hermiticity check
  mutable int herm_ = 0;         // the current call's input is Hermitian (kernels.hpp: KronView::herm)
  int herm_mode_ = 1;            // set_hermitian_mode
  std::vector<DeviceBuffer<double2>> kron_wt_;  // factored + one GPU: row-major W_k for the Hermitian path
  DeviceBuffer<double2> kron_axt_;               // kernels.hpp: KronView::axt
  mutable Workspace ws_;
  // build_local / build_global inputs, re-run by set_omega on a fixed partition
  std::function<std::unique_ptr<Liouvillian>(double, const std::vector<std::int64_t>*)> rebuild_;
  void adopt(Liouvillian& o);  // take o's operator, keep this handle's stream
};

/// L-QSW (liouvillian.hpp:65-71, liouvillian.cpp:129-210).
std::unique_ptr<Liouvillian> build_local(double omega, const SparseMatrix& h, const SparseMatrix& m_l,
                                         const std::vector<SourceArc>& sources,
                                         const std::vector<SinkArc>& sinks, const DeviceConfig& cfg);
/// G-QSW / NM-G-QSW (liouvillian.hpp:73-85, liouvillian.cpp:212-307).
std::unique_ptr<Liouvillian> build_global(double omega, const SparseMatrix& h,
                                          const std::vector<SparseMatrix>& lindblads,
                                          const std::optional<SparseMatrix>& h_rot,
                                          const DeviceConfig& cfg);

}  // namespace qswg
