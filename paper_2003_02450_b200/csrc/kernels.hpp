// Launch interface between the C++ host layer (host/*.cpp) and the sm_100a
// kernels (cuda/*.cu).  Plain structs of device pointers; no torch types.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>

namespace qswg::dev {

inline constexpr int kMaxKron = 8;      // Lindblad operators per G-QSW
inline constexpr int kMaxSeriesD = 128; // super-step outputs (d <= floor(1e280^(1/55)) = 123)
inline constexpr int kSeriesRegD = 4;   // running sums updated per chunk in the series kernel
inline constexpr int kStageSlots = 5;   // column tiles a 32-row tile of an operand may name on the staged path
inline constexpr int kPendMax = 64;     // series terms held back before one batched sum update

// A "multi-CSR" over the n x n operator space: rows sorted by column with
// duplicates kept adjacent in emission order (they are summed on the device
// in that order).  ptr == nullptr means the list is empty.
struct KronList {
  const int* ptr = nullptr;
  const int* col = nullptr;
  const double2* val = nullptr;
};

// Every superoperator variant of the reference (liouvillian.cpp:129-307) is
//   L = I (x) A + B (x) I + sum_k P_k (x) Q_k + T_diag + decay
// in the column-major vec convention: row r = n*j + i of L picks up
//   A(i, c)           at column n*j + c,
//   B(j, c)           at column n*c + i,
//   P_k(j,a) Q_k(i,b) at column n*a + b,
//   T(i, c)           at column n*c + c     (only when i == j),
//   -0.5*(omega*(dl_i + dl_j) + ds_i + ds_j) at column r (when d_loc != null).
struct KronOperands {
  int n = 0;
  KronList a, b;
  int nk = 0;
  KronList p[kMaxKron], q[kMaxKron];
  KronList t;
  const double* d_loc = nullptr;
  const double* d_ss = nullptr;
  double omega = 0.0;
};

// Row block [row0, row0 + rows) of a device CSR: int64 row pointers (local,
// starting at 0), int32 global column indices, complex128 values.
struct CsrView {
  const std::int64_t* rowptr = nullptr;
  const int* col = nullptr;
  const double2* val = nullptr;
  std::int64_t rows = 0;
  std::int64_t row0 = 0;
};

// Sliced ELLPACK with slices of kSlice = 32 consecutive rows: entry k of the
// rows of slice s lives at slice_ptr[s] + k * 32 + lane (lane = row % 32),
// k < (slice_ptr[s+1] - slice_ptr[s]) / 32; rows shorter than the slice's
// longest row are padded with (col = row, val = 0).  Entries of a row keep
// the canonical CSR order.  One warp per slice, one lane per row: the matrix
// stream, the x gathers of structured (lattice) superoperators and the
// epilogue vectors are all coalesced.
// SELL-C-sigma: with `perm`, slot t (= 32 s + lane) holds local row perm[t];
// rows are sorted by length (descending, stable) inside windows of sigma rows
// so the slices of irregular superoperators pad little (c3: 1.24 -> ~1.02).
inline constexpr int kSlice = 32;
struct SellView {
  const std::int64_t* slice_ptr = nullptr;
  const int* col = nullptr;
  const double2* val = nullptr;
  const int* perm = nullptr;  // slot -> local row; nullptr = identity
  // Column panels: the row sums of the earlier panels, added to this
  // panel's sum (nullptr: a single panel).
  const double2* part_in = nullptr;
  // Dynamic slice scheduling: a device counter the warps of one launch draw
  // chunks of consecutive slices from (the launch's last draw zeroes it again);
  // nullptr = the static grid-stride assignment.
  unsigned* work = nullptr;
  // Fused B (x) I part (one GPU, sigma-sorted rows; nullptr = none): the
  // panel's B (x) I entries — for the 32 consecutive rows (i .. i + 31, j) of a
  // slice the same operand row j, their gathers x[n c + i .. i + 31] one
  // coalesced 512-byte segment — kept in a second sliced ELL in NATURAL row
  // order (no padding between rows of one rho column), while col / val hold
  // the remaining entries in the sorted order.  A block works through
  // windows of win_slices slices (sigma = 32 win_slices rows, so the sort
  // permutes inside a window): the natural-order sums of the window go to
  // shared memory, then the sorted slices add them to theirs.  win_work: the
  // device counter the blocks draw windows from.
  const std::int64_t* b_slice_ptr = nullptr;
  const int* b_col = nullptr;
  const double2* b_val = nullptr;
  int win_slices = 0;
  unsigned* win_work = nullptr;
  std::int64_t rows = 0;
  std::int64_t row0 = 0;
  std::int64_t n_slices = 0;
};

enum class Format : int { Csr = 0, Sell = 1, Kron = 2 };

// Matrix-free Kronecker action (no superoperator stored):
//   (L x)[n*j + i] = sum_c A(i,c) X(c,j) + sum_c B(j,c) X(i,c)
//                  + sum_k sum_a P_k(j,a) W_k(i,a)          with W_k = Q_k X
//                  + [i == j] sum_c T(i,c) X(c,c) - decay(i,j) X(i,j)
// for X(i,j) = x[n*j + i] (column-major vec).  A, B, T are the summed
// (canonical) operand lists of KronOperands; W_k are full-length work
// vectors filled by kron_prepare() before every product.
// Row-indexed n x n operand in sliced ELL (32 rows per slice, entry k of the
// rows of slice s at sptr[s] + 32 k + lane, padded with col = row, val = 0):
// the 32 lanes of a warp handle 32 consecutive rows i, so their operand
// loads are coalesced.
struct KronEll {
  const int* sptr = nullptr;  // n_slices + 1 entry offsets
  const int* col = nullptr;
  const double2* val = nullptr;
};

// Value class of an operand (KronView::vk_*): every stored value purely real,
// purely imaginary, or general complex.  The kernels multiply the first two
// with half the FMAs; the products they drop are exact zeros.
// kValConst (or-ed in): every entry of the operand equals KronView::cv_*.
inline constexpr int kValComplex = 0, kValReal = 1, kValImag = 2, kValConst = 4;

// Tile grid of the KRON kernels (32 x 32 tiles of X over the local columns),
// precomputed on the host: herm_tiles lists the upper tiles (I, J), I <= J,
// in launch order (one GPU).
struct KronTiles {
  int nc = 0, c0 = 0, nti = 0, ntj = 0;
  long long ntiles = 0, ntiles_herm = 0;
  const int2* herm_tiles = nullptr;
};

struct KronView {
  int n = 0;
  std::int64_t rows = 0;  // local rows [row0, row0 + rows), multiples of n
  std::int64_t row0 = 0;
  // Row-indexed operands come in sliced ELL when its padding is small (lattice
  // operators), else in CSR (their `ell.sptr` is then null).
  KronEll a_ell;  // I (x) A, indexed by the rho row i
  KronList a;
  KronList b;     // B (x) I, indexed by the rho column j (warp-uniform)
  KronList t;     // transfer onto the diagonal (rows i == j)
  // a and b hold no diagonal entries: (A_ii + B_jj) X(i, j) is one term
  // (nullptr: both diagonals vanish)
  const double2* da = nullptr;
  const double2* db = nullptr;
  int nk = 0;
  KronList p[kMaxKron];      // indexed by j (warp-uniform)
  KronEll q_ell[kMaxKron];   // W_k = Q_k X, indexed by i
  KronList q[kMaxKron];
  // Factored G-QSW dissipator (a, b then hold only the coherent parts):
  //   + sum_b R_k(i,b) W_k(b,j)      R_k = -w/2 L_k'   (column j of W_k)
  //   + sum_a S_k(j,a) V_k(i,a)      S_k = -w/2 L_k^T  (columns of V_k)
  //   with V_k(:, a) = sum_c U_k(a,c) X(:, c),  U_k = conj(L_k).
  int factored = 0;
  KronList r[kMaxKron], s[kMaxKron], u[kMaxKron];
  double2* v[kMaxKron] = {};
  const double* d_loc = nullptr;
  const double* d_ss = nullptr;
  double omega = 0.0;
  double2* w[kMaxKron] = {};
  // One GPU only.  Every superoperator here maps Hermitian X to Hermitian
  // L(X) (Lindblad form); when the input of a call is exactly Hermitian
  // (kron_hermitian_check, herm = 1) the kernels compute the upper-triangular
  // 32 x 32 tiles only and write each one twice (Y(j,i) = conj Y(i,j), real
  // diagonal), so the iterates stay exactly Hermitian.  herm_flag: device int
  // for the check (nullptr in row-partitioned runs: always the full product).
  int* herm_flag = nullptr;
  int herm = 0;
  double2* wt[kMaxKron] = {};  // factored + Hermitian: row-major copies of W_k
  // p_rows (factored, one GPU, padding-free P_k ELL): the Hermitian tiles
  // apply P_k in the transposed section, P_k(j, a) W_k(i, a) = P_k(j, a)
  // Wt_k[n i + a], lane = j, so the column-major W_k is never read (nor written).
  int p_rows = 0;
  KronEll p_ell[kMaxKron];
  // b_rows (one GPU, padding-free B ELL): B applied there too, lane = j,
  // B(j, c) X(i, c) = B(j, c) conj x[n i + c].
  int b_rows = 0;
  KronEll b_ell;
  // a_len > 0 (one GPU, uniform A slices of a_len <= 8 entries): the
  // transposed A part fetches its four rows' column indices with one warp load
  // and shuffles them out.
  int a_len = 0;
  KronEll a_ellu;
  // The same for R_k and S_k (factored) and Q_k (Hermitian W kernel): uniform
  // ELL slices of r_len / s_len / q_len <= 8 entries (0: the CSR rows).
  int r_len[kMaxKron] = {}, s_len[kMaxKron] = {}, q_len[kMaxKron] = {};
  KronEll r_ellu[kMaxKron], s_ellu[kMaxKron], q_ellu[kMaxKron];
  // value classes: A, B, T, the merged diagonal (da, db), and per Lindblad
  // term P_k, Q_k, R_k, S_k, U_k
  int vk_a = kValComplex, vk_b = kValComplex, vk_t = kValComplex, vk_d = kValComplex;
  int vk_p[kMaxKron] = {}, vk_q[kMaxKron] = {}, vk_r[kMaxKron] = {}, vk_s[kMaxKron] = {}, vk_u[kMaxKron] = {};
  double2 cv_a{}, cv_b{}, cv_p[kMaxKron] = {}, cv_q[kMaxKron] = {}, cv_r[kMaxKron] = {}, cv_s[kMaxKron] = {};
  // Column offsets: the lists gathered as base + c * n hold c * n already —
  // b, p, s, u, every *_ellu and the Hermitian-path copies a_sc, r_sc, q_sc
  // (a, r, q, a_ell, q_ell, p_ell, b_ell and t hold plain columns).
  KronList a_sc, r_sc[kMaxKron], q_sc[kMaxKron];
  KronTiles tg;
  // ax (one GPU, factored, one Lindblad operator): A's pattern lies inside
  // Q_0's and B = conj(A) entrywise (a Hermitian H / H_rot).  The Hermitian W
  // kernel then also forms AX = A X from the gathers of W_0 = Q_0 X (A's
  // values aligned to Q_0's entries: aq_ellu_val / aq_sc_val, class vk_aq,
  // constant cv_aq) into axt (row-major, axt[n i + j] = AX(i, j)); the
  // Hermitian term kernel reads A's part as AX(i, j) and B's as conj AX(j, i)
  // — Sum_c B(j, c) X(i, c) = conj Sum_c A(j, c) X(c, i) exactly, term by
  // term.  b_sep: the general path sums B's part on its own before adding
  // it, the association the Hermitian path has.
  // d_const: every decay coefficient 0.5 (w (dl_i + dl_j) + ds_i + ds_j) is
  // the same value d_val (constant dl, no sources / sinks: regular graphs)
  int d_const = 0;
  double d_val = 0.0;
  int ax = 0, b_sep = 0;
  double2* axt = nullptr;
  // Staged Hermitian tiles (one GPU, n % 32 == 0, operands whose rows of one
  // 32-row tile name at most kStageSlots column tiles: lattices in their
  // natural labelling).  Every operand-weighted gather of a tile (I, J) then
  // falls in a few 32 x 32 tiles of ONE row-major source F (Wt_0 for the
  // factored G-QSW with one Lindblad operator, x itself for L-QSW):
  //   pattern 0  F(T, J), T in st_nbr[0][I]   rows c of R_0 / A, lane = j
  //   pattern 1  F(I, T), T in st_nbr[1][J]   columns a of P_0 / B, lane = j
  //   pattern 2  F(T, I), T in st_nbr[2][J]   rows c of S_0, lane = i
  // which the staged term kernel copies into shared memory a tile ahead
  // (cp.async, 16 bytes per thread, one copy group per phase), so the
  // operand-index -> gather -> FMA chains run against shared memory.  Opt-in
  // (QSWG_KRON_STAGED=1): measured slower than the global gathers.
  // st_col[p]: the operand's ELL column array (layout of r_ellu[0] / a_ellu,
  // p_ell[0] / b_ell, s_ellu[0]) with every column replaced by its element
  // offset inside the pattern's shared-memory region.
  int staged = 0;
  int st_slots[3] = {};           // tiles per region (max over the tile rows)
  const int* st_nbr[3] = {};      // [n / 32][kStageSlots] tile indices, -1 = none
  const int* st_col[3] = {};
  int st_len[3] = {};             // row length of each pattern's operand (the same in every row, <= 8)
  const double2* aq_ellu_val = nullptr;
  const double2* aq_sc_val = nullptr;
  int vk_aq = kValComplex;
  double2 cv_aq{};
};

// The device superoperator block as the Taylor kernels see it.  group: CSR
// lanes per row (2..32); group == 1 selects the bitwise reference-order mode
// for either format.
// SELL split into column panels (one GPU, x beyond L2): the earlier panels
// accumulate row sums in `part`; the last one (DevMatrix::sell) adds them.
inline constexpr int kMaxSellPanels = 16;
inline constexpr int kSellWindowSlices = 64;  // fused B (x) I windows: 2048 rows, 32 KB of sums per block

struct DevMatrix {
  Format format = Format::Csr;
  int group = 8;
  CsrView csr;
  SellView sell;
  KronView kron;
  int n_pre = 0;                           // SELL column panels before `sell`
  SellView sell_pre[kMaxSellPanels - 1];
  double2* part = nullptr;                 // their row sums (local rows)
  int local_first = 0;                     // sell_pre[0 .. local_first) = this rank's own columns (no halo)
  int pre_done = 0;                        // panels already summed for this product (sell_local_panel)
  std::int64_t rows() const {
    return format == Format::Csr ? csr.rows : format == Format::Sell ? sell.rows : kron.rows;
  }
};

struct RealCsrView {
  const std::int64_t* rowptr = nullptr;
  const int* col = nullptr;
  const double* val = nullptr;
  std::int64_t rows = 0;
  std::int64_t row0 = 0;
};

// ---- assembly (cuda/assemble.cu) -------------------------------------------
// Entries per row; with [c_lo, c_hi) only those of that column panel.
void assemble_count(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                    std::int64_t* counts, cudaStream_t s, std::int64_t c_lo = 0,
                    std::int64_t c_hi = INT64_MAX);
// counts (rows + 1 entries, last one ignored) -> exclusive prefix sum.
void exclusive_scan(const std::int64_t* counts, std::int64_t* rowptr, std::int64_t n,
                    void* tmp, std::size_t& tmp_bytes, cudaStream_t s);
// dst[k] = src[k] - base, k < n (local row pointers of a row block).
void rebase_rowptr(const std::int64_t* src, std::int64_t base, std::int64_t* dst, std::int64_t n,
                   cudaStream_t s);
void assemble_fill(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                   const std::int64_t* rowptr, int* col, double2* val, cudaStream_t s);
// slice_entries[s] = 32 * (longest row of slice s), s < ceil(rows / 32);
// grp_local holds rows + 1 row offsets (any base).
// perm (slot -> row) may be nullptr (identity).
void sell_slice_entries(const std::int64_t* grp_local, std::int64_t rows, const int* perm,
                        std::int64_t* slice_entries, cudaStream_t s);
void assemble_fill_sell(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                        const std::int64_t* slice_ptr, const int* perm, int* col, double2* val, cudaStream_t s,
                        std::int64_t c_lo = 0, std::int64_t c_hi = INT64_MAX);
// perm[0..rows): inside each window of sigma rows, the rows by descending
// length (grp_local[r+1] - grp_local[r]), equal lengths in row order.
void sell_sort_rows(const std::int64_t* grp_local, std::int64_t rows, int sigma, int* perm, cudaStream_t s);
void assemble_fill_abs(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                       const std::int64_t* rowptr, int* col, double* val, cudaStream_t s);

// Halo hulls: for every peer q != rank, lo[q] / hi[q] = min / max+1 of the
// columns in col[0..n) owned by q (starts: world + 1 global row starts, on
// the device).  lo must be preset to INT64_MAX and hi to INT64_MIN.
void halo_hulls(const int* col, std::int64_t n, const std::int64_t* starts, int world, int rank,
                std::int64_t* lo, std::int64_t* hi, cudaStream_t s);

// ---- norms (cuda/norms.cu) ---------------------------------------------------
// Exact ||L^p||_1 (p = 1..9) through dense powers of L applied to the
// identity; dim <= 4096.  work: 2 * dim * dim double2 + dim doubles.
void exact_norms(const CsrView& l, std::int64_t dim, double2* work0, double2* work1,
                 double* colsum, double* norms9_host, cudaStream_t s);
// next[r] = sum_c v[c] |L^T|(r, c), ascending c, no FMA (liouvillian.cpp:321-343).
void abs_transpose_product(const RealCsrView& lt, const double* v, double* next,
                           cudaStream_t s);
// max over n non-negative doubles -> *out (device); uses the uint64 bit order.
void max_reduce(const double* v, std::int64_t n, unsigned long long* out_bits, cudaStream_t s);

// ---- Taylor loop (cuda/taylor.cu) -----------------------------------------
struct StepCtl {
  unsigned long long term_bits;
  unsigned long long sum_bits;
  unsigned int arrivals;
  int done;
  int error;
  int spmvs;
  double c1;
  double last_nf;
};

// Series control block.  Running sums are updated lazily and per output:
// term kernels only write K_p (into a ring of pend_max + 1 vectors) and
// ||K_p||; the stop test of every active output is first evaluated against
// a rigorous upper bound of ||S_k|| (its last exact norm + the sum of its
// pending terms' norms, rounded up).  An output whose test is settled
// ("continues") keeps its terms pending; an undecidable test marks that
// output, and the flush kernel then adds its pending terms in order
// (bit-identical to per-term updates) and runs its exact test.  A full ring
// or the super-step's last term marks every active output.
struct SeriesCtl {
  unsigned long long term_bits;               // adjacent to sum_bits: one
  unsigned long long sum_bits[kMaxSeriesD];   // allreduce covers both
  unsigned int arrivals;
  int n_active;
  int error;
  int spmvs;
  int count;
  int flush;       // the flush kernel after this term must run (some output marked)
  int pend_max;    // ring capacity in use (<= kPendMax); ring slots = pend_max + 1
  int slots;
  double z_norm;
  double tn_last;  // ||K_p|| of the newest term
  double factor[kMaxSeriesD];
  double c1[kMaxSeriesD];
  double nf_last[kMaxSeriesD];  // exact ||S_k|| at its last flush (||Z|| at the start)
  double bound[kMaxSeriesD];    // upper bound of the pending terms' contribution
  double fac_ring[kPendMax + 1][kMaxSeriesD];  // k^q of the term in ring slot q % slots
  int p0[kMaxSeriesD];          // first pending term of output k
  int mark[kMaxSeriesD];        // output k is flushed after this term
  int fresh[kMaxSeriesD];       // output k's first flush starts from Z
  int active[kMaxSeriesD];
  // Stop settled by the lower bound: the output is done (no more tests) but
  // its terms p0 .. p_end are still pending; the next flush adds them.
  // n_active counts active + pending outputs.
  int pending[kMaxSeriesD];
  int p_end[kMaxSeriesD];
};

// Term vectors of a series super-step: term p lives in k[p % slots]
// (full-length, SpMV inputs); slots = pend_max + 1.
struct SeriesRing {
  double2* k[kPendMax + 1];
  int slots;
};

struct SeriesSums {
  double2* s[kMaxSeriesD];
};

// Multi-GPU overlap: the partial sums of the own-column panels
// (DevMatrix::local_first of them) of the next product with x, launched while
// x's halo is exchanged; the product then runs with pre_done = local_first.  The skip test is the
// term kernel's: series control (series != nullptr) or step control.
void sell_local_panel(const DevMatrix& m, const double2* x, const SeriesCtl* series, const StepCtl* step,
                      int first_of_stage, cudaStream_t s);

// Lanes per row for the row-group SpMV kernels: 2, 4, 8, 16 or 32; 1 selects
// the bitwise reference-order mode (sequential rows, no FMA).
int valid_group(int g);

// Every reduction kernel below takes `decide`: true on one GPU (the last
// block to arrive runs the control step); false under multi-GPU, where the
// kernel leaves its local maxima in the control block for an allreduce(max)
// and the matching *_control / *_fin kernel then runs the same control step.

// ctl->c1 = ||v||_inf over n local elements (`error`/`spmvs` are sticky).
void step_init(const double2* v, std::int64_t n, StepCtl* ctl, bool decide, cudaStream_t s);
void step_init_fin(StepCtl* ctl, cudaStream_t s);
void step_control(StepCtl* ctl, bool first_of_stage, int stage, double tol, cudaStream_t s);
void series_init_fin(SeriesCtl* ctl, int count, int pend_max, cudaStream_t s);
// One Taylor term of `step` (expm.cpp:175-195):
//   y = scale * (L x);  sum_out = sum_in + y;  c2 = ||y||, nf = ||sum_out||;
//   stop test c1 + c2 <= tol * nf decided on the device.  Skips itself when
//   the stage is already done (unless first_of_stage) or on error.
void step_term(const DevMatrix& l, const double2* x, double2* y, const double2* sum_in,
               double2* sum_out, double scale, bool first_of_stage, int stage, double tol,
               StepCtl* ctl, bool decide, cudaStream_t s);
// Super-step start of `series` (expm.cpp:267-276): z_norm = ||Z||, count
// outputs active, factor_k = k, c1_k = z_norm; pend_max terms may be held back.
void series_init(const double2* z, std::int64_t n, int count, int pend_max, SeriesCtl* ctl, bool decide,
                 cudaStream_t s);
// K_p = scale * (L K_{p-1}) and ||K_p|| (expm.cpp:283-293); the control then
// decides which stop tests are already settled and whether a flush is due
// (always on the super-step's `last` term).
void series_term(const DevMatrix& l, const double2* x, double2* kp, int p, bool last, double scale,
                 double tol, SeriesCtl* ctl, bool decide, cudaStream_t s);
void series_term_control(SeriesCtl* ctl, int p, int last, double tol, cudaStream_t s);
// Several GPUs, after term p and one allreduce of [term_bits, sum_bits]: the
// exact tests of the flush after term p - 1 (when one ran), then term p's
// control (skipped when term p is not part of the series).
void series_flush_term_control(SeriesCtl* ctl, int p, int last, double tol, cudaStream_t s);
// When ctl->flush: for every marked output k, S_k = (fresh_k ? Z : S_k) +
// sum over its pending terms q of k^q K_q, in term order (expm.cpp:300-305),
// then its exact stop test of term p (expm.cpp:306-316).  No-op otherwise.
// herm_n > 0 (KRON Hermitian path on one GPU, n x n states): the Hermitian
// tile flush, which reads the upper elements only and mirrors them.
void series_flush(const SeriesRing& ring, std::int64_t row0, std::int64_t rows, const double2* z,
                  const SeriesSums& sums, int herm_n, int p, bool strict, double tol, SeriesCtl* ctl,
                  bool decide, cudaStream_t s);
void series_flush_control(SeriesCtl* ctl, int p, double tol, cudaStream_t s);
// Kron format: W_k = Q_k X on the local columns (call before every product
// with input x; multi-GPU callers then exchange the W_k halos).
void kron_prepare(const DevMatrix& l, const double2* x, cudaStream_t s);
// One GPU, Kron with Lindblad terms: kron_prepare(x) for the next term fused
// in one launch with series_flush(..., p, decide = true) for the term just
// computed (the flush streams from HBM while W gathers from L2).  Returns
// false (nothing launched) for other matrices.
bool kron_prepare_flush(const DevMatrix& l, const double2* x, const SeriesRing& ring, std::int64_t row0,
                        std::int64_t rows, const double2* z, const SeriesSums& sums, int p, double tol,
                        SeriesCtl* ctl, cudaStream_t s);
// Kron format, one GPU: whether x (dim) is exactly Hermitian as an n x n
// matrix (synchronises the stream).  false for other formats / multi-GPU.
bool kron_hermitian_check(const DevMatrix& l, const double2* x, cudaStream_t s);
// y = scale * (L x) (liouvillian.cpp:346-360).
void spmv(const DevMatrix& l, const double2* x, double2* y, double scale, cudaStream_t s);
// pops[i] = Re v[i*(n+1)] for the diagonal elements inside [row0, row0+rows).
void diag_real(const double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
               double* pops, cudaStream_t s);
// *out = max(*out, max |v(i, j)| over the local off-diagonal elements) as
// the uint64 pattern of a non-negative double (max_coherence, walk.cpp:32-40).
void coherence_bits(const double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
                    unsigned long long* out, cudaStream_t s);
// Deterministic non-zero test pattern (benchmark inputs).
void fill_pattern(double2* v, std::int64_t n, cudaStream_t s);
// Deterministic Hermitian n x n test pattern (column-major, n*n entries).
void fill_pattern_hermitian(double2* v, std::int64_t n, cudaStream_t s);
// v = 0 except v[i*(n+1)] = p[i] (walk.cpp:101-126 without the dense host rho).
void state_from_probabilities(double2* v_local, std::int64_t row0, std::int64_t rows,
                              std::int64_t n, const double* p, cudaStream_t s);

}  // namespace qswg::dev
