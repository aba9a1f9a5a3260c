// Host control flow of the exponential action.  Mirrors expm.cpp:146-325
// step for step; every Taylor term is one fused kernel launch and every stop
// test is evaluated on the device (see cuda/taylor.cu).
//
// One GPU: a whole step or series is enqueued without host round-trips and
// synchronised once — the last block of each term kernel decides.
// Several GPUs (one process each): each term kernel leaves its local maxima,
// an allreduce(max) over NCCL combines them, a one-thread control kernel runs
// the same decision, and the host reads the stop flag before exchanging the
// new term's halo (so terms after the stop are neither computed nor sent).
#include "expm.hpp"

#include <algorithm>
#include <array>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstddef>
#include <cstring>
#include <functional>
#include <memory>
#include <utility>
#include <vector>

#include "comm.hpp"

namespace qswg {

namespace {

// Workspace slots.
enum Slot : std::size_t {
  kT0 = 0, kT1 = 1, kSOther = 2, kNext = 3, kZ = 4, kXStage = 5, kZFull = 6, kSums = 8,
  kRing = kSums + dev::kMaxSeriesD  // series term ring slots 2.. (slots 0, 1 are kT0, kT1)
};

std::size_t ring_slot(int i) { return i < 2 ? static_cast<std::size_t>(i) : kRing + static_cast<std::size_t>(i - 2); }

// Terms a series super-step may hold back (kernels.hpp: SeriesCtl): kPendMax,
// fewer when the ring of pend_max + 1 full-length vectors would take more
// than 30% of the free device memory; QSWG_PEND_MAX overrides (1 = update
// the sums after every term).
int series_pend_max(std::int64_t dim) {
  int pm = dev::kPendMax;
  if (const char* e = std::getenv("QSWG_PEND_MAX")) pm = std::max(1, std::min(dev::kPendMax, std::atoi(e)));
  std::size_t free_b = 0, total_b = 0;
  if (cudaMemGetInfo(&free_b, &total_b) == cudaSuccess) {
    const double vec_b = static_cast<double>(dim) * sizeof(double2);
    while (pm > 1 && (pm - 1) * vec_b > 0.3 * static_cast<double>(free_b)) --pm;
  }
  return pm;
}

dev::StepCtl* step_ctl(const Liouvillian& l) {
  Workspace& ws = l.workspace();
  if (!ws.step_ctl.get()) ws.step_ctl.resize(1);
  return ws.step_ctl.get();
}

dev::SeriesCtl* series_ctl(const Liouvillian& l) {
  Workspace& ws = l.workspace();
  if (!ws.series_ctl.get()) ws.series_ctl.resize(1);
  return ws.series_ctl.get();
}

struct Flags {
  int error = 0;
  std::int64_t spmvs = 0;
};

// The error flags and SpMV counters of the call, read into pinned memory
// (asynchronous copies) after the caller's own reads, one synchronisation.
Flags read_flags(const Liouvillian& l, bool with_series, const std::function<void()>& before_sync = {}) {
  Workspace& ws = l.workspace();
  if (!ws.flags) ws.flags = std::make_shared<PinnedBuffer<int>>(4);
  int* h = ws.flags->get();
  h[0] = h[1] = h[2] = h[3] = 0;
  cudaStream_t s = l.stream();
  if (before_sync) before_sync();
  static_assert(offsetof(dev::StepCtl, spmvs) == offsetof(dev::StepCtl, error) + sizeof(int), "error, spmvs adjacent");
  QSWG_CHECK(cudaMemcpyAsync(h, &step_ctl(l)->error, 2 * sizeof(int), cudaMemcpyDeviceToHost, s));
  if (with_series) {
    QSWG_CHECK(cudaMemcpyAsync(h + 2, &series_ctl(l)->error, sizeof(int), cudaMemcpyDeviceToHost, s));
    QSWG_CHECK(cudaMemcpyAsync(h + 3, &series_ctl(l)->spmvs, sizeof(int), cudaMemcpyDeviceToHost, s));
  }
  QSWG_CHECK(cudaStreamSynchronize(s));
  return {h[0] | h[2], static_cast<std::int64_t>(h[1]) + h[3]};
}

void reset_ctls(const Liouvillian& l, bool with_series) {
  QSWG_CHECK(cudaMemsetAsync(step_ctl(l), 0, sizeof(dev::StepCtl), l.stream()));
  if (with_series) QSWG_CHECK(cudaMemsetAsync(series_ctl(l), 0, sizeof(dev::SeriesCtl), l.stream()));
}

// Execution context: one GPU, or one rank of a row-partitioned run.
struct Exec {
  const Liouvillian& l;
  Comm* comm;
  cudaStream_t s;
  bool single;
  std::int64_t row0, rows, dim;

  explicit Exec(const Liouvillian& lv)
      : l(lv), comm(lv.comm()), s(lv.stream()), single(!lv.comm() || lv.comm()->world() == 1),
        row0(lv.block().row0), rows(lv.block().rows), dim(lv.dim()) {}

  // Full-length (dim) vectors are SpMV inputs; local (rows) vectors are states.
  double2* full(std::size_t slot) const { return l.workspace().get(slot, static_cast<std::size_t>(dim)); }
  double2* local(std::size_t slot) const {
    return l.workspace().get(slot, static_cast<std::size_t>(std::max<std::int64_t>(rows, 1)));
  }

  // Receive every peer segment this block's columns reference.
  void exchange(double2* full_vec) const {
    if (!single) comm->exchange_ranges(full_vec, l.halo_lo(), l.halo_hi(), sizeof(double2), s);
  }

  // Halo exchange of the next product's input; with an own-column SELL panel
  // (row-partitioned stored superoperator) that panel's partial sums run on
  // the library stream while the exchange runs on a side stream.  Returns
  // the number of panels launched (the product then runs with pre_done = it).
  int exchange_overlap(double2* full_vec, const dev::DevMatrix& m, const dev::SeriesCtl* series,
                       const dev::StepCtl* step, int first_of_stage) const {
    if (single) return 0;
    if (m.format != dev::Format::Sell || m.local_first < 1) {
      exchange(full_vec);
      return 0;
    }
    cudaEvent_t ev[2];
    cudaStream_t side = l.side_stream(ev);
    QSWG_CHECK(cudaEventRecord(ev[0], s));  // the input's own rows are final
    QSWG_CHECK(cudaStreamWaitEvent(side, ev[0], 0));
    dev::sell_local_panel(m, full_vec, series, step, first_of_stage, s);
    comm->exchange_ranges(full_vec, l.halo_lo(), l.halo_hi(), sizeof(double2), side);
    QSWG_CHECK(cudaEventRecord(ev[1], side));
    QSWG_CHECK(cudaStreamWaitEvent(s, ev[1], 0));
    return std::min(m.local_first, m.n_pre);
  }

  // SpMV input from a local state: on one GPU the state itself; otherwise
  // its rows copied into a full-length buffer whose halo is then exchanged.
  const double2* spmv_input(const double2* local_vec, std::size_t slot) const {
    if (single) return local_vec;
    double2* f = full(slot);
    QSWG_CHECK(cudaMemcpyAsync(f + row0, local_vec, static_cast<std::size_t>(rows) * sizeof(double2),
                               cudaMemcpyDeviceToDevice, s));
    exchange(f);
    return f;
  }

  // Before every product with input x (full-length, halo filled): the Kron
  // format builds W_k = Q_k x on the local columns and exchanges their halos.
  void prepare(const dev::DevMatrix& m, const double2* x) const {
    if (m.format != dev::Format::Kron) return;
    dev::kron_prepare(m, x, s);
    if (!single)
      for (int k = 0; k < m.kron.nk; ++k) {
        comm->exchange_ranges(m.kron.w[k], l.w_halo_lo(), l.w_halo_hi(), sizeof(double2), s);
        if (m.kron.factored) comm->exchange_ranges(m.kron.v[k], l.v_halo_lo(), l.v_halo_hi(), sizeof(double2), s);
      }
  }

  template <class T>
  T read(const T* dev_ptr) const {
    T v{};
    QSWG_CHECK(cudaMemcpyAsync(&v, dev_ptr, sizeof(T), cudaMemcpyDeviceToHost, s));
    QSWG_CHECK(cudaStreamSynchronize(s));
    return v;
  }
};

// Several GPUs: the host enqueues every term without reading the stop flags
// (each kernel and control skips itself once its stage or super-step is
// done).  To stop enqueueing soon after the end, the flag of every term is
// copied asynchronously into pinned memory behind an event; the host looks at
// the copy from kLag terms back and waits for it only when the device is that
// far behind — the stream never waits on the host.
struct FlagPoll {
  static constexpr int kLag = 4, kRing = 8;
  cudaEvent_t ev[kRing] = {};
  PinnedBuffer<int> flags{kRing};
  int tags[kRing] = {};
  long long recorded = 0;
  std::int64_t waits = 0;  // host waits on an event (reported as SeriesInfo::host_waits)
  FlagPoll() {
    for (auto& e : ev) QSWG_CHECK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  ~FlagPoll() {
    for (auto& e : ev)
      if (e) cudaEventDestroy(e);
  }
  FlagPoll(const FlagPoll&) = delete;
  FlagPoll& operator=(const FlagPoll&) = delete;
  void record(const int* dev_flag, int tag, cudaStream_t s) {
    const int k = static_cast<int>(recorded % kRing);
    tags[k] = tag;
    QSWG_CHECK(cudaMemcpyAsync(flags.get() + k, dev_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
    QSWG_CHECK(cudaEventRecord(ev[k], s));
    ++recorded;
  }
  // The flag recorded kLag records ago (waiting for it if needed); false if
  // there is none yet.
  bool lagged(int& value, int& tag) {
    if (recorded < kLag) return false;
    const int k = static_cast<int>((recorded - kLag) % kRing);
    if (cudaEventQuery(ev[k]) == cudaErrorNotReady) {
      ++waits;
      QSWG_CHECK(cudaEventSynchronize(ev[k]));
    }
    cudaGetLastError();
    value = flags.get()[k];
    tag = tags[k];
    return true;
  }
};

// Enqueues one step (expm.cpp:146-212).  `out` (local) receives the result;
// scratch vectors come from the workspace.
StepParameters enqueue_step(const Exec& ex, const double2* v, double t, const TaylorParameters& params,
                            double2* out, std::int64_t& launches, std::int64_t& host_waits) {
  const Liouvillian& l = ex.l;
  cudaStream_t s = ex.s;
  const StepParameters sp = select_parameters(l.one_norms().data(), t, params);
  if (sp.m_star == 0) {  // expm.cpp:152
    QSWG_CHECK(cudaMemcpyAsync(out, v, static_cast<std::size_t>(ex.rows) * sizeof(double2),
                               cudaMemcpyDeviceToDevice, s));
    return sp;
  }
  double2* term[2] = {ex.full(kT0), ex.full(kT1)};
  double2* sums[2];
  // stage st accumulates into sums[st % 2]; the last stage lands in `out`.
  sums[(sp.s - 1) % 2] = out;
  sums[sp.s % 2] = ex.local(kSOther);
  dev::StepCtl* ctl = step_ctl(l);
  const dev::DevMatrix mat = l.matrix();
  dev::step_init(v, ex.rows, ctl, ex.single, s);  // c1 = ||v||_inf (expm.cpp:165-170)
  if (!ex.single) {
    ex.comm->allreduce_max_u64(&ctl->term_bits, 1, s);
    dev::step_init_fin(ctl, s);
  }
  launches += 1 + sp.s * sp.m_star * (1 + (mat.format == dev::Format::Kron ? mat.kron.nk * (1 + (mat.kron.factored && !mat.kron.herm)) : 0));
  const double s_count = static_cast<double>(sp.s);
  // One GPU, very many stages (a huge ||t L||: test_expm.cpp:234-244 reaches 10^5 stages before
  // it overflows): the error flag is polled every kErrStride stages, lagged like the stop
  // flags of several GPUs, so a step that has already failed stops being enqueued.  Not under
  // stream capture (events of a capture cannot be queried).
  constexpr std::int64_t kErrStride = 64, kErrMinStages = 512;
  std::unique_ptr<FlagPoll> err_poll;
  if (ex.single && sp.s >= kErrMinStages) {
    cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
    QSWG_CHECK(cudaStreamIsCapturing(s, &cap));
    if (cap == cudaStreamCaptureStatusNone) err_poll = std::make_unique<FlagPoll>();
  }
  for (std::int64_t st = 0; st < sp.s; ++st) {
    if (err_poll && st % kErrStride == 0) {
      int err = 0, tag = 0;
      if (err_poll->lagged(err, tag) && err != 0) break;  // failed kLag polls ago: step() reports it
      err_poll->record(&ctl->error, static_cast<int>(st / kErrStride), s);
    }
    // stage input: v, then the previous stage's sum (term = sum, expm.cpp:197-205)
    const double2* x_stage = st == 0 ? v : sums[(st - 1) % 2];
    const double2* x_stage_full = ex.spmv_input(x_stage, kXStage);
    double2* acc = sums[st % 2];
    int pre = 0;  // own-column panels of this product already summed (overlapped exchange)
    std::unique_ptr<FlagPoll> poll;
    if (!ex.single) poll = std::make_unique<FlagPoll>();
    for (std::int64_t j = 1; j <= sp.m_star; ++j) {
      if (!ex.single) {
        int done = 0, tag = 0;
        if (poll->lagged(done, tag) && done != 0) break;  // this stage stopped kLag terms ago
      }
      const double2* x = j == 1 ? x_stage_full : term[(j - 1) % 2];
      double2* y = term[j % 2] + ex.row0;
      const double scale = t / (s_count * static_cast<double>(j));  // expm.cpp:174
      ex.prepare(mat, x);
      dev::DevMatrix mj = mat;
      mj.pre_done = pre;
      dev::step_term(mj, x, y, j == 1 ? x_stage : acc, acc, scale, j == 1, static_cast<int>(st),
                     params.tolerance, ctl, ex.single, s);
      pre = 0;
      if (!ex.single) {
        ex.comm->allreduce_max_u64(&ctl->term_bits, 2, s);  // term_bits, sum_bits
        dev::step_control(ctl, j == 1, static_cast<int>(st), params.tolerance, s);  // (error sets done)
        poll->record(&ctl->done, static_cast<int>(j), s);
        if (j < sp.m_star) pre = ex.exchange_overlap(term[j % 2], mat, nullptr, ctl, 0);
      }
    }
    if (poll) host_waits += poll->waits;
  }
  return sp;
}

}  // namespace

StepInfo step(const Liouvillian& l, const double2* v, double t, const TaylorParameters& params,
              double2* out, int herm_known) {
  DeviceGuard g(l.device());
  const Exec ex(l);
  reset_ctls(l, false);
  l.set_hermitian_input(v, herm_known);  // Hermitian input: the iterates stay Hermitian
  std::int64_t launches = 0;
  std::int64_t host_waits = 0;
  const StepParameters sp = enqueue_step(ex, v, t, params, out, launches, host_waits);
  const Flags f = read_flags(l, false);
  if (f.error) throw NumericalError("non-finite values encountered in exponential action");
  return {sp.m_star, sp.s, f.spmvs, launches};
}

namespace {

// Everything one `series` call enqueues after the Hermiticity check; no host
// synchronisation on one GPU (capturable).
SeriesInfo enqueue_series(const Liouvillian& l, const Exec& ex, const double2* v, double t1, double tq,
                          std::int64_t steps, const TaylorParameters& params,
                          const std::function<void(std::int64_t, const double2*)>& emit_fn) {
  cudaStream_t s = ex.s;
  const std::int64_t q = steps;
  const double h = (tq - t1) / static_cast<double>(q);
  reset_ctls(l, true);
  SeriesInfo info;
  auto emit = [&](std::int64_t k, const double2* state) {
    ++info.emits;
    emit_fn(k, state);
  };

  // states[0] = step(v, t1) (expm.cpp:225)
  double2* z = ex.local(kZ);
  enqueue_step(ex, v, t1, params, z, info.launches, info.host_waits);
  emit(0, z);

  const StepParameters span = select_parameters(l.one_norms().data(), tq - t1, params);
  info.span_m_star = span.m_star;
  info.span_s = span.s;
  if (span.m_star == 0) {  // zero generator (expm.cpp:228-232)
    info.path = 0;
    for (std::int64_t k = 1; k <= q; ++k) emit(k, z);
  } else if (q <= span.s) {  // q sequential steps (expm.cpp:234-240)
    info.path = 1;
    double2* cur = z;
    double2* nxt = ex.local(kNext);
    for (std::int64_t k = 1; k <= q; ++k) {
      enqueue_step(ex, cur, h, params, nxt, info.launches, info.host_waits);
      emit(k, nxt);
      std::swap(cur, nxt);
    }
  } else {  // super-steps sharing K_p = (hL)^p Z / p! (expm.cpp:242-323)
    info.path = 2;
    std::int64_t d = q / span.s;
    const double d_cap = std::pow(1e280, 1.0 / static_cast<double>(TaylorParameters::m_max));
    d = std::min(d, static_cast<std::int64_t>(d_cap));
    const std::int64_t n_super = q / d;
    const std::int64_t remainder = q - d * n_super;
    const StepParameters sub = select_parameters(l.one_norms().data(), h * static_cast<double>(d), params);
    const std::int64_t m_star = std::max<std::int64_t>(sub.m_star, 1);  // sub.s unused, as in the reference
    info.d = d;
    info.n_super = n_super;
    info.remainder = remainder;
    info.sub_m_star = m_star;
    if (d > dev::kMaxSeriesD) throw std::logic_error("super-step size exceeds the device limit");

    dev::SeriesCtl* ctl = series_ctl(l);
    const dev::DevMatrix mat = l.matrix();
    const int pend_max = series_pend_max(ex.dim);
    dev::SeriesRing ring{};
    ring.slots = pend_max + 1;
    for (int i = 0; i < ring.slots; ++i) ring.k[i] = ex.full(ring_slot(i));
    std::vector<double2*> sums(static_cast<std::size_t>(d));
    for (std::int64_t k = 0; k < d; ++k) sums[static_cast<std::size_t>(k)] = ex.local(kSums + static_cast<std::size_t>(k));
    const bool strict = mat.group == 1;
    // KRON Hermitian path (one GPU): every term and sum is exactly Hermitian
    const int herm_n = (ex.single && mat.format == dev::Format::Kron && mat.kron.herm) ? static_cast<int>(l.n()) : 0;
    // One GPU, Kron with Lindblad terms: the flush after term p runs in the
    // launch that prepares W for term p + 1.
    const bool fused = ex.single && mat.format == dev::Format::Kron && mat.kron.nk > 0;
    const std::int64_t per_term =
        (fused ? 1 : 2) +
        (mat.format == dev::Format::Kron ? mat.kron.nk * (1 + (mat.kron.factored && !mat.kron.herm)) : 0);
    for (std::int64_t super = 0; super <= n_super; ++super) {
      const std::int64_t count = super < n_super ? d : remainder;
      if (count == 0) break;
      dev::series_init(z, ex.rows, static_cast<int>(count), pend_max, ctl, ex.single, s);
      if (!ex.single) {
        ex.comm->allreduce_max_u64(&ctl->term_bits, 1, s);
        dev::series_init_fin(ctl, static_cast<int>(count), pend_max, s);
      }
      info.launches += 1 + m_star * per_term + (fused ? 1 : 0);
      dev::SeriesSums ss{};
      for (std::int64_t k = 0; k < count; ++k) ss.s[k] = sums[static_cast<std::size_t>(k)];
      const double2* z_full = ex.spmv_input(z, kZFull);
      int pre = 0;  // own-column panels of this term already summed (overlapped exchange)
      std::int64_t p_last = 0;  // the last term enqueued (several GPUs)
      std::unique_ptr<FlagPoll> poll;
      if (!ex.single) poll = std::make_unique<FlagPoll>();
      for (std::int64_t p = 1; p <= m_star; ++p) {
        const double2* x = p == 1 ? z_full : ring.k[(p - 1) % ring.slots];
        double2* kp = ring.k[p % ring.slots] + ex.row0;
        const bool last = p == m_star;
        if (!ex.single) {
          int active = 1, tag = 0;
          if (poll->lagged(active, tag) && active == 0) break;  // the super-step ended kLag terms ago
          if (p > 1)  // the flush after term p - 1 when its control asked for one (a no-op otherwise);
                      // its norms join term p's allreduce
            dev::series_flush(ring, ex.row0, ex.rows, z, ss, herm_n, static_cast<int>(p - 1), strict,
                              params.tolerance, ctl, false, s);
        }
        p_last = p;
        if (!fused || p == 1) ex.prepare(mat, x);
        dev::DevMatrix mp = mat;
        mp.pre_done = pre;
        pre = 0;
        dev::series_term(mp, x, kp, static_cast<int>(p), last, h / static_cast<double>(p), params.tolerance, ctl,
                         ex.single, s);
        if (ex.single) {
          if (!(fused && !last &&
                dev::kron_prepare_flush(mat, ring.k[p % ring.slots], ring, ex.row0, ex.rows, z, ss,
                                        static_cast<int>(p), params.tolerance, ctl, s)))
            dev::series_flush(ring, ex.row0, ex.rows, z, ss, herm_n, static_cast<int>(p), strict,
                              params.tolerance, ctl, true, s);
          continue;
        }
        // one allreduce: term p's maximum and the sums of the flush after p - 1 (adjacent fields)
        ex.comm->allreduce_max_u64(&ctl->term_bits, 1 + static_cast<std::size_t>(count), s);
        dev::series_flush_term_control(ctl, static_cast<int>(p), last ? 1 : 0, params.tolerance, s);
        poll->record(&ctl->n_active, static_cast<int>(p), s);
        if (p < m_star) pre = ex.exchange_overlap(ring.k[p % ring.slots], mat, ctl, nullptr, 1);
      }
      if (!ex.single && p_last > 0) {  // the flush after the last term enqueued (a no-op unless asked for)
        dev::series_flush(ring, ex.row0, ex.rows, z, ss, herm_n, static_cast<int>(p_last), strict,
                          params.tolerance, ctl, false, s);
        ex.comm->allreduce_max_u64(&ctl->sum_bits[0], static_cast<std::size_t>(count), s);
        dev::series_flush_control(ctl, static_cast<int>(p_last), params.tolerance, s);
      }
      if (poll) info.host_waits += poll->waits;
      for (std::int64_t k = 1; k <= count; ++k) emit(super * d + k, sums[static_cast<std::size_t>(k - 1)]);
      // the next super-step starts from states[(super + 1) d] = the last output
      std::swap(z, sums[static_cast<std::size_t>(count - 1)]);
      // (an error skips every later kernel on the device; the call reports it at its end)
    }
  }
  return info;
}

// Captured series launch sequences of one Liouvillian, most recent first
// (a few, so alternating callers, e.g. two input states, keep theirs).
struct SeriesGraph {
  struct Entry {
    std::vector<double> key;
    cudaGraphExec_t exec = nullptr;
    SeriesInfo info;
  };
  static constexpr std::size_t kKeep = 4;
  std::vector<Entry> entries;
  std::vector<double> last;
  Entry* find(const std::vector<double>& key) {
    for (std::size_t i = 0; i < entries.size(); ++i)
      if (entries[i].key == key) {
        std::rotate(entries.begin(), entries.begin() + static_cast<std::ptrdiff_t>(i),
                    entries.begin() + static_cast<std::ptrdiff_t>(i) + 1);
        return &entries.front();
      }
    return nullptr;
  }
  void add(std::vector<double> key, cudaGraphExec_t exec, const SeriesInfo& info) {
    if (entries.size() == kKeep) {
      cudaGraphExecDestroy(entries.back().exec);
      entries.pop_back();
    }
    entries.insert(entries.begin(), Entry{std::move(key), exec, info});
  }
  ~SeriesGraph() {
    for (Entry& e : entries) cudaGraphExecDestroy(e.exec);
  }
};

}  // namespace

SeriesInfo series(const Liouvillian& l, const double2* v, double t1, double tq, std::int64_t steps,
                  const TaylorParameters& params,
                  const std::function<void(std::int64_t, const double2*)>& emit,
                  const std::vector<const void*>& graph_key, int herm_known,
                  const std::function<void()>& before_sync) {
  // expm.cpp:216-217
  if (!(tq > t1)) throw std::invalid_argument("series requires tq > t1");
  if (steps < 1) throw std::invalid_argument("series requires at least one step");
  DeviceGuard g(l.device());
  const Exec ex(l);
  cudaStream_t s = ex.s;
  l.set_hermitian_input(v, herm_known);  // Hermitian input: every state stays Hermitian
  static const bool graphs_off = [] {
    const char* e = std::getenv("QSWG_GRAPH");
    return e != nullptr && e[0] == '0';
  }();
  SeriesInfo info;
  if (ex.single && !graph_key.empty() && !graphs_off) {
    Workspace& ws = l.workspace();
    if (!ws.series_graph) ws.series_graph = std::make_shared<SeriesGraph>();
    auto* gr = static_cast<SeriesGraph*>(ws.series_graph.get());
    std::vector<double> key = {static_cast<double>(reinterpret_cast<std::uintptr_t>(v)), t1, tq,
                               static_cast<double>(steps), params.tolerance,
                               static_cast<double>(l.matrix().kron.herm), static_cast<double>(series_pend_max(ex.dim))};
    for (const void* b : graph_key) key.push_back(static_cast<double>(reinterpret_cast<std::uintptr_t>(b)));
    if (SeriesGraph::Entry* e = gr->find(key)) {
      QSWG_CHECK(cudaGraphLaunch(e->exec, s));
      info = e->info;
      info.graph = true;
    } else if (gr->last == key) {  // second identical call: its workspace exists, capture it
      if (std::getenv("QSWG_DEBUG_GRAPH")) std::fprintf(stderr, "qswg: capturing a series graph\n");
      cudaGraph_t graph = nullptr;
      QSWG_CHECK(cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal));
      try {
        info = enqueue_series(l, ex, v, t1, tq, steps, params, emit);
      } catch (...) {
        cudaStreamEndCapture(s, &graph);
        if (graph) cudaGraphDestroy(graph);
        throw;
      }
      QSWG_CHECK(cudaStreamEndCapture(s, &graph));
      cudaGraphExec_t exec = nullptr;
      const cudaError_t ie = cudaGraphInstantiate(&exec, graph, 0);
      cudaGraphDestroy(graph);
      QSWG_CHECK(ie);
      gr->add(key, exec, info);
      QSWG_CHECK(cudaGraphLaunch(exec, s));
      info.graph = true;
    } else {
      info = enqueue_series(l, ex, v, t1, tq, steps, params, emit);
      gr->last = key;
    }
  } else {
    info = enqueue_series(l, ex, v, t1, tq, steps, params, emit);
  }
  const Flags f = read_flags(l, info.path == 2, before_sync);
  info.spmvs = f.spmvs;
  if (f.error) throw NumericalError("non-finite values encountered in series evolution");
  return info;
}

// Mean device ms of the parts of one series term over `iters` terms: [0] the
// Kron prepare kernels (W_k, V_k; 0 for stored formats), [1] the term
// kernel, [2] the flush kernel (amortised: it runs its sum update once per
// ring, as in the converging part of a real series) and [3] the whole term.
std::array<double, 4> time_series_parts(const Liouvillian& l, int iters, int count) {
  if (count < 1 || count > dev::kMaxSeriesD) throw std::invalid_argument("count out of range");
  if (iters < 1) throw std::invalid_argument("iters must be >= 1");
  DeviceGuard g(l.device());
  const Exec ex(l);
  cudaStream_t s = ex.s;
  const int pend_max = series_pend_max(ex.dim);
  dev::SeriesRing ring{};
  ring.slots = pend_max + 1;
  for (int i = 0; i < ring.slots; ++i) ring.k[i] = ex.full(ring_slot(i));
  double2* z = ex.local(kZ);
  dev::SeriesSums ss{};
  for (int c = 0; c < count; ++c) ss.s[c] = ex.local(kSums + static_cast<std::size_t>(c));
  if (l.matrix().format == dev::Format::Kron && l.matrix().kron.herm_flag) {  // density-matrix-like input, as in a real series
    dev::fill_pattern_hermitian(ring.k[0], l.n(), s);
  } else {
    dev::fill_pattern(ring.k[0], ex.dim, s);
  }
  l.set_hermitian_input(ring.k[0]);
  const dev::DevMatrix mat = l.matrix();
  dev::fill_pattern(z, ex.rows, s);
  for (int c = 0; c < count; ++c) dev::fill_pattern(ss.s[c], ex.rows, s);
  dev::SeriesCtl* ctl = series_ctl(l);
  QSWG_CHECK(cudaMemsetAsync(ctl, 0, sizeof(dev::SeriesCtl), s));
  dev::series_init(z, ex.rows, count, pend_max, ctl, true, s);
  // tol = -1 keeps every output active and settles every test without the
  // sums (c1 + c2 > -ub); scale 1/||L||_1 keeps the iterates bounded.  Local
  // kernel time only (no exchange), as the per-GPU roofline needs.
  const double scale = 1.0 / std::max(l.one_norms()[0], 1e-300);
  // every launch of the timed terms is bracketed by events; one
  // synchronisation at the end (the stream runs back to back, as in a series)
  std::vector<cudaEvent_t> ev(static_cast<std::size_t>(4 * iters));
  for (auto& e : ev) QSWG_CHECK(cudaEventCreate(&e));
  for (int i = 0; i < pend_max + iters; ++i) {  // the first ring is warm-up
    const int it = i - pend_max;
    const double2* x = ring.k[i % ring.slots];
    auto mark = [&](int k) {
      if (it >= 0) QSWG_CHECK(cudaEventRecord(ev[static_cast<std::size_t>(4 * it + k)], s));
    };
    mark(0);
    dev::kron_prepare(mat, x, s);
    mark(1);
    dev::series_term(mat, x, ring.k[(i + 1) % ring.slots] + ex.row0, i + 1, false, scale, -1.0, ctl, true, s);
    mark(2);
    dev::series_flush(ring, ex.row0, ex.rows, z, ss,
                      (ex.single && mat.format == dev::Format::Kron && mat.kron.herm) ? static_cast<int>(l.n()) : 0,
                      i + 1, mat.group == 1, -1.0, ctl, true, s);
    mark(3);
  }
  QSWG_CHECK(cudaEventSynchronize(ev.back()));
  std::array<double, 4> acc{};
  for (int it = 0; it < iters; ++it)
    for (int k = 0; k < 3; ++k) {
      float t = 0.f;
      QSWG_CHECK(cudaEventElapsedTime(&t, ev[static_cast<std::size_t>(4 * it + k)], ev[static_cast<std::size_t>(4 * it + k + 1)]));
      acc[static_cast<std::size_t>(k)] += t;
    }
  float total = 0.f;
  QSWG_CHECK(cudaEventElapsedTime(&total, ev.front(), ev.back()));
  for (auto& e : ev) cudaEventDestroy(e);
  for (int k = 0; k < 3; ++k) acc[static_cast<std::size_t>(k)] /= iters;
  acc[3] = static_cast<double>(total) / iters;  // first prepare to last flush, per term
  return acc;
}

double time_series_term(const Liouvillian& l, int iters, int count) { return time_series_parts(l, iters, count)[3]; }

}  // namespace qswg
