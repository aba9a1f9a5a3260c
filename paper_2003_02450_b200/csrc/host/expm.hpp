// Exponential action on the device: the B200 counterparts of qsw::step and
// qsw::series (proj/core/include/qsw/expm.hpp:47-63).
//
// Vectors are device pointers to the caller's local segment of vec(rho)
// (column-major, expm state layout of state.hpp:10-12).  All launches go to
// the Liouvillian's stream; the host does not synchronise between Taylor
// terms on one GPU — the stop tests run on the device (cuda/taylor.cu).
#pragma once

#include <array>
#include <functional>
#include <vector>

#include "liouvillian.hpp"
#include "taylor.hpp"

namespace qswg {

struct StepInfo {
  std::int64_t m_star = 0;
  std::int64_t s = 1;
  std::int64_t spmvs = 0;     // Taylor terms actually evaluated
  std::int64_t launches = 0;  // kernels enqueued
};

struct SeriesInfo {
  int path = 0;  // 0: zero generator, 1: q sequential steps, 2: shared-term super-steps
  std::int64_t span_m_star = 0, span_s = 1;
  std::int64_t d = 0, n_super = 0, remainder = 0, sub_m_star = 0;
  std::int64_t spmvs = 0;
  std::int64_t launches = 0;  // kernels enqueued (emit() launches excluded)
  std::int64_t emits = 0;     // emit() calls
  bool graph = false;         // replayed from a captured CUDA graph
  // Several GPUs: times the host waited for the device (an event of a term's
  // stop flag kLag terms back, when the device was that far behind).  The
  // stream itself is synchronised once per call (the error / SpMV counters).
  std::int64_t host_waits = 0;
};

/// out = exp(t L) v.  `out` must not alias `v`.  Throws NumericalError on
/// non-finite values (expm.cpp:191-193).
StepInfo step(const Liouvillian& l, const double2* v, double t, const TaylorParameters& params,
              double2* out, int herm_known = -1);

/// Outputs at t1 + k (tq - t1)/steps, k = 0..steps (expm.cpp:214-325).  Each
/// output is handed to `emit(k, state)` as a device pointer valid until the
/// call returns (stream-ordered: enqueue copies on l.stream()).
///
/// A non-empty `graph_key` declares that `emit` only enqueues stream-ordered
/// device work whose targets are exactly the buffers listed in graph_key; then
/// a one-GPU call that repeats the previous call exactly (same v, times,
/// tolerance, graph_key buffers and Hermitian mode) is captured once into a CUDA graph and replayed by
/// later identical calls — the same kernels with the same arguments, minus the
/// per-launch host overhead (QSWG_GRAPH=0 disables).
/// herm_known: as Liouvillian::set_hermitian_input.  before_sync: enqueues
/// the caller's stream-ordered reads (D2H of the outputs) before the one
/// synchronisation of the call.
SeriesInfo series(const Liouvillian& l, const double2* v, double t1, double tq, std::int64_t steps,
                  const TaylorParameters& params,
                  const std::function<void(std::int64_t, const double2*)>& emit,
                  const std::vector<const void*>& graph_key = {}, int herm_known = -1,
                  const std::function<void()>& before_sync = {});

/// Mean device time (ms) of one fused series-term launch with `count`
/// active outputs (p > 1 traffic: K read, K write, count sums read+write),
/// `iters` back-to-back launches on the Liouvillian's stream.
double time_series_term(const Liouvillian& l, int iters, int count);
std::array<double, 4> time_series_parts(const Liouvillian& l, int iters, int count);

}  // namespace qswg
