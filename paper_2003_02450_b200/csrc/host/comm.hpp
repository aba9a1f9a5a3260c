// Multi-GPU exchange interface (one process per GPU).
//
// Replaces the reference's in-process "communication" — direct reads of other
// workers' segments into `ext` (liouvillian.cpp:110-113, plan from
// partition.cpp:26-59) and host max-reductions over workers
// (expm.cpp:137-142) — with stream-ordered collectives.  The NCCL
// implementation lives in comm_nccl.cpp; world == 1 runs use no Comm at all.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <memory>
#include <vector>

namespace qswg {

class Comm {
 public:
  virtual ~Comm() = default;
  virtual int rank() const = 0;
  virtual int world() const = 0;
  /// `full` holds `starts.back()` elements of `elem_bytes`; rank r owns
  /// [starts[r], starts[r+1]).  Every rank's segment is broadcast in place.
  virtual void allgather_rows(void* full, const std::vector<std::int64_t>& starts, std::size_t elem_bytes,
                              cudaStream_t s) = 0;
  /// Halo exchange for the SpMV input: rank r needs, from every peer q, the
  /// contiguous global range needs[r][q] = {lo, hi} of q's segment.
  virtual void exchange_ranges(void* full, const std::vector<std::vector<std::int64_t>>& lo,
                               const std::vector<std::vector<std::int64_t>>& hi, std::size_t elem_bytes,
                               cudaStream_t s) = 0;
  /// Elementwise max over ranks of n uint64 (bit patterns of non-negative doubles).
  virtual void allreduce_max_u64(unsigned long long* buf, std::size_t n, cudaStream_t s) = 0;
  /// Elementwise sum over ranks of n doubles (populations).
  virtual void allreduce_sum_f64(double* buf, std::size_t n, cudaStream_t s) = 0;
};

/// `world` linked in-process communicators (comm_local.cpp): the multi-GPU
/// control flow driven by `world` host threads, e.g. on one GPU in tests.
std::vector<std::unique_ptr<Comm>> make_local_comms(int world);

}  // namespace qswg

/// C-ABI handle (include/qswg.h).
struct qswg_comm {
  std::unique_ptr<qswg::Comm> c;
};
