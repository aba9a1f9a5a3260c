// In-process communicator: `world` ranks driven by `world` host threads of
// one process, all sharing one GPU (or several GPUs of one process).
//
// It exists to run the multi-GPU control flow of expm.cpp — partition, halo
// plan, per-term halo exchanges, allreduce(max) of the stop-test maxima,
// allreduce(sum) of populations — on a single device: every collective is a
// host-side rendezvous (each rank first drains its own stream, the last rank
// to arrive moves the data with cudaMemcpy, everyone resumes), so no kernel
// ever waits on another rank's kernel.  Production multi-GPU runs use
// comm_nccl.cpp.
#include <condition_variable>
#include <cstring>
#include <functional>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <vector>

#include "../../../include/qswg.h"
#include "comm.hpp"
#include "device.hpp"

namespace qswg {

namespace {

struct LocalGroup {
  explicit LocalGroup(int w) : world(w), slot(static_cast<std::size_t>(w)) {}
  int world;
  std::mutex m;
  std::condition_variable cv;
  int arrived = 0;
  unsigned long long generation = 0;
  std::vector<void*> slot;  // per-rank buffer of the current collective
};

class LocalComm final : public Comm {
 public:
  LocalComm(std::shared_ptr<LocalGroup> g, int rank) : g_(std::move(g)), rank_(rank) {}
  int rank() const override { return rank_; }
  int world() const override { return g_->world; }

  void allgather_rows(void* full, const std::vector<std::int64_t>& starts, std::size_t elem_bytes,
                      cudaStream_t s) override {
    collective(full, s, [&](const std::vector<void*>& bufs) {
      for (int r = 0; r < g_->world; ++r) {
        const std::size_t off = static_cast<std::size_t>(starts[static_cast<std::size_t>(r)]) * elem_bytes;
        const std::size_t cnt =
            static_cast<std::size_t>(starts[static_cast<std::size_t>(r) + 1] - starts[static_cast<std::size_t>(r)]) *
            elem_bytes;
        for (int q = 0; q < g_->world; ++q)
          if (q != r && cnt)
            QSWG_CHECK(cudaMemcpy(static_cast<char*>(bufs[static_cast<std::size_t>(q)]) + off,
                                  static_cast<char*>(bufs[static_cast<std::size_t>(r)]) + off, cnt,
                                  cudaMemcpyDefault));
      }
    });
  }

  void exchange_ranges(void* full, const std::vector<std::vector<std::int64_t>>& lo,
                       const std::vector<std::vector<std::int64_t>>& hi, std::size_t elem_bytes,
                       cudaStream_t s) override {
    collective(full, s, [&](const std::vector<void*>& bufs) {
      for (int r = 0; r < g_->world; ++r)
        for (int q = 0; q < g_->world; ++q) {
          const auto ur = static_cast<std::size_t>(r), uq = static_cast<std::size_t>(q);
          if (r == q || hi[ur][uq] <= lo[ur][uq]) continue;
          const std::size_t off = static_cast<std::size_t>(lo[ur][uq]) * elem_bytes;
          const std::size_t cnt = static_cast<std::size_t>(hi[ur][uq] - lo[ur][uq]) * elem_bytes;
          QSWG_CHECK(cudaMemcpy(static_cast<char*>(bufs[ur]) + off, static_cast<char*>(bufs[uq]) + off, cnt,
                                cudaMemcpyDefault));
        }
    });
  }

  void allreduce_max_u64(unsigned long long* buf, std::size_t n, cudaStream_t s) override {
    reduce<unsigned long long>(buf, n, s, [](unsigned long long& a, unsigned long long b) { a = a > b ? a : b; });
  }

  void allreduce_sum_f64(double* buf, std::size_t n, cudaStream_t s) override {
    reduce<double>(buf, n, s, [](double& a, double b) { a += b; });  // rank order: deterministic
  }

 private:
  template <class T, class Op>
  void reduce(T* buf, std::size_t n, cudaStream_t s, Op op) {
    collective(buf, s, [&](const std::vector<void*>& bufs) {
      std::vector<T> acc(n), tmp(n);
      QSWG_CHECK(cudaMemcpy(acc.data(), bufs[0], n * sizeof(T), cudaMemcpyDefault));
      for (std::size_t r = 1; r < bufs.size(); ++r) {
        QSWG_CHECK(cudaMemcpy(tmp.data(), bufs[r], n * sizeof(T), cudaMemcpyDefault));
        for (std::size_t i = 0; i < n; ++i) op(acc[i], tmp[i]);
      }
      for (void* b : bufs) QSWG_CHECK(cudaMemcpy(b, acc.data(), n * sizeof(T), cudaMemcpyDefault));
    });
  }

  // Rendezvous of all ranks on this collective; the last to arrive runs `fn`.
  void collective(void* mine, cudaStream_t s, const std::function<void(const std::vector<void*>&)>& fn) {
    QSWG_CHECK(cudaStreamSynchronize(s));
    std::unique_lock<std::mutex> lk(g_->m);
    g_->slot[static_cast<std::size_t>(rank_)] = mine;
    const unsigned long long gen = g_->generation;
    if (++g_->arrived == g_->world) {
      fn(g_->slot);
      // device-to-device cudaMemcpy may return before the copy completes and
      // the ranks' non-blocking streams do not order against it: drain it
      QSWG_CHECK(cudaDeviceSynchronize());
      g_->arrived = 0;
      ++g_->generation;
      g_->cv.notify_all();
    } else {
      g_->cv.wait(lk, [&] { return g_->generation != gen; });
    }
  }

  std::shared_ptr<LocalGroup> g_;
  int rank_;
};

}  // namespace

// Creates `world` linked in-process communicators (see file comment).
std::vector<std::unique_ptr<Comm>> make_local_comms(int world) {
  if (world < 1) throw std::invalid_argument("world size must be at least 1");
  auto g = std::make_shared<LocalGroup>(world);
  std::vector<std::unique_ptr<Comm>> out;
  for (int r = 0; r < world; ++r) out.push_back(std::make_unique<LocalComm>(g, r));
  return out;
}

}  // namespace qswg
