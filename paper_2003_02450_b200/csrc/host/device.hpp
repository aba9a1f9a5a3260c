// RAII device memory and the per-handle CUDA context (device, stream).
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <stdexcept>
#include <string>
#include <utility>

namespace qswg {

class CudaError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    if (e == cudaErrorMemoryAllocation) {
      cudaGetLastError();
      throw std::bad_alloc();
    }
    throw CudaError(std::string(what) + ": " + cudaGetErrorString(e));
  }
}
#define QSWG_CHECK(x) ::qswg::cuda_check((x), #x)

template <class T>
class DeviceBuffer {
 public:
  DeviceBuffer() = default;
  explicit DeviceBuffer(std::size_t n) { resize(n); }
  ~DeviceBuffer() { reset(); }
  DeviceBuffer(const DeviceBuffer&) = delete;
  DeviceBuffer& operator=(const DeviceBuffer&) = delete;
  DeviceBuffer(DeviceBuffer&& o) noexcept : p_(std::exchange(o.p_, nullptr)), n_(std::exchange(o.n_, 0)) {}
  DeviceBuffer& operator=(DeviceBuffer&& o) noexcept {
    if (this != &o) {
      reset();
      p_ = std::exchange(o.p_, nullptr);
      n_ = std::exchange(o.n_, 0);
    }
    return *this;
  }
  void resize(std::size_t n) {
    if (n == n_) return;
    reset();
    if (n) {
      QSWG_CHECK(cudaMalloc(&p_, n * sizeof(T)));
      n_ = n;
    }
  }
  void reset() {
    if (p_) cudaFree(p_);
    p_ = nullptr;
    n_ = 0;
  }
  T* get() const { return p_; }
  std::size_t size() const { return n_; }
  std::size_t bytes() const { return n_ * sizeof(T); }

 private:
  T* p_ = nullptr;
  std::size_t n_ = 0;
};

// Page-locked host memory (cudaHostAlloc): stream-ordered copies into it stay
// asynchronous, so several small reads share one synchronisation.
template <class T>
class PinnedBuffer {
 public:
  PinnedBuffer() = default;
  explicit PinnedBuffer(std::size_t n) { QSWG_CHECK(cudaHostAlloc(reinterpret_cast<void**>(&p_), n * sizeof(T), 0)); }
  ~PinnedBuffer() {
    if (p_) cudaFreeHost(p_);
  }
  PinnedBuffer(const PinnedBuffer&) = delete;
  PinnedBuffer& operator=(const PinnedBuffer&) = delete;
  T* get() const { return p_; }

 private:
  T* p_ = nullptr;
};

// Makes `device` current for the scope and restores the previous device.
class DeviceGuard {
 public:
  explicit DeviceGuard(int device) {
    cudaGetDevice(&prev_);
    if (device != prev_) QSWG_CHECK(cudaSetDevice(device));
  }
  ~DeviceGuard() { cudaSetDevice(prev_); }

 private:
  int prev_ = 0;
};

}  // namespace qswg
