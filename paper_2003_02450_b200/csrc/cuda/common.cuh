// Shared device helpers for the sm_100a kernels.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <stdexcept>
#include <string>

#include "../host/device.hpp"

namespace qswg::dev {

inline void check(cudaError_t e, const char* what) { ::qswg::cuda_check(e, what); }

#define QSWG_CUDA(x) ::qswg::dev::check((x), #x)
#define QSWG_LAUNCH_CHECK(name) ::qswg::dev::check(cudaGetLastError(), name)

constexpr int kThreads = 256;

// Resident blocks per SM of `kernel` at kThreads threads (cached per device
// and kernel: the occupancy query costs microseconds of host time, which
// would otherwise bound short launches).
inline int blocks_per_sm(const void* kernel, std::size_t smem = 0, int threads = 256) {
  struct Key {
    int dev;
    const void* k;
    std::size_t smem;
  };
  static thread_local Key keys[64];
  static thread_local int vals[64];
  static thread_local int used = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < used; ++i)
    if (keys[i].dev == dev && keys[i].k == kernel && keys[i].smem == smem) return vals[i];
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem);
  if (per_sm < 1) per_sm = 1;
  if (used < 64) {
    keys[used] = {dev, kernel, smem};
    vals[used++] = per_sm;
  }
  return per_sm;
}

inline int sm_count() {
  static thread_local int cached_dev = -1, cached = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev != cached_dev) {
    cudaDeviceGetAttribute(&cached, cudaDevAttrMultiProcessorCount, dev);
    cached_dev = dev;
  }
  return cached > 0 ? cached : 148;
}

// Non-negative doubles order like their uint64 bit patterns; NaN patterns
// sort above +Inf, so a max over bits flags any non-finite value.
__device__ __forceinline__ unsigned long long dbits(double x) {
  return static_cast<unsigned long long>(__double_as_longlong(x));
}
__device__ __forceinline__ double bitsd(unsigned long long b) {
  return __longlong_as_double(static_cast<long long>(b));
}
__device__ __forceinline__ unsigned long long umax64(unsigned long long a, unsigned long long b) {
  return a > b ? a : b;
}
__device__ __forceinline__ unsigned long long warp_max_bits(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = umax64(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
// Block-wide max of bit patterns; result valid in thread 0. `red` holds >= 32.
__device__ __forceinline__ unsigned long long block_max_bits(unsigned long long v,
                                                             unsigned long long* red) {
  v = warp_max_bits(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  if (w == 0) {
    v = l < static_cast<int>(blockDim.x >> 5) ? red[l] : 0ull;
    v = warp_max_bits(v);
  }
  return v;
}

// Streaming loads for data touched once per SpMV (values, columns): no L1
// allocation and an L2 evict-first policy, so L2 keeps the gathered vector.
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double2 ld_stream(const double2* p, unsigned long long pol) {
#ifdef QSWG_NO_HINTS
  (void)pol;
  return __ldg(p);
#endif
  double2 r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
      : "=d"(r.x), "=d"(r.y)
      : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_stream(const int* p, unsigned long long pol) {
#ifdef QSWG_NO_HINTS
  (void)pol;
  return __ldg(p);
#endif
  int r;
  asm("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ unsigned long long evict_last_policy() {
  unsigned long long pol;
  asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
// Gathered SpMV input (reused ~nnz/row times): read-only path, L2 evict-last.
__device__ __forceinline__ double2 ld_gather(const double2* p, unsigned long long pol) {
#ifdef QSWG_GATHER_HINT
  double2 r;
  asm("ld.global.nc.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;" : "=d"(r.x), "=d"(r.y) : "l"(p), "l"(pol));
  return r;
#else
  (void)pol;  // plain read-only load: measured faster than the L2 evict-last hint (c2 1.38x, c3 1.24x)
#ifdef QSWG_GATHER_FOLD  // experiment (wrong results): fold every 1 MB onto its first 512 B (L1-resident gathers)
#ifndef QSWG_GATHER_FOLD_MASK
#define QSWG_GATHER_FOLD_MASK 0xFFE00ull
#endif
  p = reinterpret_cast<const double2*>(reinterpret_cast<unsigned long long>(p) & ~QSWG_GATHER_FOLD_MASK);
#endif
  return __ldg(p);
#endif
}
// Read-modify-write vectors touched once per kernel (running sums): no L1
// allocation, L2 evict-first.  Volatile keeps the issue order the caller
// wrote (all loads of a chunk before its stores).
__device__ __forceinline__ double2 ld_once(const double2* p, unsigned long long pol) {
#ifdef QSWG_NO_HINTS
  (void)pol;
  return *p;
#endif
  double2 r;
  asm volatile("ld.global.L1::no_allocate.L2::cache_hint.v2.f64 {%0, %1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ void st_hint(double2* p, double2 v, unsigned long long pol) {
#ifdef QSWG_NO_HINTS
  (void)pol;
  *p = v;
  return;
#endif
  asm volatile("st.global.L1::no_allocate.L2::cache_hint.v2.f64 [%0], {%1, %2}, %3;" ::"l"(p), "d"(v.x),
               "d"(v.y), "l"(pol)
               : "memory");
}

// Programmatic dependent launch: every kernel of the Taylor loop is launched
// with programmatic stream serialisation.  Each kernel first waits for its
// predecessor's completion and memory (griddepcontrol.wait; a no-op without a
// programmatic predecessor); once its main work is done (before the final
// reductions and the stop test) it lets its dependents' CTAs be scheduled, so
// their launch overlaps this kernel's tail (triggering at the start was
// measured slower on c2: the waiting CTAs compete for SM slots).
__device__ __forceinline__ void pdl_prologue() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

template <class... KArgs, class... Args>
inline void launch_pdl(void (*kernel)(KArgs...), int grid, int block, std::size_t smem, cudaStream_t s,
                       Args... args) {
  static const bool off = [] {  // experiment knob: QSWG_PDL=0 launches plainly
    const char* e = std::getenv("QSWG_PDL");
    return e != nullptr && e[0] == '0';
  }();
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(static_cast<unsigned>(block));
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = off ? 0 : 1;
  QSWG_CUDA(cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...));
}

}  // namespace qswg::dev
