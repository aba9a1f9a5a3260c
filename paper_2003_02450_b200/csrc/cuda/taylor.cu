// The truncated-Taylor loop on sm_100a: fused SpMV + axpy + infinity-norm
// reductions + the early-termination test, all on the device.
//
// Replaces the reference's per-term WorkerPool rounds
//   worker_multiply (liouvillian.cpp:105-127) + the step axpy/norm loop
//   (expm.cpp:175-195) and the series lazy-term SpMV + per-k axpy/norm loops
//   (expm.cpp:283-316).
// The path is HBM-bound complex128 SpMV (~0.4 flop/B), so there are no
// tensor-core ops here.  Each block owns tiles of kTile = 256 consecutive
// rows (persistent grid-stride over tiles):
//   phase A  row groups of G lanes (G in {2,4,8,16,32}, autotuned per matrix)
//            compute the tile's row dot products from a shared-memory copy of
//            the tile's row pointers; values/columns stream with an L2
//            evict-first policy so the gathered vector stays L2-resident;
//   phase B  one thread per row runs the fused epilogue (scale, term write,
//            running-sum axpys for every active output, inf-norms) with fully
//            coalesced 16-byte accesses and all sum loads in flight at once.
// Grid-wide maxima use the uint64 bit order of non-negative doubles
// (order-independent, hence deterministic); the LAST block to arrive
// evaluates the stop test c1 + c2 <= tol * ||sum|| and publishes it for the
// next launch, so the host never synchronises inside a step or a series.
#include <cstdlib>
#include <string>
#include <utility>

#include "../kernels.hpp"
#include "common.cuh"

namespace qswg::dev {

namespace {

constexpr int kTile = kThreads;  // rows per block tile

__device__ __forceinline__ double cabs2(double2 v) { return hypot(v.x, v.y); }

// m = max(m, bits of |v|) with |v| = hypot as std::abs (expm.cpp:167, 182-183),
// evaluated only when it can raise the maximum: hypot(x, y) <= |x| + |y|
// (and CUDA's hypot is within 2 ulp), so an element with
// (|x| + |y|)(1 + 2^-48) <= max cannot change it.  NaN/Inf fail the test and
// reach hypot, so non-finite values are still flagged.
__device__ __forceinline__ void max_abs_bits(unsigned long long& m, double2 v) {
  if (!((fabs(v.x) + fabs(v.y)) * (1.0 + 0x1p-48) <= bitsd(m))) m = umax64(m, dbits(cabs2(v)));
}

// Sum of one row, computed by the G lanes of a group; every lane returns the
// full sum.  G == 1 is the bitwise "reference order" mode: one thread per
// row, columns in CSR order, every product and sum rounded separately (no
// FMA) — exactly `acc += vals[k] * x[...]` of liouvillian.cpp:120-124 in a
// no-FMA build.
template <int G>
__device__ __forceinline__ double2 row_dot(const CsrView& l, long long b, long long e,
                                           const double2* __restrict__ x, int lane,
                                           unsigned long long pol, unsigned long long xpol) {
  double2 acc = make_double2(0.0, 0.0);
  if constexpr (G == 1) {
    for (long long k = b; k < e; ++k) {
      const double2 v = ld_stream(l.val + k, pol);
      const double2 xv = ld_gather(x + ld_stream(l.col + k, pol), xpol);
      acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(v.x, xv.x), __dmul_rn(v.y, xv.y)));
      acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(v.x, xv.y), __dmul_rn(v.y, xv.x)));
    }
    return acc;
  } else {
    constexpr int U = G <= 8 ? 4 : 2;  // independent loads in flight per lane
    long long k = b + lane;
    for (; k + (U - 1) * G < e; k += U * G) {
      int c[U];
      double2 v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = ld_stream(l.col + k + u * G, pol);
#ifdef QSWG_GATHER_MASK  // experiment: confine the gathers to an L2-sized window
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] &= QSWG_GATHER_MASK;
#endif
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream(l.val + k + u * G, pol);
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = ld_gather(x + c[u], xpol);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x = fma(v[u].x, xv[u].x, acc.x);
        acc.x = fma(-v[u].y, xv[u].y, acc.x);
        acc.y = fma(v[u].x, xv[u].y, acc.y);
        acc.y = fma(v[u].y, xv[u].x, acc.y);
      }
    }
    for (; k < e; k += G) {
      int c0 = ld_stream(l.col + k, pol);
#ifdef QSWG_GATHER_MASK
      c0 &= QSWG_GATHER_MASK;
#endif
      const double2 v0 = ld_stream(l.val + k, pol);
      const double2 x0 = ld_gather(x + c0, xpol);
      acc.x = fma(v0.x, x0.x, acc.x);
      acc.x = fma(-v0.y, x0.y, acc.x);
      acc.y = fma(v0.x, x0.y, acc.y);
      acc.y = fma(v0.y, x0.x, acc.y);
    }
#pragma unroll
    for (int o = G / 2; o > 0; o >>= 1) {
      acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
      acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
    }
    return acc;
  }
}

// s + f * k; separately rounded in the bitwise mode (G == 1).
template <int G>
__device__ __forceinline__ double2 axpy(double2 s, double f, double2 k) {
  if constexpr (G == 1) {
    return make_double2(__dadd_rn(s.x, __dmul_rn(f, k.x)), __dadd_rn(s.y, __dmul_rn(f, k.y)));
  } else {
    return make_double2(s.x + f * k.x, s.y + f * k.y);
  }
}

// Persistent loop over row tiles.  Phase A fills tile_acc[] with the raw row
// sums (L x)_r of the tile; phase B calls epi(row, acc, valid) on every
// thread (one row each; `valid` is false past the last row, so epilogues may
// use full-warp shuffles).  Every thread of the block reaches both barriers.
template <int G, class Epi>
__device__ __forceinline__ void tile_loop(const CsrView& l, const double2* __restrict__ x, Epi&& epi) {
  __shared__ long long tile_ptr[kTile + 1];
  __shared__ double2 tile_acc[kTile];
  const unsigned long long pol = evict_first_policy(), xpol = evict_last_policy();
  constexpr int kGroups = kThreads / G;
  const int g = threadIdx.x / G, lane = threadIdx.x % G;
  for (long long base = static_cast<long long>(blockIdx.x) * kTile; base < l.rows;
       base += static_cast<long long>(gridDim.x) * kTile) {
    const int n_rows = static_cast<int>(min(static_cast<long long>(kTile), l.rows - base));
    __syncthreads();  // previous tile's phase B is done with tile_acc / tile_ptr
    for (int t = threadIdx.x; t <= n_rows; t += blockDim.x) tile_ptr[t] = __ldg(l.rowptr + base + t);
    __syncthreads();
#pragma unroll 1
    for (int j = 0; j < kTile / kGroups; ++j) {
      const int r = j * kGroups + g;
      const bool valid = r < n_rows;
      const long long b = valid ? tile_ptr[r] : 0, e = valid ? tile_ptr[r + 1] : 0;
      const double2 acc = row_dot<G>(l, b, e, x, lane, pol, xpol);
      if (lane == 0 && valid) tile_acc[r] = acc;
    }
    __syncthreads();
    const bool valid = static_cast<int>(threadIdx.x) < n_rows;
    epi(base + threadIdx.x, valid ? tile_acc[threadIdx.x] : make_double2(0.0, 0.0), valid);
  }
}

// ---------------------------------------------------------------- step term
// Stop test after one step term (expm.cpp:188-195), run by one thread of the
// last block to arrive.
__device__ void step_control(StepCtl* ctl, int first_of_stage, int stage, double tol) {
  const double c2 = bitsd(*(volatile unsigned long long*)&ctl->term_bits);
  const double nf = bitsd(*(volatile unsigned long long*)&ctl->sum_bits);
  ctl->spmvs += 1;
  if (!isfinite(c2) || !isfinite(nf)) {  // expm.cpp:191-193
    ctl->error = 1;
    ctl->done = 1;
  } else {
    // stage start: c1 = ||v|| (stage 0, from step_init) or ||sum|| of the
    // previous stage (expm.cpp:197-205), which is that stage's last nf.
    const double c1 = first_of_stage ? (stage == 0 ? ctl->c1 : ctl->last_nf) : ctl->c1;
    ctl->done = (c1 + c2 <= tol * nf) ? 1 : 0;  // expm.cpp:194
    ctl->c1 = c2;
    ctl->last_nf = nf;
  }
  ctl->term_bits = 0;
  ctl->sum_bits = 0;
  ctl->arrivals = 0;
}

struct StepTermArgs {
  CsrView l;
  const double2* x;
  double2* y;
  const double2* sum_in;
  double2* sum_out;
  double scale;
  double tol;
  StepCtl* ctl;
  int first_of_stage;
  int stage;
  int decide;
};

template <int G>
__global__ void __launch_bounds__(kThreads) step_term_kernel(StepTermArgs a) {
  pdl_prologue();
  StepCtl* ctl = a.ctl;
  if (*(volatile int*)&ctl->error) return;
  if (!a.first_of_stage && *(volatile int*)&ctl->done) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0, smax = 0;
  const unsigned long long once = evict_first_policy(), keep = evict_last_policy();
  tile_loop<G>(a.l, a.x, [&](long long row, double2 acc, bool valid) {
    if (!valid) return;
    // y = scale * acc with scale = Complex{t/(s*j), 0} (liouvillian.cpp:125)
    const double2 yv = make_double2(__dmul_rn(a.scale, acc.x), __dmul_rn(a.scale, acc.y));
    const double2 sv0 = ld_once(a.sum_in + row, once);
    st_hint(a.y + row, yv, keep);  // next term's SpMV input
    const double2 sv = make_double2(sv0.x + yv.x, sv0.y + yv.y);  // expm.cpp:181
    st_hint(a.sum_out + row, sv, once);
    max_abs_bits(tmax, yv);
    max_abs_bits(smax, sv);
  });
  pdl_trigger();
  tmax = block_max_bits(tmax, red);
  smax = block_max_bits(smax, red);
  if (threadIdx.x == 0) {
    atomicMax(&ctl->term_bits, tmax);
    atomicMax(&ctl->sum_bits, smax);
    __threadfence();
    if (atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1) {
      __threadfence();
      if (a.decide) {
        step_control(ctl, a.first_of_stage, a.stage, a.tol);
      } else {
        ctl->arrivals = 0;  // maxima stay for the allreduce + step_control_kernel
      }
    }
  }
}

// ------------------------------------------------------------- series term
// Stop tests of the super-step terms (expm.cpp:298-316, evaluated p-major)
// with deferred running sums (kernels.hpp: SeriesCtl).  Both controls run on
// the whole last block to arrive, one thread per output (or in a one-block
// kernel after the multi-GPU allreduce); every thread of the block calls them.
//
// After term p: c2_k = k^p ||K_p||.  The exact test c1_k + c2_k <= tol ||S_k||
// is settled without S_k when c1_k + c2_k > tol * ub_k, where
//   ub_k = (||S_k at the last flush|| + sum of the pending k^q ||K_q||) (1 + 2^-30)
// is computed with upward rounding: ||S_k|| <= ub_k holds through every
// rounding of the pending axpys and norms (each at most (1 + 2^-53)), so the
// settled outcome "continue" is the one the exact test would give.  Likewise
// "stop" is settled without S_k when c1_k + c2_k <= tol * lb_k,
//   lb_k = (||S_k at the last flush|| - pending bound) (1 - 2^-30)
// (downward rounding; used only while the pending bound is below 2^-20 of
// ||S_k||, where the 2^-30 slack covers the rounding of <= 64 pending axpys):
// the output stops at term p exactly as the reference's, and its pending
// terms join the next flush.  In the stop regime the terms are ~2^-53 ||S_k||,
// so an output's stop rarely needs a flush of its own.
__device__ void series_term_control(SeriesCtl* ctl, int p, int last, double tol) {
  static_assert(kMaxSeriesD <= kThreads, "one thread per output");
  __shared__ int pmin_sh;
  const int k = threadIdx.x;
  // every field this step reads, loaded up front: the control block sits in L2 and
  // this step is the tail of the term kernel that the next kernel's blocks wait for, so
  // its global round trips are taken once, in parallel, instead of one after another
  const double tn = bitsd(*(volatile unsigned long long*)&ctl->term_bits);
  const int count = ctl->count;
  const int slots_l = ctl->slots, pend_max_l = ctl->pend_max;
  const int kk = k < kMaxSeriesD ? k : 0;
  const int active_l = ctl->active[kk], pending_l = ctl->pending[kk], p0_l = ctl->p0[kk];
  const double factor_l = ctl->factor[kk], bound_l = ctl->bound[kk], nf_last_l = ctl->nf_last[kk], c1_l = ctl->c1[kk];
  if (k == 0) pmin_sh = p;
  __syncthreads();
  if (!isfinite(tn)) {  // expm.cpp:293-295
    if (k == 0) {
      ctl->spmvs += 1;
      ctl->error = 1;
      ctl->n_active = 0;
      ctl->term_bits = 0;
      ctl->arrivals = 0;
    }
    return;
  }
  const int slot = p % slots_l;
  const bool act = k < count && active_l;
  const bool pend = k < count && pending_l;
  if (act || pend) atomicMin(&pmin_sh, p0_l);
  __syncthreads();
  // the next term must not overwrite a pending one
  const bool full = last || p - pmin_sh + 1 >= pend_max_l;
  double f = 0.0;
  bool und = false, stop = false;
  if (act) {
    f = factor_l;
    ctl->fac_ring[slot][k] = f;
    const double bnd = __dadd_ru(bound_l, __dmul_ru(f, tn));
    ctl->bound[k] = bnd;
    const double nf0 = nf_last_l;
    const double ub = __dmul_ru(__dadd_ru(nf0, bnd), 1.0 + 0x1p-30);
    if (!(c1_l + f * tn > tol * ub)) {  // "continue" not settled (expm.cpp:310, 315)
      const double lb = bnd <= nf0 * 0x1p-20 ? __dmul_rd(__dsub_rd(nf0, bnd), 1.0 - 0x1p-30) : 0.0;
      stop = __dadd_rn(c1_l, __dmul_rn(f, tn)) <= __dmul_rd(tol, lb);  // c1 + c2 as expm.cpp:310-315 rounds it
#ifdef QSWG_NO_SETTLED_STOP  // experiment: every stop through a flush and the exact test
      stop = false;
#endif
      und = !stop;
    }
  }
  const bool running = __syncthreads_or(act && !stop);
  const bool pending_any = __syncthreads_or(pend || stop);
  // One undecidable test flushes every active output: each pending term is
  // then read once per super-step, and a large ring keeps flushes to the
  // outputs' stop events (measured cheaper than flushing the undecidable
  // outputs alone, which re-reads the shared terms per output).  When the
  // last active output stops, the pending ones are flushed right away.
  const bool any = __syncthreads_or(und) || full || (!running && pending_any);
  if (stop) {  // settled stop: done testing, terms p0 .. p pending
    ctl->active[k] = 0;
    ctl->pending[k] = 1;
    ctl->p_end[k] = p;
    ctl->mark[k] = 0;
  } else if (act) {
    ctl->mark[k] = any;
    if (!any) {  // every test settled: continue
      ctl->c1[k] = f * tn;
      ctl->factor[k] = f * static_cast<double>(k + 1);  // factor *= k for p + 1
    }
  }
  if (k == 0) {
    ctl->spmvs += 1;
    ctl->tn_last = tn;
    ctl->flush = any;
    ctl->term_bits = 0;
    ctl->arrivals = 0;
  }
}

// Exact tests of term p for the marked outputs after the flush wrote their sums.
__device__ void series_flush_control(SeriesCtl* ctl, int p, double tol) {
  __shared__ int stopped, err;
  const int k = threadIdx.x;
  const int count = ctl->count;
  const int slot = p % ctl->slots;
  const double tn = ctl->tn_last;
  if (k == 0) stopped = err = 0;
  __syncthreads();
  if (k < count && ctl->active[k] && ctl->mark[k]) {
    const double f = ctl->fac_ring[slot][k];
    const double c2 = f * tn;  // expm.cpp:310
    const double nf = bitsd(*(volatile unsigned long long*)&ctl->sum_bits[k]);
    if (!isfinite(nf)) {  // expm.cpp:312-314
      err = 1;
    } else if (ctl->c1[k] + c2 <= tol * nf) {  // expm.cpp:315
      ctl->active[k] = 0;
      atomicAdd(&stopped, 1);
    } else {
      ctl->c1[k] = c2;
    }
    ctl->factor[k] = f * static_cast<double>(k + 1);
    ctl->nf_last[k] = nf;
    ctl->bound[k] = 0.0;
    ctl->sum_bits[k] = 0;
    ctl->p0[k] = p + 1;
    ctl->fresh[k] = 0;
    ctl->mark[k] = 0;
  } else if (k < count && ctl->pending[k]) {  // stopped earlier, now summed
    ctl->pending[k] = 0;
    ctl->sum_bits[k] = 0;
    atomicAdd(&stopped, 1);
  }
  __syncthreads();
  if (k == 0) {
    if (err) ctl->error = 1;
    ctl->n_active = ctl->error ? 0 : ctl->n_active - stopped;
    ctl->flush = 0;
    ctl->arrivals = 0;
  }
}

struct SeriesTermArgs {
  const double2* x;
  double2* kp;
  int p;
  int last;
  double scale;
  double tol;
  SeriesCtl* ctl;
  int decide;
};

__device__ __forceinline__ bool series_skip(const SeriesCtl* ctl) {
  return *(volatile const int*)&ctl->error || *(volatile const int*)&ctl->n_active == 0;
}

// Term-kernel epilogue of one row: K_p = (h/p) L K_{p-1} (expm.cpp:286-287),
// kept in L2 for the next term's gathers and the flush.
__device__ __forceinline__ void series_store(double2* kp, double scale, long long row, double2 acc, bool valid,
                                             unsigned long long keep, unsigned long long& tmax) {
  if (!valid) return;
  const double2 kv = make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y));
  st_hint(kp + row, kv, keep);
  max_abs_bits(tmax, kv);
}

// Grid-wide ||K_p|| and the term control (last block).
__device__ __forceinline__ void series_term_finish(const SeriesTermArgs& a, unsigned long long tmax,
                                                   unsigned long long* red) {
  pdl_trigger();  // the main work is done: let the next kernel's CTAs in
  __shared__ int is_last;
  tmax = block_max_bits(tmax, red);
  SeriesCtl* ctl = a.ctl;
  if (threadIdx.x == 0) {
    atomicMax(&ctl->term_bits, tmax);
    __threadfence();
    is_last = atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1;
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
  if (a.decide) {
    series_term_control(ctl, a.p, a.last, a.tol);
  } else if (threadIdx.x == 0) {
    ctl->arrivals = 0;  // maximum stays for the allreduce + series_term_control_kernel
  }
}

template <int G>
__global__ void __launch_bounds__(kThreads) series_term_kernel(SeriesTermArgs a, CsrView l) {
  pdl_prologue();
  if (series_skip(a.ctl)) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0;
  const unsigned long long keep = evict_last_policy();
  double2* const kp = a.kp;
  const double scale = a.scale;
  tile_loop<G>(l, a.x, [&](long long row, double2 acc, bool valid) { series_store(kp, scale, row, acc, valid, keep, tmax); });
  series_term_finish(a, tmax, red);
}

struct SeriesFlushArgs {
  SeriesRing ring;
  long long row0, rows;
  const double2* z;
  SeriesSums sums;
  int p;
  double tol;
  SeriesCtl* ctl;
  int decide;
  int herm_n = 0;  // > 0: Hermitian tile flush over an n x n state (one GPU)
};

// Batched running-sum update of the marked outputs (kernels.hpp:
// series_flush).  The marked outputs are walked in chunks of kSeriesRegD
// with all their sum loads in flight; per chunk the pending terms are read
// once, oldest first (each output adds only terms from its own first pending
// one), so every output sums in term order as with per-term updates.
// Whether the flush after term a.p must run (block-uniform: the flag was set
// by the previous kernel).
__device__ __forceinline__ bool flush_due(const SeriesFlushArgs& a) {
  return *(volatile const int*)&a.ctl->flush && !series_skip(a.ctl);
}

// The outputs a flush updates (marked active and stopped-pending ones), with
// their pending-term ranges; built by thread 0, block-shared.
struct FlushList {
  int list[kMaxSeriesD];
  int q0[kMaxSeriesD];  // first pending term
  int q1[kMaxSeriesD];  // last pending term
  int fr[kMaxSeriesD];  // first flush: starts from Z
  unsigned long long smax[kMaxSeriesD];
  int nm;
};

__device__ __forceinline__ void flush_prepare(const SeriesFlushArgs& a, FlushList& L) {
  const SeriesCtl* ctl = a.ctl;
  if (threadIdx.x == 0) {
    int nm = 0;
    for (int k = 0; k < ctl->count; ++k) {
      const bool pend = ctl->pending[k];
      if ((ctl->active[k] && ctl->mark[k]) || pend) {
        L.list[nm] = k;
        L.q0[nm] = ctl->p0[k];
        L.q1[nm] = pend ? ctl->p_end[k] : a.p;
        L.fr[nm] = ctl->fresh[k];
        ++nm;
      }
    }
    L.nm = nm;
  }
  __syncthreads();
  for (int u = threadIdx.x; u < L.nm; u += blockDim.x) L.smax[u] = 0;
  __syncthreads();
}

// Norms into the control block; the last block to arrive runs the exact
// stop tests (kCoop: the caller does, after a grid barrier).
template <bool kCoop>
__device__ __forceinline__ void flush_finish(const SeriesFlushArgs& a, FlushList& L) {
  SeriesCtl* ctl = a.ctl;
  pdl_trigger();
  __syncthreads();
  for (int u = threadIdx.x; u < L.nm; u += blockDim.x) atomicMax(&ctl->sum_bits[L.list[u]], L.smax[u]);
  __syncthreads();
  if constexpr (kCoop) return;
  __shared__ int is_last;
  if (threadIdx.x == 0) {
    __threadfence();
    is_last = atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1;
    if (is_last) __threadfence();
  }
  __syncthreads();
  if (!is_last) return;
  if (a.decide) {
    series_flush_control(ctl, a.p, a.tol);
  } else if (threadIdx.x == 0) {
    ctl->arrivals = 0;
  }
}

#ifndef QSWG_FLUSH_UNROLL
#define QSWG_FLUSH_UNROLL 4  // c5 flush part 463 -> 425 us (1: 463, 8: 434); the full c5 series is unchanged (15.0 s)
#endif
constexpr int kFlushUnroll = QSWG_FLUSH_UNROLL;  // pending terms read per flush-loop step

// Sum updates of one element row (local index) for the outputs u0 .. u0 +
// kSeriesRegD of the list: sv[v] = S (or Z) + sum over its pending terms of
// k^q K_q, oldest first.
template <bool kStrict>
__device__ __forceinline__ void flush_element(const SeriesFlushArgs& a, const FlushList& L, int u0, long long row,
                                              bool valid, unsigned long long once, double2* sv) {
  const SeriesCtl* ctl = a.ctl;
  const int slots = ctl->slots, p = a.p, nm = L.nm;
  int lo = p + 1;
#pragma unroll
  for (int v = 0; v < kSeriesRegD; ++v) {
    const int u = u0 + v;
    sv[v] = make_double2(0.0, 0.0);
    if (u < nm) {
      lo = L.q0[u] < lo ? L.q0[u] : lo;
      if (valid) sv[v] = ld_once((L.fr[u] ? a.z : a.sums.s[L.list[u]]) + row, once);
    }
  }
#pragma unroll kFlushUnroll
  for (int q = lo; q <= p; ++q) {  // sum += k^q K_q (expm.cpp:300-305)
    const int sl = q % slots;
    const double2 kv = valid ? __ldg(a.ring.k[sl] + a.row0 + row) : make_double2(0.0, 0.0);
#pragma unroll
    for (int v = 0; v < kSeriesRegD; ++v) {
      const int u = u0 + v;
      if (u < nm && q >= L.q0[u] && q <= L.q1[u] && valid) {
        const double f = ctl->fac_ring[sl][L.list[u]];  // block-uniform
        sv[v] = kStrict ? axpy<1>(sv[v], f, kv) : axpy<2>(sv[v], f, kv);
      }
    }
  }
}

// Norm maxima of the outputs a flush updates.  kReg: per-thread maxima of the
// first 2 kSeriesRegD outputs in registers, reduced once per block (the
// flush fused into the 64-register W kernel: c2 flush 8.0 -> 6.2 us per
// term); otherwise (and past those outputs) a warp reduction per element,
// which keeps the stand-alone streaming flush kernel at 46 registers (its
// occupancy is its bandwidth: with the register maxima at 60-71 registers
// the c5 flush went from 437 to 550-690 us per term).
template <bool kReg>
struct FlushMax {
  unsigned long long m[2][kSeriesRegD];
  __device__ __forceinline__ FlushMax() {
    if constexpr (kReg) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < kSeriesRegD; ++v) m[c][v] = 0;
    }
  }
  // the norm of the output u0 + v (v a constant) from element value sv
  __device__ __forceinline__ void add(FlushList& L, int u0, int v, double2 sv, bool valid) {
    if (kReg && u0 == 0) {
      if (valid) max_abs_bits(m[0][v], sv);
    } else if (kReg && u0 == kSeriesRegD) {
      if (valid) max_abs_bits(m[1][v], sv);
    } else {
      unsigned long long mk = valid ? dbits(cabs2(sv)) : 0ull;
      mk = warp_max_bits(mk);
      if ((threadIdx.x & 31) == 0 && mk) atomicMax(&L.smax[u0 + v], mk);
    }
  }
  __device__ __forceinline__ void done(FlushList& L) {
    if constexpr (kReg) {
#pragma unroll
      for (int c = 0; c < 2; ++c)
#pragma unroll
        for (int v = 0; v < kSeriesRegD; ++v) {
          const int u = c * kSeriesRegD + v;
          if (u >= L.nm) continue;  // block-uniform
          const unsigned long long mk = warp_max_bits(m[c][v]);
          if ((threadIdx.x & 31) == 0 && mk) atomicMax(&L.smax[u], mk);
        }
    }
  }
};

// The flush work of one block over all local rows (every thread calls it).
template <bool kStrict, bool kCoop = false, bool kReg = false>
__device__ __forceinline__ void flush_body(const SeriesFlushArgs& a) {
  __shared__ FlushList L;
  flush_prepare(a, L);
  const int nm = L.nm;
  const unsigned long long once = evict_first_policy();
  const long long stride = static_cast<long long>(gridDim.x) * blockDim.x;
  FlushMax<kReg> fm;
  for (long long base = static_cast<long long>(blockIdx.x) * blockDim.x; base < a.rows; base += stride) {
    const long long row = base + threadIdx.x;
    const bool valid = row < a.rows;
#pragma unroll 1
    for (int u0 = 0; u0 < nm; u0 += kSeriesRegD) {
      double2 sv[kSeriesRegD];
      flush_element<kStrict>(a, L, u0, row, valid, once, sv);
#pragma unroll
      for (int v = 0; v < kSeriesRegD; ++v) {
        const int u = u0 + v;
        if (u >= nm) break;  // block-uniform
        if (valid) st_hint(a.sums.s[L.list[u]] + row, sv[v], once);
        fm.add(L, u0, v, sv[v], valid);
      }
    }
  }
  fm.done(L);
  flush_finish<kCoop>(a, L);
}

// Hermitian flush (KRON Hermitian path, one GPU: every pending term and sum is
// exactly Hermitian, a.herm_n = n): only the upper elements i <= j are
// computed, in 32 x 8 sub-tiles of the upper 32 x 32 tiles, and each is
// written twice, S(j, i) = conj S(i, j), through a shared-memory transpose.
// The mirrored element is bit-identical to what the element-wise flush
// computes (conj is exact and the axpys are symmetric in the sign of the
// imaginary parts), so the pending terms and sums are read for half the
// elements only.
// One upper 32 x 32 tile t of the Hermitian flush (in 32 x 8 sub-tiles).
using FlushTr = double2[kSeriesRegD][8][33];
template <bool kReg>
__device__ __forceinline__ void flush_herm_tile(const SeriesFlushArgs& a, FlushList& L, FlushTr& tr, long long t,
                                                FlushMax<kReg>& fm, unsigned long long once) {
  const int nm = L.nm, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int n = a.herm_n;
  int J = static_cast<int>((sqrt(8.0 * static_cast<double>(t) + 1.0) - 1.0) * 0.5);
  while (static_cast<long long>(J) * (J + 1) / 2 > t) --J;
  while (static_cast<long long>(J + 1) * (J + 2) / 2 <= t) ++J;
  const int I = static_cast<int>(t - static_cast<long long>(J) * (J + 1) / 2);
#pragma unroll 1
  for (int sub = 0; sub < 4; ++sub) {
    const int i = I * 32 + lane, j = J * 32 + sub * 8 + w;
    const bool upper = i < n && j < n && i <= j;
    const long long row = static_cast<long long>(j) * n + i;
    // mirror target of this thread after the transpose: row i2 of the
    // sub-tile's columns, column j2 (8 consecutive j per 8 threads)
    const int i2 = I * 32 + (threadIdx.x >> 3), j2 = J * 32 + sub * 8 + (threadIdx.x & 7);
    const bool mirror = i2 < n && j2 < n && i2 < j2;
#pragma unroll 1
    for (int u0 = 0; u0 < nm; u0 += kSeriesRegD) {
      double2 sv[kSeriesRegD];
      flush_element<false>(a, L, u0, row, upper, once, sv);
#pragma unroll
      for (int v = 0; v < kSeriesRegD; ++v) {
        const int u = u0 + v;
        if (u >= nm) break;  // block-uniform
        if (upper) st_hint(a.sums.s[L.list[u]] + row, sv[v], once);
        fm.add(L, u0, v, sv[v], upper);
        tr[v][w][lane] = sv[v];
      }
      __syncthreads();
#pragma unroll
      for (int v = 0; v < kSeriesRegD; ++v) {
        const int u = u0 + v;
        if (u >= nm) break;
        if (mirror) {  // element (j2, i2) = conj of the computed (i2, j2)
          const double2 m = tr[v][threadIdx.x & 7][threadIdx.x >> 3];
          st_hint(a.sums.s[L.list[u]] + static_cast<long long>(i2) * n + j2, make_double2(m.x, -m.y), once);
        }
      }
      __syncthreads();
    }
  }
}

template <bool kReg = false, bool kCoop = false>
__device__ __forceinline__ void flush_body_herm(const SeriesFlushArgs& a) {
  __shared__ FlushList L;
  __shared__ FlushTr tr;
  flush_prepare(a, L);
  const int nt = (a.herm_n + 31) / 32;
  const long long ntiles = static_cast<long long>(nt) * (nt + 1) / 2;
  const unsigned long long once = evict_first_policy();
  FlushMax<kReg> fm;
  for (long long t = blockIdx.x; t < ntiles; t += gridDim.x) flush_herm_tile(a, L, tr, t, fm, once);
  fm.done(L);
  flush_finish<kCoop>(a, L);
}

template <bool kStrict>
__global__ void __launch_bounds__(kThreads) series_flush_kernel(SeriesFlushArgs a) {
  pdl_prologue();
  if (!flush_due(a)) return;
  if (a.herm_n > 0) {
    flush_body_herm(a);
  } else {
    flush_body<kStrict>(a);
  }
}

// ------------------------------------------------------------- SELL path
// One warp per 32-row slice, one lane per row (kernels.hpp: SellView).
template <bool kStrict>
__device__ __forceinline__ double2 sell_dot(const int* __restrict__ col, const double2* __restrict__ val, long long b,
                                            int len, int lane, const double2* __restrict__ x, unsigned long long pol,
                                            unsigned long long xpol) {
  double2 acc = make_double2(0.0, 0.0);
  const int* cp = col + b + lane;
  const double2* vp = val + b + lane;
  int k = 0;
  if constexpr (!kStrict) {
#ifndef QSWG_SELL_U
#define QSWG_SELL_U 4
#endif
    constexpr int U = QSWG_SELL_U;  // entries per lane in flight
    for (; k + U <= len; k += U) {
      int c[U];
      double2 v[U], xv[U];
#pragma unroll
      for (int u = 0; u < U; ++u) c[u] = ld_stream(cp + (k + u) * kSlice, pol);
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = ld_stream(vp + (k + u) * kSlice, pol);
#pragma unroll
      for (int u = 0; u < U; ++u) xv[u] = ld_gather(x + c[u], xpol);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        acc.x = fma(v[u].x, xv[u].x, acc.x);
        acc.x = fma(-v[u].y, xv[u].y, acc.x);
        acc.y = fma(v[u].x, xv[u].y, acc.y);
        acc.y = fma(v[u].y, xv[u].x, acc.y);
      }
    }
  }
  for (; k < len; ++k) {
    const double2 v = ld_stream(vp + k * kSlice, pol);
    const double2 xv = ld_gather(x + ld_stream(cp + k * kSlice, pol), xpol);
    if constexpr (kStrict) {  // CSR order, separately rounded (liouvillian.cpp:120-124)
      acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(v.x, xv.x), __dmul_rn(v.y, xv.y)));
      acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(v.x, xv.y), __dmul_rn(v.y, xv.x)));
    } else {
      acc.x = fma(v.x, xv.x, acc.x);
      acc.x = fma(-v.y, xv.y, acc.x);
      acc.y = fma(v.x, xv.y, acc.y);
      acc.y = fma(v.y, xv.x, acc.y);
    }
  }
  return acc;
}

// Warp-uniform loop over slices; epi(row, acc, valid) runs on every lane.
//
// Static path (SellView::work == nullptr): warp w takes slices w, w + nwarps,
// ... and loads values and columns through registers (sell_dot).
//
// Streamed path (SellView::work): the matrix stream never passes through
// registers.  Every warp owns a ring of kSellStages shared-memory stages; one
// lane keeps the ring full with 1-D bulk copies (cp.async.bulk, completion on
// an mbarrier per stage) of kSellPiece slots at a time — the values and
// columns of consecutive slices are contiguous, so a chunk of slices is one
// byte range — while the warp consumes the oldest stage: columns and values
// from shared memory, the gathers of x from L2.  The bytes in flight per SM
// (what an HBM-bound kernel needs: bandwidth x latency) are then set by the
// ring depth instead of by registers and occupancy, and they no longer drain
// at the end of every slice (the column panels of c4 have ~30 entries per row).
// Chunks of consecutive slices are drawn from a device counter, so no warp
// idles while another still holds a long share and the warps of the grid walk
// the matrix (and the gathered columns of x) front to front; the first chunk
// of a warp is its own index (no draw), the next chunk's descriptor is loaded
// and the one after is drawn while the current one is processed.  Every warp
// makes exactly one draw past the end, so the draw returning the launch's
// last value zeroes the counter for the next launch.
// Per row the entries are accumulated in slot order on both paths (identical
// results).
#ifndef QSWG_SELL_MIN_BLOCKS
#define QSWG_SELL_MIN_BLOCKS 2  // two CTAs of 8 rings per SM (<= 128 registers: no spills)
#endif
#ifndef QSWG_SELL_PIECE
#define QSWG_SELL_PIECE 4
#endif
constexpr int kSellPiece = QSWG_SELL_PIECE;                            // slots (32 entries each) per bulk copy
#ifndef QSWG_SELL_STAGES
#define QSWG_SELL_STAGES 4
#endif
constexpr int kSellStages = QSWG_SELL_STAGES;
#ifndef QSWG_SELL_GROUP
#define QSWG_SELL_GROUP 2
#endif
constexpr int kSellGroup = QSWG_SELL_GROUP;  // pieces consumed per round (their gathers in flight together)
constexpr int kSellStageVal = kSellPiece * kSlice * 16;  // bytes of values per stage
constexpr int kSellStageCol = kSellPiece * kSlice * 4;
constexpr int kSellWarpBytes = kSellStages * (kSellStageVal + kSellStageCol);
constexpr int kSellWarps = kThreads / 32;
constexpr std::size_t kSellSmemBytes = static_cast<std::size_t>(kSellWarps) * (kSellWarpBytes + kSellStages * 8);
constexpr int kSellTargetSlots = 96;  // slots per chunk aimed at
constexpr int kSellMaxChunk = 31;     // slices per chunk (their slice_ptr entries fit one warp load)

__device__ __forceinline__ unsigned smem_addr(const void* p) {
  return static_cast<unsigned>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned ok;
  do {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(ok)
        : "r"(bar), "r"(parity)
        : "memory");
  } while (!ok);
}
__device__ __forceinline__ void bulk_load(unsigned dst, const void* src, unsigned bytes, unsigned bar,
                                          unsigned long long pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(bar), "l"(pol)
      : "memory");
}
__device__ __forceinline__ unsigned draw_chunk(unsigned* ctr, int lane) {
  unsigned v = 0;
  if (lane == 0) v = atomicAdd(ctr, 1u);
  return __shfl_sync(0xffffffffu, v, 0);
}

template <bool kStrict>
__device__ __forceinline__ void sell_mac(double2& acc, double2 v, double2 xv) {
  if constexpr (kStrict) {  // CSR order, separately rounded (liouvillian.cpp:120-124)
    acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(v.x, xv.x), __dmul_rn(v.y, xv.y)));
    acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(v.x, xv.y), __dmul_rn(v.y, xv.x)));
  } else {
    acc.x = fma(v.x, xv.x, acc.x);
    acc.x = fma(-v.y, xv.y, acc.x);
    acc.y = fma(v.x, xv.y, acc.y);
    acc.y = fma(v.y, xv.x, acc.y);
  }
}

// A chunk of consecutive slices as the streamed path sees it.
struct SellChunk {
  long long s0 = 0;   // first slice
  long long e0 = 0;   // first entry
  int ns = 0;         // slices (0: no chunk)
  int nslots = 0;     // 32-entry slots
  int npieces = 0;
  int issued = 0;     // pieces handed to the copy engine
};

template <bool kStrict, class Epi>
__device__ __forceinline__ void slice_stream(const SellView& m, const double2* __restrict__ x, Epi&& epi) {
  extern __shared__ __align__(128) unsigned char sell_smem[];
  const unsigned long long pol = evict_first_policy();
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* const ring = sell_smem + wib * kSellWarpBytes;
  const double2* const sval = reinterpret_cast<const double2*>(ring);
  const int* const scol = reinterpret_cast<const int*>(ring + kSellStages * kSellStageVal);
  const unsigned ring_a = smem_addr(ring);
  const unsigned bar_a = smem_addr(sell_smem + kSellWarps * kSellWarpBytes) + wib * kSellStages * 8;
  if (lane == 0) {
#pragma unroll
    for (int st = 0; st < kSellStages; ++st) mbar_init(bar_a + 8 * st, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncwarp();

  const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
  const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
  // Slices per chunk (grid-uniform): ~kSellTargetSlots slots, but at least ~8 chunks per warp.
  const long long total_slots = __ldg(m.slice_ptr + m.n_slices) / kSlice;
  long long chunk = total_slots > 0 ? (kSellTargetSlots * m.n_slices) / total_slots : kSellMaxChunk;
  const long long fair = m.n_slices / (8 * nwarps);
  if (chunk > fair) chunk = fair;
  chunk = chunk < 1 ? 1 : (chunk > kSellMaxChunk ? kSellMaxChunk : chunk);
  const long long n_chunks = (m.n_slices + chunk - 1) / chunk;
  const unsigned last_draw =
      static_cast<unsigned>((n_chunks > nwarps ? n_chunks - nwarps : 0) + nwarps - 1);

  // Descriptor of chunk c; sp = this lane's slice_ptr entry (lane k: start of slice k of the chunk).
  auto describe = [&](long long c, SellChunk& ch, long long& sp) {
    ch = SellChunk{};
    if (c >= n_chunks) return;
    ch.s0 = c * chunk;
    const long long left = m.n_slices - ch.s0;
    ch.ns = static_cast<int>(left < chunk ? left : chunk);
    sp = lane <= ch.ns ? __ldg(m.slice_ptr + ch.s0 + lane) : 0;
    ch.e0 = __shfl_sync(0xffffffffu, sp, 0);
    ch.nslots = static_cast<int>((__shfl_sync(0xffffffffu, sp, ch.ns) - ch.e0) / kSlice);
    ch.npieces = (ch.nslots + kSellPiece - 1) / kSellPiece;
  };
  unsigned issued_total = 0, consumed_total = 0;  // running piece counters: stage = n % stages, parity = (n / stages) & 1
  auto issue_piece = [&](SellChunk& ch) {
    const int p = ch.issued++;
    const int st = static_cast<int>(issued_total % kSellStages);
    ++issued_total;
    if (lane == 0) {
      const int slots = ch.nslots - p * kSellPiece < kSellPiece ? ch.nslots - p * kSellPiece : kSellPiece;
      const long long e = ch.e0 + static_cast<long long>(p) * (kSellPiece * kSlice);
      const unsigned bar = bar_a + 8 * st;
      mbar_expect_tx(bar, static_cast<unsigned>(slots) * (kSlice * 20));
      bulk_load(ring_a + st * kSellStageVal, m.val + e, static_cast<unsigned>(slots) * (kSlice * 16), bar, pol);
      bulk_load(ring_a + kSellStages * kSellStageVal + st * kSellStageCol, m.col + e,
                static_cast<unsigned>(slots) * (kSlice * 4), bar, pol);
    }
  };

  SellChunk cur, nxt;
  long long sp_cur = 0, sp_nxt = 0;
  describe(warp, cur, sp_cur);
  unsigned raw = draw_chunk(m.work, lane);  // pending draw: the chunk after nxt
  bool drawing = true;                      // false once a draw went past the end
  auto take_draw = [&](SellChunk& ch, long long& sp) {  // turns the pending draw into a descriptor, draws again
    ch = SellChunk{};
    if (!drawing) return;
    const long long c = static_cast<long long>(raw) + nwarps;
    if (c < n_chunks) {
      describe(c, ch, sp);
      raw = draw_chunk(m.work, lane);
    } else {
      drawing = false;
      if (lane == 0 && raw == last_draw) *m.work = 0u;
    }
  };
  take_draw(nxt, sp_nxt);
  auto refill = [&]() {  // fills the free stages while pieces are left
#pragma unroll 1
    while (issued_total - consumed_total < static_cast<unsigned>(kSellStages)) {
      if (cur.issued < cur.npieces) {
        issue_piece(cur);
      } else if (nxt.issued < nxt.npieces) {
        issue_piece(nxt);
      } else {
        break;
      }
    }
  };
  refill();

  while (cur.ns > 0) {
    // Walk the chunk: g = slot index in the chunk, k = slice in the chunk.
    int k = 0, g = 0;
    int slice_end = static_cast<int>((__shfl_sync(0xffffffffu, sp_cur, 1) - cur.e0) / kSlice);
    long long slot = cur.s0 * kSlice + lane;
    bool valid = slot < m.rows;
    long long row = m.perm && valid ? static_cast<long long>(__ldg(m.perm + slot)) : slot;
    double2 pp = m.part_in && valid ? ld_once(m.part_in + row, pol) : make_double2(0.0, 0.0);
    double2 acc = make_double2(0.0, 0.0);
    auto next_slice = [&]() {  // finishes slice k, starts slice k + 1
      if (m.part_in) acc = make_double2(pp.x + acc.x, pp.y + acc.y);  // earlier column panels first, then this one
      epi(row, acc, valid);
      ++k;
      acc = make_double2(0.0, 0.0);
      if (k < cur.ns) {
        slice_end = static_cast<int>((__shfl_sync(0xffffffffu, sp_cur, k + 1) - cur.e0) / kSlice);
        slot = (cur.s0 + k) * kSlice + lane;
        valid = slot < m.rows;
        row = m.perm && valid ? static_cast<long long>(__ldg(m.perm + slot)) : slot;
        pp = m.part_in && valid ? ld_once(m.part_in + row, pol) : make_double2(0.0, 0.0);
      }
    };
    // kSellGroup pieces per round: their gathers are all in flight together.
#pragma unroll 1
    for (int p = 0; p < cur.npieces; p += kSellGroup) {
      double2 v[kSellGroup][kSellPiece], xv[kSellGroup][kSellPiece];
      const int left = cur.nslots - p * kSellPiece;  // slots of this round: min(left, group * piece)
#pragma unroll
      for (int q = 0; q < kSellGroup; ++q) {
        if (q * kSellPiece < left) {
          const unsigned n = consumed_total + q;
          const int st = static_cast<int>(n % kSellStages);
          mbar_wait(bar_a + 8 * st, (n / kSellStages) & 1u);
          const int* pc = scol + st * (kSellPiece * kSlice) + lane;
#pragma unroll
          for (int u = 0; u < kSellPiece; ++u)
            if (q * kSellPiece + u < left) xv[q][u] = ld_gather(x + pc[u * kSlice], 0ull);
        }
      }
#pragma unroll
      for (int q = 0; q < kSellGroup; ++q) {
        if (q * kSellPiece < left) {
          const int st = static_cast<int>((consumed_total + q) % kSellStages);
          const double2* pv = sval + st * (kSellPiece * kSlice) + lane;
#pragma unroll
          for (int u = 0; u < kSellPiece; ++u)
            if (q * kSellPiece + u < left) v[q][u] = pv[u * kSlice];
        }
      }
      __syncwarp();  // every lane has read the stages: they can be refilled
      consumed_total += left > (kSellGroup - 1) * kSellPiece ? kSellGroup : (left + kSellPiece - 1) / kSellPiece;
      refill();
#pragma unroll
      for (int q = 0; q < kSellGroup; ++q) {
#pragma unroll
        for (int u = 0; u < kSellPiece; ++u) {
          if (q * kSellPiece + u < left) {
            while (g == slice_end) next_slice();
            sell_mac<kStrict>(acc, v[q][u], xv[q][u]);
            ++g;
          }
        }
      }
    }
    while (k < cur.ns) next_slice();  // the last slice and any empty ones after it
    cur = nxt;
    sp_cur = sp_nxt;
    take_draw(nxt, sp_nxt);
    refill();
  }
}

template <bool kStrict, class Epi>
__device__ __forceinline__ void slice_body(const SellView& m, const double2* __restrict__ x, long long sl, int lane,
                                           unsigned long long pol, unsigned long long xpol, Epi&& epi) {
  const long long b = __ldg(m.slice_ptr + sl);
  const int len = static_cast<int>((__ldg(m.slice_ptr + sl + 1) - b) / kSlice);
  double2 acc = sell_dot<kStrict>(m.col, m.val, b, len, lane, x, pol, xpol);
  const long long slot = sl * kSlice + lane;
  const bool valid = slot < m.rows;
  const long long row = m.perm && valid ? static_cast<long long>(__ldg(m.perm + slot)) : slot;
  if (m.part_in && valid) {  // earlier column panels first, then this one
    const double2 pp = ld_once(m.part_in + row, pol);
    acc = make_double2(pp.x + acc.x, pp.y + acc.y);
  }
  epi(row, acc, valid);
}

// Fused B (x) I windows (kernels.hpp: SellView::b_val).  Blocks draw windows
// of win_slices slices from a device counter (first window = the block's own
// index; the launch's last draw zeroes the counter).  Per window: the
// natural-order B (x) I sums of its rows go to shared memory (every row once:
// sums[row - window start]), then each sorted slice adds the sum of its row —
// (B part) + (the rest), then the earlier panels' partial sum as on the other
// paths.
template <bool kStrict, class Epi>
__device__ __forceinline__ void slice_windows(const SellView& m, const double2* __restrict__ x, int lane,
                                              unsigned long long pol, unsigned long long xpol, Epi&& epi) {
  __shared__ double2 sums[kSellWindowSlices * kSlice];
  __shared__ long long next_window;
  const int wib = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const long long n_windows = (m.n_slices + m.win_slices - 1) / m.win_slices;
  const long long nb = gridDim.x;
  const unsigned last_draw =
      static_cast<unsigned>((n_windows > nb ? n_windows - nb : 0) + (n_windows < nb ? n_windows : nb) - 1);
  long long win = blockIdx.x;
  while (win < n_windows) {
    const long long s0 = win * m.win_slices;
    const long long s1 = s0 + m.win_slices < m.n_slices ? s0 + m.win_slices : m.n_slices;
    for (long long sl = s0 + wib; sl < s1; sl += wpb) {  // natural order: slot = row
      const long long b = __ldg(m.b_slice_ptr + sl);
      const int len = static_cast<int>((__ldg(m.b_slice_ptr + sl + 1) - b) / kSlice);
      sums[(sl - s0) * kSlice + lane] = sell_dot<kStrict>(m.b_col, m.b_val, b, len, lane, x, pol, xpol);
    }
    __syncthreads();
    for (long long sl = s0 + wib; sl < s1; sl += wpb) {
      const long long b = __ldg(m.slice_ptr + sl);
      const int len = static_cast<int>((__ldg(m.slice_ptr + sl + 1) - b) / kSlice);
      double2 acc = sell_dot<kStrict>(m.col, m.val, b, len, lane, x, pol, xpol);
      const long long slot = sl * kSlice + lane;
      const bool valid = slot < m.rows;
      const long long row = m.perm && valid ? static_cast<long long>(__ldg(m.perm + slot)) : slot;
      if (valid) {
        const double2 bs = sums[row - s0 * kSlice];
        acc = make_double2(bs.x + acc.x, bs.y + acc.y);
        if (m.part_in) {
          const double2 pp = ld_once(m.part_in + row, pol);
          acc = make_double2(pp.x + acc.x, pp.y + acc.y);
        }
      }
      epi(row, acc, valid);
    }
    __syncthreads();  // (the sums are read; the draw below is the block's)
    if (threadIdx.x == 0) {
      const unsigned r = atomicAdd(m.win_work, 1u);
      const long long wn = static_cast<long long>(r) + nb;
      if (wn >= n_windows && r == last_draw) *m.win_work = 0u;
      next_window = wn;
    }
    __syncthreads();
    win = next_window;
  }
}

// kMode: the SELL kernels are instantiated per path, each with the register
// budget it was measured best at: kSellReg (registers, grid-stride slices),
// kSellStream (the matrix streamed through shared memory, SellView::work) and
// kSellWindows (fused B (x) I windows, SellView::b_val).
constexpr int kSellReg = 0, kSellStream = 1, kSellWindows = 2;
template <bool kStrict, int kMode, class Epi>
__device__ __forceinline__ void slice_loop(const SellView& m, const double2* __restrict__ x, Epi&& epi) {
  if constexpr (kMode == kSellStream) {
    slice_stream<kStrict>(m, x, epi);
  } else {
    const unsigned long long pol = evict_first_policy(), xpol = evict_last_policy();
    const int lane = threadIdx.x & 31;
    if constexpr (kMode == kSellWindows) {
      slice_windows<kStrict>(m, x, lane, pol, xpol, epi);
    } else {
      const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
      const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
      for (long long sl = warp; sl < m.n_slices; sl += nwarps) slice_body<kStrict>(m, x, sl, lane, pol, xpol, epi);
    }
  }
}
// Resident blocks per SM asked of ptxas: the streamed path holds its rings in
// shared memory (2 blocks of 8 rings, <= 128 registers); the register path
// hides the latency of its scattered gathers with warps (3 blocks, <= 85
// registers: c3 0.79 -> 0.82 of HBM, c4 0.70 -> 0.74; 4 blocks: 0.78 / 0.72).
#ifndef QSWG_SELL_REG_MIN_BLOCKS
#define QSWG_SELL_REG_MIN_BLOCKS 3
#endif
template <int kMode>
constexpr int sell_min_blocks() {
  return kMode == kSellStream ? QSWG_SELL_MIN_BLOCKS : QSWG_SELL_REG_MIN_BLOCKS;
}

// Skip test of the partial-panel kernels: the same early exits as the term
// kernel they precede.
struct SkipCheck {
  const SeriesCtl* series = nullptr;
  const StepCtl* step = nullptr;
  int first_of_stage = 1;
};
__device__ __forceinline__ bool skip_now(const SkipCheck& k) {
  if (k.series) return series_skip(k.series);
  if (k.step)
    return *(volatile const int*)&k.step->error || (!k.first_of_stage && *(volatile const int*)&k.step->done);
  return false;
}

// One earlier column panel: part[row] (=|+=) its row sums.
template <bool kFirst, int kMode>
__global__ void __launch_bounds__(kThreads, sell_min_blocks<kMode>())
    sell_partial_kernel(SellView m, const double2* x, double2* part, SkipCheck sk) {
  pdl_prologue();
  if (skip_now(sk)) return;
  const unsigned long long once = evict_first_policy();
  slice_loop<false, kMode>(m, x, [&](long long row, double2 acc, bool valid) {
    if (!valid) return;
    if constexpr (!kFirst) {
      const double2 pp = ld_once(part + row, once);
      acc = make_double2(pp.x + acc.x, pp.y + acc.y);
    }
    part[row] = acc;
  });
  pdl_trigger();
}

template <bool kStrict, int kMode>
__global__ void __launch_bounds__(kThreads, sell_min_blocks<kMode>())
    sell_spmv_kernel(SellView m, const double2* x, double2* y, double scale) {
  pdl_prologue();
  slice_loop<kStrict, kMode>(m, x, [&](long long row, double2 acc, bool valid) {
    if (valid) y[row] = make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y));
  });
}

struct SellStepArgs {
  SellView m;
  const double2* x;
  double2* y;
  const double2* sum_in;
  double2* sum_out;
  double scale;
  double tol;
  StepCtl* ctl;
  int first_of_stage;
  int stage;
  int decide;
};

template <bool kStrict, int kMode>
__global__ void __launch_bounds__(kThreads, sell_min_blocks<kMode>()) sell_step_term_kernel(SellStepArgs a) {
  pdl_prologue();
  StepCtl* ctl = a.ctl;
  if (*(volatile int*)&ctl->error) return;
  if (!a.first_of_stage && *(volatile int*)&ctl->done) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0, smax = 0;
  const unsigned long long once = evict_first_policy(), keep = evict_last_policy();
  slice_loop<kStrict, kMode>(a.m, a.x, [&](long long row, double2 acc, bool valid) {
    if (!valid) return;
    const double2 yv = make_double2(__dmul_rn(a.scale, acc.x), __dmul_rn(a.scale, acc.y));
    const double2 sv0 = ld_once(a.sum_in + row, once);
    st_hint(a.y + row, yv, keep);
    const double2 sv = make_double2(sv0.x + yv.x, sv0.y + yv.y);  // expm.cpp:181
    st_hint(a.sum_out + row, sv, once);
    max_abs_bits(tmax, yv);
    max_abs_bits(smax, sv);
  });
  pdl_trigger();
  tmax = block_max_bits(tmax, red);
  smax = block_max_bits(smax, red);
  if (threadIdx.x == 0) {
    atomicMax(&ctl->term_bits, tmax);
    atomicMax(&ctl->sum_bits, smax);
    __threadfence();
    if (atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1) {
      __threadfence();
      if (a.decide) {
        step_control(ctl, a.first_of_stage, a.stage, a.tol);
      } else {
        ctl->arrivals = 0;  // maxima stay for the allreduce + step_control_kernel
      }
    }
  }
}

template <bool kStrict, int kMode>
__global__ void __launch_bounds__(kThreads, sell_min_blocks<kMode>())
    sell_series_term_kernel(SeriesTermArgs a, SellView m) {
  pdl_prologue();
  if (series_skip(a.ctl)) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0;
  const unsigned long long keep = evict_last_policy();
  double2* const kp = a.kp;
  const double scale = a.scale;
  slice_loop<kStrict, kMode>(m, a.x, [&](long long row, double2 acc, bool valid) { series_store(kp, scale, row, acc, valid, keep, tmax); });
  series_term_finish(a, tmax, red);
}

// ------------------------------------------------------------ Kron path
#ifndef QSWG_KRON_MIN_BLOCKS
#define QSWG_KRON_MIN_BLOCKS 4  // <= 64 registers: 4 resident blocks of 256 threads per SM
#endif

// Matrix-free action (kernels.hpp: KronView), in 32 x 32 tiles of X.
// Per element the terms are summed in the order
//   A, R_1 .. R_nk (row-indexed operands),  P_1 .. P_nk, B, S_1 .. S_nk,
//   (A_ii + B_jj), T, decay (column-indexed operands and the diagonal terms;
//   A and B of G-QSW are stored without their diagonals),
// in every path, so the Hermitian path reproduces the general one bit for bit.
//
// General path: lane = rho row i, warp w = rho columns j0 + 4w .. j0 + 4w + 3.
// Row-indexed operands are per lane (sliced ELL when padding is small, so the
// operand loads are coalesced), each entry loaded once for 4 columns with 4
// gathers in flight; column-indexed operand rows are warp-uniform and their
// gathers X(i, c), W_k(i, a), V_k(i, a) stream coalesced columns.
//
// Hermitian path (X = X', one GPU): only tiles I <= J, and the row-indexed
// part is computed transposed — warp w = rows i0 + 4w + r, lane = column j —
// from X(c, j) = conj X(j, c) = conj x[n c + j], so those gathers are
// coalesced too and every operand row is warp-uniform; the partial sums meet
// in shared memory, the column-indexed part continues in the normal
// orientation, and the tile is written twice (Y(j, i) = conj Y(i, j)).
constexpr int kKT = 32;                      // tile edge
constexpr int kKR = kKT / (kThreads / 32);   // columns (rows) per thread (4)

__device__ __forceinline__ void cfma(double2& acc, double2 v, double2 xv) {
  acc.x = fma(v.x, xv.x, acc.x);
  acc.x = fma(-v.y, xv.y, acc.x);
  acc.y = fma(v.x, xv.y, acc.y);
  acc.y = fma(v.y, xv.x, acc.y);
}
__device__ __forceinline__ double2 conj2(double2 v) { return make_double2(v.x, -v.y); }

// Operand value classes (KronView::vk_*).  Every operand of the BASELINE
// configs is purely real (R_k, P_k, S_k, Q_k, T) or purely imaginary (A, B
// and their diagonals: the coherent -i(1-w)H parts): those multiply with 2
// FMAs instead of 4 and load 8 bytes instead of 16.  The products dropped are
// exact zeros, so every class gives the complex formula's values.  With
// kValConst every entry holds the same value (unweighted lattices, the
// coherent part of any unweighted graph), taken from the kernel parameters
// instead of being loaded.
template <int K, bool C>
__device__ __forceinline__ double2 opv(const double2* p, double2 cv) {
  if constexpr (C) {
    return cv;
  } else if constexpr (K == kValReal) {
    return make_double2(__ldg(&p->x), 0.0);
  } else if constexpr (K == kValImag) {
    return make_double2(0.0, __ldg(&p->y));
  } else {
    return __ldg(p);
  }
}
template <int K>
__device__ __forceinline__ double2 ldv(const double2* p) {
  return opv<K, false>(p, double2{});
}
template <int K>
__device__ __forceinline__ void cfmak(double2& acc, double2 v, double2 xv) {
  if constexpr (K == kValReal) {
    acc.x = fma(v.x, xv.x, acc.x);
    acc.y = fma(v.x, xv.y, acc.y);
  } else if constexpr (K == kValImag) {
    acc.x = fma(-v.y, xv.y, acc.x);
    acc.y = fma(v.y, xv.x, acc.y);
  } else {
    cfma(acc, v, xv);
  }
}
template <int K>
using ValK = std::integral_constant<int, K>;
template <bool C>
using ConstK = std::integral_constant<bool, C>;
// f(ValK<class>{}, ConstK<constant>{}) for the runtime (warp-uniform) code k.
template <class F>
__device__ __forceinline__ void by_kind(int k, F&& f) {
  const bool c = (k & kValConst) != 0;
  switch (k & 3) {
    case kValReal:
      if (c) {
        f(ValK<kValReal>{}, ConstK<true>{});
      } else {
        f(ValK<kValReal>{}, ConstK<false>{});
      }
      break;
    case kValImag:
      if (c) {
        f(ValK<kValImag>{}, ConstK<true>{});
      } else {
        f(ValK<kValImag>{}, ConstK<false>{});
      }
      break;
    default:
      f(ValK<kValComplex>{}, ConstK<false>{});
  }
}
#define QSWG_KC(kc, cc)                     \
  constexpr int K = decltype(kc)::value;    \
  constexpr bool C = decltype(cc)::value;   \
  (void)0

// Element offsets are 32-bit (dim <= 46340^2 < 2^31): base + unsigned offset
// is one wide multiply-add.  Column lists the gathers scale by n hold c * n
// already (kernels.hpp: KronView).
__device__ __forceinline__ double2 gat(const double2* base, unsigned off, unsigned long long pol) {
  (void)pol;  // plain read-only load (common.cuh: ld_gather)
  double2 r;
  // one IMAD.WIDE.U32 for the address: written out, so the compiler does not
  // re-associate base + off into 64-bit index arithmetic
  asm("{\n\t.reg .b64 qa;\n\tmad.wide.u32 qa, %2, 16, %3;\n\tld.global.nc.v2.f64 {%0, %1}, [qa];\n\t}"
      : "=d"(r.x), "=d"(r.y)
      : "r"(off), "l"(base));
  return r;
}

// Row-indexed part at (i, j[r]), lane = row i: A then R_k (general path).
// kF: the factored G-QSW dissipator is present (1) or not (0); the kernels
// are instantiated per case (KronView::factored).
template <int kF>
__device__ __forceinline__ void kron_rows_lane(const KronView& m, const double2* __restrict__ x, int i,
                                               const int* j, double2* acc, unsigned long long xpol) {
  const unsigned n = static_cast<unsigned>(m.n);
  unsigned jn[kKR];
#pragma unroll
  for (int r = 0; r < kKR; ++r) jn[r] = static_cast<unsigned>(j[r]) * n;
  if (m.a_ell.sptr) {  // I (x) A: columns j of X, operand rows in sliced ELL
    const int sl = i >> 5, lane = i & 31;
    const int b = __ldg(m.a_ell.sptr + sl), len = (__ldg(m.a_ell.sptr + sl + 1) - b) >> 5;
    const int* cp = m.a_ell.col + b + lane;
    const double2* vp = m.a_ell.val + b + lane;
    // (padded slices: the padding's zero values must be loaded, not the constant)
    by_kind(m.vk_a & 3, [&](auto kc, auto cc) {
      QSWG_KC(kc, cc);
#pragma unroll 2
      for (int e = 0; e < len; ++e) {
        const unsigned c = static_cast<unsigned>(__ldg(cp + 32 * e));
        const double2 v = opv<K, C>(vp + 32 * e, m.cv_a);
#pragma unroll
        for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(x, jn[r] + c, xpol));
      }
    });
  } else if (m.a.ptr) {
    const int e0 = __ldg(m.a.ptr + i), e1 = __ldg(m.a.ptr + i + 1);
    by_kind(m.vk_a, [&](auto kc, auto cc) {
      QSWG_KC(kc, cc);
#pragma unroll 2
      for (int e = e0; e < e1; ++e) {
        const unsigned c = static_cast<unsigned>(__ldg(m.a.col + e));
        const double2 v = opv<K, C>(m.a.val + e, m.cv_a);
#pragma unroll
        for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(x, jn[r] + c, xpol));
      }
    });
  }
  if constexpr (kF == 1) {
    for (int k = 0; k < m.nk; ++k) {  // -w/2 L'(L X): columns j of W_k
      const KronList& rk = m.r[k];
      if (rk.ptr == nullptr) continue;
      const int e0 = __ldg(rk.ptr + i), e1 = __ldg(rk.ptr + i + 1);
      const double2* wk = m.w[k];
      by_kind(m.vk_r[k], [&](auto kc, auto cc) {
        QSWG_KC(kc, cc);
#pragma unroll 2
        for (int e = e0; e < e1; ++e) {
          const unsigned c = static_cast<unsigned>(__ldg(rk.col + e));
          const double2 v = opv<K, C>(rk.val + e, m.cv_r[k]);
#pragma unroll
          for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(wk, jn[r] + c, xpol));
        }
      });
    }
  }
}

// acc += sum over operand row `row` of val * g(col) (warp-uniform row).
#ifndef QSWG_ROW_UNROLL
#define QSWG_ROW_UNROLL 4
#endif
constexpr int kRowUnroll = QSWG_ROW_UNROLL;
template <int K, bool C, class G>
__device__ __forceinline__ void uniform_row(const KronList& l, double2 cv, int row, double2& acc, G&& g) {
  if (l.ptr == nullptr) return;
  const int e1 = __ldg(l.ptr + row + 1);
#pragma unroll kRowUnroll
  for (int e = __ldg(l.ptr + row); e < e1; ++e)
    cfmak<K>(acc, opv<K, C>(l.val + e, cv), g(static_cast<unsigned>(__ldg(l.col + e))));
}

// acc[r] += sum over operand row rows[r] of val * g(col) for r < kKR, one
// row after the other.  (Walking the kKR rows in lockstep was measured
// slower on c2-c4.)
template <int K, bool C, class G>
__device__ __forceinline__ void uniform_rows(const KronList& l, double2 cv, const int* rows, double2* acc, G&& g) {
  if (l.ptr == nullptr) return;  // an operand without entries (e.g. a zero Lindblad operator)
#pragma unroll
  for (int r = 0; r < kKR; ++r) uniform_row<K, C>(l, cv, rows[r], acc[r], g);
}

// acc[r] += sum_k E(row0 + r, k) g(col) over the kKR consecutive rows row0 ..
// row0 + 3 (row0 = 32 slice + l0) of a uniform-slice ELL operand of len <= 8
// entries per row: one warp load fetches all their column indices, which are
// shuffled out, so the index -> gather chain skips an L1 round trip.  The
// entries of each row are added in their stored order.
template <int K, bool C, int L, class G>
__device__ __forceinline__ void shfl_rows_len(const KronEll& e, double2 cv, int len, int base, int mycol, int l0,
                                              double2* acc, G&& g) {
  // L > 0: the row length as a constant (fully unrolled, constant shuffle lanes)
  const int n_e = L > 0 ? L : len;
#pragma unroll(L > 0 ? L : 2)
  for (int k = 0; k < n_e; ++k) {
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const unsigned c = static_cast<unsigned>(__shfl_sync(0xffffffffu, mycol, kKR * k + r));
      cfmak<K>(acc[r], opv<K, C>(e.val + base + 32 * k + l0 + r, cv), g(c));
    }
  }
}
template <int K, bool C, class G>
__device__ __forceinline__ void shfl_rows(const KronEll& e, double2 cv, int len, int slice, int l0, double2* acc,
                                          G&& g) {
  const int lane = threadIdx.x & 31;
  const int base = slice * 32 * len;  // one row length in every slice (host: uniform_row_length)
  const int kt = lane >> 2, rt = lane & 3;
  const int mycol = kt < len ? __ldg(e.col + base + 32 * kt + l0 + rt) : 0;
  if (len == 4) {  // square lattices (c2)
    shfl_rows_len<K, C, 4>(e, cv, len, base, mycol, l0, acc, g);
  } else if (len == 6) {  // cubic lattices (c5)
    shfl_rows_len<K, C, 6>(e, cv, len, base, mycol, l0, acc, g);
  } else {
    shfl_rows_len<K, C, 0>(e, cv, len, base, mycol, l0, acc, g);
  }
}

// shfl_rows with the slice's entry offset and this lane's column index
// already in registers (the staged path loads them a tile ahead).
template <int K, bool C, class G>
__device__ __forceinline__ void shfl_rows_pre(const double2* val, double2 cv, int len, int base, int mycol, int l0,
                                              double2* acc, G&& g) {
  const KronEll e{nullptr, nullptr, val};
  if (len == 4) {
    shfl_rows_len<K, C, 4>(e, cv, len, base, mycol, l0, acc, g);
  } else if (len == 6) {
    shfl_rows_len<K, C, 6>(e, cv, len, base, mycol, l0, acc, g);
  } else {
    shfl_rows_len<K, C, 0>(e, cv, len, base, mycol, l0, acc, g);
  }
}

// W_0 = Q_0 X and AX = A X from the same gathers (KronView::ax): acc from
// Q's values, aacc from A's values aligned to Q's entries; the same per-row
// entry order as shfl_rows / uniform_rows, so each sum is the one its own
// list would give.
template <int KQ, bool CQ, int KA, bool CA, int L, class G>
__device__ __forceinline__ void shfl_rows2_len(const KronEll& e, const double2* aval, double2 cvq, double2 cva, int len,
                                               int base, int mycol, int l0, double2* acc, double2* aacc, G&& g) {
  const int n_e = L > 0 ? L : len;
#pragma unroll(L > 0 ? L : 2)
  for (int k = 0; k < n_e; ++k) {
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const unsigned c = static_cast<unsigned>(__shfl_sync(0xffffffffu, mycol, kKR * k + r));
      const double2 xv = g(c);
      cfmak<KQ>(acc[r], opv<KQ, CQ>(e.val + base + 32 * k + l0 + r, cvq), xv);
      cfmak<KA>(aacc[r], opv<KA, CA>(aval + base + 32 * k + l0 + r, cva), xv);
    }
  }
}
template <int KQ, bool CQ, int KA, bool CA, class G>
__device__ __forceinline__ void shfl_rows2(const KronEll& e, const double2* aval, double2 cvq, double2 cva, int len,
                                           int slice, int l0, double2* acc, double2* aacc, G&& g) {
  const int lane = threadIdx.x & 31;
  const int base = slice * 32 * len;
  const int kt = lane >> 2, rt = lane & 3;
  const int mycol = kt < len ? __ldg(e.col + base + 32 * kt + l0 + rt) : 0;
  if (len == 4) {
    shfl_rows2_len<KQ, CQ, KA, CA, 4>(e, aval, cvq, cva, len, base, mycol, l0, acc, aacc, g);
  } else if (len == 6) {
    shfl_rows2_len<KQ, CQ, KA, CA, 6>(e, aval, cvq, cva, len, base, mycol, l0, acc, aacc, g);
  } else {
    shfl_rows2_len<KQ, CQ, KA, CA, 0>(e, aval, cvq, cva, len, base, mycol, l0, acc, aacc, g);
  }
}
template <int KQ, bool CQ, int KA, bool CA, class G>
__device__ __forceinline__ void uniform_rows2(const KronList& l, const double2* aval, double2 cvq, double2 cva,
                                              const int* rows, double2* acc, double2* aacc, G&& g) {
  if (l.ptr == nullptr) return;
#pragma unroll
  for (int r = 0; r < kKR; ++r) {
    const int e1 = __ldg(l.ptr + rows[r] + 1);
#pragma unroll kRowUnroll
    for (int e = __ldg(l.ptr + rows[r]); e < e1; ++e) {
      const double2 xv = g(static_cast<unsigned>(__ldg(l.col + e)));
      cfmak<KQ>(acc[r], opv<KQ, CQ>(l.val + e, cvq), xv);
      cfmak<KA>(aacc[r], opv<KA, CA>(aval + e, cva), xv);
    }
  }
}
// f(ValK<Q class>, ConstK<Q const>, ValK<A class>, ConstK<A const>) for the
// AX combination (Q real, A imaginary; KronView::ax guarantees it).
template <class F>
__device__ __forceinline__ void by_kind_ax(int kq, int ka, F&& f) {
  const bool cq = (kq & kValConst) != 0, ca = (ka & kValConst) != 0;
  if (cq) {
    if (ca) {
      f(ValK<kValReal>{}, ConstK<true>{}, ValK<kValImag>{}, ConstK<true>{});
    } else {
      f(ValK<kValReal>{}, ConstK<true>{}, ValK<kValImag>{}, ConstK<false>{});
    }
  } else {
    if (ca) {
      f(ValK<kValReal>{}, ConstK<false>{}, ValK<kValImag>{}, ConstK<true>{});
    } else {
      f(ValK<kValReal>{}, ConstK<false>{}, ValK<kValImag>{}, ConstK<false>{});
    }
  }
}

// Row-indexed part, transposed (Hermitian path): acc[r] at (i[r], j), warp-
// uniform rows i[r], lane = column j: A from conj X(j, c), R_k from the
// row-major copy Wt_k (Wt_k[n b + j] = W_k(b, j)).  Column lists pre-scaled.
template <int kF>
__device__ __forceinline__ void kron_rows_uniform(const KronView& m, const double2* __restrict__ x, const int* i,
                                                  int j, double2* acc, unsigned long long xpol) {
  const unsigned n = static_cast<unsigned>(m.n);
  const double2* xj = x + j;
  // rows i[r] = I*32 + 4w + r: lanes 4w .. 4w+3 of ELL slice I (clamped edge rows read
  // that slice's padding lanes, whose results are discarded)
  const int sl = i[0] >> 5, l0 = (threadIdx.x >> 5) * kKR;
  if (m.ax) {  // A's part = AX(i, j), formed by the W kernel (KronView::ax)
#pragma unroll
    for (int r = 0; r < kKR; ++r) acc[r] = gat(m.axt + j, static_cast<unsigned>(i[r]) * n, xpol);
  } else {
    by_kind(m.vk_a, [&](auto kc, auto cc) {
      QSWG_KC(kc, cc);
      const auto g = [&](unsigned cn) { return conj2(gat(xj, cn, xpol)); };
      if (m.a_len > 0) {
        shfl_rows<K, C>(m.a_ellu, m.cv_a, m.a_len, sl, l0, acc, g);
      } else if (m.a_sc.ptr) {
        uniform_rows<K, C>(m.a_sc, m.cv_a, i, acc, g);
      }
    });
  }
  if constexpr (kF == 1) {
    for (int k = 0; k < m.nk; ++k) {
      const double2* wtj = m.wt[k] + j;
      by_kind(m.vk_r[k], [&](auto kc, auto cc) {
        QSWG_KC(kc, cc);
        const auto g = [&](unsigned cn) { return gat(wtj, cn, xpol); };
        if (m.r_len[k] > 0) {
          shfl_rows<K, C>(m.r_ellu[k], m.cv_r[k], m.r_len[k], sl, l0, acc, g);
        } else {
          uniform_rows<K, C>(m.r_sc[k], m.cv_r[k], i, acc, g);
        }
      });
    }
  }
  if (m.p_rows) {  // P_k(j, a) W_k(i, a), lane = j: padding-free ELL rows of P_k, rows i of Wt_k
    const int sj = j >> 5, ln = j & 31;
    for (int k = 0; k < m.nk; ++k) {
      const KronEll& pe = m.p_ell[k];
      const double2* wr[kKR];
#pragma unroll
      for (int r = 0; r < kKR; ++r) wr[r] = m.wt[k] + static_cast<unsigned>(i[r]) * n;
      const int b = __ldg(pe.sptr + sj), len = (__ldg(pe.sptr + sj + 1) - b) >> 5;
      by_kind(m.vk_p[k], [&](auto kc, auto cc) {
        QSWG_KC(kc, cc);
#pragma unroll 2
        for (int e = 0; e < len; ++e) {
          const unsigned a = static_cast<unsigned>(__ldg(pe.col + b + 32 * e + ln));
          const double2 v = opv<K, C>(pe.val + b + 32 * e + ln, m.cv_p[k]);
#pragma unroll
          for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(wr[r], a, xpol));
        }
      });
    }
  }
  if (m.b_rows && !m.ax) {  // B(j, c) X(i, c) = B(j, c) conj x[n i + c], lane = j: padding-free ELL rows of B
    const int sj = j >> 5, ln = j & 31;
    const KronEll& be = m.b_ell;
    const double2* xr[kKR];
#pragma unroll
    for (int r = 0; r < kKR; ++r) xr[r] = x + static_cast<unsigned>(i[r]) * n;
    const int b = __ldg(be.sptr + sj), len = (__ldg(be.sptr + sj + 1) - b) >> 5;
    by_kind(m.vk_b, [&](auto kc, auto cc) {
      QSWG_KC(kc, cc);
#pragma unroll 2
      for (int e = 0; e < len; ++e) {
        const unsigned c = static_cast<unsigned>(__ldg(be.col + b + 32 * e + ln));
        const double2 v = opv<K, C>(be.val + b + 32 * e + ln, m.cv_b);
#pragma unroll
        for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, conj2(gat(xr[r], c, xpol)));
      }
    });
  }
}

// Column-indexed part and diagonal terms at (i, j[r]), lane = row i.
// kHerm: V_k = X L_k' = W_k' for Hermitian X, so V_k(i, a) = conj Wt_k[n a + i]
// and no V_k is built.  (B, P_k, S_k lists and the S_k uniform ELL hold c * n.)
template <class XL>
__device__ __forceinline__ void kron_tail(const KronView& m, const double2* __restrict__ x, int i, const int* j,
                                          double2* acc, unsigned long long xpol, XL&& xl);

template <bool kHerm, int kF>
__device__ __forceinline__ void kron_cols(const KronView& m, const double2* __restrict__ x, int i, const int* j,
                                          double2* acc, unsigned long long xpol) {
  const unsigned n = static_cast<unsigned>(m.n);
  if (!(kHerm && m.p_rows)) {  // (the Hermitian tiles applied P_k in the transposed section)
    for (int k = 0; k < m.nk; ++k) {
      const double2* wi = m.w[k] + i;  // P_k (x) Q_k = P_k applied to the columns of W_k = Q_k X
      by_kind(m.vk_p[k], [&](auto kc, auto cc) {
        QSWG_KC(kc, cc);
        uniform_rows<K, C>(m.p[k], m.cv_p[k], j, acc, [&](unsigned cn) { return gat(wi, cn, xpol); });
      });
    }
  }
  if (kHerm && m.ax) {  // B's part = conj AX(j, i) (KronView::ax), added as one sum
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const double2 b = gat(m.axt + i, static_cast<unsigned>(j[r]) * n, xpol);
      acc[r].x += b.x;
      acc[r].y -= b.y;
    }
  } else if (m.b.ptr && !(kHerm && m.b_rows)) {  // B (x) I: coalesced columns c of X
    const double2* xi = x + i;
    by_kind(m.vk_b, [&](auto kc, auto cc) {
      QSWG_KC(kc, cc);
      const auto g = [&](unsigned cn) { return gat(xi, cn, xpol); };
      if (m.b_sep) {  // summed on its own, then added: the association of the AX path
#pragma unroll
        for (int r = 0; r < kKR; ++r) {
          double2 bs = make_double2(0.0, 0.0);
          uniform_row<K, C>(m.b, m.cv_b, j[r], bs, g);
          acc[r].x += bs.x;
          acc[r].y += bs.y;
        }
      } else {
        uniform_rows<K, C>(m.b, m.cv_b, j, acc, g);
      }
    });
  }
  if constexpr (kF == 1) {
    for (int k = 0; k < m.nk; ++k) {  // -w/2 (X L') L: columns of V_k
      by_kind(m.vk_s[k], [&](auto kc, auto cc) {
        QSWG_KC(kc, cc);
        if constexpr (kHerm) {
          const double2* vi = m.wt[k] + i;
          const auto g = [&](unsigned cn) { return conj2(gat(vi, cn, xpol)); };
          if (m.s_len[k] > 0) {  // rows j[r] = J*32 + 4w + r: lanes 4w .. 4w+3 of slice J
            shfl_rows<K, C>(m.s_ellu[k], m.cv_s[k], m.s_len[k], j[0] >> 5, (threadIdx.x >> 5) * kKR, acc, g);
          } else {
            uniform_rows<K, C>(m.s[k], m.cv_s[k], j, acc, g);
          }
        } else {
          const double2* vi = m.v[k] + i;
          uniform_rows<K, C>(m.s[k], m.cv_s[k], j, acc, [&](unsigned cn) { return gat(vi, cn, xpol); });
        }
      });
    }
  }
  const double2* xij[kKR];
#pragma unroll
  for (int r = 0; r < kKR; ++r) xij[r] = x + (static_cast<unsigned>(j[r]) * n + static_cast<unsigned>(i));
  kron_tail(m, x, i, j, acc, xpol, [&](int r) { return ld_gather(xij[r], xpol); });
}

// The diagonal terms at (i, j[r]), lane = row i, after the operand parts:
// (A_ii + B_jj), T, decay.  xl(r) = X(i, j[r]) (a gather, or the staged tile).
template <class XL>
__device__ __forceinline__ void kron_tail(const KronView& m, const double2* __restrict__ x, int i, const int* j,
                                          double2* acc, unsigned long long xpol, XL&& xl) {
  const unsigned n = static_cast<unsigned>(m.n);
  if (m.da) {  // the diagonals of A and B: (A_ii + B_jj) X(i, j), one gather
    const double2 dai = __ldg(m.da + i);
    by_kind(m.vk_d & 3, [&](auto kc, auto) {
      constexpr int K = decltype(kc)::value;
#pragma unroll
      for (int r = 0; r < kKR; ++r) {
        const double2 dbj = __ldg(m.db + j[r]);
        const double2 c = make_double2(dai.x + dbj.x, dai.y + dbj.y);
        if (c.x != 0.0 || c.y != 0.0) cfmak<K>(acc[r], c, xl(r));
      }
    });
  }
  if (m.t.ptr) {
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      if (i == j[r]) {  // transfer onto the diagonal
        const int e1 = __ldg(m.t.ptr + i + 1);
        by_kind(m.vk_t & 3, [&](auto kc, auto) {
          constexpr int K = decltype(kc)::value;
          for (int e = __ldg(m.t.ptr + i); e < e1; ++e)
            cfmak<K>(acc[r], ldv<K>(m.t.val + e), gat(x, static_cast<unsigned>(__ldg(m.t.col + e)) * (n + 1), xpol));
        });
      }
    }
  }
  if (m.d_const) {  // a constant coefficient (regular graphs, no sources / sinks)
    if (m.d_val != 0.0) {
#pragma unroll
      for (int r = 0; r < kKR; ++r) {
        const double2 xg = xl(r);
        acc[r].x = fma(-m.d_val, xg.x, acc[r].x);
        acc[r].y = fma(-m.d_val, xg.y, acc[r].y);
      }
    }
  } else if (m.d_loc) {  // -0.5 (w (dl_i + dl_j) + ds_i + ds_j) X(i, j)
    const double dli = __ldg(m.d_loc + i), dsi = __ldg(m.d_ss + i);
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const double d = __dmul_rn(
          0.5, __dadd_rn(__dadd_rn(__dmul_rn(m.omega, __dadd_rn(dli, __ldg(m.d_loc + j[r]))), dsi),
                         __ldg(m.d_ss + j[r])));
      if (d != 0.0) {
        const double2 xg = xl(r);
        acc[r].x = fma(-d, xg.x, acc[r].x);
        acc[r].y = fma(-d, xg.y, acc[r].y);
      }
    }
  }
}

// Tile enumeration (grid constants precomputed on the host, KronView::tg):
// J-major over all tiles (blocks launched together share the columns J), or
// in Hermitian mode the upper tiles I <= J in the order of the host table
// tg.herm_tiles.
struct TileGrid {
  int n, nc, nti;
  int c0;
  long long ntiles;
};

__device__ __forceinline__ TileGrid tile_grid(const KronView& m, bool herm) {
  return TileGrid{m.n, m.tg.nc, m.tg.nti, m.tg.c0, herm ? m.tg.ntiles_herm : m.tg.ntiles};
}

__device__ __forceinline__ void tile_coords(const KronView& m, const TileGrid& g, bool herm, long long t, int& I,
                                            int& J) {
  if (herm) {
    const int2 ij = __ldg(m.tg.herm_tiles + t);
    I = ij.x;
    J = ij.y;
  } else {
    J = static_cast<int>(t / g.nti);
    I = static_cast<int>(t - static_cast<long long>(J) * g.nti);
  }
}

// Writes one computed tile (acc[r] at row I*32 + lane, column J*32 + 4w + r)
// through epi(local_row, value, valid, mirror): directly and, in Hermitian
// mode, conjugated into tile (J, I) through a shared-memory transpose
// (coalesced both ways; mirror = true: the conjugate of an element already
// emitted, same magnitude); diagonal tiles keep their upper triangle, a real
// diagonal and its mirror.  Every thread of the block calls it.
template <bool kHerm, class Epi>
__device__ __forceinline__ void kron_tile_emit(const TileGrid& g, int I, int J, const double2* acc,
                                               double2 (*tile)[kKT + 1], Epi&& epi) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned n = static_cast<unsigned>(g.n);
  const int iu = I * kKT + lane;
  const bool diag = kHerm && I == J;
  const unsigned row0 = static_cast<unsigned>(J * kKT + kKR * w) * n + static_cast<unsigned>(iu);
#pragma unroll
  for (int r = 0; r < kKR; ++r) {
    const int jt = kKR * w + r;  // column within the tile
    const int jl = J * kKT + jt;
    double2 y = acc[r];
    if (diag && lane == jt) y.y = 0.0;
    epi(row0 + static_cast<unsigned>(r) * n, y, iu < g.n && jl < g.nc && (!diag || lane <= jt), false);
    if (kHerm) tile[jt][lane] = acc[r];
  }
  if (kHerm) {
    __syncthreads();
    // mirror: element (row J*32 + lane, column I*32 + it) = conj Y(I*32 + it, J*32 + lane)
    const int jrow = J * kKT + lane;
    const unsigned mrow0 = static_cast<unsigned>(I * kKT + kKR * w) * n + static_cast<unsigned>(jrow);
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const int it = kKR * w + r;
      const double2 v = tile[lane][it];
      const int icol = I * kKT + it;
      epi(mrow0 + static_cast<unsigned>(r) * n, conj2(v), jrow < g.n && icol < g.n && (!diag || lane > it), true);
    }
    __syncthreads();
  }
}

// Persistent loop over the tiles; epi(local_row, value, valid, mirror) runs on
// every thread for every element (valid is false outside the matrix and for
// the elements a Hermitian tile takes from its mirror).
template <bool kHerm, int kF, class Epi>
__device__ __forceinline__ void kron_tiles(const KronView& m, const double2* __restrict__ x, Epi&& epi) {
  __shared__ double2 tile[kKT][kKT + 1];
  const unsigned long long xpol = evict_last_policy();
  const TileGrid g = tile_grid(m, kHerm);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (long long t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    int I, J;
    tile_coords(m, g, kHerm, t, I, J);
    const int iu = I * kKT + lane;
    const int i = iu < g.n ? iu : g.n - 1;
    int jg[kKR];
#pragma unroll
    for (int r = 0; r < kKR; ++r) {
      const int jl = J * kKT + kKR * w + r;
      jg[r] = g.c0 + (jl < g.nc ? jl : g.nc - 1);
    }
    if (m.d_loc) {  // the decay term reads the tile's own elements last: start them towards L2 now
#pragma unroll
      for (int r = 0; r < kKR; ++r)
        asm volatile("prefetch.global.L2 [%0];" ::"l"(x + (static_cast<unsigned>(jg[r]) * static_cast<unsigned>(g.n) +
                                                          static_cast<unsigned>(i))));
    }
    double2 acc[kKR];
    if constexpr (kHerm) {
      int ir[kKR];
#pragma unroll
      for (int r = 0; r < kKR; ++r) {
        const int iv = I * kKT + kKR * w + r;
        ir[r] = iv < g.n ? iv : g.n - 1;
        acc[r] = make_double2(0.0, 0.0);
      }
      const int ju = J * kKT + lane;
      kron_rows_uniform<kF>(m, x, ir, ju < g.n ? ju : g.n - 1, acc, xpol);
#pragma unroll
      for (int r = 0; r < kKR; ++r) tile[kKR * w + r][lane] = acc[r];  // [row][column] of the tile
      __syncthreads();
#pragma unroll
      for (int r = 0; r < kKR; ++r) acc[r] = tile[lane][kKR * w + r];
      __syncthreads();
    } else {
#pragma unroll
      for (int r = 0; r < kKR; ++r) acc[r] = make_double2(0.0, 0.0);
      kron_rows_lane<kF>(m, x, i, jg, acc, xpol);
    }
    kron_cols<kHerm, kF>(m, x, i, jg, acc, xpol);
    kron_tile_emit<kHerm>(g, I, J, acc, tile, epi);
  }
}

// ---- staged Hermitian tiles (KronView::staged) -------------------------------
// 16-byte asynchronous copies global -> shared (LDGSTS; a warp moves one
// 512-byte tile row per instruction).  512-byte cp.async.bulk copies were
// measured first: the per-copy cost of the bulk engine (288 copies per tile)
// made the c2 term 41.5 us against 23.7 us for the global gathers.
__device__ __forceinline__ void cp_async16(double2* dst_smem, const double2* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst_smem)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}
constexpr int kStageTile = kKT * kKT;  // elements of one staged tile (16 KB)

// The upper tiles (I, J) of one block, each computed from shared memory.
// Phase A of a tile: the tiles of F named by patterns 0 and 1 and (factored)
// AXt(I, J); phase B: pattern 2, AXt(J, I) and the tile's own elements of x.
// They are copied a tile ahead, as soon as their regions are free again —
// phase A of the next tile once the transposed section of this one is done,
// phase B after its emit — so the copies of tile t + 1 run under the second
// half and the stores of tile t; the operand column indices of the next tile
// are loaded into registers at the same distance.  With one block per SM (the
// regions take 176 - 192 KB) nothing else hides a global-memory round trip,
// so the arithmetic of a tile touches shared memory and registers only
// (constant operand values; others are loaded).  Every thread commits one
// copy group per phase in the order A, B, A, B, ...; "at most one group
// pending" therefore means the older phase has landed.  The per-element order
// of the sums is kron_tiles'.
template <int kF, class Epi>
__device__ __forceinline__ void kron_tiles_staged(const KronView& m, const double2* __restrict__ x, Epi&& epi) {
  extern __shared__ __align__(128) unsigned char st_smem[];
  __shared__ double2 tile[kKT][kKT + 1];
  const unsigned long long xpol = evict_last_policy();
  const TileGrid g = tile_grid(m, true);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, l0 = w * kKR;
  const unsigned n = static_cast<unsigned>(m.n);
  const double2* const F = kF == 1 ? m.wt[0] : x;
  double2* const reg0 = reinterpret_cast<double2*>(st_smem);
  double2* const reg1 = reg0 + m.st_slots[0] * kStageTile;
  double2* const reg2 = reg1 + m.st_slots[1] * kStageTile;
  double2* const d2 = reg2 + m.st_slots[2] * kStageTile;  // x(I-rows of columns J): [j][i]
  double2* const d0 = d2 + kStageTile;                    // factored: AXt(I, J): [i][j]
  double2* const d1 = d0 + kStageTile;                    // factored: AXt(J, I): [j][i]
  const int len0 = m.st_len[0], len1 = m.st_len[1], len2 = m.st_len[2];
  // The tile indices come in registers (loaded a phase earlier): a load
  // between two copies would wait behind the copies' data in the load/store
  // pipe and serialise them.
  struct Next {
    int t[3][kStageSlots];
    int mycol0, mycol2, pcol[8];
  };
  const int kt = lane >> 2, rt = lane & 3;
  const auto load_next = [&](int I, int J, Next& nx) {
#pragma unroll
    for (int q = 0; q < kStageSlots; ++q) {
      nx.t[0][q] = q < m.st_slots[0] ? __ldg(m.st_nbr[0] + I * kStageSlots + q) : -1;
      nx.t[1][q] = q < m.st_slots[1] ? __ldg(m.st_nbr[1] + J * kStageSlots + q) : -1;
      nx.t[2][q] = q < m.st_slots[2] ? __ldg(m.st_nbr[2] + J * kStageSlots + q) : -1;
    }
    // (uniform ELL of constant row length: slice s starts at 32 s len)
    nx.mycol0 = kt < len0 ? __ldg(m.st_col[0] + I * kKT * len0 + 32 * kt + l0 + rt) : 0;
    nx.mycol2 = kt < len2 ? __ldg(m.st_col[2] + J * kKT * len2 + 32 * kt + l0 + rt) : 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) nx.pcol[e] = e < len1 ? __ldg(m.st_col[1] + J * kKT * len1 + 32 * e + lane) : 0;
  };
  // warp w copies rows w, w + 8, ... of every tile
  const auto copy_tile = [&](double2* dst, const double2* src00) {  // src00: element (0, 0) of the 32 x 32 source tile
#pragma unroll
    for (int r = 0; r < kKT; r += kThreads / 32) {
      const int row = r + w;
      cp_async16(dst + row * kKT + lane, src00 + (static_cast<unsigned>(row) * n + static_cast<unsigned>(lane)));
    }
  };
  const auto copy_a = [&](int I, int J, const Next& nx) {
#pragma unroll
    for (int q = 0; q < kStageSlots; ++q) {
      if (nx.t[0][q] >= 0) copy_tile(reg0 + q * kStageTile, F + (static_cast<unsigned>(nx.t[0][q] * kKT) * n + static_cast<unsigned>(J * kKT)));
    }
#pragma unroll
    for (int q = 0; q < kStageSlots; ++q) {
      if (nx.t[1][q] >= 0) copy_tile(reg1 + q * kStageTile, F + (static_cast<unsigned>(I * kKT) * n + static_cast<unsigned>(nx.t[1][q] * kKT)));
    }
    if constexpr (kF == 1) copy_tile(d0, m.axt + (static_cast<unsigned>(I * kKT) * n + static_cast<unsigned>(J * kKT)));
  };
  const auto copy_b = [&](int I, int J, const Next& nx) {
#pragma unroll
    for (int q = 0; q < kStageSlots; ++q) {
      if (nx.t[2][q] >= 0) copy_tile(reg2 + q * kStageTile, F + (static_cast<unsigned>(nx.t[2][q] * kKT) * n + static_cast<unsigned>(I * kKT)));
    }
    if constexpr (kF == 1) copy_tile(d1, m.axt + (static_cast<unsigned>(J * kKT) * n + static_cast<unsigned>(I * kKT)));
    copy_tile(d2, x + (static_cast<unsigned>(J * kKT) * n + static_cast<unsigned>(I * kKT)));
  };
  long long t = blockIdx.x;
  int I = 0, J = 0;
  Next cur;
  if (t < g.ntiles) {
    tile_coords(m, g, true, t, I, J);
    load_next(I, J, cur);
    copy_a(I, J, cur);
    cp_async_commit();
    copy_b(I, J, cur);
    cp_async_commit();
  }
  for (; t < g.ntiles; t += gridDim.x) {
    const long long tn = t + gridDim.x;
    const bool more = tn < g.ntiles;
    int In = 0, Jn = 0;
    Next nx;
    if (more) {
      tile_coords(m, g, true, tn, In, Jn);
      load_next(In, Jn, nx);
    }
    const int i = I * kKT + lane;  // n % 32 == 0: no edge tiles
    int jg[kKR];
    double2 acc[kKR];
#pragma unroll
    for (int r = 0; r < kKR; ++r) jg[r] = J * kKT + l0 + r;
    cp_async_wait<1>();
    __syncthreads();  // phase A of this tile is in shared memory
    // ---- transposed section: warp-uniform rows i = I*32 + l0 + r, lane = column j
    if constexpr (kF == 1) {
#pragma unroll
      for (int r = 0; r < kKR; ++r) acc[r] = d0[(l0 + r) * kKT + lane];  // A's part = AX(i, j)
      by_kind(m.vk_r[0], [&](auto kc, auto cc) {  // R_0: rows b of Wt_0
        QSWG_KC(kc, cc);
        const double2* r0 = reg0 + lane;
        shfl_rows_pre<K, C>(m.r_ellu[0].val, m.cv_r[0], len0, I * kKT * len0, cur.mycol0, l0, acc,
                            [&](unsigned o) { return r0[o]; });
      });
      by_kind(m.vk_p[0], [&](auto kc, auto cc) {  // P_0(j, a) Wt_0(i, a)
        QSWG_KC(kc, cc);
        const double2* r1 = reg1 + l0 * kKT;
        const double2* pv = m.p_ell[0].val + J * kKT * len1 + lane;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < len1) {
            const double2 v = opv<K, C>(pv + 32 * e, m.cv_p[0]);
#pragma unroll
            for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, r1[cur.pcol[e] + r * kKT]);
          }
        }
      });
    } else {
#pragma unroll
      for (int r = 0; r < kKR; ++r) acc[r] = make_double2(0.0, 0.0);
      by_kind(m.vk_a, [&](auto kc, auto cc) {  // A(i, c) conj x[n c + j]
        QSWG_KC(kc, cc);
        const double2* r0 = reg0 + lane;
        shfl_rows_pre<K, C>(m.a_ellu.val, m.cv_a, len0, I * kKT * len0, cur.mycol0, l0, acc,
                            [&](unsigned o) { return conj2(r0[o]); });
      });
      by_kind(m.vk_b, [&](auto kc, auto cc) {  // B(j, c) conj x[n i + c]
        QSWG_KC(kc, cc);
        const double2* r1 = reg1 + l0 * kKT;
        const double2* bv = m.b_ell.val + J * kKT * len1 + lane;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          if (e < len1) {
            const double2 v = opv<K, C>(bv + 32 * e, m.cv_b);
#pragma unroll
            for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, conj2(r1[cur.pcol[e] + r * kKT]));
          }
        }
      });
    }
#pragma unroll
    for (int r = 0; r < kKR; ++r) tile[l0 + r][lane] = acc[r];
    __syncthreads();  // the transposed sums are in `tile`; the phase-A regions are free
    if (more) copy_a(In, Jn, nx);
    cp_async_commit();
#pragma unroll
    for (int r = 0; r < kKR; ++r) acc[r] = tile[lane][l0 + r];
    cp_async_wait<1>();
    __syncthreads();  // phase B of this tile is in shared memory (and `tile` is free)
    // ---- normal orientation: lane = row i, columns j = J*32 + l0 + r
    if constexpr (kF == 1) {
#pragma unroll
      for (int r = 0; r < kKR; ++r) {  // B's part = conj AX(j, i), added as one sum
        const double2 bb = d1[(l0 + r) * kKT + lane];
        acc[r].x += bb.x;
        acc[r].y -= bb.y;
      }
      by_kind(m.vk_s[0], [&](auto kc, auto cc) {  // S_0: rows a of Wt_0, conjugated
        QSWG_KC(kc, cc);
        const double2* r2 = reg2 + lane;
        shfl_rows_pre<K, C>(m.s_ellu[0].val, m.cv_s[0], len2, J * kKT * len2, cur.mycol2, l0, acc,
                            [&](unsigned o) { return conj2(r2[o]); });
      });
    }
    kron_tail(m, x, i, jg, acc, xpol, [&](int r) { return d2[(l0 + r) * kKT + lane]; });
    kron_tile_emit<true>(g, I, J, acc, tile, epi);  // (ends with a barrier: the phase-B regions are free)
    if (more) copy_b(In, Jn, nx);
    cp_async_commit();
    I = In;
    J = Jn;
    cur = nx;
  }
  cp_async_wait<0>();
}

// W_k = Q_k X on the local columns (W_k(i, a) at w[n*a + i], global index)
// in the tiles of kron_tiles.  General path: lane = row i, 4 columns a per
// thread (per-lane operand rows).  Hermitian path: warp-uniform rows i, lane
// = column a, gathers conj X(a, b) coalesced; the tile is transposed through
// shared memory for the column-major store, and (factored dissipator) also
// stored row-major into Wt_k for the transposed R_k part.
#ifndef QSWG_KRON_W_MIN_BLOCKS
#define QSWG_KRON_W_MIN_BLOCKS 4
#endif
#ifndef QSWG_WFLUSH_REG
#define QSWG_WFLUSH_REG 1  // the fused flush keeps its norm maxima in registers (FlushMax)
#endif
// kFlush: the same launch then runs the flush after the previous term
// (series_flush; its HBM streaming overlaps the gathers of W).
template <bool kHerm, bool kFlush>
__global__ void __launch_bounds__(kThreads, QSWG_KRON_W_MIN_BLOCKS) kron_w_kernel(KronView m, const double2* __restrict__ x, int k,
                                                                               SeriesFlushArgs fa) {
  pdl_prologue();
  __shared__ double2 tile[kKT][kKT + 1];
  const unsigned long long xpol = evict_last_policy();
  const unsigned n = static_cast<unsigned>(m.n);
  const TileGrid g = tile_grid(m, false);
  const KronEll& qe = m.q_ell[k];
  const KronList& q = m.q[k];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int vk = m.vk_q[k];
  const double2 cv = m.cv_q[k];
  for (long long t = blockIdx.x; t < g.ntiles; t += gridDim.x) {
    int I, J;
    tile_coords(m, g, false, t, I, J);
    double2 acc[kKR];
#pragma unroll
    for (int r = 0; r < kKR; ++r) acc[r] = make_double2(0.0, 0.0);
    if constexpr (kHerm) {
      const int au = J * kKT + lane;  // column a (single GPU: c0 = 0)
      const double2* xa = x + (au < g.n ? au : g.n - 1);
      const auto gx = [&](unsigned bn) { return conj2(gat(xa, bn, xpol)); };  // q_ellu / q_sc hold b * n
      if (k == 0 && m.ax) {  // W_0 and AX from the same gathers (KronView::ax)
        double2 aacc[kKR];
#pragma unroll
        for (int r = 0; r < kKR; ++r) aacc[r] = make_double2(0.0, 0.0);
        int ir[kKR];
#pragma unroll
        for (int r = 0; r < kKR; ++r) {
          const int iv = I * kKT + kKR * w + r;
          ir[r] = iv < g.n ? iv : g.n - 1;
        }
        by_kind_ax(vk, m.vk_aq, [&](auto kq, auto cq, auto ka, auto ca) {
          constexpr int KQ = decltype(kq)::value, KA = decltype(ka)::value;
          constexpr bool CQ = decltype(cq)::value, CA = decltype(ca)::value;
          if (m.q_len[0] > 0) {
            shfl_rows2<KQ, CQ, KA, CA>(m.q_ellu[0], m.aq_ellu_val, cv, m.cv_aq, m.q_len[0], ir[0] >> 5, kKR * w, acc,
                                       aacc, gx);
          } else {
            uniform_rows2<KQ, CQ, KA, CA>(m.q_sc[0], m.aq_sc_val, cv, m.cv_aq, ir, acc, aacc, gx);
          }
        });
        const unsigned arow = static_cast<unsigned>(I * kKT + kKR * w) * n + static_cast<unsigned>(au);
#pragma unroll
        for (int r = 0; r < kKR; ++r) {
          const int iv = I * kKT + kKR * w + r;
          if (iv < g.n && au < g.n) st_hint(m.axt + (arow + static_cast<unsigned>(r) * n), aacc[r], xpol);
        }
      } else if (m.q_len[k] > 0) {  // rows I*32 + 4w + r: lanes 4w .. 4w+3 of slice I
        const int iv0 = I * kKT + kKR * w;
        by_kind(vk, [&](auto kc, auto cc) {
          QSWG_KC(kc, cc);
          shfl_rows<K, C>(m.q_ellu[k], cv, m.q_len[k], (iv0 < g.n ? iv0 : g.n - 1) >> 5, kKR * w, acc, gx);
        });
      } else if (m.q_sc[k].ptr) {
        int ir[kKR];
#pragma unroll
        for (int r = 0; r < kKR; ++r) {
          const int iv = I * kKT + kKR * w + r;
          ir[r] = iv < g.n ? iv : g.n - 1;
        }
        by_kind(vk, [&](auto kc, auto cc) {
          QSWG_KC(kc, cc);
          uniform_rows<K, C>(m.q_sc[k], cv, ir, acc, gx);
        });
      }
      const unsigned wrow = static_cast<unsigned>(I * kKT + kKR * w) * n + static_cast<unsigned>(au);
#pragma unroll
      for (int r = 0; r < kKR; ++r) {
        const int iv = I * kKT + kKR * w + r;
        if (m.wt[k] && iv < g.n && au < g.n) st_hint(m.wt[k] + (wrow + static_cast<unsigned>(r) * n), acc[r], xpol);
        tile[kKR * w + r][lane] = acc[r];
      }
      if (!m.p_rows) {  // the column-major W_k (read by P_k in the normal orientation)
        __syncthreads();
        const int iu = I * kKT + lane;
        const unsigned wcol = static_cast<unsigned>(J * kKT + kKR * w) * n + static_cast<unsigned>(iu);
#pragma unroll
        for (int r = 0; r < kKR; ++r) {
          const int at = J * kKT + kKR * w + r;
          if (iu < g.n && at < g.n) st_hint(m.w[k] + (wcol + static_cast<unsigned>(r) * n), tile[lane][kKR * w + r], xpol);
        }
        __syncthreads();
      }
    } else {
      const int iu = I * kKT + lane;
      const bool vi = iu < m.n;
      const int i = vi ? iu : m.n - 1;
      unsigned col[kKR];
      bool vj[kKR];
#pragma unroll
      for (int r = 0; r < kKR; ++r) {
        const int jl = J * kKT + kKR * w + r;
        vj[r] = jl < g.nc;
        col[r] = static_cast<unsigned>(g.c0 + (vj[r] ? jl : g.nc - 1)) * n;
      }
      by_kind(qe.sptr ? vk & 3 : vk, [&](auto kc, auto cc) {  // (padded ELL: load the zeros)
        QSWG_KC(kc, cc);
        if (qe.sptr) {
          const int sl = i >> 5, ln = i & 31;
          const int b = __ldg(qe.sptr + sl), len = (__ldg(qe.sptr + sl + 1) - b) >> 5;
#pragma unroll 2
          for (int e = 0; e < len; ++e) {
            const unsigned c = static_cast<unsigned>(__ldg(qe.col + b + 32 * e + ln));
            const double2 v = opv<K, C>(qe.val + b + 32 * e + ln, cv);
#pragma unroll
            for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(x, col[r] + c, xpol));
          }
        } else if (q.ptr) {
          const int e1 = __ldg(q.ptr + i + 1);
#pragma unroll 2
          for (int e = __ldg(q.ptr + i); e < e1; ++e) {
            const unsigned c = static_cast<unsigned>(__ldg(q.col + e));
            const double2 v = opv<K, C>(q.val + e, cv);
#pragma unroll
            for (int r = 0; r < kKR; ++r) cfmak<K>(acc[r], v, gat(x, col[r] + c, xpol));
          }
        }
      });
#pragma unroll
      for (int r = 0; r < kKR; ++r)
        if (vi && vj[r]) st_hint(m.w[k] + (col[r] + static_cast<unsigned>(i)), acc[r], xpol);
    }
  }
  if constexpr (kFlush) {
    if (flush_due(fa)) {
      if (fa.herm_n > 0) {
        flush_body_herm<QSWG_WFLUSH_REG != 0>(fa);
      } else {
        flush_body<false, false, QSWG_WFLUSH_REG != 0>(fa);
      }
      return;
    }
  }
  pdl_trigger();
}

// V_k = X L_k' on the local columns: V_k(i, a) = sum_c conj(L_k(a, c)) X(i, c)
// (U_k lists hold c * n).
__global__ void __launch_bounds__(kThreads) kron_v_kernel(KronView m, const double2* __restrict__ x, int k) {
  pdl_prologue();
  const unsigned long long xpol = evict_last_policy();
  const long long n = m.n;
  const KronList& u = m.u[k];
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < m.rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = m.row0 + r;
    const long long a = g / n, i = g - a * n;
    double2 acc = make_double2(0.0, 0.0);
    const double2* xi = x + i;
    by_kind(m.vk_u[k] & 3, [&](auto kc, auto) {
      uniform_row<decltype(kc)::value, false>(u, double2{}, static_cast<int>(a), acc,
                                              [&](unsigned cn) { return gat(xi, cn, xpol); });
    });
    st_hint(m.v[k] + g, acc, xpol);
  }
}

template <bool kHerm, int kF>
__global__ void __launch_bounds__(kThreads) kron_spmv_kernel(KronView m, const double2* x, double2* y, double scale) {
  pdl_prologue();
  kron_tiles<kHerm, kF>(m, x, [&](unsigned row, double2 acc, bool valid, bool) {
    if (valid) y[row] = make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y));
  });
}

struct KronStepArgs {
  KronView m;
  const double2* x;
  double2* y;
  const double2* sum_in;
  double2* sum_out;
  double scale;
  double tol;
  StepCtl* ctl;
  int first_of_stage;
  int stage;
  int decide;
};

// The step term's epilogue (running sum in and out, two norms) needs more
// registers than the series term's: 3 blocks per SM (<= 80 registers) there
// (c3, whose series is 50 sequential steps: 865 -> 825 ms), 4 for the series
// term (c2 at 3 blocks: 35.2 -> 40.1 ms).
#ifndef QSWG_KRON_STEP_MIN_BLOCKS
#define QSWG_KRON_STEP_MIN_BLOCKS 3
#endif
template <bool kHerm, int kF>
__global__ void __launch_bounds__(kThreads, QSWG_KRON_STEP_MIN_BLOCKS) kron_step_term_kernel(KronStepArgs a) {
  pdl_prologue();
  StepCtl* ctl = a.ctl;
  if (*(volatile int*)&ctl->error) return;
  if (!a.first_of_stage && *(volatile int*)&ctl->done) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0, smax = 0;
  const unsigned long long once = evict_first_policy(), keep = evict_last_policy();
  kron_tiles<kHerm, kF>(a.m, a.x, [&](unsigned row, double2 acc, bool valid, bool mirror) {
    if (!valid) return;
    const double2 yv = make_double2(__dmul_rn(a.scale, acc.x), __dmul_rn(a.scale, acc.y));
    const double2 sv0 = ld_once(a.sum_in + row, once);
    st_hint(a.y + row, yv, keep);
    const double2 sv = make_double2(sv0.x + yv.x, sv0.y + yv.y);  // expm.cpp:181
    st_hint(a.sum_out + row, sv, once);
    if (!mirror) {  // a mirrored element is the conjugate of one already counted (Hermitian sums)
      max_abs_bits(tmax, yv);
      max_abs_bits(smax, sv);
    }
  });
  pdl_trigger();
  tmax = block_max_bits(tmax, red);
  smax = block_max_bits(smax, red);
  if (threadIdx.x == 0) {
    atomicMax(&ctl->term_bits, tmax);
    atomicMax(&ctl->sum_bits, smax);
    __threadfence();
    if (atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1) {
      __threadfence();
      if (a.decide) {
        step_control(ctl, a.first_of_stage, a.stage, a.tol);
      } else {
        ctl->arrivals = 0;
      }
    }
  }
}

template <bool kHerm, int kF>
__global__ void __launch_bounds__(kThreads, QSWG_KRON_MIN_BLOCKS) kron_series_term_kernel(SeriesTermArgs a, KronView m) {
  pdl_prologue();
  if (series_skip(a.ctl)) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0;
  const unsigned long long keep = evict_last_policy();
  double2* const kp = a.kp;
  const double scale = a.scale;
  kron_tiles<kHerm, kF>(m, a.x, [&](unsigned row, double2 acc, bool valid, bool mirror) {
    series_store(kp, scale, row, acc, valid && !mirror, keep, tmax);
    if (valid && mirror) st_hint(kp + row, make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y)), keep);
  });
  series_term_finish(a, tmax, red);
}

// The Hermitian series term on the staged tiles (one block per SM).
template <int kF>
__global__ void __launch_bounds__(kThreads, 1) kron_series_term_staged_kernel(SeriesTermArgs a, KronView m) {
  pdl_prologue();
  if (series_skip(a.ctl)) return;
  __shared__ unsigned long long red[32];
  unsigned long long tmax = 0;
  const unsigned long long keep = evict_last_policy();
  double2* const kp = a.kp;
  const double scale = a.scale;
  kron_tiles_staged<kF>(m, a.x, [&](unsigned row, double2 acc, bool valid, bool mirror) {
    series_store(kp, scale, row, acc, valid && !mirror, keep, tmax);
    if (valid && mirror) st_hint(kp + row, make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y)), keep);
  });
  series_term_finish(a, tmax, red);
}

// ------------------------------------------------------------ norm kernels
// Grid-wide max |v| into *bits, last block runs `fin`.
template <class Fin>
__device__ __forceinline__ void norm_body(const double2* __restrict__ v, long long n,
                                          unsigned long long* bits, unsigned int* arrivals, Fin fin) {
  __shared__ unsigned long long red[32];
  unsigned long long m = 0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    max_abs_bits(m, v[k]);
  m = block_max_bits(m, red);
  if (threadIdx.x == 0) {
    atomicMax(bits, m);
    __threadfence();
    if (atomicAdd(arrivals, 1u) == gridDim.x - 1) {
      __threadfence();
      fin(bitsd(*(volatile unsigned long long*)bits));
    }
  }
}

__device__ void step_init_apply(StepCtl* ctl, double nv) {
  ctl->c1 = nv;  // expm.cpp:165-170
  ctl->last_nf = nv;
  ctl->done = 0;  // `error` and `spmvs` are sticky across calls
  ctl->sum_bits = 0;
  ctl->term_bits = 0;
  ctl->arrivals = 0;
}

__device__ void series_init_apply(SeriesCtl* ctl, int count, int pend_max, double nz) {
  ctl->z_norm = nz;  // expm.cpp:271-276
  ctl->count = count;
  ctl->n_active = ctl->error ? 0 : count;  // `error` and `spmvs` are sticky
  for (int k = 0; k < count; ++k) {
    ctl->active[k] = 1;
    ctl->factor[k] = static_cast<double>(k + 1);  // factor *= k at p = 1
    ctl->c1[k] = nz;
    ctl->nf_last[k] = nz;  // S_k starts as Z
    ctl->bound[k] = 0.0;
    ctl->sum_bits[k] = 0;
    ctl->p0[k] = 1;
    ctl->mark[k] = 0;
    ctl->fresh[k] = 1;
    ctl->pending[k] = 0;
    ctl->p_end[k] = 0;
  }
  ctl->flush = 0;
  ctl->pend_max = pend_max < 1 ? 1 : (pend_max > kPendMax ? kPendMax : pend_max);
  ctl->slots = ctl->pend_max + 1;
  ctl->term_bits = 0;
  ctl->arrivals = 0;
}

__global__ void __launch_bounds__(kThreads) step_init_kernel(const double2* v, long long n, StepCtl* ctl, int decide) {
  pdl_prologue();
  pdl_trigger();
  norm_body(v, n, &ctl->term_bits, &ctl->arrivals, [ctl, decide](double nv) {
    if (decide) {
      step_init_apply(ctl, nv);
    } else {
      ctl->arrivals = 0;
    }
  });
}

__global__ void __launch_bounds__(kThreads) series_init_kernel(const double2* z, long long n, int count,
                                                              int pend_max, SeriesCtl* ctl, int decide) {
  pdl_prologue();
  pdl_trigger();
  norm_body(z, n, &ctl->term_bits, &ctl->arrivals, [ctl, count, pend_max, decide](double nz) {
    if (decide) {
      series_init_apply(ctl, count, pend_max, nz);
    } else {
      ctl->arrivals = 0;
    }
  });
}

// Control steps after a cross-GPU allreduce(max) of the maxima (one thread).
__global__ void step_init_fin_kernel(StepCtl* ctl) {
  pdl_prologue();
  pdl_trigger();
  step_init_apply(ctl, bitsd(ctl->term_bits));
}
__global__ void series_init_fin_kernel(SeriesCtl* ctl, int count, int pend_max) {
  pdl_prologue();
  pdl_trigger();
  series_init_apply(ctl, count, pend_max, bitsd(ctl->term_bits));
}
// The multi-GPU controls run after every term whether or not it ran (the
// host enqueues without reading the stop flags): a term the stop test or an
// error already skipped leaves the control block untouched.
__global__ void step_control_kernel(StepCtl* ctl, int first_of_stage, int stage, double tol) {
  pdl_prologue();
  pdl_trigger();
  if (ctl->error || (!first_of_stage && ctl->done)) {  // the term kernel skipped itself
    ctl->term_bits = 0;
    ctl->sum_bits = 0;
    ctl->arrivals = 0;
    return;
  }
  step_control(ctl, first_of_stage, stage, tol);
}
__global__ void __launch_bounds__(kThreads) series_term_control_kernel(SeriesCtl* ctl, int p, int last, double tol) {
  pdl_prologue();
  pdl_trigger();
  series_term_control(ctl, p, last, tol);
}
// After term p on several GPUs (one allreduce of [term_bits, sum_bits]): the
// exact tests of the flush after term p - 1 when one ran, then term p's
// control — unless term p is not part of the series (the series had ended,
// or that flush stopped every output: the term ran speculatively and is
// neither tested nor counted).
__global__ void __launch_bounds__(kThreads) series_flush_term_control_kernel(SeriesCtl* ctl, int p, int last,
                                                                            double tol) {
  pdl_prologue();
  pdl_trigger();
  __shared__ int go;
  if (*(volatile int*)&ctl->flush) series_flush_control(ctl, p - 1, tol);
  __syncthreads();
  if (threadIdx.x == 0) go = !ctl->error && ctl->n_active > 0;
  __syncthreads();
  if (go) {
    series_term_control(ctl, p, last, tol);
  } else if (threadIdx.x == 0) {
    ctl->term_bits = 0;
    ctl->arrivals = 0;
  }
}
__global__ void __launch_bounds__(kThreads) series_flush_control_kernel(SeriesCtl* ctl, int p, double tol) {
  pdl_prologue();
  pdl_trigger();
  if (!*(volatile int*)&ctl->flush) return;  // no flush was due (multi-GPU: enqueued unconditionally)
  series_flush_control(ctl, p, tol);
}

// --------------------------------------------------------------- plain SpMV
template <int G>
__global__ void __launch_bounds__(kThreads) spmv_kernel(CsrView l, const double2* x, double2* y, double scale) {
  pdl_prologue();
  pdl_trigger();
  tile_loop<G>(l, x, [&](long long row, double2 acc, bool valid) {
    if (valid) y[row] = make_double2(__dmul_rn(scale, acc.x), __dmul_rn(scale, acc.y));
  });
}

__global__ void diag_kernel(const double2* v, long long row0, long long rows, long long n, double* pops) {
  pdl_prologue();
  pdl_trigger();
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = i * (n + 1) - row0;
    if (g >= 0 && g < rows) pops[i] = v[g].x;
  }
}

// out[0] = max over the off-diagonal elements of |v| as a bit pattern
// (DensityMatrix::max_coherence, walk.cpp:32-40; hypot like std::abs).
__global__ void __launch_bounds__(kThreads) coherence_kernel(const double2* __restrict__ v, long long row0, long long rows,
                                                             long long n, unsigned long long* out) {
  pdl_prologue();
  pdl_trigger();
  __shared__ unsigned long long red[32];
  unsigned long long m = 0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = row0 + k;
    if (g % (n + 1) != 0) m = umax64(m, dbits(cabs2(__ldg(v + k))));  // g = n j + i, i == j <=> g = j (n + 1)
  }
  m = block_max_bits(m, red);
  if (threadIdx.x == 0 && m != 0) atomicMax(out, m);
}

__global__ void probs_kernel(double2* v, long long row0, long long rows, long long n, const double* p) {
  pdl_prologue();
  pdl_trigger();
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = row0 + k;
    const long long j = g / n, i = g - j * n;
    v[k] = make_double2(i == j ? p[i] : 0.0, 0.0);
  }
}

// *flag = 0 when some X(i, j) != conj X(j, i) (i <= j); one thread per
// upper element, lanes along i (the mirrored reads are strided).
__global__ void hermitian_check_kernel(const double2* __restrict__ x, long long n, int* flag) {
  pdl_prologue();
  pdl_trigger();
  const long long total = n * n;
  bool ok = true;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = k / n, i = k - j * n;
    if (i > j) continue;
    const double2 a = __ldg(x + k), b = __ldg(x + i * n + j);
    ok = ok && a.x == b.x && a.y == -b.y;
  }
  if (__any_sync(0xffffffffu, !ok) && (threadIdx.x & 31) == 0) *flag = 0;
}

__global__ void pattern_hermitian_kernel(double2* v, long long n) {
  pdl_prologue();
  pdl_trigger();
  const long long total = n * n;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < total;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long j = k / n, i = k - j * n;
    const long long a = i < j ? i : j, b = i < j ? j : i;
    const unsigned long long h = (static_cast<unsigned long long>(a * n + b) + 1) * 0x9E3779B97F4A7C15ull;
    const double re = static_cast<double>(h >> 11) * 0x1p-53 - 0.5;
    const double im = i == j ? 0.0 : static_cast<double>((h * 0xBF58476D1CE4E5B9ull) >> 11) * 0x1p-53 - 0.5;
    v[k] = make_double2(re, i <= j ? im : -im);
  }
}

__global__ void pattern_kernel(double2* v, long long n) {
  pdl_prologue();
  pdl_trigger();
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long h = (static_cast<unsigned long long>(k) + 1) * 0x9E3779B97F4A7C15ull;
    v[k] = make_double2(static_cast<double>(h >> 11) * 0x1p-53 - 0.5,
                        static_cast<double>((h * 0xBF58476D1CE4E5B9ull) >> 11) * 0x1p-53 - 0.5);
  }
}

// ------------------------------------------------------------ launch helpers
template <class K>
int persistent_grid(K kernel, long long rows) {
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel));
  const long long cap = static_cast<long long>(sm_count()) * per_sm;
  long long want = (rows + kTile - 1) / kTile;
  if (want < 1) want = 1;
  return static_cast<int>(want < cap ? want : cap);
}

// Dynamic shared memory beyond 48 KB: opt in once per device, kernel and size.
void allow_smem(const void* fn, std::size_t smem) {
  struct Key {
    int dev;
    const void* k;
    std::size_t bytes;
  };
  static thread_local Key done[64];
  static thread_local int used = 0;
  int dev = 0;
  cudaGetDevice(&dev);
  for (int i = 0; i < used; ++i)
    if (done[i].dev == dev && done[i].k == fn && done[i].bytes >= smem) return;
  QSWG_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)));
  if (used < 64) done[used++] = {dev, fn, smem};
}

// Launch of a SELL kernel: persistent grid; the streamed path (SellView::work)
// carries its rings in dynamic shared memory.
template <class... KArgs, class... Args>
void launch_sell(void (*kernel)(KArgs...), const SellView& m, cudaStream_t s, Args... args) {
  const std::size_t smem = m.work ? kSellSmemBytes : 0;
  const void* fn = reinterpret_cast<const void*>(kernel);
  if (smem) allow_smem(fn, smem);
  const int per_sm = blocks_per_sm(fn, smem);
  const long long cap = static_cast<long long>(sm_count()) * per_sm;
  long long want = m.b_val && !m.work ? (m.n_slices + m.win_slices - 1) / m.win_slices
                                      : (m.n_slices + kThreads / 32 - 1) / (kThreads / 32);
  if (want < 1) want = 1;
  launch_pdl(kernel, static_cast<int>(want < cap ? want : cap), kThreads, smem, s, args...);
}

// Persistent launch geometry of a Kron kernel (no dynamic shared memory).
template <class K>
std::pair<int, std::size_t> kron_geom(K kernel, const KronView& m, bool herm = false) {
  const int per_sm = blocks_per_sm(reinterpret_cast<const void*>(kernel));
  const long long cap = static_cast<long long>(sm_count()) * per_sm;
  long long want = herm ? m.tg.ntiles_herm : m.tg.ntiles;
  if (want < 1) want = 1;
  return {static_cast<int>(want < cap ? want : cap), std::size_t{0}};
}

int small_grid(long long n) {
  long long want = (n + kThreads - 1) / kThreads, cap = sm_count() * 4LL;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

template <template <int> class KT, class... Args>
void dispatch_group(int g, long long rows, cudaStream_t s, Args... args) {
  switch (g) {
#define QSWG_G(GV)                                                          \
  case GV: {                                                                \
    auto k = KT<GV>::fn;                                                    \
    launch_pdl(k, persistent_grid(k, rows), kThreads, 0, s, args...);              \
    break;                                                                  \
  }
    QSWG_G(1)
    QSWG_G(2)
    QSWG_G(4)
    QSWG_G(8)
    QSWG_G(16)
    QSWG_G(32)
#undef QSWG_G
    default:
      throw std::invalid_argument("row group size must be 1, 2, 4, 8, 16 or 32");
  }
}

template <int G> struct StepTermK { static constexpr auto fn = step_term_kernel<G>; };
template <int G> struct SeriesTermK { static constexpr auto fn = series_term_kernel<G>; };
template <int G> struct SpmvK { static constexpr auto fn = spmv_kernel<G>; };

}  // namespace

int valid_group(int g) { return (g == 1 || g == 2 || g == 4 || g == 8 || g == 16 || g == 32) ? g : 0; }

void step_init(const double2* v, std::int64_t n, StepCtl* ctl, bool decide, cudaStream_t s) {
  launch_pdl(step_init_kernel, small_grid(n), kThreads, 0, s, v, n, ctl, decide ? 1 : 0);
  QSWG_LAUNCH_CHECK("step_init");
}

void step_init_fin(StepCtl* ctl, cudaStream_t s) {
  launch_pdl(step_init_fin_kernel, 1, 1, 0, s, ctl);
  QSWG_LAUNCH_CHECK("step_init_fin");
}

void step_control(StepCtl* ctl, bool first_of_stage, int stage, double tol, cudaStream_t s) {
  launch_pdl(step_control_kernel, 1, 1, 0, s, ctl, first_of_stage ? 1 : 0, stage, tol);
  QSWG_LAUNCH_CHECK("step_control");
}

void series_init_fin(SeriesCtl* ctl, int count, int pend_max, cudaStream_t s) {
  launch_pdl(series_init_fin_kernel, 1, 1, 0, s, ctl, count, pend_max);
  QSWG_LAUNCH_CHECK("series_init_fin");
}

void series_term_control(SeriesCtl* ctl, int p, int last, double tol, cudaStream_t s) {
  launch_pdl(series_term_control_kernel, 1, kThreads, 0, s, ctl, p, last, tol);
  QSWG_LAUNCH_CHECK("series_term_control");
}

void series_flush_term_control(SeriesCtl* ctl, int p, int last, double tol, cudaStream_t s) {
  launch_pdl(series_flush_term_control_kernel, 1, kThreads, 0, s, ctl, p, last, tol);
  QSWG_LAUNCH_CHECK("series_flush_term_control");
}

void series_flush_control(SeriesCtl* ctl, int p, double tol, cudaStream_t s) {
  launch_pdl(series_flush_control_kernel, 1, kThreads, 0, s, ctl, p, tol);
  QSWG_LAUNCH_CHECK("series_flush_control");
}

// The partial sums of the earlier SELL column panels (no-op for one panel).
void sell_partials(const DevMatrix& m, const double2* x, const SkipCheck& sk, cudaStream_t s) {
  for (int q = m.pre_done; q < m.n_pre; ++q) {
    if (q == 0) {
      if (m.sell_pre[q].work) {
        launch_sell(sell_partial_kernel<true, kSellStream>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      } else if (m.sell_pre[q].b_val) {
        launch_sell(sell_partial_kernel<true, kSellWindows>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      } else {
        launch_sell(sell_partial_kernel<true, kSellReg>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      }
    } else {
      if (m.sell_pre[q].work) {
        launch_sell(sell_partial_kernel<false, kSellStream>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      } else if (m.sell_pre[q].b_val) {
        launch_sell(sell_partial_kernel<false, kSellWindows>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      } else {
        launch_sell(sell_partial_kernel<false, kSellReg>, m.sell_pre[q], s, m.sell_pre[q], x, m.part, sk);
      }
    }
    QSWG_LAUNCH_CHECK("sell_partials");
  }
}

void sell_local_panel(const DevMatrix& m, const double2* x, const SeriesCtl* series, const StepCtl* step,
                      int first_of_stage, cudaStream_t s) {
  if (m.format != Format::Sell || m.local_first < 1 || m.n_pre < 1) return;
  DevMatrix own = m;
  own.n_pre = m.local_first < m.n_pre ? m.local_first : m.n_pre;
  own.pre_done = 0;
  sell_partials(own, x, SkipCheck{series, step, first_of_stage}, s);
}

void step_term(const DevMatrix& m, const double2* x, double2* y, const double2* sum_in, double2* sum_out,
               double scale, bool first_of_stage, int stage, double tol, StepCtl* ctl, bool decide, cudaStream_t s) {
  if (m.format == Format::Kron) {
    KronStepArgs a{m.kron, x, y, sum_in, sum_out, scale, tol, ctl, first_of_stage ? 1 : 0, stage, decide ? 1 : 0};
    if (m.kron.herm) {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_step_term_kernel<true, 1>, m.kron, true);
        launch_pdl(kron_step_term_kernel<true, 1>, g.first, kThreads, g.second, s, a);
      } else {
        const auto g = kron_geom(kron_step_term_kernel<true, 0>, m.kron, true);
        launch_pdl(kron_step_term_kernel<true, 0>, g.first, kThreads, g.second, s, a);
      }
    } else {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_step_term_kernel<false, 1>, m.kron);
        launch_pdl(kron_step_term_kernel<false, 1>, g.first, kThreads, g.second, s, a);
      } else {
        const auto g = kron_geom(kron_step_term_kernel<false, 0>, m.kron);
        launch_pdl(kron_step_term_kernel<false, 0>, g.first, kThreads, g.second, s, a);
      }
    }
  } else if (m.format == Format::Sell) {
    sell_partials(m, x, SkipCheck{nullptr, ctl, first_of_stage ? 1 : 0}, s);
    SellStepArgs a{m.sell, x, y, sum_in, sum_out, scale, tol, ctl, first_of_stage ? 1 : 0, stage, decide ? 1 : 0};
    if (m.group == 1) {
      if (m.sell.work) {
        launch_sell(sell_step_term_kernel<true, kSellStream>, m.sell, s, a);
      } else if (m.sell.b_val) {
        launch_sell(sell_step_term_kernel<true, kSellWindows>, m.sell, s, a);
      } else {
        launch_sell(sell_step_term_kernel<true, kSellReg>, m.sell, s, a);
      }
    } else {
      if (m.sell.work) {
        launch_sell(sell_step_term_kernel<false, kSellStream>, m.sell, s, a);
      } else if (m.sell.b_val) {
        launch_sell(sell_step_term_kernel<false, kSellWindows>, m.sell, s, a);
      } else {
        launch_sell(sell_step_term_kernel<false, kSellReg>, m.sell, s, a);
      }
    }
  } else {
    StepTermArgs a{m.csr, x, y, sum_in, sum_out, scale, tol, ctl, first_of_stage ? 1 : 0, stage, decide ? 1 : 0};
    dispatch_group<StepTermK>(m.group, m.csr.rows, s, a);
  }
  QSWG_LAUNCH_CHECK("step_term");
}

void series_init(const double2* z, std::int64_t n, int count, int pend_max, SeriesCtl* ctl, bool decide,
                 cudaStream_t s) {
  if (count < 1 || count > kMaxSeriesD) throw std::invalid_argument("series super-step size out of range");
  launch_pdl(series_init_kernel, small_grid(n), kThreads, 0, s, z, n, count, pend_max, ctl, decide ? 1 : 0);
  QSWG_LAUNCH_CHECK("series_init");
}

void series_term(const DevMatrix& m, const double2* x, double2* kp, int p, bool last, double scale,
                 double tol, SeriesCtl* ctl, bool decide, cudaStream_t s) {
  const SeriesTermArgs a{x, kp, p, last ? 1 : 0, scale, tol, ctl, decide ? 1 : 0};
  if (m.format == Format::Kron) {
    if (m.kron.herm && m.kron.staged) {
      const std::size_t smem = static_cast<std::size_t>(m.kron.st_slots[0] + m.kron.st_slots[1] + m.kron.st_slots[2] +
                                                        (m.kron.factored ? 3 : 1)) *
                               (kStageTile * 16);
      const auto go = [&](auto kernel) {
        const void* fn = reinterpret_cast<const void*>(kernel);
        allow_smem(fn, smem);
        const long long cap = static_cast<long long>(sm_count()) * blocks_per_sm(fn, smem);
        const long long want = m.kron.tg.ntiles_herm < 1 ? 1 : m.kron.tg.ntiles_herm;
        launch_pdl(kernel, static_cast<int>(want < cap ? want : cap), kThreads, smem, s, a, m.kron);
      };
      if (m.kron.factored) {
        go(kron_series_term_staged_kernel<1>);
      } else {
        go(kron_series_term_staged_kernel<0>);
      }
    } else if (m.kron.herm) {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_series_term_kernel<true, 1>, m.kron, true);
        launch_pdl(kron_series_term_kernel<true, 1>, g.first, kThreads, g.second, s, a, m.kron);
      } else {
        const auto g = kron_geom(kron_series_term_kernel<true, 0>, m.kron, true);
        launch_pdl(kron_series_term_kernel<true, 0>, g.first, kThreads, g.second, s, a, m.kron);
      }
    } else {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_series_term_kernel<false, 1>, m.kron);
        launch_pdl(kron_series_term_kernel<false, 1>, g.first, kThreads, g.second, s, a, m.kron);
      } else {
        const auto g = kron_geom(kron_series_term_kernel<false, 0>, m.kron);
        launch_pdl(kron_series_term_kernel<false, 0>, g.first, kThreads, g.second, s, a, m.kron);
      }
    }
  } else if (m.format == Format::Sell) {
    sell_partials(m, x, SkipCheck{ctl, nullptr, 1}, s);
    if (m.group == 1) {
      if (m.sell.work) {
        launch_sell(sell_series_term_kernel<true, kSellStream>, m.sell, s, a, m.sell);
      } else if (m.sell.b_val) {
        launch_sell(sell_series_term_kernel<true, kSellWindows>, m.sell, s, a, m.sell);
      } else {
        launch_sell(sell_series_term_kernel<true, kSellReg>, m.sell, s, a, m.sell);
      }
    } else {
      if (m.sell.work) {
        launch_sell(sell_series_term_kernel<false, kSellStream>, m.sell, s, a, m.sell);
      } else if (m.sell.b_val) {
        launch_sell(sell_series_term_kernel<false, kSellWindows>, m.sell, s, a, m.sell);
      } else {
        launch_sell(sell_series_term_kernel<false, kSellReg>, m.sell, s, a, m.sell);
      }
    }
  } else {
    dispatch_group<SeriesTermK>(m.group, m.csr.rows, s, a, m.csr);
  }
  QSWG_LAUNCH_CHECK("series_term");
}

void series_flush(const SeriesRing& ring, std::int64_t row0, std::int64_t rows, const double2* z,
                  const SeriesSums& sums, int herm_n, int p, bool strict, double tol, SeriesCtl* ctl,
                  bool decide, cudaStream_t s) {
  const SeriesFlushArgs a{ring, row0, rows, z, sums, p, tol, ctl, decide ? 1 : 0, strict ? 0 : herm_n};
  if (strict) {
    launch_pdl(series_flush_kernel<true>, persistent_grid(series_flush_kernel<true>, rows), kThreads, 0, s, a);
  } else {
    launch_pdl(series_flush_kernel<false>, persistent_grid(series_flush_kernel<false>, rows), kThreads, 0, s, a);
  }
  QSWG_LAUNCH_CHECK("series_flush");
}

namespace {
template <bool kFlush>
void launch_w(const DevMatrix& m, const double2* x, int k, const SeriesFlushArgs& fa, cudaStream_t s) {
  if (m.kron.herm) {
    const auto g = kron_geom(kron_w_kernel<true, kFlush>, m.kron);
    launch_pdl(kron_w_kernel<true, kFlush>, g.first, kThreads, g.second, s, m.kron, x, k, fa);
  } else {
    const auto g = kron_geom(kron_w_kernel<false, kFlush>, m.kron);
    launch_pdl(kron_w_kernel<false, kFlush>, g.first, kThreads, g.second, s, m.kron, x, k, fa);
  }
}
}  // namespace

bool kron_prepare_flush(const DevMatrix& m, const double2* x, const SeriesRing& ring, std::int64_t row0,
                        std::int64_t rows, const double2* z, const SeriesSums& sums, int p, double tol,
                        SeriesCtl* ctl, cudaStream_t s) {
  if (m.format != Format::Kron || m.kron.nk == 0) return false;
  const SeriesFlushArgs fa{ring, row0, rows, z, sums, p, tol, ctl, 1, m.kron.herm ? m.kron.n : 0};
  launch_w<true>(m, x, 0, fa, s);
  QSWG_LAUNCH_CHECK("kron_prepare_flush");
  for (int k = 0; k < m.kron.nk; ++k) {
    if (k > 0) {
      launch_w<false>(m, x, k, fa, s);
      QSWG_LAUNCH_CHECK("kron_prepare_flush");
    }
    if (m.kron.factored && !m.kron.herm) {
      const auto gv = kron_geom(kron_v_kernel, m.kron);
      launch_pdl(kron_v_kernel, gv.first, kThreads, gv.second, s, m.kron, x, k);
      QSWG_LAUNCH_CHECK("kron_prepare_flush");
    }
  }
  return true;
}

void kron_prepare(const DevMatrix& m, const double2* x, cudaStream_t s) {
  if (m.format != Format::Kron) return;
  const SeriesFlushArgs none{};
  for (int k = 0; k < m.kron.nk; ++k) {
    launch_w<false>(m, x, k, none, s);
    QSWG_LAUNCH_CHECK("kron_prepare");
    if (m.kron.factored && !m.kron.herm) {  // Hermitian path: V_k = W_k', read from Wt_k
      const auto gv = kron_geom(kron_v_kernel, m.kron);
      launch_pdl(kron_v_kernel, gv.first, kThreads, gv.second, s, m.kron, x, k);
      QSWG_LAUNCH_CHECK("kron_prepare");
    }
  }
}

bool kron_hermitian_check(const DevMatrix& m, const double2* x, cudaStream_t s) {
  if (m.format != Format::Kron || m.kron.herm_flag == nullptr) return false;
  QSWG_CUDA(cudaMemsetAsync(m.kron.herm_flag, 1, sizeof(int), s));  // any non-zero value = Hermitian
  const long long n = m.kron.n;
  const long long want = (n * n + kThreads - 1) / kThreads, cap = sm_count() * 8LL;
  launch_pdl(hermitian_check_kernel, static_cast<int>(want < cap ? (want < 1 ? 1 : want) : cap), kThreads, 0, s, x, n, m.kron.herm_flag);
  QSWG_LAUNCH_CHECK("kron_hermitian_check");
  int flag = 0;
  QSWG_CUDA(cudaMemcpyAsync(&flag, m.kron.herm_flag, sizeof(int), cudaMemcpyDeviceToHost, s));
  QSWG_CUDA(cudaStreamSynchronize(s));
  return flag != 0;
}

void spmv(const DevMatrix& m, const double2* x, double2* y, double scale, cudaStream_t s) {
  if (m.format == Format::Kron) {
    kron_prepare(m, x, s);  // single-GPU product (multi-GPU callers exchange W first)
    if (m.kron.herm) {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_spmv_kernel<true, 1>, m.kron, true);
        launch_pdl(kron_spmv_kernel<true, 1>, g.first, kThreads, g.second, s, m.kron, x, y, scale);
      } else {
        const auto g = kron_geom(kron_spmv_kernel<true, 0>, m.kron, true);
        launch_pdl(kron_spmv_kernel<true, 0>, g.first, kThreads, g.second, s, m.kron, x, y, scale);
      }
    } else {
      if (m.kron.factored) {
        const auto g = kron_geom(kron_spmv_kernel<false, 1>, m.kron);
        launch_pdl(kron_spmv_kernel<false, 1>, g.first, kThreads, g.second, s, m.kron, x, y, scale);
      } else {
        const auto g = kron_geom(kron_spmv_kernel<false, 0>, m.kron);
        launch_pdl(kron_spmv_kernel<false, 0>, g.first, kThreads, g.second, s, m.kron, x, y, scale);
      }
    }
  } else if (m.format == Format::Sell) {
    sell_partials(m, x, SkipCheck{}, s);
    if (m.group == 1) {
      if (m.sell.work) {
        launch_sell(sell_spmv_kernel<true, kSellStream>, m.sell, s, m.sell, x, y, scale);
      } else if (m.sell.b_val) {
        launch_sell(sell_spmv_kernel<true, kSellWindows>, m.sell, s, m.sell, x, y, scale);
      } else {
        launch_sell(sell_spmv_kernel<true, kSellReg>, m.sell, s, m.sell, x, y, scale);
      }
    } else {
      if (m.sell.work) {
        launch_sell(sell_spmv_kernel<false, kSellStream>, m.sell, s, m.sell, x, y, scale);
      } else if (m.sell.b_val) {
        launch_sell(sell_spmv_kernel<false, kSellWindows>, m.sell, s, m.sell, x, y, scale);
      } else {
        launch_sell(sell_spmv_kernel<false, kSellReg>, m.sell, s, m.sell, x, y, scale);
      }
    }
  } else {
    dispatch_group<SpmvK>(m.group, m.csr.rows, s, m.csr, x, y, scale);
  }
  QSWG_LAUNCH_CHECK("spmv");
}

void diag_real(const double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
               double* pops, cudaStream_t s) {
  launch_pdl(diag_kernel, small_grid(n), kThreads, 0, s, v_local, row0, rows, n, pops);
  QSWG_LAUNCH_CHECK("diag_real");
}

void coherence_bits(const double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
                    unsigned long long* out, cudaStream_t s) {
  launch_pdl(coherence_kernel, small_grid(rows), kThreads, 0, s, v_local, row0, rows, n, out);
  QSWG_LAUNCH_CHECK("coherence_bits");
}

void fill_pattern(double2* v, std::int64_t n, cudaStream_t s) {
  launch_pdl(pattern_kernel, small_grid(n), kThreads, 0, s, v, n);
  QSWG_LAUNCH_CHECK("fill_pattern");
}

void fill_pattern_hermitian(double2* v, std::int64_t n, cudaStream_t s) {
  launch_pdl(pattern_hermitian_kernel, small_grid(n * n), kThreads, 0, s, v, n);
  QSWG_LAUNCH_CHECK("fill_pattern_hermitian");
}

void state_from_probabilities(double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
                              const double* p, cudaStream_t s) {
  launch_pdl(probs_kernel, small_grid(rows), kThreads, 0, s, v_local, row0, rows, n, p);
  QSWG_LAUNCH_CHECK("state_from_probabilities");
}

}  // namespace qswg::dev
