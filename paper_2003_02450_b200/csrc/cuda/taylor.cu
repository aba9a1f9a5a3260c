// The truncated-Taylor loop on sm_100a: fused SpMV + axpy + infinity-norm
// reductions + the early-termination test, all on the device.
//
// Replaces the reference's per-term WorkerPool rounds
//   worker_multiply (liouvillian.cpp:105-127) + the step axpy/norm loop
//   (expm.cpp:175-195) and the series lazy-term SpMV + per-k axpy/norm loops
//   (expm.cpp:283-316).
// The path is HBM-bound complex128 SpMV (~0.4 flop/B), so there are no
// tensor-core ops here: rows are processed by groups of G lanes (G in
// {2,4,8,16,32}, autotuned per matrix) in a persistent grid-stride loop;
// values/columns stream with an L2 evict-first policy so the gathered vector
// stays L2-resident; the axpy and both inf-norms are fused into the epilogue;
// the grid-wide maxima use the uint64 bit order of non-negative doubles
// (order-independent, hence deterministic) and the LAST block to arrive
// evaluates the stop test c1 + c2 <= tol * ||sum|| and publishes it for the
// next launch, so the host never synchronises inside a step or a series.
#include "../kernels.hpp"
#include "common.cuh"

namespace qswg::dev {

namespace {

__device__ __forceinline__ double cabs2(double2 v) { return hypot(v.x, v.y); }

// Row-group SpMV core: returns the full row sum in every lane of the group.
// G == 1 is the bitwise "reference order" mode: one thread per row, columns
// in CSR order, every product and sum rounded separately (no FMA) — exactly
// `acc += vals[k] * x[...]` of liouvillian.cpp:120-124 in a no-FMA build.
template <int G>
__device__ __forceinline__ double2 row_dot(const CsrView& l, long long row, bool valid,
                                           const double2* __restrict__ x, int lane,
                                           unsigned long long pol) {
  double2 acc = make_double2(0.0, 0.0);
  if constexpr (G == 1) {
    if (valid) {
      const long long b = __ldg(l.rowptr + row), e = __ldg(l.rowptr + row + 1);
      for (long long k = b; k < e; ++k) {
        const double2 v = ld_stream(l.val + k, pol);
        const double2 xv = __ldg(x + ld_stream(l.col + k, pol));
        acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(v.x, xv.x), __dmul_rn(v.y, xv.y)));
        acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(v.x, xv.y), __dmul_rn(v.y, xv.x)));
      }
    }
    return acc;
  }
  if (valid) {
    const long long b = __ldg(l.rowptr + row), e = __ldg(l.rowptr + row + 1);
    long long k = b + lane;
    for (; k + G < e; k += 2 * G) {
      const int c0 = ld_stream(l.col + k, pol);
      const int c1 = ld_stream(l.col + k + G, pol);
      const double2 v0 = ld_stream(l.val + k, pol);
      const double2 v1 = ld_stream(l.val + k + G, pol);
      const double2 x0 = __ldg(x + c0);
      const double2 x1 = __ldg(x + c1);
      acc.x = fma(v0.x, x0.x, acc.x);
      acc.x = fma(-v0.y, x0.y, acc.x);
      acc.y = fma(v0.x, x0.y, acc.y);
      acc.y = fma(v0.y, x0.x, acc.y);
      acc.x = fma(v1.x, x1.x, acc.x);
      acc.x = fma(-v1.y, x1.y, acc.x);
      acc.y = fma(v1.x, x1.y, acc.y);
      acc.y = fma(v1.y, x1.x, acc.y);
    }
    if (k < e) {
      const int c0 = ld_stream(l.col + k, pol);
      const double2 v0 = ld_stream(l.val + k, pol);
      const double2 x0 = __ldg(x + c0);
      acc.x = fma(v0.x, x0.x, acc.x);
      acc.x = fma(-v0.y, x0.y, acc.x);
      acc.y = fma(v0.x, x0.y, acc.y);
      acc.y = fma(v0.y, x0.x, acc.y);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    acc.x += __shfl_xor_sync(0xffffffffu, acc.x, o);
    acc.y += __shfl_xor_sync(0xffffffffu, acc.y, o);
  }
  return acc;
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

// Grid-stride iteration over rows in warp-uniform steps (all lanes of a warp
// run the same trip count, so the group shuffles are always convergent).
template <int G>
struct RowIter {
  long long first, stride;
  int lane, sub;
  __device__ RowIter() {
    const long long warp = (blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x) >> 5;
    const long long nwarps = (static_cast<long long>(gridDim.x) * blockDim.x) >> 5;
    const int wl = threadIdx.x & 31;
    sub = wl / G;
    lane = wl & (G - 1);
    first = warp * (32 / G);
    stride = nwarps * (32 / G);
  }
};

// ---------------------------------------------------------------- step term
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
};

template <int G>
__global__ void __launch_bounds__(kThreads) step_term_kernel(StepTermArgs a) {
  StepCtl* ctl = a.ctl;
  if (*(volatile int*)&ctl->error) return;
  if (!a.first_of_stage && *(volatile int*)&ctl->done) return;
  __shared__ unsigned long long red[32];
  __shared__ bool last;
  const unsigned long long pol = evict_first_policy();
  RowIter<G> it;
  unsigned long long tmax = 0, smax = 0;
  for (long long r0 = it.first; r0 < a.l.rows; r0 += it.stride) {
    const long long row = r0 + it.sub;
    const bool valid = row < a.l.rows;
    const double2 acc = row_dot<G>(a.l, row, valid, a.x, it.lane, pol);
    if (valid && it.lane == 0) {
      // y = scale * acc, scale = Complex{t/(s*j), 0} (liouvillian.cpp:125)
      const double2 yv = make_double2(__dmul_rn(a.scale, acc.x), __dmul_rn(a.scale, acc.y));
      a.y[row] = yv;
      const double2 sv0 = a.sum_in[row];
      const double2 sv = make_double2(sv0.x + yv.x, sv0.y + yv.y);  // expm.cpp:181
      a.sum_out[row] = sv;
      tmax = umax64(tmax, dbits(cabs2(yv)));
      smax = umax64(smax, dbits(cabs2(sv)));
    }
  }
  tmax = block_max_bits(tmax, red);
  smax = block_max_bits(smax, red);
  if (threadIdx.x == 0) {
    atomicMax(&ctl->term_bits, tmax);
    atomicMax(&ctl->sum_bits, smax);
    __threadfence();
    last = atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1;
    if (last) {
      __threadfence();
      const double c2 = bitsd(atomicAdd(&ctl->term_bits, 0ull));
      const double nf = bitsd(atomicAdd(&ctl->sum_bits, 0ull));
      ctl->spmvs += 1;
      if (!isfinite(c2) || !isfinite(nf)) {  // expm.cpp:191-193
        ctl->error = 1;
        ctl->done = 1;
      } else {
        // stage start: c1 = ||v|| (stage 0, from step_init) or ||sum|| of the
        // previous stage (expm.cpp:197-205) which is that stage's last nf.
        const double c1 = a.first_of_stage ? (a.stage == 0 ? ctl->c1 : ctl->last_nf) : ctl->c1;
        ctl->done = (c1 + c2 <= a.tol * nf) ? 1 : 0;  // expm.cpp:194
        ctl->c1 = c2;
        ctl->last_nf = nf;
      }
      ctl->term_bits = 0;
      ctl->sum_bits = 0;
      ctl->arrivals = 0;
    }
  }
}

// ------------------------------------------------------------- series term
// Per-k stop tests after term p (expm.cpp:298-316, evaluated p-major): run
// by one thread of the last block to arrive.
__device__ void series_control(SeriesCtl* ctl, int count, double tol) {
  ctl->spmvs += 1;
  const double tn = bitsd(*(volatile unsigned long long*)&ctl->term_bits);
  if (!isfinite(tn)) ctl->error = 1;  // expm.cpp:293-295
  for (int k = 0; k < count; ++k) {
    if (!ctl->active[k]) continue;
    const double f = ctl->factor[k];
    const double c2 = f * tn;  // expm.cpp:310
    const double nf = bitsd(*(volatile unsigned long long*)&ctl->sum_bits[k]);
    if (!isfinite(nf)) {  // expm.cpp:312-314
      ctl->error = 1;
    } else if (ctl->c1[k] + c2 <= tol * nf) {  // expm.cpp:315
      ctl->active[k] = 0;
      ctl->n_active -= 1;
    } else {
      ctl->c1[k] = c2;
    }
    ctl->factor[k] = f * static_cast<double>(k + 1);  // factor *= k for p + 1
    ctl->sum_bits[k] = 0;
  }
  if (ctl->error) ctl->n_active = 0;
  ctl->term_bits = 0;
  ctl->arrivals = 0;
}


struct SeriesTermArgs {
  CsrView l;
  const double2* x;
  double2* kp;
  const double2* z;
  SeriesSums sums;
  int count;
  int p;
  double scale;
  double tol;
  SeriesCtl* ctl;
};

template <int G>
__global__ void __launch_bounds__(kThreads) series_term_kernel(SeriesTermArgs a) {
  SeriesCtl* ctl = a.ctl;
  if (*(volatile int*)&ctl->error || *(volatile int*)&ctl->n_active == 0) return;
  __shared__ unsigned long long red[32];
  __shared__ double fac[kMaxSeriesD];
  __shared__ int act[kMaxSeriesD];
  __shared__ unsigned long long smax_sh[kMaxSeriesD];
  for (int k = threadIdx.x; k < a.count; k += blockDim.x) {
    fac[k] = ctl->factor[k];
    act[k] = ctl->active[k];
    smax_sh[k] = 0;
  }
  __syncthreads();
  const unsigned long long pol = evict_first_policy();
  RowIter<G> it;
  unsigned long long tmax = 0;
  unsigned long long smax[kSeriesRegD];
#pragma unroll
  for (int k = 0; k < kSeriesRegD; ++k) smax[k] = 0;
  const bool first = a.p == 1;
  for (long long r0 = it.first; r0 < a.l.rows; r0 += it.stride) {
    const long long row = r0 + it.sub;
    const bool valid = row < a.l.rows;
    const double2 acc = row_dot<G>(a.l, row, valid, a.x, it.lane, pol);
    if (valid && it.lane == 0) {
      const double2 kv = make_double2(__dmul_rn(a.scale, acc.x), __dmul_rn(a.scale, acc.y));  // (h/p) L K_{p-1}
      a.kp[row] = kv;
      tmax = umax64(tmax, dbits(cabs2(kv)));
      const double2 zv = first ? a.z[row] : make_double2(0.0, 0.0);
#pragma unroll
      for (int k = 0; k < kSeriesRegD; ++k) {
        if (k < a.count && act[k]) {
          double2* s = a.sums.s[k];
          const double2 sv0 = first ? zv : s[row];
          const double f = fac[k];
          const double2 sv = axpy<G>(sv0, f, kv);  // expm.cpp:303
          s[row] = sv;
          smax[k] = umax64(smax[k], dbits(cabs2(sv)));
        }
      }
      for (int k = kSeriesRegD; k < a.count; ++k) {
        if (act[k]) {
          double2* s = a.sums.s[k];
          const double2 sv0 = first ? zv : s[row];
          const double f = fac[k];
          const double2 sv = axpy<G>(sv0, f, kv);
          s[row] = sv;
          atomicMax(&smax_sh[k], dbits(cabs2(sv)));
        }
      }
    }
  }
  tmax = block_max_bits(tmax, red);
  if (threadIdx.x == 0) atomicMax(&ctl->term_bits, tmax);
#pragma unroll
  for (int k = 0; k < kSeriesRegD; ++k) {
    if (k < a.count) {  // block-uniform
      const unsigned long long m = block_max_bits(smax[k], red);
      if (threadIdx.x == 0 && act[k]) atomicMax(&ctl->sum_bits[k], m);
    }
  }
  __syncthreads();
  for (int k = kSeriesRegD + threadIdx.x; k < a.count; k += blockDim.x)
    if (act[k]) atomicMax(&ctl->sum_bits[k], smax_sh[k]);
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(&ctl->arrivals, 1u) == gridDim.x - 1) {
      __threadfence();
      series_control(ctl, a.count, a.tol);
    }
  }
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
    m = umax64(m, dbits(cabs2(v[k])));
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

__global__ void __launch_bounds__(kThreads) step_init_kernel(const double2* v, long long n, StepCtl* ctl) {
  norm_body(v, n, &ctl->term_bits, &ctl->arrivals, [ctl](double nv) {
    ctl->c1 = nv;  // expm.cpp:165-170
    ctl->last_nf = nv;
    ctl->done = 0;  // `error` and `spmvs` are sticky across calls
    ctl->sum_bits = 0;
    ctl->term_bits = 0;
    ctl->arrivals = 0;
  });
}

__global__ void __launch_bounds__(kThreads) series_init_kernel(const double2* z, long long n, int count,
                                                              SeriesCtl* ctl) {
  norm_body(z, n, &ctl->term_bits, &ctl->arrivals, [ctl, count](double nz) {
    ctl->z_norm = nz;  // expm.cpp:271-276
    ctl->count = count;
    ctl->n_active = ctl->error ? 0 : count;  // `error` and `spmvs` are sticky
    for (int k = 0; k < count; ++k) {
      ctl->active[k] = 1;
      ctl->factor[k] = static_cast<double>(k + 1);  // factor *= k at p = 1
      ctl->c1[k] = nz;
      ctl->sum_bits[k] = 0;
    }
    ctl->term_bits = 0;
    ctl->arrivals = 0;
  });
}

// --------------------------------------------------------------- plain SpMV
template <int G>
__global__ void __launch_bounds__(kThreads) spmv_kernel(CsrView l, const double2* x, double2* y, double scale) {
  const unsigned long long pol = evict_first_policy();
  RowIter<G> it;
  for (long long r0 = it.first; r0 < l.rows; r0 += it.stride) {
    const long long row = r0 + it.sub;
    const bool valid = row < l.rows;
    const double2 acc = row_dot<G>(l, row, valid, x, it.lane, pol);
    if (valid && it.lane == 0) y[row] = make_double2(scale * acc.x, scale * acc.y);
  }
}

__global__ void diag_kernel(const double2* v, long long row0, long long rows, long long n, double* pops) {
  for (long long i = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = i * (n + 1) - row0;
    if (g >= 0 && g < rows) pops[i] = v[g].x;
  }
}

__global__ void probs_kernel(double2* v, long long row0, long long rows, long long n, const double* p) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < rows;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long g = row0 + k;
    const long long j = g / n, i = g - j * n;
    v[k] = make_double2(i == j ? p[i] : 0.0, 0.0);
  }
}

__global__ void pattern_kernel(double2* v, long long n) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const unsigned long long h = (static_cast<unsigned long long>(k) + 1) * 0x9E3779B97F4A7C15ull;
    v[k] = make_double2(static_cast<double>(h >> 11) * 0x1p-53 - 0.5,
                        static_cast<double>((h * 0xBF58476D1CE4E5B9ull) >> 11) * 0x1p-53 - 0.5);
  }
}

// ------------------------------------------------------------ launch helpers
template <class K>
int persistent_grid(K kernel, long long work_items) {
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, 0);
  if (per_sm < 1) per_sm = 1;
  const long long cap = static_cast<long long>(sm_count()) * per_sm;
  long long want = (work_items + kThreads - 1) / kThreads;
  if (want < 1) want = 1;
  return static_cast<int>(want < cap ? want : cap);
}

int small_grid(long long n) {
  long long want = (n + kThreads - 1) / kThreads, cap = sm_count() * 4LL;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

template <template <int> class KT, class... Args>
void dispatch_group(int g, long long rows, cudaStream_t s, Args... args) {
  switch (g) {
#define QSWG_G(GV)                                                                   \
  case GV: {                                                                         \
    auto k = KT<GV>::fn;                                                             \
    k<<<persistent_grid(k, rows * GV), kThreads, 0, s>>>(args...);                  \
    break;                                                                           \
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

void step_init(const double2* v, std::int64_t n, StepCtl* ctl, cudaStream_t s) {
  step_init_kernel<<<small_grid(n), kThreads, 0, s>>>(v, n, ctl);
  QSWG_LAUNCH_CHECK("step_init");
}

void step_term(const CsrView& l, int group, const double2* x, double2* y, const double2* sum_in,
               double2* sum_out, double scale, bool first_of_stage, int stage, double tol,
               StepCtl* ctl, cudaStream_t s) {
  StepTermArgs a{l, x, y, sum_in, sum_out, scale, tol, ctl, first_of_stage ? 1 : 0, stage};
  dispatch_group<StepTermK>(group, l.rows, s, a);
  QSWG_LAUNCH_CHECK("step_term");
}

void series_init(const double2* z, std::int64_t n, int count, SeriesCtl* ctl, cudaStream_t s) {
  if (count < 1 || count > kMaxSeriesD) throw std::invalid_argument("series super-step size out of range");
  series_init_kernel<<<small_grid(n), kThreads, 0, s>>>(z, n, count, ctl);
  QSWG_LAUNCH_CHECK("series_init");
}

void series_term(const CsrView& l, int group, const double2* x, double2* kp, const double2* z,
                 const SeriesSums& sums, int count, int p, double scale, double tol,
                 SeriesCtl* ctl, cudaStream_t s) {
  SeriesTermArgs a{l, x, kp, z, sums, count, p, scale, tol, ctl};
  dispatch_group<SeriesTermK>(group, l.rows, s, a);
  QSWG_LAUNCH_CHECK("series_term");
}

void spmv(const CsrView& l, int group, const double2* x, double2* y, double scale, cudaStream_t s) {
  dispatch_group<SpmvK>(group, l.rows, s, l, x, y, scale);
  QSWG_LAUNCH_CHECK("spmv");
}

void diag_real(const double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
               double* pops, cudaStream_t s) {
  diag_kernel<<<small_grid(n), kThreads, 0, s>>>(v_local, row0, rows, n, pops);
  QSWG_LAUNCH_CHECK("diag_real");
}

void fill_pattern(double2* v, std::int64_t n, cudaStream_t s) {
  pattern_kernel<<<small_grid(n), kThreads, 0, s>>>(v, n);
  QSWG_LAUNCH_CHECK("fill_pattern");
}

void state_from_probabilities(double2* v_local, std::int64_t row0, std::int64_t rows, std::int64_t n,
                              const double* p, cudaStream_t s) {
  probs_kernel<<<small_grid(rows), kThreads, 0, s>>>(v_local, row0, rows, n, p);
  QSWG_LAUNCH_CHECK("state_from_probabilities");
}

}  // namespace qswg::dev
