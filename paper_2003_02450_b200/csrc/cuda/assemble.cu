// Device assembly of the N^2 x N^2 superoperator in canonical CSR.
//
// Replaces LiouvillianBuilder::build + the build_local / build_global row
// emitters + SparseMatrix::from_triplets (liouvillian.cpp:37-84, 129-307;
// sparse.cpp:25-64).  Instead of emitting O(nnz) triplets and sorting them,
// each row r = n*j + i is produced by a k-way merge of already-sorted column
// streams (see KronOperands in kernels.hpp), summing equal columns and
// dropping exact zeros on the fly:
//   pass 1 (count) -> exclusive scan -> pass 2 (fill).
// One thread per row; the operand lists are the small n x n operators and
// stay L1/L2 resident.  The same kernel assembles |L^T| (for the 1-norm
// bound) from transposed operand lists.
#include <cub/device/device_scan.cuh>
#include <cub/device/device_segmented_sort.cuh>

#include <climits>

#include "../kernels.hpp"
#include "common.cuh"

namespace qswg::dev {

namespace {

struct Cursor {
  int pos, end;
};

struct RowMerge {
  long long n, i, j, r;
  Cursor a, b, t;
  int pa[kMaxKron], pe[kMaxKron], qb[kMaxKron], qe[kMaxKron], qpos[kMaxKron];
  bool decay_pending;
  double decay;
};

__device__ __forceinline__ double2 cadd(double2 x, double2 y) { return make_double2(x.x + y.x, x.y + y.y); }
// std::complex<double> product (expm/liouvillian use it for finite values).
__device__ __forceinline__ double2 cmul(double2 x, double2 y) {
  return make_double2(__dsub_rn(__dmul_rn(x.x, y.x), __dmul_rn(x.y, y.y)),
                      __dadd_rn(__dmul_rn(x.x, y.y), __dmul_rn(x.y, y.x)));
}

__device__ __forceinline__ void merge_init(const KronOperands& o, long long r, RowMerge& m) {
  m.n = o.n;
  m.j = r / o.n;
  m.i = r - m.j * o.n;
  m.r = r;
  const int i = static_cast<int>(m.i), j = static_cast<int>(m.j);
  m.a = o.a.ptr ? Cursor{__ldg(o.a.ptr + i), __ldg(o.a.ptr + i + 1)} : Cursor{0, 0};
  m.b = o.b.ptr ? Cursor{__ldg(o.b.ptr + j), __ldg(o.b.ptr + j + 1)} : Cursor{0, 0};
  m.t = (o.t.ptr && i == j) ? Cursor{__ldg(o.t.ptr + i), __ldg(o.t.ptr + i + 1)} : Cursor{0, 0};
#pragma unroll
  for (int k = 0; k < kMaxKron; ++k) {
    if (k < o.nk) {
      m.pa[k] = __ldg(o.p[k].ptr + j);
      m.pe[k] = __ldg(o.p[k].ptr + j + 1);
      m.qb[k] = __ldg(o.q[k].ptr + i);
      m.qe[k] = __ldg(o.q[k].ptr + i + 1);
      if (m.qb[k] == m.qe[k]) m.pa[k] = m.pe[k];  // empty Q row: no products
      m.qpos[k] = m.qb[k];
    } else {
      m.pa[k] = m.pe[k] = 0;
      m.qb[k] = m.qe[k] = m.qpos[k] = 0;
    }
  }
  m.decay_pending = false;
  m.decay = 0.0;
  if (o.d_loc) {
    // liouvillian.cpp:180-183, same expression order.
    // 0.5 * (omega * (dl_i + dl_j) + ds_i + ds_j), evaluated without contraction
    const double d = __dmul_rn(
        0.5, __dadd_rn(__dadd_rn(__dmul_rn(o.omega, __dadd_rn(__ldg(o.d_loc + i), __ldg(o.d_loc + j))),
                                 __ldg(o.d_ss + i)),
                       __ldg(o.d_ss + j)));
    if (d != 0.0) {
      m.decay_pending = true;
      m.decay = -d;
    }
  }
}

// Emits the next summed column of the row; returns false when exhausted.
// Contributions to one column are added in stream order A, B, P(x)Q, decay, T.
__device__ __forceinline__ bool merge_next(const KronOperands& o, RowMerge& m, long long& col,
                                           double2& val) {
  while (true) {
    long long c = LLONG_MAX;
    if (m.a.pos < m.a.end) c = min(c, m.n * m.j + __ldg(o.a.col + m.a.pos));
    if (m.b.pos < m.b.end) c = min(c, m.n * __ldg(o.b.col + m.b.pos) + m.i);
#pragma unroll
    for (int k = 0; k < kMaxKron; ++k)
      if (k < o.nk && m.pa[k] < m.pe[k])
        c = min(c, m.n * __ldg(o.p[k].col + m.pa[k]) + __ldg(o.q[k].col + m.qpos[k]));
    if (m.decay_pending) c = min(c, m.r);
    if (m.t.pos < m.t.end) {
      const long long tc = __ldg(o.t.col + m.t.pos);
      c = min(c, m.n * tc + tc);
    }
    if (c == LLONG_MAX) return false;

    double2 s = make_double2(0.0, 0.0);
    while (m.a.pos < m.a.end && m.n * m.j + __ldg(o.a.col + m.a.pos) == c) s = cadd(s, __ldg(o.a.val + m.a.pos++));
    while (m.b.pos < m.b.end && m.n * __ldg(o.b.col + m.b.pos) + m.i == c) s = cadd(s, __ldg(o.b.val + m.b.pos++));
#pragma unroll
    for (int k = 0; k < kMaxKron; ++k) {
      if (k < o.nk && m.pa[k] < m.pe[k] &&
          m.n * __ldg(o.p[k].col + m.pa[k]) + __ldg(o.q[k].col + m.qpos[k]) == c) {
        s = cadd(s, cmul(__ldg(o.p[k].val + m.pa[k]), __ldg(o.q[k].val + m.qpos[k])));
        if (++m.qpos[k] == m.qe[k]) {
          m.qpos[k] = m.qb[k];
          ++m.pa[k];
        }
      }
    }
    if (m.decay_pending && m.r == c) {
      s.x = s.x + m.decay;
      m.decay_pending = false;
    }
    while (m.t.pos < m.t.end) {
      const long long tc = __ldg(o.t.col + m.t.pos);
      if (m.n * tc + tc != c) break;
      s = cadd(s, __ldg(o.t.val + m.t.pos++));
    }
    if (s.x != 0.0 || s.y != 0.0) {
      col = c;
      val = s;
      return true;
    }
  }
}

// Entries of each row with column in [c_lo, c_hi) (a column panel; the
// whole row for [0, LLONG_MAX)).  Columns come out of the merge increasing.
__global__ void __launch_bounds__(kThreads) count_kernel(KronOperands o, long long row0, long long rows,
                                                         long long* counts, long long c_lo, long long c_hi) {
  for (long long lr = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; lr < rows;
       lr += static_cast<long long>(gridDim.x) * blockDim.x) {
    RowMerge m;
    merge_init(o, row0 + lr, m);
    long long c;
    double2 v;
    long long cnt = 0;
    while (merge_next(o, m, c, v)) {
      if (c >= c_hi) break;
      cnt += c >= c_lo;
    }
    counts[lr] = cnt;
  }
}

template <bool kAbs>
__global__ void __launch_bounds__(kThreads) fill_kernel(KronOperands o, long long row0, long long rows,
                                                        const long long* rowptr, int* col, void* val) {
  for (long long lr = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; lr < rows;
       lr += static_cast<long long>(gridDim.x) * blockDim.x) {
    RowMerge m;
    merge_init(o, row0 + lr, m);
    long long c;
    double2 v;
    long long k = rowptr[lr];
    while (merge_next(o, m, c, v)) {
      col[k] = static_cast<int>(c);
      if constexpr (kAbs) {
        static_cast<double*>(val)[k] = hypot(v.x, v.y);
      } else {
        static_cast<double2*>(val)[k] = v;
      }
      ++k;
    }
  }
}

__global__ void __launch_bounds__(kThreads) fill_sell_kernel(KronOperands o, long long row0, long long rows,
                                                             const long long* slice_ptr, const int* perm, int* col,
                                                             double2* val, long long c_lo, long long c_hi) {
  // every lane of every slice, including the lanes past the last row of a
  // partial final slice (pure padding)
  const long long padded_rows = (rows + kSlice - 1) / kSlice * kSlice;
  for (long long lr = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; lr < padded_rows;
       lr += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long sl = lr / kSlice;
    const long long base = slice_ptr[sl] + (lr - sl * kSlice);
    const long long len = (slice_ptr[sl + 1] - slice_ptr[sl]) / kSlice;
    long long k = 0;
    const long long row = lr < rows ? (perm ? perm[lr] : lr) : rows - 1;
    if (lr < rows) {
      RowMerge m;
      merge_init(o, row0 + row, m);
      long long c;
      double2 v;
      while (merge_next(o, m, c, v)) {
        if (c >= c_hi) break;
        if (c < c_lo) continue;
        col[base + k * kSlice] = static_cast<int>(c);
        val[base + k * kSlice] = v;
        ++k;
      }
    }
    const int pad_col = static_cast<int>(row0 + row);
    for (; k < len; ++k) {  // padding: x[row] * 0
      col[base + k * kSlice] = pad_col;
      val[base + k * kSlice] = make_double2(0.0, 0.0);
    }
  }
}

__global__ void slice_len_kernel(const long long* grp, long long rows, const int* perm, long long n_slices,
                                 long long* out) {
  for (long long sl = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; sl < n_slices;
       sl += static_cast<long long>(gridDim.x) * blockDim.x) {
    long long mx = 0;
    const long long t1 = min(rows, (sl + 1) * kSlice);
    for (long long t = sl * kSlice; t < t1; ++t) {
      const long long r = perm ? perm[t] : t;
      mx = max(mx, grp[r + 1] - grp[r]);
    }
    out[sl] = mx * kSlice;
  }
}

__global__ void row_len_kernel(const long long* grp, long long rows, int sigma, int* len, int* idx, int* seg) {
  for (long long r = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; r < rows;
       r += static_cast<long long>(gridDim.x) * blockDim.x) {
    len[r] = static_cast<int>(grp[r + 1] - grp[r]);
    idx[r] = static_cast<int>(r);
    if (r % sigma == 0) seg[r / sigma] = static_cast<int>(r);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) seg[(rows + sigma - 1) / sigma] = static_cast<int>(rows);
}

__global__ void rebase_kernel(const long long* src, long long base, long long* dst, long long n) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    dst[k] = src[k] - base;
}

__global__ void hull_kernel(const int* col, long long n, const long long* starts, int world, int rank,
                            long long* lo, long long* hi) {
  long long mn[8], mx[8];
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    mn[q] = LLONG_MAX;
    mx[q] = LLONG_MIN;
  }
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long c = col[k];
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q < world && q != rank && c >= starts[q] && c < starts[q + 1]) {
        mn[q] = min(mn[q], c);
        mx[q] = max(mx[q], c + 1);
      }
    }
  }
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    if (q < world && mn[q] != LLONG_MAX) {
      atomicMin(lo + q, mn[q]);
      atomicMax(hi + q, mx[q]);
    }
  }
}

int grid_for(long long rows) {
  long long want = (rows + kThreads - 1) / kThreads;
  long long cap = static_cast<long long>(sm_count()) * 8;
  return static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap));
}

}  // namespace

void assemble_count(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                    std::int64_t* counts, cudaStream_t s, std::int64_t c_lo, std::int64_t c_hi) {
  if (rows <= 0) return;
  count_kernel<<<grid_for(rows), kThreads, 0, s>>>(o, row0, rows, reinterpret_cast<long long*>(counts), c_lo, c_hi);
  QSWG_LAUNCH_CHECK("assemble_count");
}

void exclusive_scan(const std::int64_t* counts, std::int64_t* rowptr, std::int64_t n, void* tmp,
                    std::size_t& tmp_bytes, cudaStream_t s) {
  QSWG_CUDA(cub::DeviceScan::ExclusiveSum(tmp, tmp_bytes, counts, rowptr, n, s));
}

void halo_hulls(const int* col, std::int64_t n, const std::int64_t* starts, int world, int rank, std::int64_t* lo,
                std::int64_t* hi, cudaStream_t s) {
  if (world > 8) throw std::invalid_argument("at most 8 ranks per communicator");
  if (n <= 0) return;
  hull_kernel<<<grid_for(n), kThreads, 0, s>>>(col, n, reinterpret_cast<const long long*>(starts), world, rank,
                                               reinterpret_cast<long long*>(lo), reinterpret_cast<long long*>(hi));
  QSWG_LAUNCH_CHECK("halo_hulls");
}

void rebase_rowptr(const std::int64_t* src, std::int64_t base, std::int64_t* dst, std::int64_t n,
                   cudaStream_t s) {
  rebase_kernel<<<grid_for(n), kThreads, 0, s>>>(reinterpret_cast<const long long*>(src), base,
                                                 reinterpret_cast<long long*>(dst), n);
  QSWG_LAUNCH_CHECK("rebase_rowptr");
}

void assemble_fill(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                   const std::int64_t* rowptr, int* col, double2* val, cudaStream_t s) {
  if (rows <= 0) return;
  fill_kernel<false><<<grid_for(rows), kThreads, 0, s>>>(
      o, row0, rows, reinterpret_cast<const long long*>(rowptr), col, val);
  QSWG_LAUNCH_CHECK("assemble_fill");
}

void sell_slice_entries(const std::int64_t* grp_local, std::int64_t rows, const int* perm,
                        std::int64_t* slice_entries, cudaStream_t s) {
  const long long n_slices = (rows + kSlice - 1) / kSlice;
  if (n_slices <= 0) return;
  slice_len_kernel<<<grid_for(n_slices), kThreads, 0, s>>>(reinterpret_cast<const long long*>(grp_local), rows, perm,
                                                           n_slices, reinterpret_cast<long long*>(slice_entries));
  QSWG_LAUNCH_CHECK("sell_slice_entries");
}

void assemble_fill_sell(const KronOperands& o, std::int64_t row0, std::int64_t rows, const std::int64_t* slice_ptr,
                        const int* perm, int* col, double2* val, cudaStream_t s, std::int64_t c_lo,
                        std::int64_t c_hi) {
  if (rows <= 0) return;
  fill_sell_kernel<<<grid_for(rows + kSlice), kThreads, 0, s>>>(o, row0, rows, reinterpret_cast<const long long*>(slice_ptr),
                                                       perm, col, val, c_lo, c_hi);
  QSWG_LAUNCH_CHECK("assemble_fill_sell");
}

void sell_sort_rows(const std::int64_t* grp_local, std::int64_t rows, int sigma, int* perm, cudaStream_t s) {
  if (rows <= 0) return;
  const long long nseg = (rows + sigma - 1) / sigma;
  int *len = nullptr, *len_out = nullptr, *idx = nullptr, *seg = nullptr;
  QSWG_CHECK(cudaMallocAsync(&len, sizeof(int) * rows, s));
  QSWG_CHECK(cudaMallocAsync(&len_out, sizeof(int) * rows, s));
  QSWG_CHECK(cudaMallocAsync(&idx, sizeof(int) * rows, s));
  QSWG_CHECK(cudaMallocAsync(&seg, sizeof(int) * (nseg + 1), s));
  row_len_kernel<<<grid_for(rows), kThreads, 0, s>>>(reinterpret_cast<const long long*>(grp_local), rows, sigma, len,
                                                     idx, seg);
  QSWG_LAUNCH_CHECK("row_len");
  std::size_t bytes = 0;
  QSWG_CHECK(cub::DeviceSegmentedSort::StableSortPairsDescending(nullptr, bytes, len, len_out, idx, perm,
                                                                  static_cast<int>(rows), static_cast<int>(nseg), seg,
                                                                  seg + 1, s));
  void* tmp = nullptr;
  QSWG_CHECK(cudaMallocAsync(&tmp, bytes, s));
  QSWG_CHECK(cub::DeviceSegmentedSort::StableSortPairsDescending(tmp, bytes, len, len_out, idx, perm,
                                                                  static_cast<int>(rows), static_cast<int>(nseg), seg,
                                                                  seg + 1, s));
  for (void* p : {static_cast<void*>(len), static_cast<void*>(len_out), static_cast<void*>(idx),
                  static_cast<void*>(seg), tmp})
    QSWG_CHECK(cudaFreeAsync(p, s));
}

void assemble_fill_abs(const KronOperands& o, std::int64_t row0, std::int64_t rows,
                       const std::int64_t* rowptr, int* col, double* val, cudaStream_t s) {
  if (rows <= 0) return;
  fill_kernel<true><<<grid_for(rows), kThreads, 0, s>>>(
      o, row0, rows, reinterpret_cast<const long long*>(rowptr), col, val);
  QSWG_LAUNCH_CHECK("assemble_fill_abs");
}

}  // namespace qswg::dev
