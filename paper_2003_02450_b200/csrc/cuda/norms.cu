// 1-norm power series ||L^p||_1, p = 1..9 (liouvillian.cpp:309-344).
//
// dim <= 4096: exact.  The reference forms sparse powers on the host,
// P <- P * L by Gustavson (sparse.cpp:178-208); here P is dense and
// Y[i][c] = sum over k of P[i][k] L[k][c] is summed in the same order —
// ascending k, zero P entries skipped (the reference drops them), complex
// products rounded like std::complex (no contraction) — so every power is
// bit-identical to the reference's; then per-column sums of |.| in ascending
// row order (the reference's one_norm order, sparse.cpp:134-140).
// dim > 4096: the bound max(1^T |L|^p): v <- |L|^T v from v = 1.  |L^T| is
// assembled by the same merge kernel from transposed operands, so each
// next[r] is a plain row-ordered sum in ascending original-row order with no
// FMA — the reference's accumulation order (liouvillian.cpp:327-339),
// deterministic and without fp64 atomics.
#include "../kernels.hpp"
#include <cstring>
#include <vector>

#include "common.cuh"

namespace qswg::dev {

namespace {

// Y[i][c] = sum_k X[i][k] L[k][c], k ascending over column c of L (CSC:
// lcp / lrow / lval); X, Y row-major dim x dim.
__global__ void __launch_bounds__(kThreads) dense_power_kernel(const long long* __restrict__ lcp,
                                                               const int* __restrict__ lrow,
                                                               const double2* __restrict__ lval, long long dim,
                                                               const double2* __restrict__ x,
                                                               double2* __restrict__ y) {
  const long long i = blockIdx.y;
  const double2* xi = x + i * dim;
  for (long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; c < dim;
       c += static_cast<long long>(gridDim.x) * blockDim.x) {
    double2 acc = make_double2(0.0, 0.0);
    const long long b = __ldg(lcp + c), e = __ldg(lcp + c + 1);
    for (long long k = b; k < e; ++k) {
      const double2 w = xi[__ldg(lrow + k)];
      if (w.x == 0.0 && w.y == 0.0) continue;  // not stored in the reference's power
      const double2 a = __ldg(lval + k);
      acc.x = __dadd_rn(acc.x, __dsub_rn(__dmul_rn(w.x, a.x), __dmul_rn(w.y, a.y)));
      acc.y = __dadd_rn(acc.y, __dadd_rn(__dmul_rn(w.x, a.y), __dmul_rn(w.y, a.x)));
    }
    y[i * dim + c] = acc;
  }
}

__global__ void __launch_bounds__(kThreads) colsum_kernel(const double2* __restrict__ y, long long dim,
                                                          double* __restrict__ colsum) {
  const long long c = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x;
  if (c >= dim) return;
  double s = 0.0;
  for (long long r = 0; r < dim; ++r) {
    const double2 v = y[r * dim + c];
    s = __dadd_rn(s, hypot(v.x, v.y));
  }
  colsum[c] = s;
}

__global__ void identity_kernel(double2* x, long long dim) {
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < dim * dim;
       k += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long r = k / dim, c = k - r * dim;
    x[k] = make_double2(r == c ? 1.0 : 0.0, 0.0);
  }
}

__global__ void __launch_bounds__(kThreads) max_kernel(const double* __restrict__ v, long long n,
                                                       unsigned long long* out) {
  __shared__ unsigned long long red[32];
  unsigned long long m = 0;
  for (long long k = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; k < n;
       k += static_cast<long long>(gridDim.x) * blockDim.x)
    m = umax64(m, dbits(v[k]));
  m = block_max_bits(m, red);
  if (threadIdx.x == 0) atomicMax(out, m);
}

// next[r] = sum over row r of |L^T| of v[c] * a, ascending c, round-to-nearest
// multiply then add (no contraction), matching `next[c] += vr * |L_rc|`.
__global__ void __launch_bounds__(kThreads) abs_product_kernel(RealCsrView lt, const double* __restrict__ v,
                                                               double* __restrict__ next) {
  for (long long lr = blockIdx.x * static_cast<long long>(blockDim.x) + threadIdx.x; lr < lt.rows;
       lr += static_cast<long long>(gridDim.x) * blockDim.x) {
    const long long b = lt.rowptr[lr], e = lt.rowptr[lr + 1];
    double acc = 0.0;
    for (long long k = b; k < e; ++k) {
      const double vc = __ldg(v + lt.col[k]);
      if (vc == 0.0) continue;  // liouvillian.cpp:330
      acc = __dadd_rn(acc, __dmul_rn(vc, lt.val[k]));
    }
    next[lr] = acc;
  }
}

}  // namespace

void exact_norms(const CsrView& l, std::int64_t dim, double2* w0, double2* w1, double* colsum,
                 double* norms9_host, cudaStream_t s) {
  // CSC of L (rows ascending in each column), transposed on the host: the
  // matrix is small here (dim <= 4096)
  std::vector<long long> rp(static_cast<std::size_t>(dim) + 1);
  QSWG_CUDA(cudaMemcpyAsync(rp.data(), l.rowptr, rp.size() * sizeof(long long), cudaMemcpyDeviceToHost, s));
  QSWG_CUDA(cudaStreamSynchronize(s));
  const long long nz = rp.back();
  std::vector<int> col(static_cast<std::size_t>(nz)), row(static_cast<std::size_t>(nz));
  std::vector<double2> val(static_cast<std::size_t>(nz)), tval(static_cast<std::size_t>(nz));
  if (nz > 0) {
    QSWG_CUDA(cudaMemcpyAsync(col.data(), l.col, col.size() * sizeof(int), cudaMemcpyDeviceToHost, s));
    QSWG_CUDA(cudaMemcpyAsync(val.data(), l.val, val.size() * sizeof(double2), cudaMemcpyDeviceToHost, s));
    QSWG_CUDA(cudaStreamSynchronize(s));
  }
  std::vector<long long> cp(static_cast<std::size_t>(dim) + 1, 0);
  for (long long k = 0; k < nz; ++k) ++cp[static_cast<std::size_t>(col[k]) + 1];
  for (long long c = 0; c < dim; ++c) cp[c + 1] += cp[c];
  std::vector<long long> fill(cp.begin(), cp.end() - 1);
  for (long long r = 0; r < dim; ++r)
    for (long long k = rp[r]; k < rp[r + 1]; ++k) {
      const long long d = fill[col[k]]++;
      row[d] = static_cast<int>(r);
      tval[d] = val[k];
    }
  long long* dcp = nullptr;
  int* drow = nullptr;
  double2* dval = nullptr;
  QSWG_CUDA(cudaMallocAsync(&dcp, cp.size() * sizeof(long long), s));
  QSWG_CUDA(cudaMallocAsync(&drow, (row.size() + 1) * sizeof(int), s));
  QSWG_CUDA(cudaMallocAsync(&dval, (tval.size() + 1) * sizeof(double2), s));
  QSWG_CUDA(cudaMemcpyAsync(dcp, cp.data(), cp.size() * sizeof(long long), cudaMemcpyHostToDevice, s));
  if (nz > 0) {
    QSWG_CUDA(cudaMemcpyAsync(drow, row.data(), row.size() * sizeof(int), cudaMemcpyHostToDevice, s));
    QSWG_CUDA(cudaMemcpyAsync(dval, tval.data(), tval.size() * sizeof(double2), cudaMemcpyHostToDevice, s));
  }
  identity_kernel<<<sm_count() * 4, kThreads, 0, s>>>(w0, dim);
  QSWG_LAUNCH_CHECK("identity");
  unsigned long long* dmax = nullptr;
  QSWG_CUDA(cudaMallocAsync(&dmax, 9 * sizeof(unsigned long long), s));
  QSWG_CUDA(cudaMemsetAsync(dmax, 0, 9 * sizeof(unsigned long long), s));
  double2* x = w0;
  double2* y = w1;
  const int gx = static_cast<int>((dim + kThreads - 1) / kThreads);
  for (int p = 0; p < 9; ++p) {
    dense_power_kernel<<<dim3(gx, static_cast<unsigned>(dim)), kThreads, 0, s>>>(dcp, drow, dval, dim, x, y);
    QSWG_LAUNCH_CHECK("dense_power");
    colsum_kernel<<<gx, kThreads, 0, s>>>(y, dim, colsum);
    QSWG_LAUNCH_CHECK("colsum");
    max_kernel<<<1, kThreads, 0, s>>>(colsum, dim, dmax + p);
    QSWG_LAUNCH_CHECK("max");
    double2* t = x;
    x = y;
    y = t;
  }
  unsigned long long bits[9];
  QSWG_CUDA(cudaMemcpyAsync(bits, dmax, sizeof(bits), cudaMemcpyDeviceToHost, s));
  QSWG_CUDA(cudaFreeAsync(dmax, s));
  QSWG_CUDA(cudaFreeAsync(dcp, s));
  QSWG_CUDA(cudaFreeAsync(drow, s));
  QSWG_CUDA(cudaFreeAsync(dval, s));
  QSWG_CUDA(cudaStreamSynchronize(s));
  for (int p = 0; p < 9; ++p) std::memcpy(norms9_host + p, bits + p, sizeof(double));
}

void abs_transpose_product(const RealCsrView& lt, const double* v, double* next, cudaStream_t s) {
  if (lt.rows <= 0) return;
  long long want = (lt.rows + kThreads - 1) / kThreads, cap = sm_count() * 16LL;
  abs_product_kernel<<<static_cast<int>(want < cap ? want : cap), kThreads, 0, s>>>(lt, v, next);
  QSWG_LAUNCH_CHECK("abs_transpose_product");
}

void max_reduce(const double* v, std::int64_t n, unsigned long long* out_bits, cudaStream_t s) {
  long long want = (n + kThreads - 1) / kThreads, cap = sm_count() * 4LL;
  max_kernel<<<static_cast<int>(want < 1 ? 1 : (want < cap ? want : cap)), kThreads, 0, s>>>(v, n, out_bits);
  QSWG_LAUNCH_CHECK("max_reduce");
}

}  // namespace qswg::dev
