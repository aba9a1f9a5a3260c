#include "taylor.hpp"

#include <algorithm>
#include <cmath>
#include <limits>
#include <map>
#include <mutex>
#include <vector>

#include "theta_table.inc"

namespace qswg {

namespace {

constexpr double kThetaDouble[55] = QSWG_THETA_DOUBLE;
constexpr double kThetaSingle[55] = QSWG_THETA_SINGLE;

// theta_m for an arbitrary tolerance in double precision.  e^{-x} T_m(x) =
// 1 + sum_{k>m} a_k x^k with a_k = (-1)^(k-m) / (m! (k-m-1)! k); c_k are the
// coefficients of its logarithm (f * (log f)' = f'); theta_m is the root of
// sum_k |c_k| theta^(k-1) = tol, found by bisection.  Same published
// construction as expm.cpp:20-59 / tools/gen_theta.py.
double solve_theta(int m, double tol) {
  const int kmax = m + 150;
  std::vector<double> a(static_cast<std::size_t>(kmax) + 1, 0.0), c(a.size(), 0.0);
  for (int k = m + 1; k <= kmax; ++k) {
    const double log_mag = -(std::lgamma(m + 1.0) + std::lgamma(static_cast<double>(k - m)) +
                             std::log(static_cast<double>(k)));
    a[static_cast<std::size_t>(k)] = ((k - m) % 2 ? -1.0 : 1.0) * std::exp(log_mag);
  }
  for (int k = m + 1; k <= kmax; ++k) {
    double acc = 0.0;
    for (int u = m + 1; u + m + 1 <= k; ++u)
      acc += a[static_cast<std::size_t>(u)] * (k - u) * c[static_cast<std::size_t>(k - u)];
    c[static_cast<std::size_t>(k)] = a[static_cast<std::size_t>(k)] - acc / k;
  }
  auto excess = [&](double th) {
    double s = 0.0, pw = std::pow(th, static_cast<double>(m));
    for (int k = m + 1; k <= kmax; ++k) {
      s += std::abs(c[static_cast<std::size_t>(k)]) * pw;
      pw *= th;
      if (pw == 0.0 || !std::isfinite(pw)) break;
    }
    return s - tol;
  };
  double lo = 0.0, hi = 1e-280;
  while (excess(hi) < 0.0) {
    lo = hi;
    hi *= 2.0;
  }
  for (int it = 0; it < 300; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid == lo || mid == hi) break;
    (excess(mid) > 0.0 ? hi : lo) = mid;
  }
  return lo;
}

}  // namespace

const TaylorParameters& build_theta_table(double tolerance) {
  if (!(tolerance > 0.0 && tolerance < 1.0))
    throw std::invalid_argument("tolerance must lie in (0, 1)");
  static std::mutex mu;
  static std::map<double, TaylorParameters> cache;
  std::lock_guard<std::mutex> lock(mu);
  auto it = cache.find(tolerance);
  if (it != cache.end()) return it->second;
  TaylorParameters p;
  p.tolerance = tolerance;
  if (tolerance == kDoublePrecisionTol) {
    std::copy(std::begin(kThetaDouble), std::end(kThetaDouble), p.theta.begin());
  } else if (tolerance == kSinglePrecisionTol) {
    std::copy(std::begin(kThetaSingle), std::end(kThetaSingle), p.theta.begin());
  } else {
    for (int m = 1; m <= TaylorParameters::m_max; ++m) p.theta[static_cast<std::size_t>(m - 1)] = solve_theta(m, tolerance);
  }
  return cache.emplace(tolerance, p).first->second;
}

// expm.cpp:87-125.  Evaluation order of every floating-point expression is
// kept so (m*, s) is bit-for-bit the reference's for identical norms.
StepParameters select_parameters(const double* norms, double t, const TaylorParameters& p) {
  const double at = std::abs(t);
  if (at * norms[0] == 0.0) return {0, 1};
  constexpr int m_max = TaylorParameters::m_max, p_max = TaylorParameters::p_max;
  double alpha[p_max - 1];
  const double norm1 = at * norms[0];
  const bool small = norm1 <= 4.0 * p.theta[m_max - 1] * static_cast<double>(p_max) *
                                 static_cast<double>(p_max + 3) / static_cast<double>(m_max);
  for (int q = 2; q <= p_max; ++q) {
    if (small) {
      alpha[q - 2] = norm1;
    } else {
      const double dp = at * std::pow(norms[q - 1], 1.0 / static_cast<double>(q));
      const double dp1 = at * std::pow(norms[q], 1.0 / static_cast<double>(q + 1));
      alpha[q - 2] = std::max(dp, dp1);
    }
  }
  StepParameters best{0, 1};
  double best_cost = std::numeric_limits<double>::infinity();
  for (int q = 2; q <= p_max; ++q) {
    for (int m = q * (q - 1) - 1; m <= m_max; ++m) {
      const double s_real = std::max(std::ceil(alpha[q - 2] / p.theta[static_cast<std::size_t>(m - 1)]), 1.0);
      const double cost = static_cast<double>(m) * s_real;
      if (cost < best_cost) {
        best_cost = cost;
        best = {m, static_cast<std::int64_t>(s_real)};
      }
    }
  }
  return best;
}

}  // namespace qswg
