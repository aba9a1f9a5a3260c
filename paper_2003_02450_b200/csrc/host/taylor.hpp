// Truncated-Taylor parameters: theta tables and the (m*, s) selection.
//
// Mirrors proj/core/include/qsw/expm.hpp:13-45.  The 2^-53 / 2^-24 tables
// are regenerated independently by tools/gen_theta.py (bit-identical to the
// shipped theta_tables.cpp:8-122, pinned by tests/test_theta.py); other
// tolerances are solved at runtime from the same backward-error series.
#pragma once

#include <array>
#include <cstdint>
#include <stdexcept>

namespace qswg {

/// Raised when an evolution produces non-finite values (expm.hpp:13-17).
class NumericalError : public std::runtime_error {
 public:
  using std::runtime_error::runtime_error;
};

inline constexpr double kDoublePrecisionTol = 0x1p-53;
inline constexpr double kSinglePrecisionTol = 0x1p-24;

struct TaylorParameters {
  static constexpr int m_max = 55;
  static constexpr int p_max = 8;
  double tolerance = kDoublePrecisionTol;
  std::array<double, m_max> theta{};
};

/// Memoised per tolerance; throws std::invalid_argument outside (0, 1).
const TaylorParameters& build_theta_table(double tolerance = kDoublePrecisionTol);

struct StepParameters {
  std::int64_t m_star = 0;  // 0 means exp(tA)v = v
  std::int64_t s = 1;
};

/// Cost-minimising (m*, s) from ||A^n||_1, n = 1..9 (expm.cpp:87-125).
StepParameters select_parameters(const double* one_norms9, double t, const TaylorParameters& p);

}  // namespace qswg
