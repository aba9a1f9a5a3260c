#include "dist.hpp"

#include <algorithm>
#include <stdexcept>

namespace qswg {

std::vector<std::int64_t> partition_rows(const std::vector<std::int64_t>& colptr, std::int64_t n, int world) {
  if (world < 1) throw std::invalid_argument("world size must be at least 1");
  if (static_cast<std::int64_t>(colptr.size()) != n + 1) throw std::invalid_argument("colptr must have n + 1 entries");
  std::vector<std::int64_t> starts(static_cast<std::size_t>(world) + 1, 0);
  starts[static_cast<std::size_t>(world)] = n * n;
  const std::int64_t total = colptr.back();
  std::int64_t j = 0;
  for (int w = 1; w < world; ++w) {
    const long double target = static_cast<long double>(total) * w / world;
    // advance while the midpoint of column j lies before the target
    while (j < n && static_cast<long double>(colptr[static_cast<std::size_t>(j)]) +
                            (colptr[static_cast<std::size_t>(j) + 1] - colptr[static_cast<std::size_t>(j)]) / 2.0L <
                        target)
      ++j;
    starts[static_cast<std::size_t>(w)] = std::max(j * n, starts[static_cast<std::size_t>(w) - 1]);
  }
  return starts;
}

std::vector<HaloRange> halo_needs_host(const std::int64_t* cols, std::int64_t nnz,
                                       const std::vector<std::int64_t>& starts, int rank) {
  const int world = static_cast<int>(starts.size()) - 1;
  std::vector<HaloRange> out(static_cast<std::size_t>(world));
  std::vector<std::int64_t> mn(static_cast<std::size_t>(world), INT64_MAX), mx(static_cast<std::size_t>(world), INT64_MIN);
  for (std::int64_t k = 0; k < nnz; ++k) {
    const std::int64_t c = cols[k];
    const auto it = std::upper_bound(starts.begin(), starts.end(), c);
    const int q = static_cast<int>(it - starts.begin()) - 1;
    if (q < 0 || q >= world || q == rank) continue;
    mn[static_cast<std::size_t>(q)] = std::min(mn[static_cast<std::size_t>(q)], c);
    mx[static_cast<std::size_t>(q)] = std::max(mx[static_cast<std::size_t>(q)], c + 1);
  }
  for (int q = 0; q < world; ++q)
    if (mn[static_cast<std::size_t>(q)] != INT64_MAX) out[static_cast<std::size_t>(q)] = {mn[static_cast<std::size_t>(q)], mx[static_cast<std::size_t>(q)]};
  return out;
}

}  // namespace qswg
