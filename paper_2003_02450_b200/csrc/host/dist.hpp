// Row partition and halo plan for the multi-GPU superoperator.
//
// The reference partitions rows evenly over worker threads
// (RowPartition::even, partition.cpp:8-19) and derives per-peer receive lists
// of remote columns (plan_communication, partition.cpp:26-59).  Here rows are
// split on rho-column boundaries (rows n*j .. n*j+n-1 share rho column j)
// balanced by nnz, and each rank receives from each peer the contiguous hull
// [lo, hi) of the peer's columns it references: whole ranges move with one
// ncclSend/ncclRecv pair (lattices need a few neighbouring rho columns, ER
// graphs the whole peer segment, i.e. an allgather).
#pragma once

#include <cstdint>
#include <vector>

namespace qswg {

/// starts[w] = first row of rank w (world + 1 entries), on multiples of n,
/// from colptr[j] = nnz prefix at rho column j (n + 1 entries).
std::vector<std::int64_t> partition_rows(const std::vector<std::int64_t>& colptr, std::int64_t n, int world);

struct HaloRange {
  std::int64_t lo = 0, hi = 0;  // global rows [lo, hi); empty when lo >= hi
};

/// Host reference of the device hull kernel: for every peer q != rank, the
/// hull of the columns in cols[0..nnz) that rank q owns.
std::vector<HaloRange> halo_needs_host(const std::int64_t* cols, std::int64_t nnz,
                                       const std::vector<std::int64_t>& starts, int rank);

}  // namespace qswg
