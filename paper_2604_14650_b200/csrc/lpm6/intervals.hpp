// 2D -> 1D transform: prefix rules -> sorted elementary-interval starts.
//
// Contract of the reference's build_intervals (intervals.hpp:18-34,
// intervals.cpp:33-93): boundaries[0] == 0, strictly increasing,
// none equal to the sentinel, next_hops[i] = next hop of the longest rule
// covering interval i (or the FIB default), adjacent equal next hops merged by
// default, at most 2N+1 intervals. Output is bit-identical to the reference's;
// the construction is our own (see intervals.cpp).
#pragma once

#include <span>
#include <vector>

#include "lpm6/fib.hpp"

namespace lpm6 {

struct IntervalMap {
  std::vector<u64> boundaries;
  std::vector<u32> next_hops;
  u32 default_next_hop = 0;
  size_t size() const { return boundaries.size(); }
};

struct IntervalBuildOptions {
  bool merge_adjacent = true;  // intervals.hpp:26-29
};

IntervalMap build_intervals(std::span<const Prefix> rules, u32 default_next_hop,
                            const IntervalBuildOptions& opt = {});

inline IntervalMap build_intervals(const FibTable& fib, const IntervalBuildOptions& opt = {}) {
  return build_intervals(std::span<const Prefix>(fib.entries()), fib.default_next_hop(), opt);
}

}  // namespace lpm6
