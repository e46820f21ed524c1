// Interval construction by a single sweep over the prefix nesting forest.
//
// The reference builds 2N start/end events, sorts them with a four-way
// comparator and sweeps them with a next-hop stack (intervals.cpp:33-93).
// CIDR ranges are laminar (any two are nested or disjoint), so we instead sort
// the N rules once by (start, length) — a pre-order walk of the nesting forest
// — and keep a stack of open ranges ordered by end. Before a rule is pushed,
// every open range that ends at or before its start is closed. Every start and
// every close emits (address, next hop after the event); emissions at one
// address coalesce to the last, which is exactly the reference's "stack top
// after all events at this address" (intervals.cpp:58-73): closes
// at an address precede starts there (End-before-Start), nested closes come
// innermost first (Ends by descending length) and equal-start rules arrive
// shortest first (Starts by ascending length). The close at 2^64 is dropped
// (intervals.cpp:70), the origin gets the default (intervals.cpp:51-54), the
// sentinel check runs before merging (intervals.cpp:76-79) and the merge keeps
// the first of each run of equal next hops (intervals.cpp:81-91).
#include "lpm6/intervals.hpp"

#include <algorithm>

namespace lpm6 {

namespace {

struct Rule {
  u64 start;
  u32 length;
  u32 next_hop;
};

struct Open {
  u128 end;
  u32 next_hop;
};

}  // namespace

IntervalMap build_intervals(std::span<const Prefix> rules, u32 default_next_hop,
                            const IntervalBuildOptions& opt) {
  std::vector<Rule> sorted;
  sorted.reserve(rules.size());
  for (const Prefix& p : rules) {
    if (p.length < 0 || p.length > 64)
      throw Error(Errc::UnsupportedPrefixLength,
                  "unsupported prefix length /" + std::to_string(p.length) + " (keys cover /0../64)");
    if (p.next_hop == kUnresolved)
      throw Error(Errc::ReservedNextHop, "rule uses the reserved next hop: " + format_ipv6(p.value) +
                                             "/" + std::to_string(p.length));
    const u128 mask = p.length == 0 ? u128(0) : ~u128(0) << (128 - p.length);
    if ((p.value & mask) != p.value)
      throw Error(Errc::InvalidArgument, "non-canonical prefix (host bits set): " +
                                             format_ipv6(p.value) + "/" + std::to_string(p.length));
    sorted.push_back(Rule{p.top64(), static_cast<u32>(p.length), p.next_hop});
  }
  std::sort(sorted.begin(), sorted.end(), [](const Rule& a, const Rule& b) {
    return a.start != b.start ? a.start < b.start : a.length < b.length;
  });
  for (size_t i = 1; i < sorted.size(); ++i)
    if (sorted[i].start == sorted[i - 1].start && sorted[i].length == sorted[i - 1].length)
      throw Error(Errc::DuplicatePrefix, "duplicate prefix " + format_ipv6(u128(sorted[i].start) << 64) +
                                             "/" + std::to_string(sorted[i].length));

  IntervalMap map;
  map.default_next_hop = default_next_hop;
  std::vector<u64>& bnd = map.boundaries;
  std::vector<u32>& nhs = map.next_hops;
  bnd.reserve(2 * sorted.size() + 1);
  nhs.reserve(2 * sorted.size() + 1);

  constexpr u128 kTop = u128(1) << 64;
  bool have_last = false;
  u128 last_addr = 0;
  auto emit = [&](u128 addr, u32 nh) {
    if (have_last && addr == last_addr) {
      nhs.back() = nh;  // coalesce: the state after the last event at this address wins
      return;
    }
    if (addr == kTop) return;  // nothing starts at the top of the key space
    bnd.push_back(static_cast<u64>(addr));
    nhs.push_back(nh);
    have_last = true;
    last_addr = addr;
  };

  if (sorted.empty() || sorted.front().start != 0) emit(0, default_next_hop);

  std::vector<Open> stack;
  stack.reserve(65);
  auto close_until = [&](u128 limit) {
    while (!stack.empty() && stack.back().end <= limit) {
      const u128 end = stack.back().end;
      stack.pop_back();
      emit(end, stack.empty() ? default_next_hop : stack.back().next_hop);
    }
  };
  for (const Rule& r : sorted) {
    close_until(r.start);
    stack.push_back(Open{u128(r.start) + (u128(1) << (64 - r.length)), r.next_hop});
    emit(r.start, r.next_hop);
  }
  close_until(kTop);

  for (u64 b : bnd)
    if (b == kSentinelKey)
      throw Error(Errc::SentinelCollision,
                  "rule set produces a boundary at the sentinel key ffff:ffff:ffff:ffff::");

  if (opt.merge_adjacent && !bnd.empty()) {
    size_t w = 1;
    for (size_t r = 1; r < bnd.size(); ++r) {
      if (nhs[r] == nhs[w - 1]) continue;
      bnd[w] = bnd[r];
      nhs[w] = nhs[r];
      ++w;
    }
    bnd.resize(w);
    nhs.resize(w);
  }
  return map;
}

}  // namespace lpm6
