// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// Scalar stand-in for the reference's absent `src/kernels.hpp` (the per-ISA
// backend table). The interface is inferred from its only call site,
// /root/reference/proj/src/intervals.cpp:110-121:
//   - detail::RuleScan{start, mask, rank}, rank = (len+1)<<32 | next_hop  (:117)
//   - detail::OracleScanFn(rules, keys, n, best)                          (:120)
//   - detail::vector_backend().oracle_scan                                 (:120)
// `best` arrives zeroed (:119) and receives the maximal rank of every rule
// whose masked start matches the key; 0 means "no rule" (:137-138).
#pragma once

#include <cstddef>
#include <vector>

#include "lpm6/types.hpp"

namespace lpm6::detail {

struct RuleScan {
  std::vector<u64> start;
  std::vector<u64> mask;
  std::vector<u64> rank;
};

using OracleScanFn = void (*)(const RuleScan& rules, const u64* keys, size_t n, u64* best);

struct VectorBackend {
  OracleScanFn oracle_scan;
};

inline void scalar_oracle_scan(const RuleScan& rules, const u64* keys, size_t n, u64* best) {
  const size_t nr = rules.start.size();
  for (size_t i = 0; i < n; ++i) {
    u64 b = best[i];
    const u64 key = keys[i];
    for (size_t r = 0; r < nr; ++r)
      if ((key & rules.mask[r]) == rules.start[r] && rules.rank[r] > b) b = rules.rank[r];
    best[i] = b;
  }
}

inline const VectorBackend& vector_backend() {
  static const VectorBackend backend{&scalar_oracle_scan};
  return backend;
}

}  // namespace lpm6::detail
