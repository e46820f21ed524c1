// Synthetic workloads C0-C4 (BASELINE.json "configs").
//
// The paper's RIPE/RouteViews tables are not available here, so every FIB and
// every query stream is synthetic, seeded and deterministic. Generator choices
// the BASELINE text leaves open are pinned in workload.cpp and DESIGN.md §3.
#pragma once

#include <span>
#include <vector>

#include "lpm6/fib.hpp"
#include "lpm6/querygen.h"

namespace lpm6 {

enum WorkloadId : int { kC0 = 0, kC1 = 1, kC2 = 2, kC3a = 3, kC3b = 4, kC4 = 5, kNumWorkloads = 6 };

struct WorkloadConfig {
  int id = 0;
  const char* name = "";
  int fib_kind = 0;           // 0: C0 FIB, 1: C1 FIB (200K), 2: C2 FIB (1M)
  u64 n_queries = 0;
  u64 chunk = 0;              // queries per chunk (C4: 64M), 0 = one chunk
  u64 query_seed = 0;
  double in_prefix_frac = 0;  // share of queries drawn inside a FIB prefix
  u32 uniform_kind = kUniform128;
  u32 pick = kPickUniform;
  double zipf_s = 0;
  u32 value_bytes = 1;        // next-hop bytes out (w)
};

WorkloadConfig workload_config(int id);

// FIB of fib_kind 0/1/2 (C0, C1 = C3 = 200K backbone, C2 = C4 = 1M projected).
FibTable make_fib(int fib_kind);

// Host-side tables a QuerySpec points into.
struct QueryTables {
  std::vector<u64> top;
  std::vector<u8> len;
  std::vector<double> cdf;
  std::vector<u32> perm;
};

QueryTables make_query_tables(std::span<const Prefix> rules, const WorkloadConfig& cfg);
inline QueryTables make_query_tables(const FibTable& fib, const WorkloadConfig& cfg) {
  return make_query_tables(std::span<const Prefix>(fib.entries()), cfg);
}
QuerySpec make_query_spec(const WorkloadConfig& cfg, const QueryTables& t);

// Addresses [first, first+n) of a workload as 2n little-endian u64 words (lo, hi).
void gen_queries_host(const QuerySpec& spec, u64 first, u64 n, u64* out, int threads);

}  // namespace lpm6
