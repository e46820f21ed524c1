// TEST / BENCH INFRASTRUCTURE ONLY — the synthetic workload generator for the
// reference arm of bench.py.
//
// `bench.py --impl reference` must time the reference's CPU lookup in a process
// that never maps the product library (paper_2604_14650_b200/lib/liblpm6cu.so).
// The seeded FIBs and query streams of BASELINE.json's configs come from our own
// generator (csrc/lpm6/workload.cpp); this file compiles that
// generator a second time, on its own, into oracle/liblpm6work.so. No lookup code
// is in here: the arm then builds intervals and looks up with the reference's
// own code (oracle/_ref/liblpm6ref.so).
#include <cstring>
#include <exception>
#include <span>

#include "lpm6/workload.hpp"

namespace {
thread_local char g_err[256];
template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::exception& e) {
    std::strncpy(g_err, e.what(), sizeof g_err - 1);
    return 1;
  }
}
struct RuleRec {  // lpm6::Prefix / lpm6cu_prefix layout (fib.hpp:22-29)
  uint64_t value_lo, value_hi;
  int32_t length;
  uint32_t next_hop;
  uint64_t reserved;
};
static_assert(sizeof(RuleRec) == 32);
}  // namespace

extern "C" {

const char* wl_last_error() { return g_err; }

// id, fib_kind, value_bytes, n_queries, chunk; name (8 bytes)
int wl_info(int workload, int* fib_kind, uint32_t* value_bytes, uint64_t* n_queries, uint64_t* chunk, char* name8) {
  return guarded([&] {
    const lpm6::WorkloadConfig c = lpm6::workload_config(workload);
    *fib_kind = c.fib_kind;
    *value_bytes = c.value_bytes;
    *n_queries = c.n_queries;
    *chunk = c.chunk;
    std::memset(name8, 0, 8);
    std::strncpy(name8, c.name, 7);
  });
}

int wl_fib(int fib_kind, RuleRec* out, uint64_t capacity, uint64_t* n_out, uint32_t* default_nh) {
  return guarded([&] {
    const lpm6::FibTable fib = lpm6::make_fib(fib_kind);
    *n_out = fib.size();
    *default_nh = fib.default_next_hop();
    if (!out) return;
    if (capacity < fib.size()) throw std::runtime_error("capacity");
    for (size_t i = 0; i < fib.size(); ++i) {
      const lpm6::Prefix& p = fib.entries()[i];
      out[i] = RuleRec{static_cast<uint64_t>(p.value), static_cast<uint64_t>(p.value >> 64), p.length, p.next_hop, 0};
    }
  });
}

// Addresses [first, first + n) of a workload as n x (lo, hi) u64 words.
int wl_queries(int workload, const RuleRec* rules, uint64_t nrules, uint64_t first, uint64_t n, uint64_t* out,
               int threads) {
  return guarded([&] {
    std::vector<lpm6::Prefix> ps(nrules);
    for (uint64_t i = 0; i < nrules; ++i)
      ps[i] = lpm6::Prefix{(static_cast<lpm6::u128>(rules[i].value_hi) << 64) | rules[i].value_lo, rules[i].length,
                           rules[i].next_hop};
    const lpm6::WorkloadConfig c = lpm6::workload_config(workload);
    const lpm6::QueryTables t = lpm6::make_query_tables(std::span<const lpm6::Prefix>(ps), c);
    const lpm6::QuerySpec s = lpm6::make_query_spec(c, t);
    lpm6::gen_queries_host(s, first, n, out, threads);
  });
}

}  // extern "C"
