// TEST INFRASTRUCTURE ONLY — the C ABI of `oracle/_ref/liblpm6ref.so`.
//
// This file is ours; it links the reference's own, unmodified sources
// (/root/reference/proj/src/fib.cpp and intervals.cpp, compiled in place by
// oracle/Makefile) and exposes their entry points as plain C so the parity
// tests and bench.py's reference arm can call the reference itself:
//   ref_build_intervals   -> lpm6::build_intervals        (intervals.cpp:33-93)
//   ref_lookup_interval   -> lpm6::lookup_interval_oracle (intervals.cpp:142-145)
//   ref_lookup_linear     -> lpm6::lookup_linear_oracle   (intervals.cpp:95-107)
//   ref_linear_keys       -> lpm6::linear_oracle_keys     (intervals.cpp:109-140)
//   ref_parse_prefix      -> lpm6::parse_prefix           (fib.cpp:72-105)
//   ref_prefix_to_range   -> lpm6::prefix_to_range        (fib.cpp:66-70)
//   ref_synth_fib         -> lpm6::synth_fib              (fib.cpp:237-273)
// Errors are returned as the numeric lpm6::Errc (types.hpp:27-40) + 1; 0 = ok.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <span>
#include <string>
#include <thread>
#include <vector>

#include "lpm6/fib.hpp"
#include "lpm6/intervals.hpp"
#include "lpm6/types.hpp"

using namespace lpm6;

extern "C" {

// Same memory layout as lpm6::Prefix (fib.hpp:22-29): u128 value, int length, u32 next_hop.
struct ref_prefix {
  uint64_t value_lo;
  uint64_t value_hi;
  int32_t length;
  uint32_t next_hop;
  uint64_t reserved;
};

struct ref_map {
  IntervalMap map;
};

static thread_local std::string g_err;

const char* ref_last_error(void) { return g_err.c_str(); }

static int fail(const Error& e) {
  g_err = e.what();
  return static_cast<int>(e.code()) + 1;
}

static FibTable make_fib(const ref_prefix* rules, uint64_t n, uint32_t default_nh, int replace) {
  FibTable fib(default_nh);
  for (uint64_t i = 0; i < n; ++i) {
    Prefix p;
    p.value = (u128(rules[i].value_hi) << 64) | rules[i].value_lo;
    p.length = rules[i].length;
    p.next_hop = rules[i].next_hop;
    if (replace)
      fib.insert_or_replace(p);
    else
      fib.insert(p);
  }
  return fib;
}

int ref_build_intervals(const ref_prefix* rules, uint64_t n, uint32_t default_nh, int merge,
                        ref_map** out) {
  try {
    FibTable fib = make_fib(rules, n, default_nh, 0);
    IntervalBuildOptions opt;
    opt.merge_adjacent = merge != 0;
    auto* h = new ref_map{build_intervals(fib, opt)};
    *out = h;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

uint64_t ref_map_size(const ref_map* h) { return h->map.size(); }
uint32_t ref_map_default(const ref_map* h) { return h->map.default_next_hop; }

void ref_map_copy(const ref_map* h, uint64_t* boundaries, uint32_t* next_hops) {
  std::memcpy(boundaries, h->map.boundaries.data(), h->map.size() * sizeof(uint64_t));
  std::memcpy(next_hops, h->map.next_hops.data(), h->map.size() * sizeof(uint32_t));
}

void ref_map_free(ref_map* h) { delete h; }

// Keys are looked up on `threads` std::threads, sharding as intervals.cpp:122-134 does.
void ref_lookup_interval(const ref_map* h, const uint64_t* keys, uint64_t n, uint32_t* out,
                         int threads) {
  auto work = [&](uint64_t lo, uint64_t hi) {
    for (uint64_t i = lo; i < hi; ++i) out[i] = lookup_interval_oracle(h->map, keys[i]);
  };
  if (threads <= 1 || n < 4096) {
    work(0, n);
    return;
  }
  std::vector<std::thread> pool;
  const uint64_t chunk = (n + threads - 1) / threads;
  for (int t = 0; t < threads; ++t) {
    const uint64_t lo = std::min<uint64_t>(n, t * chunk), hi = std::min<uint64_t>(n, lo + chunk);
    if (lo == hi) break;
    pool.emplace_back(work, lo, hi);
  }
  for (auto& th : pool) th.join();
}

// Addresses are 16-byte little-endian u128 (the type lookup_linear_oracle takes).
int ref_lookup_linear(const ref_prefix* rules, uint64_t n, uint32_t default_nh,
                      const void* addrs, uint64_t naddr, uint32_t* out) {
  try {
    FibTable fib = make_fib(rules, n, default_nh, 0);
    const auto* a = static_cast<const uint64_t*>(addrs);
    for (uint64_t i = 0; i < naddr; ++i) {
      const u128 addr = (u128(a[2 * i + 1]) << 64) | a[2 * i];
      out[i] = lookup_linear_oracle(fib, addr);
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int ref_linear_keys(const ref_prefix* rules, uint64_t n, uint32_t default_nh,
                    const uint64_t* keys, uint64_t nkeys, uint32_t* out, int threads) {
  try {
    FibTable fib = make_fib(rules, n, default_nh, 0);
    auto v = linear_oracle_keys(fib, std::span<const u64>(keys, nkeys), threads);
    std::memcpy(out, v.data(), nkeys * sizeof(uint32_t));
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

int ref_parse_prefix(const char* text, ref_prefix* out, int* masked) {
  try {
    ParsedPrefix p = parse_prefix(text);
    out->value_lo = static_cast<uint64_t>(p.prefix.value);
    out->value_hi = static_cast<uint64_t>(p.prefix.value >> 64);
    out->length = p.prefix.length;
    out->next_hop = p.prefix.next_hop;
    out->reserved = 0;
    *masked = p.host_bits_masked ? 1 : 0;
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

// end_exclusive is returned as (hi, lo) since it may equal 2^64.
void ref_prefix_to_range(const ref_prefix* p, uint64_t* start, uint64_t* end_hi, uint64_t* end_lo) {
  Prefix q;
  q.value = (u128(p->value_hi) << 64) | p->value_lo;
  q.length = p->length;
  q.next_hop = p->next_hop;
  KeyRange r = prefix_to_range(q);
  *start = r.start_key;
  *end_hi = static_cast<uint64_t>(r.end_exclusive >> 64);
  *end_lo = static_cast<uint64_t>(r.end_exclusive);
}

// Reference synthetic FIB (backbone_default length mix, fib.cpp:207-224).
int ref_synth_fib(uint64_t n, uint64_t seed, ref_prefix* out) {
  try {
    FibTable fib = synth_fib(n, LengthDistribution::backbone_default(seed));
    uint64_t i = 0;
    for (const Prefix& p : fib.entries()) {
      out[i].value_lo = static_cast<uint64_t>(p.value);
      out[i].value_hi = static_cast<uint64_t>(p.value >> 64);
      out[i].length = p.length;
      out[i].next_hop = p.next_hop;
      out[i].reserved = 0;
      ++i;
    }
    return 0;
  } catch (const Error& e) {
    return fail(e);
  }
}

}  // extern "C"
