// FIB model: the input side of the lookup path.
//
// Mirrors the reference's fib-model surface (fib.hpp:17-121) that a caller of
// the batched lookup needs: Prefix (same memory layout as lpm6::Prefix,
// fib.hpp:22-29, so a reference FibTable's entries can be handed over as-is),
// prefix_to_range (fib.cpp:66-70), parse_prefix (fib.cpp:72-105) and FibTable
// (fib.hpp:74-105). Text FIB files are read by the caller (the reference's own
// load_fib, or fib.py's load_fib over parse_prefix).
#pragma once

#include <string>
#include <string_view>
#include <unordered_map>
#include <vector>

#include "lpm6/common.hpp"

namespace lpm6 {

struct Prefix {
  u128 value = 0;  // text order: first hextet is most significant; canonical (host bits zero)
  int length = 0;  // 0..64
  u32 next_hop = 0;

  u64 top64() const { return static_cast<u64>(value >> 64); }
  friend bool operator==(const Prefix&, const Prefix&) = default;
};
static_assert(sizeof(Prefix) == 32, "Prefix must keep lpm6::Prefix's 32-byte layout");

// Half-open key range [start_key, end_exclusive); end may be 2^64.
struct KeyRange {
  u64 start_key = 0;
  u128 end_exclusive = 0;
};

inline KeyRange prefix_to_range(const Prefix& p) {
  const u64 s = p.top64();
  return KeyRange{s, u128(s) + (u128(1) << (64 - p.length))};
}

u128 parse_ipv6(std::string_view text);
std::string format_ipv6(u128 addr);

struct ParsedPrefix {
  Prefix prefix;
  bool host_bits_masked = false;
};

// "<ipv6>/<len> <next_hop>"; len > 64 -> UnsupportedPrefixLength (fib.cpp:88-90).
ParsedPrefix parse_prefix(std::string_view text);

// Rule set with unique (value, length) pairs and a no-match next hop.
class FibTable {
 public:
  FibTable() = default;
  explicit FibTable(u32 default_next_hop) : default_next_hop_(default_next_hop) {}

  u32 default_next_hop() const { return default_next_hop_; }
  void set_default_next_hop(u32 nh) { default_next_hop_ = nh; }
  size_t size() const { return entries_.size(); }
  bool empty() const { return entries_.empty(); }
  const std::vector<Prefix>& entries() const { return entries_; }

  void insert(const Prefix& p);             // throws DuplicatePrefix / ReservedNextHop
  bool insert_or_replace(const Prefix& p);  // true when an existing rule was overwritten
  void erase(u128 value, int length);       // throws UnknownPrefix
  void modify(u128 value, int length, u32 next_hop);  // throws ReservedNextHop / UnknownPrefix
  const Prefix* find(u128 value, int length) const;
  bool contains(u128 value, int length) const { return find(value, length) != nullptr; }

 private:
  struct KeyHash {
    size_t operator()(const std::pair<u64, int>& k) const noexcept {
      u64 x = k.first * 0x9E3779B97F4A7C15ull ^ (u64(k.second) * 0xC2B2AE3D27D4EB4Full);
      return static_cast<size_t>(x ^ (x >> 29));
    }
  };
  std::vector<Prefix> entries_;
  std::unordered_map<std::pair<u64, int>, size_t, KeyHash> index_;
  u32 default_next_hop_ = 0;
};

}  // namespace lpm6
