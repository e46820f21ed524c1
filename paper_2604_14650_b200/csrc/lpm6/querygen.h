// Counter-based query generator shared by host and device.
//
// Query i of a workload is a pure function of (seed, i), so any 64M-address
// chunk of C4 (or any slice of C0-C3) can be generated independently on the
// GPU that looks it up and re-generated bit-identically on the host that
// verifies it. Addresses are 16-byte little-endian u128 (lo word first), the
// type the reference's lookup takes (intervals.hpp:37); the lookup key is the
// hi word (fib.hpp:27).
#pragma once

#include <stdint.h>

#if defined(__CUDACC__)
#define LPM6_HD __host__ __device__ __forceinline__
#else
#define LPM6_HD inline
#endif

namespace lpm6 {

LPM6_HD uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

// Independent 64-bit draw `j` for query `i` under `seed`.
LPM6_HD uint64_t qrand(uint64_t seed, uint64_t i, uint32_t j) {
  return mix64(mix64(seed + 0x9E3779B97F4A7C15ull * (i + 1)) ^ (0xD1B54A32D192ED03ull * (j + 1)));
}

enum QueryUniform : uint32_t {
  kUniform128 = 0,   // uniform over all 128-bit values
  kUniform2000 = 1,  // uniform inside 2000::/3
};

enum QueryPick : uint32_t {
  kPickUniform = 0,  // FIB prefix chosen uniformly
  kPickZipf = 1,     // FIB prefix chosen Zipf(s) by rank through a seeded permutation
};

struct QuerySpec {
  uint64_t seed;
  uint64_t in_prefix_thr;  // query is in-prefix iff (draw0 >> 11) < thr (a 53-bit fraction)
  uint32_t uniform_kind;   // QueryUniform
  uint32_t pick;           // QueryPick
  uint64_t n_prefixes;
  const uint64_t* pfx_top;   // top 64 bits of each FIB prefix
  const uint8_t* pfx_len;    // its length
  const double* zipf_cdf;    // n_prefixes cumulative probabilities, rank order (kPickZipf)
  const uint32_t* zipf_perm; // rank -> prefix index (kPickZipf)
};

LPM6_HD void gen_query(const QuerySpec& s, uint64_t i, uint64_t* lo, uint64_t* hi) {
  const uint64_t r0 = qrand(s.seed, i, 0);
  const uint64_t r2 = qrand(s.seed, i, 2);
  *lo = qrand(s.seed, i, 3);
  if (s.n_prefixes > 0 && (r0 >> 11) < s.in_prefix_thr) {
    const uint64_t r1 = qrand(s.seed, i, 1);
    uint64_t idx;
    if (s.pick == kPickZipf) {
      const double u = static_cast<double>(r1 >> 11) * (1.0 / 9007199254740992.0);
      uint64_t lo_i = 0, n = s.n_prefixes;  // first rank with cdf > u
      while (n > 0) {
        const uint64_t half = n >> 1;
        if (s.zipf_cdf[lo_i + half] <= u) {
          lo_i += half + 1;
          n -= half + 1;
        } else {
          n = half;
        }
      }
      if (lo_i >= s.n_prefixes) lo_i = s.n_prefixes - 1;
      idx = s.zipf_perm[lo_i];
    } else {
      idx = r1 % s.n_prefixes;
    }
    const uint32_t len = s.pfx_len[idx];
    const uint64_t keep = len == 0 ? 0ull : (~0ull << (64 - len));
    *hi = (s.pfx_top[idx] & keep) | (r2 & ~keep);
  } else if (s.uniform_kind == kUniform2000) {
    *hi = (r2 >> 3) | (1ull << 61);  // 001x... = 2000::/3
  } else {
    *hi = r2;
  }
}

}  // namespace lpm6
