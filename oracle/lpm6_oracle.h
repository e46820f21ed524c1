/* TEST INFRASTRUCTURE ONLY — the CPU oracle for the batched IPv6 LPM path.
 *
 * A plain-C restatement of the reference algorithm, used only by tests/,
 * __graft_entry__.smoke() and bench.py's CPU-baseline legs, and only as the
 * checker or the timed CPU baseline — never as the product path. Each
 * function cites the reference file:line it restates. Parity of this
 * restatement is pinned against the compiled reference (oracle/_ref) and the
 * committed golden vectors in tests/golden/ (see tests/test_oracle.py).
 */
#ifndef LPM6_ORACLE_H
#define LPM6_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* Memory layout of lpm6::Prefix (fib.hpp:22-29): u128 value, int length, u32 next_hop. */
typedef struct {
  uint64_t value_lo;
  uint64_t value_hi;
  int32_t length;
  uint32_t next_hop;
  uint64_t reserved;
} orc_prefix;

/* Error numbering = lpm6::Errc (types.hpp:27-40) + 1; 0 = ok. */
enum {
  ORC_OK = 0,
  ORC_E_MALFORMED_ADDRESS = 1,
  ORC_E_UNSUPPORTED_PREFIX_LENGTH = 2,
  ORC_E_MISSING_NEXT_HOP = 3,
  ORC_E_RESERVED_NEXT_HOP = 4,
  ORC_E_DUPLICATE_PREFIX = 5,
  ORC_E_UNKNOWN_PREFIX = 6,
  ORC_E_SENTINEL_COLLISION = 7,
  ORC_E_EXHAUSTED_PREFIX_SPACE = 8,
  ORC_E_INVALID_ARGUMENT = 9,
};

#define ORC_UNRESOLVED 0xFFFFFFFFu            /* types.hpp:17 */
#define ORC_SENTINEL 0xFFFFFFFFFFFFFFFFull    /* types.hpp:21 */
#define ORC_MAX_QUERY 0xFFFFFFFFFFFFFFFEull   /* types.hpp:25 */

/* build_intervals (intervals.cpp:33-93). boundaries/next_hops need room for 2n+1. */
int orc_build_intervals(const orc_prefix* rules, uint64_t n, uint32_t default_nh, int merge,
                        uint64_t* boundaries, uint32_t* next_hops, uint64_t* m_out);

/* lookup_interval_oracle (intervals.cpp:142-145): next_hops[upper_bound(key) - 1]. */
uint32_t orc_lookup_interval(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                             uint64_t key);

/* lookup_linear_oracle (intervals.cpp:95-107), address as (hi, lo) of the u128. */
uint32_t orc_lookup_linear(const orc_prefix* rules, uint64_t n, uint32_t default_nh,
                           uint64_t addr_hi, uint64_t addr_lo);

/* Reference tree geometry (tree.hpp:18-40). */
typedef struct {
  int32_t k, b, depth, pad;
  uint64_t num_keys;
  uint64_t allocated_leaf_nodes;
  uint64_t leaf_start;
  uint64_t level_start[16];
} orc_geometry;

void orc_plan_geometry(uint64_t m, int k, orc_geometry* g);
uint64_t orc_child_key_start(const orc_geometry* g, int level, uint64_t node, int child);
uint64_t orc_total_key_slots(const orc_geometry* g);

/* build_tree (tree.hpp:70-74, Alg. 2) into caller arrays sized
 * orc_total_key_slots() keys and allocated_leaf_nodes*k values. */
void orc_build_tree(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, int k,
                    const orc_geometry* g, uint64_t* keys, uint32_t* values);

/* Search variants over the reference layout; return interval ordinal. */
uint64_t orc_search_scalar(const uint64_t* keys, const orc_geometry* g, uint64_t key);
uint64_t orc_search_branchfree(const uint64_t* keys, const orc_geometry* g, uint64_t key);

/* Batched multi-threaded lookups of 16-byte little-endian u128 addresses.
 * variant: 0 = interval oracle (binary search over boundaries),
 *          1 = branch-free scalar tree search,
 *          2 = restated PlanB AVX-512 Listing 1 + B=16 batching (k=8 only; falls back
 *              to variant 1 when the CPU lacks AVX-512F).
 * out receives the next hop as u32. Returns the variant actually run. */
typedef struct {
  const uint64_t* boundaries;
  const uint32_t* next_hops;
  uint64_t m;
  const uint64_t* keys;   /* tree keys (variants 1, 2) */
  const uint32_t* values; /* tree values (variants 1, 2) */
  const orc_geometry* g;
} orc_index;

int orc_lookup_batch(int variant, const orc_index* ix, const void* addrs, uint64_t n,
                     uint32_t* out, int threads);
int orc_have_avx512(void);

/* Internal: AVX-512 batch kernel (lpm6_oracle_avx512.c). */
void orc_avx512_batch(const uint64_t* keys, const uint32_t* values, const orc_geometry* g,
                      const uint64_t* addrs, uint64_t n, uint32_t* out);

#ifdef __cplusplus
}
#endif
#endif
