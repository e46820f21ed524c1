/* TEST INFRASTRUCTURE ONLY — restated PlanB CPU search, the CPU baseline.
 *
 * The reference's own search_avx512.cpp is absent from /root/reference
 * (CMakeLists.txt:35 names it, the file is not in the snapshot), so this is a
 * restatement of its published algorithm: Listing 1 (broadcast the
 * key, one 8x64-bit unsigned >= compare per 64-byte node, popcount, descend with
 * i = (k+1) i + (c+1) k) combined with batching (B = 16
 * interleaved descents) and depth-templated full unrolling.
 * Ordinal = leaf rank - 1. Nodes are 64-byte aligned (one cache line,
 * tree.hpp:42-74; oracle.py allocates the key array so), and the next batch's
 * trace records are prefetched while the current batch descends.
 * Compiled with -mavx512f/dq/bw only in this TU
 * and selected at run time, as CMakeLists.txt:18-46 does for the reference. */
#include <immintrin.h>

#include "lpm6_oracle.h"

#define B 16

#define DEFINE_BATCH(D)                                                                    \
  static void batch_d##D(const uint64_t* keys, const uint32_t* values, uint64_t leaf_start, \
                         const uint64_t* addrs, uint32_t* out) {                           \
    int64_t i[B], c[B];                                                                     \
    __m512i q[B];                                                                           \
    /* the next batch's trace records are fetched ahead of use */            \
    for (int b = 0; b < B; b += 4) _mm_prefetch((const char*)(addrs + 2 * (B + b)), _MM_HINT_T0); \
    for (int b = 0; b < B; ++b) {                                                           \
      uint64_t key = addrs[2 * b + 1];                                                      \
      if (key > ORC_MAX_QUERY) key = ORC_MAX_QUERY;                                         \
      q[b] = _mm512_set1_epi64((long long)key);                                             \
      i[b] = 0;                                                                             \
      c[b] = -1;                                                                            \
    }                                                                                       \
    for (int l = 0; l <= (D); ++l) {                                                        \
      for (int b = 0; b < B; ++b) {                                                         \
        i[b] = 9 * i[b] + (c[b] + 1) * 8;                                                   \
        const __m512i node = _mm512_loadu_si512((const void*)(keys + i[b]));                 \
        c[b] = __builtin_popcount((unsigned)_mm512_cmpge_epu64_mask(q[b], node));           \
      }                                                                                     \
    }                                                                                       \
    for (int b = 0; b < B; ++b) out[b] = values[i[b] - (int64_t)leaf_start + c[b] - 1];    \
  }

DEFINE_BATCH(0)
DEFINE_BATCH(1)
DEFINE_BATCH(2)
DEFINE_BATCH(3)
DEFINE_BATCH(4)
DEFINE_BATCH(5)
DEFINE_BATCH(6)
DEFINE_BATCH(7)

typedef void (*batch_fn)(const uint64_t*, const uint32_t*, uint64_t, const uint64_t*, uint32_t*);
static const batch_fn kBatch[8] = {batch_d0, batch_d1, batch_d2, batch_d3,
                                   batch_d4, batch_d5, batch_d6, batch_d7};

void orc_avx512_batch(const uint64_t* keys, const uint32_t* values, const orc_geometry* g,
                      const uint64_t* addrs, uint64_t n, uint32_t* out) {
  const batch_fn fn = kBatch[g->depth & 7];
  uint64_t i = 0;
  for (; i + B <= n; i += B) fn(keys, values, g->leaf_start, addrs + 2 * i, out + i);
  if (i < n) { /* pad the tail with key 0 and discard the pad results */
    uint64_t pad[2 * B] = {0};
    uint32_t tmp[B];
    for (uint64_t j = i; j < n; ++j) {
      pad[2 * (j - i)] = addrs[2 * j];
      pad[2 * (j - i) + 1] = addrs[2 * j + 1];
    }
    fn(keys, values, g->leaf_start, pad, tmp);
    for (uint64_t j = i; j < n; ++j) out[j] = tmp[j - i];
  }
}
