/* TEST INFRASTRUCTURE ONLY — see lpm6_oracle.h. Plain-C restatement of the
 * reference's interval engine and linearized-tree search. */
#define _GNU_SOURCE
#include "lpm6_oracle.h"

#include <pthread.h>
#include <stdlib.h>
#include <string.h>

typedef unsigned __int128 u128;

/* ---- interval engine: intervals.cpp:14-93 -------------------------------- */

typedef struct {
  u128 address; /* 0 .. 2^64 inclusive */
  int is_end;
  int length;
  uint32_t next_hop;
} orc_event;

/* event_before (intervals.cpp:24-29): address; End before Start; Ends by
 * descending length; Starts by ascending length. */
static int event_cmp(const void* pa, const void* pb) {
  const orc_event* a = (const orc_event*)pa;
  const orc_event* b = (const orc_event*)pb;
  if (a->address != b->address) return a->address < b->address ? -1 : 1;
  if (a->is_end != b->is_end) return a->is_end ? -1 : 1;
  if (a->is_end) return (a->length > b->length) ? -1 : (a->length < b->length ? 1 : 0);
  return (a->length < b->length) ? -1 : (a->length > b->length ? 1 : 0);
}

int orc_build_intervals(const orc_prefix* rules, uint64_t n, uint32_t default_nh, int merge,
                        uint64_t* boundaries, uint32_t* next_hops, uint64_t* m_out) {
  orc_event* ev = (orc_event*)malloc(sizeof(orc_event) * (2 * n + 1));
  if (!ev) return ORC_E_INVALID_ARGUMENT;
  uint64_t ne = 0;
  for (uint64_t i = 0; i < n; ++i) {
    const orc_prefix* p = &rules[i];
    if (p->next_hop == ORC_UNRESOLVED) { /* intervals.cpp:36-37 */
      free(ev);
      return ORC_E_RESERVED_NEXT_HOP;
    }
    if (p->length < 0 || p->length > 64) {
      free(ev);
      return ORC_E_UNSUPPORTED_PREFIX_LENGTH;
    }
    /* prefix_to_range (fib.cpp:66-70): [top64, top64 + 2^(64-L)) */
    const uint64_t start = p->value_hi;
    const u128 end = (u128)start + ((u128)1 << (64 - p->length));
    ev[ne].address = start; ev[ne].is_end = 0; ev[ne].length = p->length; ev[ne].next_hop = p->next_hop; ++ne;
    ev[ne].address = end; ev[ne].is_end = 1; ev[ne].length = p->length; ev[ne].next_hop = ORC_UNRESOLVED; ++ne;
  }
  qsort(ev, ne, sizeof(orc_event), event_cmp);

  uint64_t m = 0;
  /* intervals.cpp:51-54: the key space starts on the default route. */
  if (ne == 0 || ev[0].address != 0) {
    boundaries[m] = 0;
    next_hops[m] = default_nh;
    ++m;
  }
  /* Sweep with a stack of next hops (intervals.cpp:56-73). */
  uint32_t* stack = (uint32_t*)malloc(sizeof(uint32_t) * (n + 1));
  uint64_t sp = 0;
  const u128 top = (u128)1 << 64;
  uint64_t i = 0;
  while (i < ne) {
    const u128 addr = ev[i].address;
    for (; i < ne && ev[i].address == addr; ++i) {
      if (ev[i].is_end)
        --sp;
      else
        stack[sp++] = ev[i].next_hop;
    }
    if (addr == top) continue; /* intervals.cpp:70 */
    boundaries[m] = (uint64_t)addr;
    next_hops[m] = sp ? stack[sp - 1] : default_nh;
    ++m;
  }
  free(stack);
  free(ev);

  /* intervals.cpp:76-79: reject a boundary at the sentinel (checked before merging). */
  for (uint64_t j = 0; j < m; ++j)
    if (boundaries[j] == ORC_SENTINEL) return ORC_E_SENTINEL_COLLISION;

  if (merge) { /* intervals.cpp:81-91 */
    uint64_t w = 1;
    for (uint64_t r = 1; r < m; ++r) {
      if (next_hops[r] == next_hops[w - 1]) continue;
      boundaries[w] = boundaries[r];
      next_hops[w] = next_hops[r];
      ++w;
    }
    m = w;
  }
  *m_out = m;
  return ORC_OK;
}

/* intervals.cpp:142-145 */
uint32_t orc_lookup_interval(const uint64_t* b, const uint32_t* nh, uint64_t m, uint64_t key) {
  uint64_t lo = 0, len = m; /* upper_bound: first element > key */
  while (len > 0) {
    const uint64_t half = len / 2;
    if (b[lo + half] <= key) {
      lo += half + 1;
      len -= half + 1;
    } else {
      len = half;
    }
  }
  return nh[lo - 1];
}

/* intervals.cpp:95-107 */
uint32_t orc_lookup_linear(const orc_prefix* rules, uint64_t n, uint32_t default_nh,
                           uint64_t addr_hi, uint64_t addr_lo) {
  const u128 addr = ((u128)addr_hi << 64) | addr_lo;
  int best_len = -1;
  uint32_t best = default_nh;
  for (uint64_t i = 0; i < n; ++i) {
    const int len = rules[i].length;
    if (len <= best_len) continue;
    const u128 mask = len == 0 ? (u128)0 : ~(u128)0 << (128 - len);
    const u128 v = ((u128)rules[i].value_hi << 64) | rules[i].value_lo;
    if ((addr & mask) == v) {
      best_len = len;
      best = rules[i].next_hop;
    }
  }
  return best;
}

/* ---- linearized tree: tree.hpp:18-74, S:179-223, P:560-578 --------------- */

static uint64_t ipow(uint64_t b, int e) {
  uint64_t r = 1;
  while (e-- > 0) r *= b;
  return r;
}

/* plan_geometry: minimal depth with k*b^depth >= m. */
void orc_plan_geometry(uint64_t m, int k, orc_geometry* g) {
  memset(g, 0, sizeof(*g));
  g->k = k;
  g->b = k + 1;
  int d = 0;
  while ((uint64_t)k * ipow((uint64_t)g->b, d) < m) ++d;
  g->depth = d;
  g->num_keys = m;
  g->allocated_leaf_nodes = (m + k - 1) / k;
  for (int l = 0; l <= d; ++l) /* level_start(l) = k(b^l - 1)/(b - 1) */
    g->level_start[l] = (uint64_t)k * (ipow((uint64_t)g->b, l) - 1) / (uint64_t)(g->b - 1);
  g->leaf_start = g->level_start[d];
}

/* child_start(d, j, c) = level_start(d+1) + (j*b + c)*k. */
uint64_t orc_child_key_start(const orc_geometry* g, int level, uint64_t node, int child) {
  return g->level_start[level + 1] + (node * (uint64_t)g->b + (uint64_t)child) * (uint64_t)g->k;
}

uint64_t orc_total_key_slots(const orc_geometry* g) {
  return g->leaf_start + g->allocated_leaf_nodes * (uint64_t)g->k;
}

/* build_tree: leaves = boundaries then sentinels; internal separator j (0-based)
 * of node g at level l = first key of child g*b + j + 1, i.e.
 * boundaries[(g*b + j + 1) * b^(depth-l-1) * k], sentinel when out of range
 * ("the j-th separator (j = 1..k) ... first key of its (j+1)-th
 * child"; decision S:244). Values replicate the last real value. */
void orc_build_tree(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, int k,
                    const orc_geometry* g, uint64_t* keys, uint32_t* values) {
  const uint64_t b = (uint64_t)g->b;
  for (int l = 0; l < g->depth; ++l) {
    const uint64_t nodes = ipow(b, l);
    const uint64_t span = ipow(b, g->depth - l - 1) * (uint64_t)k; /* keys under one child */
    for (uint64_t nd = 0; nd < nodes; ++nd)
      for (int j = 0; j < k; ++j) {
        const uint64_t idx = (nd * b + (uint64_t)j + 1) * span;
        keys[g->level_start[l] + nd * (uint64_t)k + (uint64_t)j] = idx < m ? boundaries[idx] : ORC_SENTINEL;
      }
  }
  const uint64_t slots = g->allocated_leaf_nodes * (uint64_t)k;
  for (uint64_t s = 0; s < slots; ++s) {
    keys[g->leaf_start + s] = s < m ? boundaries[s] : ORC_SENTINEL;
    values[s] = s < m ? next_hops[s] : next_hops[m - 1];
  }
}

/* node_rank: count of node keys <= key. */
static inline int node_rank_scalar(const uint64_t* node, int k, uint64_t key) {
  int c = 0;
  while (c < k && node[c] <= key) ++c; /* sorted, sentinels trailing */
  return c;
}

/* search_scalar = Alg. 1 with the rank-1 convention. */
uint64_t orc_search_scalar(const uint64_t* keys, const orc_geometry* g, uint64_t key) {
  if (key > ORC_MAX_QUERY) key = ORC_MAX_QUERY;
  uint64_t node = 0;
  for (int l = 0; l < g->depth; ++l) {
    const uint64_t start = g->level_start[l] + node * (uint64_t)g->k;
    node = node * (uint64_t)g->b + (uint64_t)node_rank_scalar(keys + start, g->k, key);
  }
  const uint64_t leaf = g->leaf_start + node * (uint64_t)g->k;
  return node * (uint64_t)g->k + (uint64_t)node_rank_scalar(keys + leaf, g->k, key) - 1;
}

/* search_branchfree: Listing 1's recurrence
 * i = (k+1) i + (c+1) k from i = 0, c = -1, rank by flag accumulation. */
uint64_t orc_search_branchfree(const uint64_t* keys, const orc_geometry* g, uint64_t key) {
  if (key > ORC_MAX_QUERY) key = ORC_MAX_QUERY;
  const int64_t k = g->k;
  int64_t i = 0, c = -1;
  for (int l = 0; l <= g->depth; ++l) {
    i = (k + 1) * i + (c + 1) * k;
    const uint64_t* node = keys + i;
    int64_t r = 0;
    for (int64_t j = 0; j < k; ++j) r += (int64_t)(node[j] <= key);
    c = r;
  }
  return (uint64_t)(i - (int64_t)g->leaf_start + c - 1);
}

/* ---- threaded batch driver (bench.py cpu_baseline / tests) -------------- */

typedef struct {
  int variant;
  const orc_index* ix;
  const uint64_t* addrs; /* 2 words per address: lo, hi */
  uint64_t lo, hi;
  uint32_t* out;
} orc_job;

static void* orc_worker(void* arg) {
  orc_job* j = (orc_job*)arg;
  const orc_index* ix = j->ix;
  if (j->variant == 0) {
    for (uint64_t i = j->lo; i < j->hi; ++i)
      j->out[i] = orc_lookup_interval(ix->boundaries, ix->next_hops, ix->m, j->addrs[2 * i + 1]);
  } else if (j->variant == 1) {
    for (uint64_t i = j->lo; i < j->hi; ++i)
      j->out[i] = ix->values[orc_search_branchfree(ix->keys, ix->g, j->addrs[2 * i + 1])];
  } else {
    orc_avx512_batch(ix->keys, ix->values, ix->g, j->addrs + 2 * j->lo, j->hi - j->lo, j->out + j->lo);
  }
  return NULL;
}

int orc_have_avx512(void) {
  __builtin_cpu_init();
  return __builtin_cpu_supports("avx512f") && __builtin_cpu_supports("avx512dq") &&
         __builtin_cpu_supports("avx512bw");
}

int orc_lookup_batch(int variant, const orc_index* ix, const void* addrs, uint64_t n,
                     uint32_t* out, int threads) {
  if (variant == 2 && (!orc_have_avx512() || ix->g->k != 8 || ix->g->depth > 7)) variant = 1;
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  orc_job jobs[256];
  const uint64_t chunk = (n + (uint64_t)threads - 1) / (uint64_t)threads;
  int started = 0;
  for (int t = 0; t < threads; ++t) {
    uint64_t lo = (uint64_t)t * chunk;
    if (lo > n) lo = n;
    uint64_t hi = lo + chunk;
    if (hi > n) hi = n;
    jobs[t].variant = variant;
    jobs[t].ix = ix;
    jobs[t].addrs = (const uint64_t*)addrs;
    jobs[t].lo = lo;
    jobs[t].hi = hi;
    jobs[t].out = out;
    if (threads == 1) {
      orc_worker(&jobs[t]);
    } else {
      pthread_create(&tid[t], NULL, orc_worker, &jobs[t]);
      ++started;
    }
  }
  for (int t = 0; t < started; ++t) pthread_join(tid[t], NULL);
  return variant;
}
