// Host half of the C ABI (include/lpm6cu.h): FIB build, layout, workloads.
// Everything here runs without a GPU.
#include <cstring>

#include "capi_internal.hpp"
#include "lpm6/fib.hpp"
#include "lpm6/intervals.hpp"
#include "lpm6/layout.hpp"
#include "lpm6/workload.hpp"
#include "lpm6cu.h"

namespace lpm6::capi {

static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }
void clear_error() { g_last_error.clear(); }

std::vector<Prefix> to_prefixes(const lpm6cu_prefix* rules, uint64_t n) {
  static_assert(sizeof(lpm6cu_prefix) == sizeof(Prefix));
  std::vector<Prefix> v(n);
  for (uint64_t i = 0; i < n; ++i) {
    v[i].value = (u128(rules[i].value_hi) << 64) | rules[i].value_lo;
    v[i].length = rules[i].length;
    v[i].next_hop = rules[i].next_hop;
  }
  return v;
}

void export_geometry(const TreeLayout& t, lpm6cu_geometry* g) {
  std::memset(g, 0, sizeof(*g));
  g->k = t.k;
  g->b = t.b;
  g->depth = t.depth;
  g->value_bytes = t.value_bytes;
  g->leaf_keys = t.leaf_keys;
  g->num_keys = t.num_keys;
  g->leaf_nodes = t.leaf_nodes;
  g->total_words = t.total_words;
  g->image_levels = t.image_levels;
  g->image_start = t.image_start;
  g->leaf_image = t.leaf_image;
  g->leaf_words = t.leaf_words;
  for (int l = 0; l < kMaxLevels; ++l) {
    g->level_nodes[l] = t.level_nodes[l];
    g->level_start[l] = t.level_start[l];
  }
  g->default_next_hop = t.default_next_hop;
}

Tree build_device_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                       const lpm6cu_build_opts* opts) {
  IntervalBuildOptions io;
  u32 vb = 0, lf = kLeafAuto;
  if (opts) {
    io.merge_adjacent = opts->merge_adjacent != 0;
    vb = opts->value_bytes;
    lf = opts->leaf_format;
  }
  auto prefixes = to_prefixes(rules, n);
  IntervalMap map = build_intervals(std::span<const Prefix>(prefixes), default_nh, io);
  return build_tree(map, vb, lf);
}

}  // namespace lpm6::capi

using namespace lpm6;
using namespace lpm6::capi;

extern "C" {

const char* lpm6cu_last_error(void) { return g_last_error.c_str(); }

const char* lpm6cu_status_name(int s) {
  static const char* names[] = {"Ok",
                                "MalformedAddress",
                                "UnsupportedPrefixLength",
                                "MissingNextHop",
                                "ReservedNextHop",
                                "DuplicatePrefix",
                                "UnknownPrefix",
                                "SentinelCollision",
                                "ExhaustedPrefixSpace",
                                "InvalidArgument",
                                "BadTraceFile",
                                "BadSnapshotFile",
                                "Io",
                                "CudaError",
                                "NcclError"};
  return (s >= 0 && s < static_cast<int>(sizeof(names) / sizeof(names[0]))) ? names[s] : "Unknown";
}

const char* lpm6cu_version(void) { return "lpm6cu 0.1 (sm_100a)"; }

int lpm6_build_intervals(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh, int merge,
                         uint64_t* boundaries, uint32_t* next_hops, uint64_t capacity,
                         uint64_t* m_out) {
  return guard([&] {
    if (n > 0 && !rules) throw Error(Errc::InvalidArgument, "rules is NULL");
    if (capacity < 2 * n + 1) throw Error(Errc::InvalidArgument, "capacity must be >= 2n+1");
    auto prefixes = to_prefixes(rules, n);
    IntervalBuildOptions io;
    io.merge_adjacent = merge != 0;
    IntervalMap map = build_intervals(std::span<const Prefix>(prefixes), default_nh, io);
    std::memcpy(boundaries, map.boundaries.data(), map.size() * sizeof(u64));
    std::memcpy(next_hops, map.next_hops.data(), map.size() * sizeof(u32));
    *m_out = map.size();
  });
}

int lpm6_plan_layout(uint64_t m, uint32_t value_bytes, lpm6cu_geometry* g) {
  return lpm6_plan_layout_ex(m, value_bytes, kLeafAuto, g);
}

int lpm6_plan_layout_ex(uint64_t m, uint32_t value_bytes, uint32_t leaf_format, lpm6cu_geometry* g) {
  return guard([&] {
    if (!g) throw Error(Errc::InvalidArgument, "NULL geometry");
    export_geometry(plan_layout(m, value_bytes, leaf_format), g);
  });
}

int lpm6_build_tree(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                    uint32_t default_nh, uint32_t value_bytes, lpm6cu_geometry* g, uint64_t* lines,
                    uint32_t* leaf_values) {
  return lpm6_build_tree_ex(boundaries, next_hops, m, default_nh, value_bytes, kLeafAuto, g, lines, leaf_values);
}

int lpm6_build_tree_ex(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                       uint32_t default_nh, uint32_t value_bytes, uint32_t leaf_format, lpm6cu_geometry* g,
                       uint64_t* lines, uint32_t* leaf_values) {
  return guard([&] {
    if (!g) throw Error(Errc::InvalidArgument, "NULL geometry");
    if (m < 1 || !boundaries || !next_hops) throw Error(Errc::InvalidArgument, "empty interval map");
    IntervalMap map;
    map.boundaries.assign(boundaries, boundaries + m);
    map.next_hops.assign(next_hops, next_hops + m);
    map.default_next_hop = default_nh;
    Tree t = build_tree(map, value_bytes, leaf_format);
    export_geometry(t.g, g);
    if (lines) std::memcpy(lines, t.lines.data(), t.lines.size() * sizeof(u64));
    if (leaf_values) std::memcpy(leaf_values, t.leaf_values.data(), t.leaf_values.size() * sizeof(u32));
  });
}

int lpm6_parse_prefix(const char* text, lpm6cu_prefix* out, int* masked) {
  return guard([&] {
    ParsedPrefix p = parse_prefix(text ? text : "");
    out->value_lo = static_cast<uint64_t>(p.prefix.value);
    out->value_hi = static_cast<uint64_t>(p.prefix.value >> 64);
    out->length = p.prefix.length;
    out->next_hop = p.prefix.next_hop;
    out->reserved = 0;
    if (masked) *masked = p.host_bits_masked ? 1 : 0;
  });
}

int lpm6_workload_info_get(int workload, lpm6_workload_info* info) {
  return guard([&] {
    if (!info) throw Error(Errc::InvalidArgument, "NULL info");
    WorkloadConfig c = workload_config(workload);
    std::memset(info, 0, sizeof(*info));
    info->id = c.id;
    info->fib_kind = c.fib_kind;
    info->n_queries = c.n_queries;
    info->chunk = c.chunk;
    info->value_bytes = c.value_bytes;
    std::strncpy(info->name, c.name, sizeof(info->name) - 1);
  });
}

int lpm6_workload_fib(int fib_kind, lpm6cu_prefix* out, uint64_t capacity, uint64_t* n_out,
                      uint32_t* default_nh) {
  return guard([&] {
    if (!n_out) throw Error(Errc::InvalidArgument, "NULL n_out");
    FibTable fib = make_fib(fib_kind);
    *n_out = fib.size();
    if (default_nh) *default_nh = fib.default_next_hop();
    if (!out) return;
    if (capacity < fib.size()) throw Error(Errc::InvalidArgument, "capacity too small");
    const auto& e = fib.entries();
    for (size_t i = 0; i < e.size(); ++i) {
      out[i].value_lo = static_cast<uint64_t>(e[i].value);
      out[i].value_hi = static_cast<uint64_t>(e[i].value >> 64);
      out[i].length = e[i].length;
      out[i].next_hop = e[i].next_hop;
      out[i].reserved = 0;
    }
  });
}

int lpm6_workload_queries_host(int workload, const lpm6cu_prefix* rules, uint64_t nrules,
                               uint64_t first, uint64_t n, void* out, int threads) {
  return guard([&] {
    if ((nrules && !rules) || (n && !out)) throw Error(Errc::InvalidArgument, "NULL argument");
    WorkloadConfig c = workload_config(workload);
    auto prefixes = to_prefixes(rules, nrules);
    QueryTables t = make_query_tables(std::span<const Prefix>(prefixes), c);
    QuerySpec s = make_query_spec(c, t);
    gen_queries_host(s, first, n, static_cast<u64*>(out), threads);
  });
}

}  // extern "C"
