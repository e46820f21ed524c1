#include "lpm6/layout.hpp"

#include <cstring>

namespace lpm6 {

TreeLayout plan_layout(u64 m, u32 k) {
  if (m < 1) throw Error(Errc::InvalidArgument, "a tree needs at least one boundary");
  if (k < 2) throw Error(Errc::InvalidArgument, "k must be >= 2");
  TreeLayout g;
  g.k = k;
  g.b = k + 1;
  g.num_keys = m;
  // Minimal depth with k * b^depth >= m.
  u32 d = 0;
  for (unsigned __int128 cap = k; cap < m; cap *= g.b) ++d;
  if (d + 1 > static_cast<u32>(kMaxLevels))
    throw Error(Errc::InvalidArgument, "tree deeper than supported (" + std::to_string(d) + ")");
  g.depth = d;
  g.leaf_nodes = (m + k - 1) / k;
  g.level_nodes[d] = g.leaf_nodes;
  for (int l = static_cast<int>(d) - 1; l >= 0; --l)
    g.level_nodes[l] = (g.level_nodes[l + 1] + g.b - 1) / g.b;
  u64 off = 0;
  for (u32 l = 0; l <= d; ++l) {
    g.level_start[l] = off;
    off += g.level_nodes[l] * k;
  }
  g.total_keys = off;
  return g;
}

Tree build_tree(const IntervalMap& map, u32 k, u32 value_bytes) {
  const u64 m = map.size();
  Tree t;
  t.g = plan_layout(m, k);
  t.g.default_next_hop = map.default_next_hop;
  if (map.boundaries.front() != 0)
    throw Error(Errc::InvalidArgument, "interval map must start at key 0");
  for (u64 b : map.boundaries)
    if (b == kSentinelKey) throw Error(Errc::SentinelCollision, "boundary at the sentinel key");

  u32 max_nh = 0;
  for (u32 nh : map.next_hops) max_nh = nh > max_nh ? nh : max_nh;
  const u32 need = max_nh <= 0xFFu ? 1 : (max_nh <= 0xFFFFu ? 2 : 4);
  if (value_bytes == 0) value_bytes = need;
  if (value_bytes != 1 && value_bytes != 2 && value_bytes != 4)
    throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
  if (value_bytes < need)
    throw Error(Errc::InvalidArgument, "next hop " + std::to_string(max_nh) + " does not fit in " +
                                           std::to_string(value_bytes) + " byte(s)");
  t.g.value_bytes = value_bytes;

  const TreeLayout& g = t.g;
  t.keys.assign(g.total_keys, kSentinelKey);
  const u64* bnd = map.boundaries.data();

  // Internal level l: separator j of node n = first key of child n*b + j + 1,
  // i.e. boundary[(n*b + j + 1) * span], span = keys under one child = k*b^(d-l-1).
  u64 span = k;
  for (int l = static_cast<int>(g.depth) - 1; l >= 0; --l) {
    u64* lvl = t.keys.data() + g.level_start[l];
    for (u64 n = 0; n < g.level_nodes[l]; ++n)
      for (u32 j = 0; j < k; ++j) {
        const unsigned __int128 idx = (static_cast<unsigned __int128>(n) * g.b + j + 1) * span;
        lvl[n * k + j] = idx < m ? bnd[static_cast<u64>(idx)] : kSentinelKey;
      }
    span *= g.b;
  }
  // Leaves: the boundaries, then sentinels.
  std::memcpy(t.keys.data() + g.level_start[g.depth], bnd, m * sizeof(u64));

  // Values parallel to leaf slots; padding replicates the last real value.
  const u64 slots = g.leaf_nodes * k;
  t.values.assign(slots * value_bytes, 0);
  for (u64 s = 0; s < slots; ++s) {
    const u32 v = map.next_hops[s < m ? s : m - 1];
    std::memcpy(t.values.data() + s * value_bytes, &v, value_bytes);  // little-endian
  }
  return t;
}

}  // namespace lpm6
