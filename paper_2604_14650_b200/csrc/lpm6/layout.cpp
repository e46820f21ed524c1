#include "lpm6/layout.hpp"

#include <cstring>

namespace lpm6 {

namespace {

TreeLayout plan_with(u64 m, u32 value_bytes, bool half) {
  TreeLayout g;
  g.value_bytes = value_bytes;
  g.leaf_keys = half ? kHalfLeafKeys : leaf_keys_for(value_bytes);
  g.leaf_words = half ? kHalfLeafWords : kLineWords;
  g.num_keys = m;
  u32 d = 0;
  for (unsigned __int128 cap = g.leaf_keys; cap < m; cap *= g.b) ++d;
  if (d + 1 > static_cast<u32>(kMaxLevels))
    throw Error(Errc::InvalidArgument, "tree deeper than supported (" + std::to_string(d) + ")");
  g.depth = d;
  g.leaf_nodes = (m + g.leaf_keys - 1) / g.leaf_keys;
  g.level_nodes[d] = g.leaf_nodes;
  for (int l = static_cast<int>(d) - 1; l >= 0; --l) g.level_nodes[l] = (g.level_nodes[l + 1] + g.b - 1) / g.b;
  u64 off = 0;
  for (u32 l = 0; l <= d; ++l) {
    g.level_start[l] = off;
    off += g.level_nodes[l] * (l < d ? kLineWords : g.leaf_words);
  }
  // Image of internal levels [0, S) for the largest S <= depth whose image fits the budget.
  u32 s = 0;
  while (s + 1 <= d && image_bytes(g, s + 1) <= kImageMaxBytes) ++s;
  g.image_levels = s;
  g.image_start = off;
  g.total_words = off + image_bytes(g, s) / 8;
  if (!half && s == d && d <= kMaxLeafImageDepth && image_bytes(g, d) + leaf_image_bytes(g) <= kImageMaxBytes) {
    g.leaf_image = 1;
    g.total_words = leaf_image_start(g) + leaf_image_bytes(g) / 8;
  }
  if (g.total_words >= (u64(1) << 32))
    throw Error(Errc::InvalidArgument, "tree larger than 32 GiB (word offsets are 32-bit in the kernel)");
  return g;
}

}  // namespace

TreeLayout plan_layout(u64 m, u32 value_bytes, u32 leaf_format) {
  if (m < 1) throw Error(Errc::InvalidArgument, "a tree needs at least one boundary");
  if (value_bytes != 1 && value_bytes != 2 && value_bytes != 4)
    throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
  if (leaf_format > kLeafHalf) throw Error(Errc::InvalidArgument, "leaf_format must be 0 (auto), 1 (full) or 2 (half)");
  if (leaf_format == kLeafHalf && value_bytes != 2)
    throw Error(Errc::InvalidArgument, "half-line leaves hold 2-byte next hops");
  const TreeLayout full = plan_with(m, value_bytes, false);
  if (leaf_format == kLeafFull || value_bytes != 2) return full;
  const TreeLayout half = plan_with(m, value_bytes, true);
  if (leaf_format == kLeafHalf) return half;
  const bool keeps = half.depth == full.depth && half.image_levels == full.image_levels;
  return keeps && !full.leaf_image && full.image_levels < full.depth ? half : full;
}

Tree build_tree(const IntervalMap& map, u32 value_bytes, u32 leaf_format) {
  const u64 m = map.size();
  if (m < 1) throw Error(Errc::InvalidArgument, "empty interval map");
  if (map.boundaries.front() != 0) throw Error(Errc::InvalidArgument, "interval map must start at key 0");
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

  Tree t;
  t.g = plan_layout(m, value_bytes, leaf_format);
  t.g.default_next_hop = map.default_next_hop;
  const TreeLayout& g = t.g;
  const u32 kl = g.leaf_keys;
  t.lines.assign(g.total_words, kSentinelKey);
  const u64* bnd = map.boundaries.data();

  // Internal levels, deepest first: span = boundaries under one child.
  u64 span = kl;
  for (int l = static_cast<int>(g.depth) - 1; l >= 0; --l) {
    u64* lvl = t.lines.data() + g.level_start[l];
    for (u64 n = 0; n < g.level_nodes[l]; ++n)
      for (u32 j = 0; j < g.k; ++j) {
        const unsigned __int128 idx = (static_cast<unsigned __int128>(n) * g.b + j + 1) * span;
        lvl[n * kLineWords + j] = idx < m ? bnd[static_cast<u64>(idx)] : kSentinelKey;
      }
    span *= g.b;
  }

  // Leaf lines (or half lines): kL keys (sentinel past m), then kL little-endian
  // next hops (padding replicates the last real value), then zero padding.
  t.leaf_values.resize(g.leaf_nodes * kl);
  u64* leaves = t.lines.data() + g.level_start[g.depth];
  for (u64 n = 0; n < g.leaf_nodes; ++n) {
    u64* line = leaves + n * g.leaf_words;
    unsigned char bytes[128];
    std::memset(bytes, 0, sizeof bytes);
    for (u32 j = 0; j < kl; ++j) {
      const u64 s = n * kl + j;
      const u64 key = s < m ? bnd[s] : kSentinelKey;
      const u32 v = map.next_hops[s < m ? s : m - 1];
      t.leaf_values[s] = v;
      std::memcpy(bytes + 8 * j, &key, 8);
      std::memcpy(bytes + 8 * kl + value_bytes * j, &v, value_bytes);
    }
    std::memcpy(line, bytes, g.leaf_words * 8);
  }

  // Shared-memory image: internal levels [0, image_levels), 15 keys per node.
  for (u32 l = 0; l < g.image_levels; ++l) {
    const u64* src = t.lines.data() + g.level_start[l];
    u64* dst = t.lines.data() + g.image_start + image_level_start(g, l);
    for (u64 n = 0; n < g.level_nodes[l]; ++n)
      for (u32 p = 0; p < kNodeKeys; ++p) dst[image_slot(n, p)] = src[n * kLineWords + p];
  }
  // Leaf image (small trees): leaf lines at a 17-word stride; the pad word stays sentinel.
  if (g.leaf_image) {
    u64* dst = t.lines.data() + leaf_image_start(g);
    for (u64 n = 0; n < g.leaf_nodes; ++n)
      std::memcpy(dst + n * kLeafImageStride, leaves + n * kLineWords, kLineWords * 8);
  }
  return t;
}

}  // namespace lpm6
