// B200 layout of the linearized B+-tree.
//
// The reference lays the tree out as one dense key array of 64-byte, 8-key
// nodes — internal levels breadth-first and fully allocated, then the leaves
// (tree.hpp:14-74). On B200 the node is one 128-byte L2
// line: k = 16 keys, arity b = 17 (the paper's own rule for 128-byte lines,
// P:601-604). Two changes from the reference layout, neither of which changes a
// single lookup result:
//   * each level holds only its reachable prefix of nodes, ceil(leaves / b^(d-l))
//     (the reference allocates b^l; the extra nodes are all-sentinel and never
//     visited), so level l starts at level_start[l] in a compact array
//     and child c of node j at level l is node j*b + c of level l+1;
//   * values are stored at the narrowest width that holds every next hop (u8 for
//     C0/C1/C3, u16 for C2/C4) instead of u32.
// Separators, sentinel padding, the leaf fill and the rank-1 ordinal are the
// reference's.
#pragma once

#include <cstddef>
#include <vector>

#include "lpm6/intervals.hpp"

namespace lpm6 {

inline constexpr int kMaxLevels = 9;  // depth <= 8

struct TreeLayout {
  u32 k = 16;
  u32 b = 17;
  u32 depth = 0;        // internal levels; a lookup visits depth + 1 nodes
  u32 value_bytes = 1;  // 1, 2 or 4
  u64 num_keys = 0;     // m, real boundaries
  u64 leaf_nodes = 0;   // ceil(m / k)
  u64 level_nodes[kMaxLevels] = {};  // reachable nodes per level; level depth = leaves
  u64 level_start[kMaxLevels] = {};  // key offset of each level in the key array
  u64 total_keys = 0;
  u32 default_next_hop = 0;
};

template <class T, size_t Align>
struct AlignedAllocator {
  using value_type = T;
  template <class U>
  struct rebind {
    using other = AlignedAllocator<U, Align>;
  };
  AlignedAllocator() = default;
  template <class U>
  AlignedAllocator(const AlignedAllocator<U, Align>&) {}
  T* allocate(size_t n) { return static_cast<T*>(::operator new(n * sizeof(T), std::align_val_t(Align))); }
  void deallocate(T* p, size_t) noexcept { ::operator delete(p, std::align_val_t(Align)); }
  template <class U>
  bool operator==(const AlignedAllocator<U, Align>&) const { return true; }
};

struct Tree {
  TreeLayout g;
  std::vector<u64, AlignedAllocator<u64, 128>> keys;  // total_keys
  std::vector<u8, AlignedAllocator<u8, 128>> values;  // leaf_nodes * k * value_bytes
};

// Minimal depth with k * b^depth >= m and the compact level table.
TreeLayout plan_layout(u64 m, u32 k = 16);

// value_bytes = 0 picks the narrowest of {1, 2, 4} holding every next hop;
// an explicit width that cannot hold one throws InvalidArgument.
Tree build_tree(const IntervalMap& map, u32 k = 16, u32 value_bytes = 0);

}  // namespace lpm6
