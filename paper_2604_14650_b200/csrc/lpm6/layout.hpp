// B200 layout of the linearized B+-tree.
//
// The reference lays the tree out as one dense key array of 64-byte, 8-key
// nodes — internal levels breadth-first and fully allocated, then the leaves —
// with next hops in a separate array indexed by leaf slot (tree.hpp:14-74,
// S:179-223). On B200 every node is one 128-byte L2 line:
//
//   * internal nodes hold k = 15 separator keys and a sentinel pad word, arity
//     b = 16 (the paper sizes nodes to the cache line: a 128-byte line
//     holds 16 keys; we give up the 16th separator so that the fan-out is a power
//     of two — a node rank is then exactly 4 binary-search probes and the child
//     index a shift; for the BASELINE FIBs the depth is the same as with b = 17);
//   * a leaf line holds kL boundary keys followed by their kL next hops
//     (kL = 14 for 1-byte, 12 for 2-byte, 8 for 4-byte next hops), so the
//     final value load of the reference (values[i - leaf_start])
//     is served by the leaf line the search already fetched;
//   * each level holds only its reachable prefix of nodes, ceil(leaves/b^(d-l))
//     (the reference allocates b^l; the extra nodes are all-sentinel and never
//     visited), and child c of node j is node j*b + c of the next level.
//
// Separators, sentinel padding, the query clamp and the rank-1 ordinal are the
// reference's: separator j of internal node n at
// level l is the first key of child n*b + j + 1, i.e. boundary[(n*b + j + 1) *
// span_l] with span_l = kL * b^(d-l-1), or the sentinel past the last boundary.
#pragma once

#include <cstddef>
#include <vector>

#include "lpm6/intervals.hpp"

namespace lpm6 {

inline constexpr int kMaxLevels = 9;  // depth <= 8
inline constexpr u32 kNodeKeys = 15;  // internal separator keys per 128-byte line (word 15 = pad)
inline constexpr u32 kLineWords = 16;  // u64 words per line

// Keys per leaf line for a next-hop width (leaf = kL keys + kL values <= 128 B).
constexpr u32 leaf_keys_for(u32 value_bytes) { return value_bytes == 1 ? 14 : value_bytes == 2 ? 12 : 8; }

// Half-line leaves (64 bytes, 2-byte next hops): 6 keys (words 0-5) and their
// next hops in words 6-7 (12 bytes), so that in a lookup the fourth lane of a 4-lane group holds
// exactly the values and the other three exactly the keys (16 bytes each). A query
// then reads one 64-byte leaf instead of a 128-byte one: one texture fetch or one
// 16-byte load per lane, half the L2 bytes. Used where it keeps the tree's depth and
// its shared-memory levels (plan_layout's automatic rule), i.e. deep trees whose
// last internal level is read from L2 anyway (the 1M-prefix C2 FIB).
inline constexpr u32 kHalfLeafKeys = 6;
inline constexpr u32 kHalfLeafWords = 8;
enum LeafFormat : u32 { kLeafAuto = 0, kLeafFull = 1, kLeafHalf = 2 };

struct TreeLayout {
  u32 k = kNodeKeys;    // internal keys per node
  u32 b = kNodeKeys + 1;
  u32 depth = 0;        // internal levels; a lookup visits depth + 1 lines
  u32 value_bytes = 1;  // 1, 2 or 4
  u32 leaf_keys = 14;   // kL
  u32 leaf_words = kLineWords;  // 16: one 128-byte line per leaf; 8: half-line leaves
  u64 num_keys = 0;     // m, real boundaries
  u64 leaf_nodes = 0;   // ceil(m / kL)
  u64 level_nodes[kMaxLevels] = {};  // reachable nodes per level; level depth = leaves
  u64 level_start[kMaxLevels] = {};  // u64-word offset of each level in the line array
  u64 total_words = 0;               // tree lines (16 words each), then the smem image
  // Packed copy of internal levels [0, image_levels) that the kernel stages
  // into shared memory with one TMA bulk copy: the 15 separators of each node,
  // 120 bytes per node (no pad word). The 15-word node stride also skews the
  // shared-memory banks: key p of node n lives in 8-byte bank pair
  // (15n + p) mod 16, so threads probing the same position of different nodes
  // hit different banks. Level l of the image starts at image word
  // image_level_start(l) = (level_start[l] / 16) * 15.
  u32 image_levels = 0;
  u64 image_start = 0;
  // Small trees only: when every internal level is imaged and the leaves fit
  // too, a second image follows the first — each leaf line's 16 words at a
  // 17-word stride (the odd stride skews banks like the 15-word internal nodes)
  // — and the kernel serves the whole lookup from shared memory.
  u32 leaf_image = 0;
  u32 default_next_hop = 0;
};

inline constexpr u64 kImageMaxBytes = 232448 - 1024;  // B200 opt-in smem per CTA minus static smem
inline constexpr u32 kLeafImageStride = 17;              // words per leaf in the leaf image
inline constexpr u32 kMaxLeafImageDepth = 3;             // leaf-image kernels are instantiated for depth <= 3

// Word offset of level l / of key p of node n (within its level) in the image.
constexpr u64 image_level_start(const TreeLayout& g, u32 l) { return g.level_start[l] / kLineWords * kNodeKeys; }
constexpr u64 image_slot(u64 n, u32 p) { return n * kNodeKeys + p; }
// Bytes the kernel stages for `levels` imaged levels (TMA sizes are 16-byte multiples).
constexpr u64 image_bytes(const TreeLayout& g, u32 levels) { return (image_level_start(g, levels) * 8 + 15) / 16 * 16; }
// The leaf image: word offset in the line array and bytes (16-byte multiple).
constexpr u64 leaf_image_start(const TreeLayout& g) { return g.image_start + image_bytes(g, g.depth) / 8; }
constexpr u64 leaf_image_bytes(const TreeLayout& g) { return (g.leaf_nodes * kLeafImageStride * 8 + 15) / 16 * 16; }

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
  std::vector<u64, AlignedAllocator<u64, 128>> lines;  // total_words: the device image
  std::vector<u32> leaf_values;                         // next hop per leaf slot (inspection only)
};

// Minimal depth with kL * b^depth >= m and the compact level table. leaf_format:
// kLeafFull, kLeafHalf (2-byte next hops only), or kLeafAuto = half-line
// leaves when they leave the depth and the number of shared-memory levels unchanged
// and the tree has an internal level in L2 (no leaf image), full lines otherwise.
TreeLayout plan_layout(u64 m, u32 value_bytes, u32 leaf_format = kLeafAuto);

// value_bytes = 0 picks the narrowest of {1, 2, 4} holding every next hop;
// an explicit width that cannot hold one throws InvalidArgument.
Tree build_tree(const IntervalMap& map, u32 value_bytes = 0, u32 leaf_format = kLeafAuto);

}  // namespace lpm6
