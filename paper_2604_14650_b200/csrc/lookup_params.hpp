// Launch interface of the lookup kernels (lookup_kernel.cuh), shared by the host
// half (lookup.cu) and the per-width instantiation units (lookup_vb{1,2,4}.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "lpm6cu.h"

namespace lpm6::kern {

// Input formats of the lookup kernel.
enum : int { kInAddr = 0, kInKey = 1, kInPacket = 2, kInKeyOrd = 3 };  // kInKeyOrd: keys in, ordinals out too

constexpr int kMaxKernelDepth = 7;
constexpr int kAllPlanes = 8;  // PLANES value: every staged level below the root as planes

struct LookupParams {
  const unsigned long long* lines;                     // the tree, 16 u64 words per line
  unsigned long long level_start[LPM6CU_MAX_LEVELS];  // word offset of each level
  const uint4* addrs;               // kInAddr: 16-byte addresses (lookup_batch), or
  const unsigned long long* keys;   // kInKey / kInKeyOrd: 8-byte keys (search_batch's input), or
  unsigned int* ord;                // kInKeyOrd: interval ordinal per query (SearchResult::interval_ordinal)
  const unsigned char* pkts;        // kInPacket: frames, destination address at pkt_off of each
  unsigned long long pkt_stride;    //   bytes between frames
  unsigned int pkt_off;             //   byte offset of the IPv6 destination address in a frame
  unsigned int pkt_align;           //   16, 8, 4, 2 or 1: alignment of every frame start
  unsigned char* out;
  unsigned long long n;
  const unsigned long long* image;  // packed 15-key copy of internal levels 0.. (layout.hpp)
  unsigned int smem_levels;  // phase A levels [0, smem_levels), <= depth
  unsigned int smem_bytes;   // image bytes staged for those levels (+ the leaf image when LEAFS)
  unsigned int leaf_image_off;  // LEAFS: word offset of the leaf image in shared memory
  unsigned long long level_nodes[LPM6CU_MAX_LEVELS];  // checked mode: node-index bounds
  unsigned int* err;         // checked mode: OR of violation bits (1 smem level, 2 line level, 4 leaf rank)
  unsigned long long root[16];  // the root's 15 separators (+ sentinel), read from the constant bank
  unsigned long long tex;       // texture object over the line array (int4 texels), 0 = none
  // Phase A address walk (lookup_kernel.cuh), with off(l) = byte offset of level l
  // in the shared-memory image: img_step[0] = off(1); img_step[l] = off(l+1) -
  // 16 off(l) for 1 <= l < smem_levels - 1; img_step[smem_levels - 1] = -16 off(l).
  unsigned int img_step[LPM6CU_MAX_LEVELS];
  // Split-plane Phase A (PLANES kernels; lpm6cu_kernel_config.plane_levels): the plane
  // levels are stored as their nodes' high words (15 u32 per node) followed, lo_delta[l]
  // bytes further, by their low words; deeper staged levels stay packed.
  unsigned int lo_delta[LPM6CU_MAX_LEVELS];
  unsigned int pl2pk;  // off(P) - 32 off(P - 1): the walk's step from the last plane level to a packed one
};

using KernelFn = void (*)(const LookupParams);

// Which kernel: tree depth, shape (32-query tiles per warp, threads per CTA, min
// CTAs per SM), checked mode, input format, leaf image, line path (texl: internal
// L2 levels 0 LSU / 1 texture / 2 split; leaftex: leaves 0 LSU / 1 texture / 2 split).
struct PickArgs {
  int depth = 0, tiles = 1, threads = 1024, minb = 1;
  bool checked = false;
  int input = kInAddr;
  bool leafs = false;
  int texl = 0, leaftex = 0;
  bool half = false;  // half-line leaves (layout.hpp kHalfLeafWords; 2-byte next hops)
  int ta = 0;         // staged levels (smem_levels) of the launch: compile-time in the texture line-path kernels
  int planes = 0;  // split-plane Phase A (2 or 4 tiles per warp on the texture leaf paths): 0, 2, 3 or kAllPlanes
};

KernelFn pick_kernel_vb1(const PickArgs& a);  // lookup_vb1.cu
KernelFn pick_kernel_vb2(const PickArgs& a);  // lookup_vb2.cu
KernelFn pick_kernel_vb4(const PickArgs& a);  // lookup_vb4.cu

// nullptr when that combination is not instantiated.
inline KernelFn pick_kernel(int vb, int depth, int tiles, int threads, int minb, bool checked = false,
                            int input = kInAddr, bool leafs = false, int texl = 0, int leaftex = 0,
                            bool half = false, int ta = 0, int planes = 0) {
  PickArgs a;
  a.depth = depth;
  a.tiles = tiles;
  a.threads = threads;
  a.minb = minb;
  a.checked = checked;
  a.input = input;
  a.leafs = leafs;
  a.texl = texl;
  a.leaftex = leaftex;
  a.half = half;
  a.ta = ta;
  a.planes = planes;
  switch (vb) {
    case 1: return pick_kernel_vb1(a);
    case 2: return pick_kernel_vb2(a);
    case 4: return pick_kernel_vb4(a);
    default: return nullptr;
  }
}

}  // namespace lpm6::kern
