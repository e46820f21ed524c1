// sm_100a batched LPM lookup kernel and the device half of the C ABI.
//
// One query = one predecessor search down the B200 tree (layout.hpp): internal
// 128-byte lines of 15 separators (arity 16), leaf lines of kL keys + kL next
// hops. The kernel is the GPU form of the reference's search_batch
// over Listing 1's node search, in two
// phases per 32-query warp tile (lane L owns query L):
//
//  Phase A — top `smem_levels` levels, one thread per query. A packed image of
//    these levels is staged into shared memory once per CTA by cp.async.bulk
//    (TMA bulk copy) on an mbarrier. Each thread ranks its own query in a node
//    with a branch-free 4-probe binary search (count of keys <= q, i.e.
//    Listing 1's popcnt(cmpge)), reading 8 bytes per probe instead of a whole
//    128-byte node.
//  Phase B — the remaining levels through L1/L2, four lanes per query: lane j of
//    a 4-lane group loads bytes [32j, 32j+32) of the line with one 256-bit load,
//    so a warp-wide load fetches exactly one full 128-byte line per query; the
//    lanes compare their keys against the broadcast query and __ballot_sync +
//    __popc give the rank. Each group carries its 4 queries at once and the
//    descent is unrolled over the depth (template), so every level has 4
//    independent line loads in flight per group (the batching of P:812-847 as
//    memory-level parallelism).
//  Leaf — the leaf line carries the next hops (P:695-705 folded into the leaf
//    fetch): after the leaf rank, the lane holding the value bytes extracts the
//    group's 4 next hops and writes them with one coalesced streaming store.
//
// Query addresses are read with coalesced 16-byte-stride loads of the top word
// (L1::no_allocate, L2 evict_first), one tile ahead of their use — each step
// streams GBs of addresses through L2 while the tree stays resident
// (evict_last on tree lines). CTAs are persistent (grid = SMs x resident CTAs,
// default one 1024-thread CTA per SM) and stride over tiles.
//
// Results are the reference's: key = min(addr >> 64, 0xFFFF...FFFE)
// (types.hpp:25), internal child = node * 16 + rank, leaf ordinal =
// rank - 1, next hop = the value of that leaf slot.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "capi_internal.hpp"
#include "lpm6/workload.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

constexpr int kMaxKernelDepth = 7;
constexpr unsigned kFull = 0xFFFFFFFFu;

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// ---- PTX helpers ------------------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}

__device__ __forceinline__ uint4 ld_stream_v4(const uint4* p, uint64_t pol) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}


// Input formats of the lookup kernel.
enum : int { kInAddr = 0, kInKey = 1, kInPacket = 2, kInKeyOrd = 3 };  // kInKeyOrd: keys in, ordinals out too

template <class T>
__device__ __forceinline__ T ld_stream(const void* p, uint64_t pol);
template <>
__device__ __forceinline__ unsigned long long ld_stream<unsigned long long>(const void* p, uint64_t pol) {
  unsigned long long r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u64 %0, [%1], %2;" : "=l"(r) : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ unsigned ld_stream<unsigned>(const void* p, uint64_t pol) {
  unsigned r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
template <>
__device__ __forceinline__ unsigned short ld_stream<unsigned short>(const void* p, uint64_t pol) {
  unsigned short r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.u16 %0, [%1], %2;" : "=h"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ unsigned long long bswap64(unsigned long long v) {
  const unsigned lo = static_cast<unsigned>(v), hi = static_cast<unsigned>(v >> 32);
  return (static_cast<unsigned long long>(__byte_perm(lo, 0, 0x0123)) << 32) | __byte_perm(hi, 0, 0x0123);
}


// Bytes [sh, sh + 8) of the little-endian pair (w0, w1), sh in 0..8.
__device__ __forceinline__ unsigned long long extract8(unsigned long long w0, unsigned long long w1, unsigned sh) {
  return sh == 0 ? w0 : sh >= 8 ? w1 : (w0 >> (8 * sh)) | (w1 << (64 - 8 * sh));
}

// Top 64 bits of an IPv6 address stored in network byte order (the first 8
// bytes of the destination field) at frame + off, where every frame start is
// aligned to `align` bytes (16, 8, 4, 2 or 1; uniform across the launch). The
// 8 key bytes are fetched with as few aligned loads as cover them — one 16-byte
// load when they sit inside one aligned 16-byte chunk — because every load
// instruction of a warp costs one L1 wavefront per distinct line it touches.
__device__ __forceinline__ unsigned long long load_dst_key(const unsigned char* frame, unsigned off, unsigned align,
                                                           uint64_t pol) {
  unsigned long long le;  // the 8 bytes as a little-endian integer
  if (align >= 16) {
    const unsigned sh = off & 15u;
    const unsigned char* c = frame + (off - sh);
    const uint4 v = ld_stream_v4(reinterpret_cast<const uint4*>(c), pol);
    const unsigned long long w0 = v.x | (static_cast<unsigned long long>(v.y) << 32);
    const unsigned long long w1 = v.z | (static_cast<unsigned long long>(v.w) << 32);
    if (sh <= 8) {
      le = extract8(w0, w1, sh);
    } else {
      const unsigned long long w2 = ld_stream<unsigned long long>(c + 16, pol);
      le = extract8(w1, w2, sh - 8);
    }
  } else if (align >= 8) {
    const unsigned sh = off & 7u;
    const unsigned char* c = frame + (off - sh);
    const unsigned long long w0 = ld_stream<unsigned long long>(c, pol);
    le = sh ? extract8(w0, ld_stream<unsigned long long>(c + 8, pol), sh) : w0;
  } else if (align >= 4 && (off & 3u) == 0) {
    const unsigned char* a = frame + off;
    le = ld_stream<unsigned>(a, pol) | (static_cast<unsigned long long>(ld_stream<unsigned>(a + 4, pol)) << 32);
  } else if (align >= 2 && (off & 1u) == 0) {
    const unsigned char* a = frame + off;
    le = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      le |= static_cast<unsigned long long>(ld_stream<unsigned short>(a + 2 * i, pol)) << (16 * i);
  } else {
    const unsigned char* a = frame + off;
    le = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i) le |= static_cast<unsigned long long>(__ldg(a + i)) << (8 * i);
  }
  return bswap64(le);  // network order: first byte is the most significant
}

// 32 bytes of a line through the texture path (two 16-byte texels at texel index t, t+1).
__device__ __forceinline__ void tex_line_quarter(unsigned long long tex, unsigned t, unsigned long long (&w)[4]) {
  int a0, a1, a2, a3, b0, b1, b2, b3;
  asm volatile("tex.1d.v4.s32.s32 {%0,%1,%2,%3}, [%4, {%5}];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "l"(tex), "r"(t));
  asm volatile("tex.1d.v4.s32.s32 {%0,%1,%2,%3}, [%4, {%5}];"
               : "=r"(b0), "=r"(b1), "=r"(b2), "=r"(b3) : "l"(tex), "r"(t + 1));
  w[0] = static_cast<unsigned>(a0) | (static_cast<unsigned long long>(static_cast<unsigned>(a1)) << 32);
  w[1] = static_cast<unsigned>(a2) | (static_cast<unsigned long long>(static_cast<unsigned>(a3)) << 32);
  w[2] = static_cast<unsigned>(b0) | (static_cast<unsigned long long>(static_cast<unsigned>(b1)) << 32);
  w[3] = static_cast<unsigned>(b2) | (static_cast<unsigned long long>(static_cast<unsigned>(b3)) << 32);
}

__device__ __forceinline__ void ld_line_quarter(const unsigned long long* p, unsigned long long (&w)[4]) {
  asm volatile("ld.global.nc.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];"
               : "=l"(w[0]), "=l"(w[1]), "=l"(w[2]), "=l"(w[3])
               : "l"(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "LAB_WAIT:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra LAB_WAIT;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(phase)
      : "memory");
}

// ---- kernel -----------------------------------------------------------------

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
};

// Count of the 15 separators of node n of a shared-memory image level that are
// <= q: a branch-free 4-probe binary search (16 outcomes). The probe positions
// 7, c|3, c|1, c are ORs of the bits found so far (one predicated OR per step).
// Nodes are packed at a 15-word stride (layout.hpp), which puts the same
// position of different nodes in different shared-memory banks.
__device__ __forceinline__ unsigned node_rank_smem(const unsigned long long* lvl, unsigned n, unsigned long long q) {
  const unsigned long long* nd = lvl + n * 15u;
  unsigned c = (nd[7] <= q) ? 8u : 0u;
  c |= (nd[c | 3u] <= q) ? 4u : 0u;
  c |= (nd[c | 1u] <= q) ? 2u : 0u;
  c |= (nd[c] <= q) ? 1u : 0u;
  return c;
}

// The same search on a shared-memory byte address: each probe is one LDS at an
// immediate offset, one 64-bit compare and one predicated add of the address
// (4 instructions; the compiler's own lowering of the index form takes 6).
// Returns the byte offset of the final position, 8 * rank.
__device__ __forceinline__ unsigned node_rank_saddr(uint32_t a, unsigned long long q) {
  const uint32_t a0 = a;
  asm("{\n\t.reg .pred p;\n\t.reg .b64 k;\n\t"
      "ld.shared.u64 k, [%0+56];\n\tsetp.le.u64 p, k, %1;\n\t@p add.u32 %0, %0, 64;\n\t"
      "ld.shared.u64 k, [%0+24];\n\tsetp.le.u64 p, k, %1;\n\t@p add.u32 %0, %0, 32;\n\t"
      "ld.shared.u64 k, [%0+8];\n\tsetp.le.u64 p, k, %1;\n\t@p add.u32 %0, %0, 16;\n\t"
      "ld.shared.u64 k, [%0];\n\tsetp.le.u64 p, k, %1;\n\t@p add.u32 %0, %0, 8;\n\t}"
      : "+r"(a)
      : "l"(q));
  return a - a0;
}

// Rank of q over the 4-lane group's line quarter: lane j holds keys 4j..4j+3;
// `nvalid` of them (per lane) are keys. Listing 1's popcnt(cmpge(q, node)).
__device__ __forceinline__ unsigned group_rank(unsigned long long q, const unsigned long long (&w)[4], unsigned nvalid,
                                               unsigned gmask) {
  unsigned r = 0;
#pragma unroll
  for (int t = 0; t < 4; ++t) r += __popc(__ballot_sync(kFull, (t < static_cast<int>(nvalid)) && q >= w[t]) & gmask);
  return r;
}

template <int VB>
struct LeafFmt {
  static constexpr int kL = VB == 1 ? 14 : VB == 2 ? 12 : 8;  // keys per leaf line
  static constexpr int kValueLane = (kL * 8) / 32;             // lane holding the next hops
  static constexpr int kValueOff = kL * 8 - kValueLane * 32;   // their byte offset in that lane's 32 B
};

template <int VB>
__device__ __forceinline__ unsigned leaf_value(const unsigned long long (&w)[4], unsigned ord) {
  const unsigned o = LeafFmt<VB>::kValueOff + ord * VB;  // byte offset within the lane's quarter
  const unsigned wi = o >> 3;
  const unsigned long long x = wi == 0 ? w[0] : wi == 1 ? w[1] : wi == 2 ? w[2] : w[3];
  const unsigned long long v = x >> ((o & 7u) * 8u);
  return VB == 1 ? static_cast<unsigned>(v & 0xFFu) : VB == 2 ? static_cast<unsigned>(v & 0xFFFFu)
                                                              : static_cast<unsigned>(v & 0xFFFFFFFFu);
}

template <int VB>
__device__ __forceinline__ void store_group(const LookupParams& p, unsigned long long q0, const unsigned (&v)[4]) {
  if (q0 + 3 < p.n) {
    if constexpr (VB == 1) {
      const unsigned x = v[0] | (v[1] << 8) | (v[2] << 16) | (v[3] << 24);
      asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p.out + q0), "r"(x));
    } else if constexpr (VB == 2) {
      const unsigned long long x = static_cast<unsigned long long>(v[0] | (v[1] << 16)) |
                                   (static_cast<unsigned long long>(v[2] | (v[3] << 16)) << 32);
      asm volatile("st.global.cs.u64 [%0], %1;" ::"l"(p.out + 2 * q0), "l"(x));
    } else {
      asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p.out + 4 * q0), "r"(v[0]), "r"(v[1]),
                   "r"(v[2]), "r"(v[3]));
    }
  } else {
#pragma unroll
    for (int s = 0; s < 4; ++s) {
      if (q0 + s >= p.n) break;
      if constexpr (VB == 1) p.out[q0 + s] = static_cast<unsigned char>(v[s]);
      else if constexpr (VB == 2) reinterpret_cast<unsigned short*>(p.out)[q0 + s] = static_cast<unsigned short>(v[s]);
      else reinterpret_cast<unsigned*>(p.out)[q0 + s] = v[s];
    }
  }
}

// Leaf search in the shared-memory leaf image (small trees): the same 4-probe
// binary search as an internal node over the line's 16 words, with slots past
// kL (the next-hop words) counting as greater than every query; then the next
// hop of ordinal rank - 1 read from the line's value bytes.
template <int VB>
__device__ __forceinline__ unsigned leaf_search_smem(const unsigned long long* lf, unsigned long long q,
                                                     unsigned& rank) {
  constexpr unsigned kL = LeafFmt<VB>::kL;
  auto le = [&](unsigned slot) { return slot < kL && lf[slot] <= q; };
  unsigned c = le(7) ? 8u : 0u;
  c |= le(c | 3u) ? 4u : 0u;
  c |= le(c | 1u) ? 2u : 0u;
  c |= le(c) ? 1u : 0u;
  rank = c;
  const unsigned ord = c ? c - 1u : 0u;
  const unsigned char* vals = reinterpret_cast<const unsigned char*>(lf + kL);
  if constexpr (VB == 1) return vals[ord];
  else if constexpr (VB == 2) return reinterpret_cast<const unsigned short*>(vals)[ord];
  else return reinterpret_cast<const unsigned*>(vals)[ord];
}

// TILES consecutive 32-query tiles per warp iteration (lane L owns query L of
// each); MINB > 0 caps registers so that MINB CTAs of THREADS threads fit an SM.
// CHECKED adds bounds checks on every node index and leaf rank: a violation
// (only possible with a corrupted tree) is clamped, never read out of bounds,
// and reported through p.err — the fail-loudly mode the tests run.
// LEAFS (small trees, layout.hpp leaf image): every level including the leaves
// is staged in shared memory and each thread finishes its own query there — no
// L2 line loads and no cross-lane traffic.
// TEXL: the internal L2 levels are read through the texture pipe (p.tex).
template <int DEPTH, int VB, int TILES, int THREADS, int MINB, bool CHECKED, int INPUT = kInAddr, bool LEAFS = false,
          bool TEXL = false>
__global__ void __launch_bounds__(THREADS, MINB) lpm6_lookup_kernel(const LookupParams p) {
  using F = LeafFmt<VB>;
  unsigned violations = 0;
  unsigned long long visits = 0;  // CHECKED: lines visited by this lane's own queries
  constexpr int NS = 4 * TILES;  // queries in flight per 4-lane group
  extern __shared__ __align__(128) unsigned long long s_lines[];
  __shared__ __align__(8) uint64_t s_bar;

  if (p.smem_bytes > 0) {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      mbar_arrive_expect_tx(&s_bar, p.smem_bytes);
      constexpr uint32_t kChunk = 32768;
      for (uint32_t off = 0; off < p.smem_bytes; off += kChunk) {
        const uint32_t sz = min(kChunk, p.smem_bytes - off);
        bulk_g2s(reinterpret_cast<char*>(s_lines) + off, reinterpret_cast<const char*>(p.image) + off, sz,
                 &s_bar);
      }
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);
  }

  const unsigned lane = threadIdx.x & 31u;
  const unsigned j = lane & 3u;                 // lane within the 4-lane group
  const unsigned gbase = lane & ~3u;            // first lane (= first query) of the group
  const unsigned gmask = 0xFu << gbase;
  const unsigned long long warp0 = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pol_stream = policy_evict_first();
  const unsigned TA = p.smem_levels;
  const uint32_t s_base = smem_u32(s_lines);  // shared-space byte address of the image
  const unsigned leaf_valid = (F::kL - 4 * static_cast<int>(j)) < 0 ? 0u
                              : (F::kL - 4 * static_cast<int>(j)) > 4 ? 4u
                                                                      : static_cast<unsigned>(F::kL - 4 * j);

  // Top 64 bits of query address (st, t, lane); the address stream comes from
  // DRAM, so each warp loads the next tile's addresses one iteration ahead.
  auto load_key = [&](unsigned long long st_, int t) -> unsigned long long {
    const unsigned long long qi = (st_ * TILES + t) * 32ull + lane;
    unsigned long long k = 0;
    if (qi < p.n) {
      if constexpr (INPUT == kInKey || INPUT == kInKeyOrd) {
        k = ld_stream<unsigned long long>(p.keys + qi, pol_stream);
      } else if constexpr (INPUT == kInPacket) {
        k = load_dst_key(p.pkts + qi * p.pkt_stride, p.pkt_off, p.pkt_align, pol_stream);
      } else {
        const uint4 a = ld_stream_v4(p.addrs + qi, pol_stream);
        k = (static_cast<unsigned long long>(a.w) << 32) | a.z;
      }
    }
    return k;
  };
  unsigned long long next_key[TILES];
#pragma unroll
  for (int t = 0; t < TILES; ++t) next_key[t] = load_key(warp0, t);

  for (unsigned long long st = warp0; st * (32ull * TILES) < p.n; st += nwarps) {
    unsigned long long key[TILES];
    unsigned node[TILES];
#pragma unroll
    for (int t = 0; t < TILES; ++t) {
      key[t] = next_key[t] > kMaxQueryKey ? kMaxQueryKey : next_key[t];  // types.hpp:25
      node[t] = 0;
      next_key[t] = load_key(st + nwarps, t);  // prefetch; consumed next iteration
    }

    // Phase A: this thread's own queries through the shared-memory levels.
#pragma unroll
    for (int l = 0; l < DEPTH; ++l)
      if (static_cast<unsigned>(l) < TA) {
#pragma unroll
        for (int t = 0; t < TILES; ++t) {
          if (l == 0) {
            // Root from the kernel-parameter constant bank: all lanes start at the
            // same node, so the probes are (nearly) uniform LDCs and keep the
            // shared-memory data pipe free for the deeper levels.
            const unsigned long long q = key[t];
            unsigned c = (p.root[7] <= q) ? 8u : 0u;
            c |= (p.root[c | 3u] <= q) ? 4u : 0u;
            c |= (p.root[c | 1u] <= q) ? 2u : 0u;
            c |= (p.root[c] <= q) ? 1u : 0u;
            node[t] = c;
          } else {
            const uint32_t lvl = s_base + static_cast<uint32_t>(p.level_start[l] >> 4) * 120u;
            node[t] = node[t] * 16u + (node_rank_saddr(lvl + node[t] * 120u, key[t]) >> 3);
          }
          if (CHECKED && node[t] >= p.level_nodes[l + 1]) {
            violations |= 1u;
            node[t] = 0;
          }
          if (CHECKED && (st * TILES + t) * 32ull + lane < p.n) ++visits;
        }
      }

    if constexpr (LEAFS) {
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        const unsigned long long qi = (st * TILES + t) * 32ull + lane;
        if (CHECKED && node[t] >= p.level_nodes[DEPTH]) {
          violations |= 1u;
          node[t] = 0;
        }
        unsigned rank;
        const unsigned v = leaf_search_smem<VB>(s_lines + p.leaf_image_off + node[t] * kLeafImageStride, key[t], rank);
        if (CHECKED && rank == 0) violations |= 4u;
        if (CHECKED && qi < p.n) ++visits;
        if (qi < p.n) {
          if constexpr (VB == 1) asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p.out + qi), "h"((unsigned short)v));
          else if constexpr (VB == 2) asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p.out + 2 * qi), "h"((unsigned short)v));
          else asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p.out + 4 * qi), "r"(v));
        }
      }
      continue;
    }

    // Phase B: the group's queries, one 128-byte line per query per level.
    unsigned long long qk[NS];
    unsigned nd[NS];
#pragma unroll
    for (int t = 0; t < TILES; ++t)
#pragma unroll
      for (int s = 0; s < 4; ++s) {
        qk[4 * t + s] = __shfl_sync(kFull, key[t], s, 4);
        nd[4 * t + s] = __shfl_sync(kFull, node[t], s, 4);
      }
    unsigned long long w[NS][4];
    // Internal L2 levels [TA, DEPTH): a runtime-count loop (one back-edge per
    // level instead of a compare-and-branch per possible level), then the leaf.
#pragma unroll
    for (int li = 0; li < DEPTH; ++li) {
      // Fully unrolled (static register indexing, scheduled across levels); the
      // level index is TA-relative so the common TA == DEPTH case skips it with
      // one uniform branch.
      if (li >= DEPTH - static_cast<int>(TA)) break;
      const unsigned l = TA + li;
      // 32-bit word offsets (the layout keeps the array below 2^32 words).
      const unsigned base_w = static_cast<unsigned>(p.level_start[l]) + j * 4u;
      if (CHECKED) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (nd[s] >= p.level_nodes[l]) {
            violations |= 2u;
            nd[s] = 0;
          }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        // Internal L2 levels through the texture pipe, leaves through the LSU:
        // the two pipes of L1TEX share the load, which helps the deep trees (C2:
        // +8 %); leaves through the texture pipe lose on L2-missing workloads
        // (C1 -17 %), so they stay on the LSU path.
        if (TEXL)
          tex_line_quarter(p.tex, (base_w + nd[s] * 16u) >> 1, w[s]);
        else
          ld_line_quarter(p.lines + (base_w + nd[s] * 16u), w[s]);
      }
      if (CHECKED) {  // one line per query: the lane owning query (t, j) counts it
#pragma unroll
        for (int t = 0; t < TILES; ++t)
          if ((st * TILES + t) * 32ull + lane < p.n) ++visits;
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) nd[s] = nd[s] * 16u + group_rank(qk[s], w[s], 4u, gmask);
    }
    unsigned leafn[INPUT == kInKeyOrd ? NS : 1];  // kInKeyOrd: leaf node of each query
    {  // the leaf line: ordinal = rank - 1
      const unsigned base_w = static_cast<unsigned>(p.level_start[DEPTH]) + j * 4u;
      if (CHECKED) {
#pragma unroll
        for (int s = 0; s < NS; ++s)
          if (nd[s] >= p.level_nodes[DEPTH]) {
            violations |= 2u;
            nd[s] = 0;
          }
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) ld_line_quarter(p.lines + (base_w + nd[s] * 16u), w[s]);
      if constexpr (INPUT == kInKeyOrd) {
#pragma unroll
        for (int s = 0; s < NS; ++s) leafn[s] = nd[s];
      }
      if (CHECKED) {
#pragma unroll
        for (int t = 0; t < TILES; ++t)
          if ((st * TILES + t) * 32ull + lane < p.n) ++visits;
      }
#pragma unroll
      for (int s = 0; s < NS; ++s) {
        const unsigned r = group_rank(qk[s], w[s], leaf_valid, gmask);
        if (CHECKED && r == 0) violations |= 4u;
        nd[s] = CHECKED && r == 0 ? 0u : r - 1u;
      }
    }

    if constexpr (INPUT == kInKeyOrd) {  // lane j stores the ordinal of its own query (4t + j of the group)
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        unsigned o = leafn[4 * t] * F::kL + nd[4 * t];
#pragma unroll
        for (int s = 1; s < 4; ++s) o = j == static_cast<unsigned>(s) ? leafn[4 * t + s] * F::kL + nd[4 * t + s] : o;
        const unsigned long long qi = (st * TILES + t) * 32ull + lane;
        if (qi < p.n) asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p.ord + qi), "r"(o));
      }
      if (p.out == nullptr) continue;  // ordinals only
    }
    // Leaf values: the value lane extracts the group's next hops and stores them.
    if (j == static_cast<unsigned>(F::kValueLane)) {
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        unsigned v[4];
#pragma unroll
        for (int s = 0; s < 4; ++s) v[s] = leaf_value<VB>(w[4 * t + s], nd[4 * t + s]);
        store_group<VB>(p, (st * TILES + t) * 32ull + gbase, v);
      }
    }
  }
  if (CHECKED) {
    if (violations) atomicOr(p.err, violations);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) visits += __shfl_xor_sync(kFull, visits, o);
    if (lane == 0 && visits) atomicAdd(reinterpret_cast<unsigned long long*>(p.err + 2), visits);
  }
}

using KernelFn = void (*)(const LookupParams);

// Instantiated shapes: (queries per lane, min CTAs per SM) for every depth and
// value width; the tuning grid below is measured by bench.py --sweep.
template <int VB>
KernelFn pick_depth_texl(int depth) {
  switch (depth) {
    case 2: return lpm6_lookup_kernel<2, VB, 1, 1024, 1, false, kInAddr, false, true>;
    case 3: return lpm6_lookup_kernel<3, VB, 1, 1024, 1, false, kInAddr, false, true>;
    case 4: return lpm6_lookup_kernel<4, VB, 1, 1024, 1, false, kInAddr, false, true>;
    case 5: return lpm6_lookup_kernel<5, VB, 1, 1024, 1, false, kInAddr, false, true>;
    case 6: return lpm6_lookup_kernel<6, VB, 1, 1024, 1, false, kInAddr, false, true>;
    case 7: return lpm6_lookup_kernel<7, VB, 1, 1024, 1, false, kInAddr, false, true>;
    default: return nullptr;
  }
}

template <int VB, bool CHECKED>
KernelFn pick_depth_leafs(int depth) {
  switch (depth) {
    case 0: return lpm6_lookup_kernel<0, VB, 1, 1024, 1, CHECKED, kInAddr, true>;
    case 1: return lpm6_lookup_kernel<1, VB, 1, 1024, 1, CHECKED, kInAddr, true>;
    case 2: return lpm6_lookup_kernel<2, VB, 1, 1024, 1, CHECKED, kInAddr, true>;
    case 3: return lpm6_lookup_kernel<3, VB, 1, 1024, 1, CHECKED, kInAddr, true>;
    default: return nullptr;
  }
}

template <int VB, int TILES, int THREADS, int MINB, bool CHECKED, int INPUT>
KernelFn pick_depth(int depth) {
  switch (depth) {
    case 0: return lpm6_lookup_kernel<0, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 1: return lpm6_lookup_kernel<1, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 2: return lpm6_lookup_kernel<2, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 3: return lpm6_lookup_kernel<3, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 4: return lpm6_lookup_kernel<4, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 5: return lpm6_lookup_kernel<5, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 6: return lpm6_lookup_kernel<6, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    case 7: return lpm6_lookup_kernel<7, VB, TILES, THREADS, MINB, CHECKED, INPUT>;
    default: return nullptr;
  }
}

template <int TILES, int THREADS, int MINB, bool CHECKED = false, int INPUT = kInAddr>
KernelFn pick_vb(int vb, int depth) {
  switch (vb) {
    case 1: return pick_depth<1, TILES, THREADS, MINB, CHECKED, INPUT>(depth);
    case 2: return pick_depth<2, TILES, THREADS, MINB, CHECKED, INPUT>(depth);
    case 4: return pick_depth<4, TILES, THREADS, MINB, CHECKED, INPUT>(depth);
    default: return nullptr;
  }
}

// Instantiated shapes (queries per lane, threads per CTA, min CTAs per SM);
// bench.py --sweep measures them. The checked variant exists for the default shape.
KernelFn pick_kernel(int vb, int depth, int tiles, int threads, int minb, bool checked = false,
                     int input = kInAddr, bool leafs = false, bool texl = false) {
  if (texl) {  // internal L2 levels via the texture pipe: address input, default shape, unchecked
    if (leafs || checked || input != kInAddr || tiles != 1 || threads != 1024 || minb != 1) return nullptr;
    switch (vb) {
      case 1: return pick_depth_texl<1>(depth);
      case 2: return pick_depth_texl<2>(depth);
      case 4: return pick_depth_texl<4>(depth);
      default: return nullptr;
    }
  }
  if (leafs) {  // leaf image: address input, default shape, depth <= kMaxLeafImageDepth
    if (input != kInAddr || tiles != 1 || threads != 1024 || minb != 1) return nullptr;
    switch (vb) {
      case 1: return checked ? pick_depth_leafs<1, true>(depth) : pick_depth_leafs<1, false>(depth);
      case 2: return checked ? pick_depth_leafs<2, true>(depth) : pick_depth_leafs<2, false>(depth);
      case 4: return checked ? pick_depth_leafs<4, true>(depth) : pick_depth_leafs<4, false>(depth);
      default: return nullptr;
    }
  }
  if (input != kInAddr) {  // key / packet input: the default shape, unchecked and checked
    if (tiles != 1 || threads != 1024 || minb != 1) return nullptr;
    if (input == kInKey)
      return checked ? pick_vb<1, 1024, 1, true, kInKey>(vb, depth) : pick_vb<1, 1024, 1, false, kInKey>(vb, depth);
    if (input == kInPacket)
      return checked ? pick_vb<1, 1024, 1, true, kInPacket>(vb, depth)
                     : pick_vb<1, 1024, 1, false, kInPacket>(vb, depth);
    if (input == kInKeyOrd)
      return checked ? pick_vb<1, 1024, 1, true, kInKeyOrd>(vb, depth)
                     : pick_vb<1, 1024, 1, false, kInKeyOrd>(vb, depth);
    return nullptr;
  }
  if (checked) return (tiles == 1 && threads == 1024 && minb == 1) ? pick_vb<1, 1024, 1, true>(vb, depth) : nullptr;
  if (tiles == 1 && threads == 256 && minb == 0) return pick_vb<1, 256, 0>(vb, depth);
  if (tiles == 1 && threads == 256 && minb == 4) return pick_vb<1, 256, 4>(vb, depth);
  if (tiles == 2 && threads == 256 && minb == 0) return pick_vb<2, 256, 0>(vb, depth);
  if (tiles == 1 && threads == 512 && minb == 2) return pick_vb<1, 512, 2>(vb, depth);
  if (tiles == 1 && threads == 1024 && minb == 1) return pick_vb<1, 1024, 1>(vb, depth);
  return nullptr;
}

// ---- query generator kernel ----------------------------------------------------

__global__ void lpm6_querygen_kernel(const QuerySpec spec, unsigned long long first, unsigned long long n,
                                     uint4* out) {
  for (unsigned long long i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    unsigned long long lo, hi;
    gen_query(spec, first + i, reinterpret_cast<uint64_t*>(&lo), reinterpret_cast<uint64_t*>(&hi));
    out[i] = make_uint4(static_cast<unsigned>(lo), static_cast<unsigned>(lo >> 32), static_cast<unsigned>(hi),
                        static_cast<unsigned>(hi >> 32));
  }
}

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    check_cuda(cudaGetDevice(&prev), "cudaGetDevice");
    if (prev != dev) check_cuda(cudaSetDevice(dev), "cudaSetDevice");
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

}  // namespace

// ---- FIB handle ------------------------------------------------------------------

struct HostPipeline {
  static constexpr int kStreams = 3;
  cudaStream_t streams[kStreams] = {};
  void* d_in[kStreams] = {};
  void* d_out[kStreams] = {};
  cudaEvent_t start = nullptr;
  unsigned long long chunk = 0;
};

// Kernel choice, occupancy and the dynamic-smem attribute for one input format
// and checked flag: resolved on the first launch, reused until the kernel
// config changes (the launch path then does no driver queries).
struct LaunchPlan {
  bool valid = false;
  void (*fn)(const LookupParams) = nullptr;
  int per_sm = 0;
};

struct lpm6cu_fib {
  int device = 0;
  lpm6cu_geometry g{};
  unsigned long long* d_lines = nullptr;
  unsigned int* d_err = nullptr;  // non-null: checked mode; [0] violation bits, [2..3] u64 node visits
  bool owns = true;
  lpm6cu_kernel_config cfg{};  // resolved
  int num_sms = 0;
  size_t max_smem_optin = 0;
  std::mutex host_mu;
  std::unique_ptr<HostPipeline> pipe;
  std::mutex plan_mu;
  LaunchPlan plans[4][2];  // [input format][checked]
  unsigned long long root[16] = {};  // host copy of the root line (kernel parameter)
  cudaTextureObject_t tex = 0;       // texture object over the line array
  bool root_ready = false;

  void invalidate_plans() {
    std::lock_guard<std::mutex> lk(plan_mu);
    for (auto& row : plans)
      for (auto& pl : row) pl = LaunchPlan{};
  }

  ~lpm6cu_fib() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    if (pipe) {
      for (int i = 0; i < HostPipeline::kStreams; ++i) {
        if (pipe->streams[i]) cudaStreamDestroy(pipe->streams[i]);
        if (pipe->d_in[i]) cudaFree(pipe->d_in[i]);
        if (pipe->d_out[i]) cudaFree(pipe->d_out[i]);
      }
      if (pipe->start) cudaEventDestroy(pipe->start);
    }
    if (tex) cudaDestroyTextureObject(tex);
    if (owns && d_lines) cudaFree(d_lines);
    if (d_err) cudaFree(d_err);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct lpm6cu_querygen {
  int device = 0;
  QuerySpec spec{};
  void* d_top = nullptr;
  void* d_len = nullptr;
  void* d_cdf = nullptr;
  void* d_perm = nullptr;
  ~lpm6cu_querygen() {
    int prev = -1;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (void* p : {d_top, d_len, d_cdf, d_perm})
      if (p) cudaFree(p);
    if (prev >= 0) cudaSetDevice(prev);
  }
};

namespace {

// Bytes of the shared-memory image for `levels` levels (layout.hpp image_bytes).
// Bytes of the shared-memory image for `levels` levels (layout.hpp image_bytes);
// levels = depth + 1 adds the leaf image of a small tree (leaf_image_bytes).
unsigned long long image_bytes_of(const lpm6cu_geometry& g, unsigned levels) {
  if (levels > g.depth)
    return image_bytes_of(g, g.depth) + (g.leaf_nodes * kLeafImageStride * 8 + 15) / 16 * 16;
  return (g.level_start[levels] / kLineWords * kNodeKeys * 8 + 15) / 16 * 16;
}

// Shape of the default kernel (the only one with the leaf-image variant).
bool default_shape(const lpm6cu_kernel_config& c) {
  return c.queries_per_lane == 1 && c.threads_per_cta == 1024 && c.min_ctas_per_sm == 1;
}

// Resolve automatic kernel settings against the device and the tree.
void resolve_config(lpm6cu_fib* f, const lpm6cu_kernel_config* req) {
  lpm6cu_kernel_config c{};
  if (req) c = *req;
  if (c.lanes_per_query == 0) c.lanes_per_query = 4;
  if (c.lanes_per_query != 4) throw Error(Errc::InvalidArgument, "lanes_per_query must be 4");
  // Default shape (measured, bench.py --sweep): one 1024-thread CTA per SM, so a
  // single shared-memory image per SM serves 32 warps and can be as large as
  // the opt-in limit (227 KiB) — all four internal levels of the 200K FIB.
  if (c.threads_per_cta == 0) c.threads_per_cta = 1024;
  if (c.queries_per_lane == 0) c.queries_per_lane = 1;
  if (c.min_ctas_per_sm == 0 && c.threads_per_cta == 512) c.min_ctas_per_sm = 2;
  if (c.min_ctas_per_sm == 0 && c.threads_per_cta == 1024) c.min_ctas_per_sm = 1;
  if (!pick_kernel(1, 0, static_cast<int>(c.queries_per_lane), static_cast<int>(c.threads_per_cta),
                   static_cast<int>(c.min_ctas_per_sm)))
    throw Error(Errc::InvalidArgument, "no kernel for queries_per_lane=" + std::to_string(c.queries_per_lane) +
                                           " threads_per_cta=" + std::to_string(c.threads_per_cta) +
                                           " min_ctas_per_sm=" + std::to_string(c.min_ctas_per_sm));
  const unsigned depth = f->g.depth;
  const size_t budget = f->max_smem_optin;
  // Phase A: imaged internal levels; depth + 1 = the leaves too (small trees, default shape).
  const unsigned tmax = f->g.leaf_image && default_shape(c) && depth <= kMaxLeafImageDepth
                            ? depth + 1
                            : std::min<unsigned>(depth, f->g.image_levels);
  if (req == nullptr || req->smem_levels == 0xFF) {
    // Auto: the deepest prefix of internal levels whose image fits the shared
    // memory one CTA may use; with 256-thread CTAs keep >= 4 CTAs per SM.
    const unsigned long long cap = c.threads_per_cta >= 1024 ? budget
                                   : c.threads_per_cta == 512 ? budget / 2 - 1024 : 48 * 1024;
    unsigned t = 0;
    for (unsigned cand = 1; cand <= tmax; ++cand) {
      if (image_bytes_of(f->g, cand) > cap) break;
      t = cand;
    }
    c.smem_levels = t;
  }
  if (c.smem_levels > tmax) c.smem_levels = tmax;
  const unsigned long long staged = image_bytes_of(f->g, c.smem_levels);
  if (staged > budget)
    throw Error(Errc::InvalidArgument, "smem_levels=" + std::to_string(c.smem_levels) + " needs " +
                                           std::to_string(staged) + " B of shared memory");
  f->cfg = c;
  f->invalidate_plans();
}

bool leaf_image_mode(const lpm6cu_fib* f) { return f->cfg.smem_levels > f->g.depth; }

struct PacketInput {
  unsigned long long stride = 0;
  unsigned off = 0, align = 8;
};

// input: kInAddr (d_in = 16-byte addresses, configured shape), kInKey (8-byte
// keys) or kInPacket (frames described by pk); the last two use the default shape.
void launch_lookup(const lpm6cu_fib* f, const void* d_in, unsigned long long n, void* d_out, cudaStream_t stream,
                   int input = kInAddr, const PacketInput* pk = nullptr, unsigned* d_ord = nullptr) {
  if (n == 0) return;
  const bool dflt = input != kInAddr;
  const unsigned tiles = dflt ? 1 : f->cfg.queries_per_lane;
  const unsigned threads_cta = dflt ? 1024 : f->cfg.threads_per_cta;
  const unsigned minb = dflt ? 1 : f->cfg.min_ctas_per_sm;
  // Leaf-image mode serves address input; key / packet input uses the internal image only.
  const bool leafs = leaf_image_mode(f) && input == kInAddr;
  // Texture pipe for internal L2 levels when the tree has any (smem_levels < depth).
  const bool texl = f->tex && !leafs && input == kInAddr && f->d_err == nullptr && f->cfg.smem_levels < f->g.depth &&
                    tiles == 1 && threads_cta == 1024 && minb == 1 && f->g.depth >= 2;
  const unsigned smem_levels = leaf_image_mode(f) && !leafs ? f->g.depth : f->cfg.smem_levels;
  const size_t smem = image_bytes_of(f->g, smem_levels);
  const int threads = static_cast<int>(threads_cta);
  LaunchPlan plan;
  {
    auto* mf = const_cast<lpm6cu_fib*>(f);
    std::lock_guard<std::mutex> lk(mf->plan_mu);
    LaunchPlan& slot = mf->plans[input][f->d_err != nullptr ? 1 : 0];
    if (!slot.valid) {
      KernelFn fn = pick_kernel(static_cast<int>(f->g.value_bytes), static_cast<int>(f->g.depth),
                                static_cast<int>(tiles), threads, static_cast<int>(minb), f->d_err != nullptr, input,
                                leafs, texl);
      if (!fn) throw Error(Errc::InvalidArgument, "no kernel instantiated for this configuration");
      if (smem > 48 * 1024)
        check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
                   "cudaFuncSetAttribute");
      int per_sm = 0;
      check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem), "occupancy");
      if (per_sm < 1) throw Error(Errc::CudaError, "lookup kernel cannot be resident with this configuration");
      if (f->cfg.ctas_per_sm > 0) per_sm = std::min<int>(per_sm, static_cast<int>(f->cfg.ctas_per_sm));
      slot.fn = fn;
      slot.per_sm = per_sm;
      slot.valid = true;
    }
    plan = slot;
  }
  LookupParams p{};
  p.lines = f->d_lines;
  for (int l = 0; l < LPM6CU_MAX_LEVELS; ++l) p.level_start[l] = f->g.level_start[l];
  if (input == kInKey || input == kInKeyOrd) {
    p.keys = static_cast<const unsigned long long*>(d_in);
    p.ord = d_ord;
  } else if (input == kInPacket) {
    p.pkts = static_cast<const unsigned char*>(d_in);
    p.pkt_stride = pk->stride;
    p.pkt_off = pk->off;
    p.pkt_align = pk->align;
  } else {
    p.addrs = static_cast<const uint4*>(d_in);
  }
  p.out = static_cast<unsigned char*>(d_out);
  p.n = n;
  p.smem_bytes = static_cast<unsigned>(smem);
  p.smem_levels = std::min<unsigned>(smem_levels, f->g.depth);
  p.leaf_image_off = static_cast<unsigned>(image_bytes_of(f->g, f->g.depth) / 8);
  p.image = f->d_lines + f->g.image_start;
  for (int l = 0; l < LPM6CU_MAX_LEVELS; ++l) p.level_nodes[l] = f->g.level_nodes[l];
  p.err = f->d_err;
  std::memcpy(p.root, f->root, sizeof p.root);
  p.tex = f->tex;
  const unsigned long long ntiles = (n + 32ull * tiles - 1) / (32ull * tiles);
  const unsigned long long warps_per_cta = threads / 32;
  unsigned long long grid = static_cast<unsigned long long>(f->num_sms) * plan.per_sm;
  grid = std::min(grid, (ntiles + warps_per_cta - 1) / warps_per_cta);
  plan.fn<<<static_cast<unsigned>(grid), threads, smem, stream>>>(p);
  check_cuda(cudaGetLastError(), "lookup launch");
}

lpm6cu_fib* new_fib(int device, const lpm6cu_geometry* g) {
  if (!g) throw Error(Errc::InvalidArgument, "geometry is NULL");
  if (g->k != kNodeKeys || g->b != kNodeKeys + 1) throw Error(Errc::InvalidArgument, "the kernels take k = 15, b = 16");
  if (g->leaf_keys != leaf_keys_for(g->value_bytes)) throw Error(Errc::InvalidArgument, "leaf_keys mismatch");
  if (g->depth > kMaxKernelDepth) throw Error(Errc::InvalidArgument, "tree depth above 7");
  if (g->value_bytes != 1 && g->value_bytes != 2 && g->value_bytes != 4)
    throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
  // The geometry must describe a line array that holds what the kernels will read.
  if (g->image_levels > g->depth || g->level_start[g->depth] + g->leaf_nodes * kLineWords > g->image_start)
    throw Error(Errc::InvalidArgument, "inconsistent geometry (levels / image offset)");
  const unsigned imaged = g->leaf_image ? g->depth + 1 : g->image_levels;
  if (g->image_start + image_bytes_of(*g, imaged) / 8 > g->total_words)
    throw Error(Errc::InvalidArgument, "inconsistent geometry (image past total_words)");
  if (g->leaf_image && (g->image_levels != g->depth || image_bytes_of(*g, g->depth + 1) > 232448 - 1024))
    throw Error(Errc::InvalidArgument, "inconsistent geometry (leaf image)");
  int ndev = 0;
  check_cuda(cudaGetDeviceCount(&ndev), "cudaGetDeviceCount");
  if (device < 0 || device >= ndev) throw Error(Errc::CudaError, "no CUDA device " + std::to_string(device));
  auto f = std::make_unique<lpm6cu_fib>();
  f->device = device;
  f->g = *g;
  check_cuda(cudaDeviceGetAttribute(&f->num_sms, cudaDevAttrMultiProcessorCount, device), "attr");
  int optin = 0;
  check_cuda(cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device), "attr");
  f->max_smem_optin = static_cast<size_t>(optin) - 1024;  // static smem + slack
  resolve_config(f.get(), nullptr);
  return f.release();
}

// The root line as kernel parameters (LookupParams::root); the line array must
// hold the tree when the handle is created.
void load_root(lpm6cu_fib* f) {
  DeviceGuard dg(f->device);
  // Texture object over the line array for the internal L2 levels (16-byte int4
  // texels). Not available (alignment, size limits): those levels use LSU loads.
  if (f->g.depth >= 1) {
    int max_w = 0, align = 0;
    cudaDeviceGetAttribute(&max_w, cudaDevAttrMaxTexture1DLinearWidth, f->device);
    cudaDeviceGetAttribute(&align, cudaDevAttrTextureAlignment, f->device);
    if (f->g.total_words / 2 <= static_cast<unsigned long long>(max_w) && align > 0 &&
        reinterpret_cast<uintptr_t>(f->d_lines) % static_cast<uintptr_t>(align) == 0) {
      cudaResourceDesc rd{};
      rd.resType = cudaResourceTypeLinear;
      rd.res.linear.devPtr = f->d_lines;
      rd.res.linear.desc = cudaCreateChannelDesc<int4>();
      rd.res.linear.sizeInBytes = f->g.total_words * 8;
      cudaTextureDesc td{};
      td.readMode = cudaReadModeElementType;
      if (cudaCreateTextureObject(&f->tex, &rd, &td, nullptr) != cudaSuccess) {
        cudaGetLastError();
        f->tex = 0;
      }
    }
  }
  check_cuda(cudaMemcpy(f->root, f->d_lines, sizeof f->root, cudaMemcpyDeviceToHost), "read root line");
  f->root_ready = true;
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

void lookup_host(lpm6cu_fib* f, const void* addrs, unsigned long long n, void* out, cudaStream_t user) {
  std::lock_guard<std::mutex> lk(f->host_mu);
  const unsigned vb = f->g.value_bytes;
  if (!f->pipe) {
    auto pipe = std::make_unique<HostPipeline>();
    pipe->chunk = 1ull << 23;  // 8M addresses = 128 MiB per staging buffer
    for (int i = 0; i < HostPipeline::kStreams; ++i) {
      check_cuda(cudaStreamCreateWithFlags(&pipe->streams[i], cudaStreamNonBlocking), "stream");
      check_cuda(cudaMalloc(&pipe->d_in[i], pipe->chunk * 16), "cudaMalloc staging");
      check_cuda(cudaMalloc(&pipe->d_out[i], pipe->chunk * 4), "cudaMalloc staging");
    }
    check_cuda(cudaEventCreateWithFlags(&pipe->start, cudaEventDisableTiming), "event");
    f->pipe = std::move(pipe);
  }
  HostPipeline& pp = *f->pipe;
  check_cuda(cudaEventRecord(pp.start, user), "event record");
  for (int i = 0; i < HostPipeline::kStreams; ++i)
    check_cuda(cudaStreamWaitEvent(pp.streams[i], pp.start, 0), "stream wait");
  const auto* src = static_cast<const unsigned char*>(addrs);
  auto* dst = static_cast<unsigned char*>(out);
  int s = 0;
  for (unsigned long long off = 0; off < n; off += pp.chunk, s = (s + 1) % HostPipeline::kStreams) {
    const unsigned long long m = std::min(pp.chunk, n - off);
    check_cuda(cudaMemcpyAsync(pp.d_in[s], src + off * 16, m * 16, cudaMemcpyHostToDevice, pp.streams[s]), "H2D");
    launch_lookup(f, pp.d_in[s], m, pp.d_out[s], pp.streams[s]);
    check_cuda(cudaMemcpyAsync(dst + off * vb, pp.d_out[s], m * vb, cudaMemcpyDeviceToHost, pp.streams[s]), "D2H");
  }
  for (int i = 0; i < HostPipeline::kStreams; ++i) check_cuda(cudaStreamSynchronize(pp.streams[i]), "sync");
}

}  // namespace

extern "C" {

int lpm6cu_fib_create(int device, const lpm6cu_geometry* g, const uint64_t* lines, lpm6cu_fib** out) {
  return guard([&] {
    if (!lines || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, g));
    const size_t bytes = g->total_words * 8;
    check_cuda(cudaMalloc(&f->d_lines, bytes), "cudaMalloc lines");
    check_cuda(cudaMemcpy(f->d_lines, lines, bytes, cudaMemcpyHostToDevice), "copy lines");
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_fib_wrap_device(int device, const lpm6cu_geometry* g, const void* d_lines, lpm6cu_fib** out) {
  return guard([&] {
    if (!d_lines || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    if (reinterpret_cast<uintptr_t>(d_lines) % 128 != 0)
      throw Error(Errc::InvalidArgument, "device lines must be 128-byte aligned");
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, g));
    f->d_lines = static_cast<unsigned long long*>(const_cast<void*>(d_lines));
    f->owns = false;
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_fib_adopt_device(int device, const lpm6cu_geometry* g, void* d_lines, lpm6cu_fib** out) {
  return guard([&] {
    if (!d_lines || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    if (reinterpret_cast<uintptr_t>(d_lines) % 128 != 0)
      throw Error(Errc::InvalidArgument, "device lines must be 128-byte aligned");
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, g));
    f->d_lines = static_cast<unsigned long long*>(d_lines);
    f->owns = true;
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_fib_build(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                     const lpm6cu_build_opts* opts, lpm6cu_fib** out) {
  return guard([&] {
    if (n > 0 && !rules) throw Error(Errc::InvalidArgument, "rules is NULL");
    Tree t = capi::build_device_tree(rules, n, default_nh, opts);
    lpm6cu_geometry g;
    capi::export_geometry(t.g, &g);
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, &g));
    check_cuda(cudaMalloc(&f->d_lines, t.lines.size() * 8), "cudaMalloc lines");
    check_cuda(cudaMemcpy(f->d_lines, t.lines.data(), t.lines.size() * 8, cudaMemcpyHostToDevice), "copy lines");
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_fib_copy_lines(const lpm6cu_fib* f, uint64_t* host_lines, uint64_t words) {
  return guard([&] {
    if (!f || !host_lines) throw Error(Errc::InvalidArgument, "NULL argument");
    if (words != f->g.total_words) throw Error(Errc::InvalidArgument, "words must equal geometry.total_words");
    DeviceGuard dg(f->device);
    check_cuda(cudaMemcpy(host_lines, f->d_lines, words * 8, cudaMemcpyDeviceToHost), "copy lines");
  });
}

int lpm6cu_fib_build_device(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                            const lpm6cu_build_opts* opts, void* stream, lpm6cu_fib** out) {
  return guard([&] {
    if (n > 0 && !rules) throw Error(Errc::InvalidArgument, "rules is NULL");
    if (!out) throw Error(Errc::InvalidArgument, "NULL out");
    DeviceGuard dg(device);
    lpm6cu_geometry g;
    void* lines = capi::device_build_tree(rules, n, default_nh, opts, static_cast<cudaStream_t>(stream), &g);
    std::unique_ptr<lpm6cu_fib> f;
    try {
      f.reset(new_fib(device, &g));
    } catch (...) {
      cudaFree(lines);
      throw;
    }
    f->d_lines = static_cast<unsigned long long*>(lines);
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_fib_geometry(const lpm6cu_fib* f, lpm6cu_geometry* g) {
  return guard([&] {
    if (!f || !g) throw Error(Errc::InvalidArgument, "NULL argument");
    *g = f->g;
  });
}

int lpm6cu_fib_device_lines(const lpm6cu_fib* f, const void** d_lines) {
  return guard([&] {
    if (!f || !d_lines) throw Error(Errc::InvalidArgument, "NULL argument");
    *d_lines = f->d_lines;
  });
}

int lpm6cu_fib_set_kernel_config(lpm6cu_fib* f, const lpm6cu_kernel_config* cfg) {
  return guard([&] {
    if (!f) throw Error(Errc::InvalidArgument, "NULL fib");
    resolve_config(f, cfg);
  });
}

int lpm6cu_fib_kernel_config(const lpm6cu_fib* f, lpm6cu_kernel_config* cfg) {
  return guard([&] {
    if (!f || !cfg) throw Error(Errc::InvalidArgument, "NULL argument");
    *cfg = f->cfg;
  });
}

void lpm6cu_fib_destroy(lpm6cu_fib* f) { delete f; }

int lpm6cu_fib_set_checked(lpm6cu_fib* f, int on) {
  return guard([&] {
    if (!f) throw Error(Errc::InvalidArgument, "NULL fib");
    DeviceGuard dg(f->device);
    if (on && !f->d_err) {
      check_cuda(cudaMalloc(&f->d_err, 4 * sizeof(unsigned)), "cudaMalloc err");
      check_cuda(cudaMemset(f->d_err, 0, 4 * sizeof(unsigned)), "memset err");
    } else if (!on && f->d_err) {
      check_cuda(cudaFree(f->d_err), "cudaFree err");
      f->d_err = nullptr;
    }
    f->invalidate_plans();
  });
}

int lpm6cu_fib_violations(lpm6cu_fib* f, uint32_t* bits, int reset) {
  return guard([&] {
    if (!f || !bits) throw Error(Errc::InvalidArgument, "NULL argument");
    *bits = 0;
    if (!f->d_err) return;
    DeviceGuard dg(f->device);
    unsigned v = 0;
    check_cuda(cudaMemcpy(&v, f->d_err, sizeof v, cudaMemcpyDeviceToHost), "read err");  // syncs the device
    *bits = v;
    if (reset) check_cuda(cudaMemset(f->d_err, 0, sizeof(unsigned)), "reset err");
  });
}

int lpm6cu_fib_node_visits(lpm6cu_fib* f, uint64_t* visits, int reset) {
  return guard([&] {
    if (!f || !visits) throw Error(Errc::InvalidArgument, "NULL argument");
    *visits = 0;
    if (!f->d_err) return;
    DeviceGuard dg(f->device);
    unsigned long long v = 0;
    check_cuda(cudaMemcpy(&v, f->d_err + 2, sizeof v, cudaMemcpyDeviceToHost), "read visits");
    *visits = v;
    if (reset) check_cuda(cudaMemset(f->d_err + 2, 0, sizeof v), "reset visits");
  });
}

int lpm6cu_lookup_batch(const lpm6cu_fib* fib, const void* addrs, uint64_t n, void* out, void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!addrs || !out) throw Error(Errc::InvalidArgument, "NULL buffer");
    DeviceGuard dg(fib->device);
    const bool da = is_device_ptr(addrs), dout = is_device_ptr(out);
    if (da != dout)
      throw Error(Errc::InvalidArgument, "addresses and results must both be device or both be host memory");
    if (reinterpret_cast<uintptr_t>(addrs) % 16 != 0)
      throw Error(Errc::InvalidArgument, "addresses must be 16-byte aligned");
    if (da)
      launch_lookup(fib, addrs, n, out, static_cast<cudaStream_t>(stream));
    else
      lookup_host(const_cast<lpm6cu_fib*>(fib), addrs, n, out, static_cast<cudaStream_t>(stream));
  });
}

int lpm6cu_lookup_keys(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, void* out, void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!keys || !out) throw Error(Errc::InvalidArgument, "NULL buffer");
    DeviceGuard dg(fib->device);
    if (!is_device_ptr(keys) || !is_device_ptr(out))
      throw Error(Errc::InvalidArgument, "lpm6cu_lookup_keys takes device buffers");
    if (reinterpret_cast<uintptr_t>(keys) % 8 != 0) throw Error(Errc::InvalidArgument, "keys must be 8-byte aligned");
    launch_lookup(fib, keys, n, out, static_cast<cudaStream_t>(stream), kInKey);
  });
}

int lpm6cu_search_batch(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, uint32_t* ordinals, void* next_hops,
                        void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!keys || !ordinals) throw Error(Errc::InvalidArgument, "NULL buffer");
    DeviceGuard dg(fib->device);
    if (!is_device_ptr(keys) || !is_device_ptr(ordinals) || (next_hops && !is_device_ptr(next_hops)))
      throw Error(Errc::InvalidArgument, "lpm6cu_search_batch takes device buffers");
    if (reinterpret_cast<uintptr_t>(keys) % 8 != 0 || reinterpret_cast<uintptr_t>(ordinals) % 4 != 0)
      throw Error(Errc::InvalidArgument, "keys must be 8-byte and ordinals 4-byte aligned");
    launch_lookup(fib, keys, n, next_hops, static_cast<cudaStream_t>(stream), kInKeyOrd, nullptr, ordinals);
  });
}

int lpm6cu_lookup_packets(const lpm6cu_fib* fib, const void* frames, uint64_t n, uint64_t stride, uint32_t dst_offset,
                          void* out, void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!frames || !out) throw Error(Errc::InvalidArgument, "NULL buffer");
    if (stride < dst_offset + 16ull) throw Error(Errc::InvalidArgument, "stride must cover dst_offset + 16 bytes");
    DeviceGuard dg(fib->device);
    if (!is_device_ptr(frames) || !is_device_ptr(out))
      throw Error(Errc::InvalidArgument, "lpm6cu_lookup_packets takes device buffers");
    PacketInput pk;
    pk.stride = stride;
    pk.off = dst_offset;
    const unsigned long long bits = reinterpret_cast<uintptr_t>(frames) | stride;  // frame-start alignment
    pk.align = (bits & 15) == 0 ? 16 : (bits & 7) == 0 ? 8 : (bits & 3) == 0 ? 4 : (bits & 1) == 0 ? 2 : 1;
    launch_lookup(fib, frames, n, out, static_cast<cudaStream_t>(stream), kInPacket, &pk);
  });
}

int lpm6cu_fib_build_from_intervals(int device, const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                                    uint32_t default_nh, const lpm6cu_build_opts* opts, void* stream,
                                    lpm6cu_fib** out) {
  return guard([&] {
    if (!boundaries || !next_hops || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    // The IntervalMap contract (intervals.hpp:18-24).
    if (m == 0) throw Error(Errc::InvalidArgument, "an interval map has at least one boundary");
    if (boundaries[0] != 0) throw Error(Errc::InvalidArgument, "boundaries[0] must be 0");
    for (uint64_t i = 0; i < m; ++i) {
      if (i && boundaries[i] <= boundaries[i - 1])
        throw Error(Errc::InvalidArgument, "boundaries must be strictly increasing");
      if (next_hops[i] == kUnresolved) throw Error(Errc::ReservedNextHop, "next hop 4294967295 is reserved");
    }
    if (boundaries[m - 1] == kSentinelKey) throw Error(Errc::SentinelCollision, "boundary equals the sentinel key");
    DeviceGuard dg(device);
    lpm6cu_geometry g;
    void* lines = capi::device_build_tree_from_intervals(boundaries, next_hops, m, default_nh, opts,
                                                         static_cast<cudaStream_t>(stream), &g);
    std::unique_ptr<lpm6cu_fib> f;
    try {
      f.reset(new_fib(device, &g));
    } catch (...) {
      cudaFree(lines);
      throw;
    }
    f->d_lines = static_cast<unsigned long long*>(lines);
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_querygen_create(int device, int workload, const lpm6cu_prefix* rules, uint64_t nrules,
                           lpm6cu_querygen** out) {
  return guard([&] {
    WorkloadConfig c = workload_config(workload);
    auto prefixes = capi::to_prefixes(rules, nrules);
    QueryTables t = make_query_tables(std::span<const Prefix>(prefixes), c);
    DeviceGuard dg(device);
    auto g = std::make_unique<lpm6cu_querygen>();
    g->device = device;
    g->spec = make_query_spec(c, t);
    auto up = [&](void** d, const void* h, size_t bytes) {
      if (bytes == 0) return;
      check_cuda(cudaMalloc(d, bytes), "cudaMalloc querygen");
      check_cuda(cudaMemcpy(*d, h, bytes, cudaMemcpyHostToDevice), "copy querygen");
    };
    up(&g->d_top, t.top.data(), t.top.size() * 8);
    up(&g->d_len, t.len.data(), t.len.size());
    up(&g->d_cdf, t.cdf.data(), t.cdf.size() * 8);
    up(&g->d_perm, t.perm.data(), t.perm.size() * 4);
    g->spec.pfx_top = static_cast<const uint64_t*>(g->d_top);
    g->spec.pfx_len = static_cast<const uint8_t*>(g->d_len);
    g->spec.zipf_cdf = static_cast<const double*>(g->d_cdf);
    g->spec.zipf_perm = static_cast<const uint32_t*>(g->d_perm);
    *out = g.release();
  });
}

int lpm6cu_querygen_run(const lpm6cu_querygen* g, uint64_t first, uint64_t n, void* d_out, void* stream) {
  return guard([&] {
    if (!g || !d_out) throw Error(Errc::InvalidArgument, "NULL argument");
    if (n == 0) return;
    DeviceGuard dg(g->device);
    int sms = 0;
    check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, g->device), "attr");
    const unsigned long long blocks = std::min<unsigned long long>((n + 255) / 256, 8ull * sms);
    lpm6_querygen_kernel<<<static_cast<unsigned>(blocks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        g->spec, first, n, static_cast<uint4*>(d_out));
    check_cuda(cudaGetLastError(), "querygen launch");
  });
}

void lpm6cu_querygen_destroy(lpm6cu_querygen* g) { delete g; }

}  // extern "C"
