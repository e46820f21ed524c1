// sm_100a batched LPM lookup kernels (device half; lookup.cu holds the host half).
//
// One query = one predecessor search down the B200 tree (layout.hpp): internal
// 128-byte lines of 15 separators (arity 16), leaf lines of kL keys + kL next
// hops. The kernel is the GPU form of the reference's search_batch
// over Listing 1's node search, per 32-query
// warp tile (lane L owns query L):
//
//  Phase A — top `smem_levels` internal levels, one thread per query. The root's
//    separators come from the kernel-parameter constant bank (every lane starts
//    there, so its probes are near-uniform LDCs); the other levels from a packed
//    image staged into shared memory once per CTA by a TMA bulk copy on an
//    mbarrier. A node is ranked with a branch-free 4-probe binary search written
//    as a pointer walk in PTX (count of keys <= q: Listing 1's popcnt(cmpge)),
//    8 bytes per probe instead of a whole 128-byte node.
//  Phase B — the remaining levels, four lanes per query: lane j of a 4-lane
//    group reads bytes [32j, 32j+32) of the line (one 256-bit LSU load, or two
//    16-byte texture fetches for internal levels — TEXL), the lanes compare
//    their keys against the broadcast query and __ballot_sync + __popc give the
//    rank. Each group carries its 4 queries at once, so every level has 4
//    independent line loads in flight per group (P:812-847's batching as
//    memory-level parallelism).
//  Leaf — the leaf line carries the next hops (P:695-705 folded into the leaf
//    fetch): the lane holding the value bytes extracts the group's 4 next hops
//    and writes them with one coalesced streaming store. Small trees (LEAFS)
//    stage the leaves too and finish each query in shared memory.
//
// With 2 or 4 tiles per warp (PBSEQ, chosen by the line-path tuner) Phase A runs
// all tiles' descents together — their dependent probe chains overlap — and Phase B
// then takes one tile at a time, so the registers holding line quarters stay those of
// one tile.
//
// PLANES (chosen by the tuner with the line path, lpm6cu_kernel_config.plane_levels): the
// upper staged levels are stored as split planes — a node's 15 high words, then its 15
// low words — and probed with one LDS.32 of the high word (32 banks instead of 16 bank
// pairs: fewer random bank conflicts); the low word is read only when some lane of the
// warp ties on the high word, a warp-uniform branch shared by the warp's tiles.
//
// Query addresses are read with coalesced loads of the top word (L1::no_allocate,
// L2 evict_first), one tile ahead of their use; tree lines use evict_last. CTAs
// are persistent (grid = SMs x resident CTAs, default one 1024-thread CTA per
// SM) and stride over tiles. Results are the reference's: key = min(addr >> 64,
// 0xFFFF...FFFE) (types.hpp:25), internal child = node * 16 + rank, leaf
// ordinal = rank - 1, next hop = the value of that leaf slot.
//
// Included by lookup_vb{1,2,4}.cu (one next-hop width each); the kernels are in an
// anonymous namespace, the launch interface in lookup_params.hpp.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "capi_internal.hpp"
#include "lookup_params.hpp"

namespace {

using namespace lpm6;
using namespace lpm6::kern;

constexpr unsigned kFull = 0xFFFFFFFFu;

// Phase B node ranking: 1 = lane-local packed counts + XOR shuffles (group_ranks),
// 0 = one ballot + popc per key slot (group_rank). Build-time switch for A/B runs.
#ifndef LPM6_RANK_MODE
#define LPM6_RANK_MODE 1
#endif
// Phase A as a shared-memory address walk (1) or the node-index form (0); the
// leaf's next hop by a branch-free word select (1) or the compiler's lowering of
// an indexed pick (0). Build-time switches for A/B runs (tools/build_variant.sh).
#ifndef LPM6_PHASEA_WALK
#define LPM6_PHASEA_WALK 1
#endif
#ifndef LPM6_LEAF_SEL
#define LPM6_LEAF_SEL 1
#endif
// Texture fetches of 1-byte-next-hop leaf lines as two sector-disjoint halves (1)
// or lane quarters (0); internal lines always as lane quarters (C2 level 4: the
// halves measured 2 % slower there).
#ifndef LPM6_TEX_SECTORS
#define LPM6_TEX_SECTORS 1
#endif
// Internal texture lines as sector-disjoint halves too (A/B switch; 0 = lane quarters).
#ifndef LPM6_INT_SECTORS
#define LPM6_INT_SECTORS 0
#endif
// PBSEQ: Phase B's per-tile passes unrolled (1: ptxas may overlap one tile's leaf
// fetch with the next tile's internal level) or kept a loop (0). A/B switch.
#ifndef LPM6_PB_UNROLL
#define LPM6_PB_UNROLL 1
#endif
// Staged-level count as a template constant in the texture line-path kernels (1) or
// always read from the launch (0). A/B switch.
#ifndef LPM6_STATIC_TA
#define LPM6_STATIC_TA 1
#endif


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

// One 16-byte texel (SASS TLD.LZ on the int4 texture object over the line array).
__device__ __forceinline__ void tex16(unsigned long long tex, unsigned texel, unsigned long long& lo,
                                      unsigned long long& hi) {
  const int4 v = tex1Dfetch<int4>(static_cast<cudaTextureObject_t>(tex), static_cast<int>(texel));
  lo = static_cast<unsigned>(v.x) | (static_cast<unsigned long long>(static_cast<unsigned>(v.y)) << 32);
  hi = static_cast<unsigned>(v.z) | (static_cast<unsigned long long>(static_cast<unsigned>(v.w)) << 32);
}

// 32 bytes of a line through the texture path: two 16-byte texels. Line texel
// t0 + 0..7; lane j of the 4-lane group fetches texels (2j, 2j+1) — words 4j..4j+3,
// the same quarter an LSU lane loads — or, with SECTORS, texels (j, j+4): words
// 2j, 2j+1, 8+2j, 9+2j. With SECTORS the group's first fetch covers sectors 0-1 of
// the line and its second sectors 2-3, so no sector is requested twice: with
// (2j, 2j+1) both fetches touch all four sectors and the second re-reads them from
// L1 — which misses when the ~30 KB of L1 a 221 KB shared-memory image leaves have
// been recycled in between (measured on C1: texture sector hit rate 25 % -> every
// line fetched ~1.5 times from L2 when the compiler spreads a slot's two fetches
// apart). Counting ranks does not depend on which lane holds which key; the leaf
// formats where it matters are handled at the call site.
// The lane's texel base of a level (line word offset / 2 + its first texel), so that
// a fetch pair is texel = base + 8 * node (one IMAD); with a per-slot address instead,
// ptxas also gave every TLD its own uniform copy of the texture handle (R2UR pairs).
template <bool SECTORS>
__device__ __forceinline__ unsigned tex_lane_base(unsigned line_w, unsigned j) {
  return (line_w >> 1) + (SECTORS ? j : 2u * j);
}
template <bool SECTORS>
__device__ __forceinline__ void tex_line_at(unsigned long long tex, unsigned base, unsigned node,
                                            unsigned long long (&w)[4]) {
  const unsigned ta = base + node * 8u;
  tex16(tex, ta, w[0], w[1]);
  tex16(tex, ta + (SECTORS ? 4u : 1u), w[2], w[3]);
}

// Half-line leaves: 16 bytes per lane (words 2j, 2j+1), by a 16-byte load or one
// texture fetch; w[2..3] are not used.
__device__ __forceinline__ void ld_half_leaf(const unsigned long long* p, unsigned long long (&w)[4]) {
  asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(w[0]), "=l"(w[1]) : "l"(p));
}
__device__ __forceinline__ void tex_half_leaf(unsigned long long tex, unsigned texel, unsigned long long (&w)[4]) {
  tex16(tex, texel, w[0], w[1]);
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



// Rank of q in the root (the kernel-parameter copy, LookupParams::root): the same
// 4-probe search. ROOT_WALK keeps the probe position as a byte offset advanced by
// predicated adds — each probe one LDC at register + immediate, two compares and one
// add — instead of rebuilding an indexed address per probe.
#ifndef LPM6_ROOT_WALK
#define LPM6_ROOT_WALK 1
#endif
__device__ __forceinline__ unsigned root_rank(const LookupParams& p, unsigned long long q) {
#if LPM6_ROOT_WALK
  unsigned o = (p.root[7] <= q) ? 64u : 0u;  // byte offset of the candidate position
  o += (p.root[(o >> 3) + 3u] <= q) ? 32u : 0u;
  o += (p.root[(o >> 3) + 1u] <= q) ? 16u : 0u;
  o += (p.root[o >> 3] <= q) ? 8u : 0u;
  return o >> 3;
#else
  unsigned c = (p.root[7] <= q) ? 8u : 0u;
  c |= (p.root[c | 3u] <= q) ? 4u : 0u;
  c |= (p.root[c | 1u] <= q) ? 2u : 0u;
  c |= (p.root[c] <= q) ? 1u : 0u;
  return c;
#endif
}

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
  asm volatile("{\n\t.reg .pred p;\n\t.reg .b64 k;\n\t"
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

// Phase B ranks of all NS queries a 4-lane group carries, without ballots: each
// lane counts its own keys <= q per query into one byte of a packed counter
// (query s -> byte s % 4 of acc[s / 4]; a count is at most 16), then two XOR
// shuffles inside the 4-lane group sum the four lanes' bytes. Per compare this is
// a 64-bit setp and one predicated add (3 SASS instructions) against the
// ballot form's compare + VOTE + LOP + POPC + add (6); the reduction costs two
// SHFL + two adds per four queries. Lane j's key slots t < 2 / t >= 2 count only
// when lo / hi is all-ones (leaf lines: slots past kL hold next hops, not keys).
template <int NS, bool MASKED, int NK = 4, int WN = 4>
__device__ __forceinline__ void group_ranks(const unsigned long long (&qk)[NS], const unsigned long long (&w)[NS][WN],
                                            unsigned lo, unsigned hi, unsigned (&r)[NS]) {
  // NK keys per lane (4: a 128-byte line, 2: a half-line leaf, where `lo` masks
  // the lane's whole count)
  constexpr int NA = (NS + 3) / 4;
  unsigned acc[NA], acc_hi[NA];
#pragma unroll
  for (int a = 0; a < NA; ++a) acc[a] = acc_hi[a] = 0u;
#pragma unroll
  for (int s = 0; s < NS; ++s) {
#pragma unroll
    for (int t = 0; t < NK; ++t) {
      unsigned& dst = (MASKED && t >= 2) ? acc_hi[s / 4] : acc[s / 4];
      asm("{\n\t.reg .pred p;\n\tsetp.ge.u64 p, %1, %2;\n\t@p add.u32 %0, %0, %3;\n\t}"
          : "+r"(dst)
          : "l"(qk[s]), "l"(w[s][t]), "r"(1u << (8 * (s % 4))));
    }
  }
#pragma unroll
  for (int a = 0; a < NA; ++a) {
    if (MASKED) acc[a] = (acc[a] & lo) + (acc_hi[a] & hi);
    if (!MASKED && NK == 2) acc[a] &= lo;
    acc[a] += __shfl_xor_sync(kFull, acc[a], 1);
    acc[a] += __shfl_xor_sync(kFull, acc[a], 2);
  }
#pragma unroll
  for (int s = 0; s < NS; ++s) r[s] = __byte_perm(acc[s / 4], 0u, 0x4440u | (s % 4));
}

template <int VB>
struct LeafFmt {
  static constexpr int kL = VB == 1 ? 14 : VB == 2 ? 12 : 8;  // keys per leaf line
  static constexpr int kValueLane = (kL * 8) / 32;             // lane holding the next hops
  static constexpr int kValueOff = kL * 8 - kValueLane * 32;   // their byte offset in that lane's 32 B
};

__device__ __forceinline__ unsigned long long sel64(bool p, unsigned long long a, unsigned long long b) {
  unsigned long long r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.u32 q, %3, 0;\n\tselp.b64 %0, %1, %2, q;\n\t}"
      : "=l"(r)
      : "l"(a), "l"(b), "r"(static_cast<unsigned>(p)));
  return r;
}

// Next hop of leaf ordinal `ord` from the value lane's 32 bytes: a branch-free
// select of the 8-byte word holding it (only the words the value bytes occupy
// are candidates) and one funnel shift. Values never straddle a word.
template <int VB, bool SELECT = (VB != 1)>
__device__ __forceinline__ unsigned leaf_value(const unsigned long long (&w)[4], unsigned ord) {
  constexpr unsigned kOff = LeafFmt<VB>::kValueOff;
  constexpr unsigned kFirst = kOff / 8;
  constexpr unsigned kLast = (kOff + LeafFmt<VB>::kL * VB - 1) / 8;
  const unsigned o = kOff + ord * VB;  // byte offset within the lane's quarter
  const unsigned wi = o >> 3;
#if LPM6_LEAF_SEL
  if constexpr (!SELECT) {
    // 1-byte next hops (unless line path 4): the compiler's own lowering of the
    // pick. With it, ptxas issues each texture leaf line's two fetches back to back;
    // with the select below it spreads them apart, and on L1-missing traffic the
    // second fetch then often misses too (C1 on texture leaves: 56 vs 85 G/s).
    // On L1-hitting traffic the select's shorter code wins (C3a 96 vs 93 G/s):
    // line path 4 = texture leaves with the select, for the tuner to choose.
    const unsigned long long x = wi == 0 ? w[0] : wi == 1 ? w[1] : wi == 2 ? w[2] : w[3];
    return static_cast<unsigned>(x >> ((o & 7u) * 8u)) & 0xFFu;
  }
  unsigned long long x = w[kFirst];
#pragma unroll
  for (unsigned i = kFirst + 1; i <= kLast; ++i) x = sel64(wi == i, w[i], x);
#else
  const unsigned long long x = wi == 0 ? w[0] : wi == 1 ? w[1] : wi == 2 ? w[2] : w[3];
#endif
  const unsigned v = static_cast<unsigned>(x >> ((o & 7u) * 8u));
  return VB == 1 ? (v & 0xFFu) : VB == 2 ? (v & 0xFFFFu) : v;
}

// Next hop of ordinal `ord` of a half-line leaf from lane 3's words 6-7 (w[0], w[1]).
template <int VB, int WN>
__device__ __forceinline__ unsigned half_leaf_value(const unsigned long long (&w)[WN], unsigned ord) {
  const unsigned o = ord * VB;  // byte offset within words 6-7
  const unsigned long long x = sel64(o >= 8u, w[1], w[0]);
  const unsigned v = static_cast<unsigned>(x >> ((o & 7u) * 8u));
  return VB == 1 ? (v & 0xFFu) : (v & 0xFFFFu);
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
// TEXL: the internal L2 levels are read through the texture pipe (p.tex) — 1:
// every line, 2: the lower half of each group's slots (the rest through the LSU).
// LEAFTEX: the leaf lines too — 1: every leaf line (3: the same with the select
// extraction of 1-byte next hops, line path 4), 2: the upper half of each
// group's slots. The halves are compile-time splits, so both L1TEX pipes work
// in every warp. Texture hits return off the LSU data pipe, which pays when
// leaf lines hit L1 often (skewed traffic: C3b +9 % with 1); on L1-missing
// traffic the texture path's miss throughput is lower (C1 -27 % with 1, +1.2 %
// with 2), so the host picks the line path by measurement
// (lpm6cu_fib_tune_line_path).
// PLANES (0 = none; 2, 3 or kAllPlanes): split-plane Phase A. With P = PLANES, staged levels 1 .. P - 1 are
// probed in the plane format (4-byte high words, 60 bytes per node; a low word only on a
// tie) and levels P .. TA - 1 in the packed format; the walk's child step between two
// plane levels is the packed one (the strides scale alike), from a plane level to a
// packed one it is 2 a + 30 a' + (off(P) - 32 off(P - 1)) (LookupParams::pl2pk).
// TAS > 0: the number of staged levels is a compile-time constant (= p.smem_levels),
// so Phase A's level loop and Phase B's internal-level loop have no runtime level
// checks (the texture line paths are instantiated for TAS = DEPTH and DEPTH - 1, the
// staging every BASELINE FIB uses; TAS = 0 reads the count from the launch).
template <int DEPTH, int VB, int TILES, int THREADS, int MINB, bool CHECKED, int INPUT = kInAddr, bool LEAFS = false,
          int TEXL = 0, int LEAFTEX = 0, bool HALF = false, int TAS = 0, bool PBSEQ = false, int PLANES = 0>
__global__ void __launch_bounds__(THREADS, MINB) lpm6_lookup_kernel(const LookupParams p) {
  using F = LeafFmt<VB>;
  // Texture leaf fetches as sector-disjoint halves (tex_line_at) for 1-byte next
  // hops. (2-byte ones would need their values gathered from lanes 2 and 3; measured
  // on C2: no gain on texture leaves, 56 vs 55 G/s, so they keep lane quarters.)
  constexpr bool kLeafSectors = LPM6_TEX_SECTORS != 0 && VB == 1;
  unsigned violations = 0;
  unsigned long long visits = 0;  // CHECKED: lines visited by this lane's own queries
  extern __shared__ __align__(128) unsigned long long s_lines[];
  __shared__ __align__(8) uint64_t s_bar;

  const unsigned lane = threadIdx.x & 31u;
  const unsigned j = lane & 3u;                 // lane within the 4-lane group
  const unsigned gbase = lane & ~3u;            // first lane (= first query) of the group
  [[maybe_unused]] const unsigned gmask = 0xFu << gbase;  // LPM6_RANK_MODE 0
  const unsigned long long warp0 = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pol_stream = policy_evict_first();
  const unsigned TA = TAS > 0 ? static_cast<unsigned>(TAS) : p.smem_levels;
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

  // Stage the image after the first addresses are requested, so their DRAM/L2
  // latency overlaps the bulk copy (it matters for small batches).
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
    if constexpr (PLANES != 0 && !CHECKED && !LEAFS) {
      constexpr unsigned PU = PLANES;
      uint32_t a[TILES];
      unsigned qh[TILES], ql[TILES];
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        const unsigned c = root_rank(p, key[t]);
        a[t] = s_base + p.img_step[0] + c * 60u;
        qh[t] = static_cast<unsigned>(key[t] >> 32);
        ql[t] = static_cast<unsigned>(key[t]);
      }
      auto lds32 = [](uint32_t addr) {
        unsigned v;
        asm volatile("ld.shared.u32 %0, [%1];" : "=r"(v) : "r"(addr));
        return v;
      };
      // One probe of every tile: high words first; low words only if a lane of the warp ties.
      auto probe = [&](uint32_t off, uint32_t step, uint32_t lod) {
        unsigned h[TILES];
        bool gt[TILES], eq[TILES];
        bool anyeq = false;
#pragma unroll
        for (int t = 0; t < TILES; ++t) h[t] = lds32(a[t] + off);
#pragma unroll
        for (int t = 0; t < TILES; ++t) {
          gt[t] = qh[t] > h[t];
          eq[t] = qh[t] == h[t];
          anyeq |= eq[t];
        }
        if (__any_sync(kFull, anyeq)) {
#pragma unroll
          for (int t = 0; t < TILES; ++t)
            if (eq[t]) gt[t] = ql[t] >= lds32(a[t] + off + lod);
        }
#pragma unroll
        for (int t = 0; t < TILES; ++t) a[t] += gt[t] ? step : 0u;
      };
#pragma unroll
      for (int l = 1; l < DEPTH; ++l) {
        if (static_cast<unsigned>(l) >= TA) break;
        if (static_cast<unsigned>(l) < PU) {
          uint32_t a0[TILES];
#pragma unroll
          for (int t = 0; t < TILES; ++t) a0[t] = a[t];
          const uint32_t lod = p.lo_delta[l];
          probe(28u, 32u, lod);
          probe(12u, 16u, lod);
          probe(4u, 8u, lod);
          probe(0u, 4u, lod);
          if (static_cast<unsigned>(l + 1) == PU && static_cast<unsigned>(l + 1) < TA) {  // next level packed
#pragma unroll
            for (int t = 0; t < TILES; ++t) a[t] = 2u * a0[t] + 30u * a[t] + (p.pl2pk - 31u * s_base);
          } else {
#pragma unroll
            for (int t = 0; t < TILES; ++t) a[t] = a0[t] + 15u * a[t] + (p.img_step[l] - 15u * s_base);
          }
        } else {
#pragma unroll
          for (int t = 0; t < TILES; ++t) {
            const uint32_t af = a[t] + node_rank_saddr(a[t], key[t]);
            a[t] = a[t] + 15u * af + (p.img_step[l] - 15u * s_base);
          }
        }
      }
      // a - s_base = 60 x node after a plane level, 120 x node after a packed one
      const unsigned sh = TA > PU ? 3u : 2u;
#pragma unroll
      for (int t = 0; t < TILES; ++t) node[t] = ((a[t] - s_base) >> sh) * 0xEEEEEEEFu;
    } else if constexpr (!CHECKED && LPM6_PHASEA_WALK) {
      // As a walk over shared-memory byte addresses: with a = the address of node
      // n of level l and a' = a + 8 * rank after the four probes, the child's
      // address in level l + 1 is img(l+1) + (16 n + rank) * 120 =
      // a + 15 a' + (img(l+1) - 16 img(l)) — one IMAD and one add per level (the
      // constants come with the launch, LookupParams::img_step); after the last
      // staged level the same step with img(l+1) := 0 leaves s_base + 120 x the
      // child's node index (an exact division by 120 recovers it).
#pragma unroll
      for (int t = 0; t < TILES; ++t) {
        if (TA == 0) break;
        const unsigned long long q = key[t];
        // Root from the kernel-parameter constant bank: all lanes start at the
        // same node, so the probes are (nearly) uniform LDCs and keep the
        // shared-memory data pipe free for the deeper levels.
        const unsigned c = root_rank(p, q);
        if (TA == 1) {
          node[t] = c;
          continue;
        }
        uint32_t a = s_base + p.img_step[0] + c * 120u;
#pragma unroll
        for (int l = 1; l < DEPTH; ++l) {
          if (static_cast<unsigned>(l) >= TA) break;
          const uint32_t af = a + node_rank_saddr(a, q);
          a = a + 15u * af + (p.img_step[l] - 15u * s_base);  // img_step: see LookupParams
        }
        // a - s_base = 120 x node: exact division (0xEEEEEEEF = 15^-1 mod 2^32)
        node[t] = ((a - s_base) >> 3) * 0xEEEEEEEFu;
      }
    } else
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

    // PBSEQ: Phase A runs TILES tiles at once (their dependent probe chains overlap)
    // and Phase B then takes one tile at a time, so its line registers stay those of
    // one tile; otherwise Phase B carries all TILES tiles together.
    constexpr int PBT = PBSEQ ? 1 : TILES;  // tiles per Phase B pass
    constexpr int NSB = 4 * PBT;            // queries in flight per 4-lane group
#if LPM6_PB_UNROLL
#pragma unroll
#else
#pragma unroll 1
#endif
    for (int pb = 0; pb < (PBSEQ ? TILES : 1); ++pb) {
      unsigned long long kcur[PBT];
      unsigned ncur[PBT];
#pragma unroll
      for (int t = 0; t < PBT; ++t) {
        kcur[t] = key[t];
        ncur[t] = node[t];
        if constexpr (PBSEQ) {
#pragma unroll
          for (int u = 1; u < TILES; ++u)
            if (pb == u) {
              kcur[t] = key[u];
              ncur[t] = node[u];
            }
        }
      }
      const int tb0 = PBSEQ ? pb : 0;
      // Phase B: the group's queries, one 128-byte line per query per level.
      unsigned long long qk[NSB];
      unsigned nd[NSB];
  #pragma unroll
      for (int t = 0; t < PBT; ++t)
  #pragma unroll
        for (int s = 0; s < 4; ++s) {
          qk[4 * t + s] = __shfl_sync(kFull, kcur[t], s, 4);
          nd[4 * t + s] = __shfl_sync(kFull, ncur[t], s, 4);
        }
      unsigned long long w[NSB][4];
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
        const unsigned line_w = static_cast<unsigned>(p.level_start[l]);
        const unsigned base_w = line_w + j * 4u;
        if (CHECKED) {
  #pragma unroll
          for (int s = 0; s < NSB; ++s)
            if (nd[s] >= p.level_nodes[l]) {
              violations |= 2u;
              nd[s] = 0;
            }
        }
  #pragma unroll
        for (int s = 0; s < NSB; ++s) {
          // Internal L2 levels through the texture pipe, leaves through the LSU:
          // the two pipes of L1TEX share the load, which helps the deep trees (C2:
          // +8 %); leaves through the texture pipe lose on L2-missing workloads
          // (C1 -17 %), so they stay on the LSU path.
          if (TEXL == 1 || (TEXL == 2 && s < NSB / 2))
            // (the per-slot texel form here: the lane-base form cost C2 0.35 %, 64 vs 60 registers)
            tex_line_at<LPM6_INT_SECTORS != 0>(p.tex, ((line_w + nd[s] * 16u) >> 1) + (LPM6_INT_SECTORS ? j : 2u * j),
                                               0u, w[s]);
          else
            ld_line_quarter(p.lines + (base_w + nd[s] * 16u), w[s]);
        }
        if (CHECKED) {  // one line per query: the lane owning query (t, j) counts it
  #pragma unroll
          for (int t = 0; t < PBT; ++t)
            if ((st * TILES + tb0 + t) * 32ull + lane < p.n) ++visits;
        }
  #if LPM6_RANK_MODE == 1
        {
          unsigned r[NSB];
          group_ranks<NSB, false>(qk, w, ~0u, ~0u, r);
  #pragma unroll
          for (int s = 0; s < NSB; ++s) nd[s] = nd[s] * 16u + r[s];
        }
  #else
  #pragma unroll
        for (int s = 0; s < NSB; ++s) nd[s] = nd[s] * 16u + group_rank(qk[s], w[s], 4u, gmask);
  #endif
      }
      unsigned leafn[INPUT == kInKeyOrd ? NSB : 1];  // kInKeyOrd: leaf node of each query
      constexpr bool half = HALF;  // the FIB's leaf format (half-line leaves: 2-byte next hops)
      if constexpr (half) {  // half-line leaves (layout.hpp): lane j reads words 2j, 2j+1 of its leaf
        const unsigned line_w = static_cast<unsigned>(p.level_start[DEPTH]);
        if (CHECKED) {
  #pragma unroll
          for (int s = 0; s < NSB; ++s)
            if (nd[s] >= p.level_nodes[DEPTH]) {
              violations |= 2u;
              nd[s] = 0;
            }
        }
  #pragma unroll
        for (int s = 0; s < NSB; ++s) {
          // 16 bytes per lane: one texture fetch, or one 16-byte load
          if (LEAFTEX == 1 || LEAFTEX == 3 || (LEAFTEX == 2 && s >= NSB / 2))
            tex_half_leaf(p.tex, ((line_w + nd[s] * kHalfLeafWords) >> 1) + j, w[s]);
          else
            ld_half_leaf(p.lines + line_w + nd[s] * kHalfLeafWords + 2u * j, w[s]);
        }
        if constexpr (INPUT == kInKeyOrd) {
  #pragma unroll
          for (int s = 0; s < NSB; ++s) leafn[s] = nd[s];
        }
        if (CHECKED) {
  #pragma unroll
          for (int t = 0; t < PBT; ++t)
            if ((st * TILES + tb0 + t) * 32ull + lane < p.n) ++visits;
        }
        unsigned r[NSB];
        group_ranks<NSB, false, 2>(qk, w, j < 3u ? ~0u : 0u, 0u, r);  // lane 3 holds the next hops
  #pragma unroll
        for (int s = 0; s < NSB; ++s) {
          if (CHECKED && r[s] == 0) violations |= 4u;
          nd[s] = CHECKED && r[s] == 0 ? 0u : r[s] - 1u;
        }
      } else {  // the leaf line: ordinal = rank - 1
        const unsigned line_w = static_cast<unsigned>(p.level_start[DEPTH]);
        const unsigned base_w = line_w + j * 4u;
        if (CHECKED) {
  #pragma unroll
          for (int s = 0; s < NSB; ++s)
            if (nd[s] >= p.level_nodes[DEPTH]) {
              violations |= 2u;
              nd[s] = 0;
            }
        }
  #pragma unroll
        for (int s = 0; s < NSB; ++s) {
          // LEAFTEX 1: every slot through the texture pipe; 2: the upper half of the
          // group's slots (compile-time split, both pipes busy in one warp).
          if (LEAFTEX == 1 || LEAFTEX == 3 || (LEAFTEX == 2 && s >= NSB / 2))
            // sector-disjoint fetches (kLeafSectors): for 1-byte next hops the leaf
            // keeps the same key slots and value lane in both orders (the values are
            // words 14-15 = lane 3's second texel either way)
            tex_line_at<kLeafSectors>(p.tex, tex_lane_base<kLeafSectors>(line_w, j), nd[s], w[s]);
          else
            ld_line_quarter(p.lines + (base_w + nd[s] * 16u), w[s]);
        }
        if constexpr (INPUT == kInKeyOrd) {
  #pragma unroll
          for (int s = 0; s < NSB; ++s) leafn[s] = nd[s];
        }
        if (CHECKED) {
  #pragma unroll
          for (int t = 0; t < PBT; ++t)
            if ((st * TILES + tb0 + t) * 32ull + lane < p.n) ++visits;
        }
  #if LPM6_RANK_MODE == 1
        {
          unsigned r[NSB];
          group_ranks<NSB, true>(qk, w, leaf_valid >= 2 ? ~0u : 0u, leaf_valid >= 4 ? ~0u : 0u, r);
  #pragma unroll
          for (int s = 0; s < NSB; ++s) {
            if (CHECKED && r[s] == 0) violations |= 4u;
            nd[s] = CHECKED && r[s] == 0 ? 0u : r[s] - 1u;
          }
        }
  #else
  #pragma unroll
        for (int s = 0; s < NSB; ++s) {
          const unsigned r = group_rank(qk[s], w[s], leaf_valid, gmask);
          if (CHECKED && r == 0) violations |= 4u;
          nd[s] = CHECKED && r == 0 ? 0u : r - 1u;
        }
  #endif
      }

      if constexpr (INPUT == kInKeyOrd) {  // lane j stores the ordinal of its own query (4t + j of the group)
  #pragma unroll
        for (int t = 0; t < PBT; ++t) {
          const unsigned kl = half ? kHalfLeafKeys : static_cast<unsigned>(F::kL);
          unsigned o = leafn[4 * t] * kl + nd[4 * t];
  #pragma unroll
          for (int s = 1; s < 4; ++s) o = j == static_cast<unsigned>(s) ? leafn[4 * t + s] * kl + nd[4 * t + s] : o;
          const unsigned long long qi = (st * TILES + tb0 + t) * 32ull + lane;
          if (qi < p.n) asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p.ord + qi), "r"(o));
        }
        if (p.out == nullptr) continue;  // ordinals only
      }
      // Leaf values: the value lane extracts the group's next hops and stores them.
      if constexpr (half) {
        if (j == 3u) {  // half-line leaves: lane 3 holds words 6-7, the next hops
  #pragma unroll
          for (int t = 0; t < PBT; ++t) {
            unsigned v[4];
  #pragma unroll
            for (int s = 0; s < 4; ++s) v[s] = half_leaf_value<VB, 4>(w[4 * t + s], nd[4 * t + s]);
            store_group<VB>(p, (st * TILES + tb0 + t) * 32ull + gbase, v);
          }
        }
      } else if (j == static_cast<unsigned>(F::kValueLane)) {
  #pragma unroll
        for (int t = 0; t < PBT; ++t) {
          unsigned v[4];
  #pragma unroll
          for (int s = 0; s < 4; ++s) v[s] = leaf_value<VB, VB != 1 || LEAFTEX == 3>(w[4 * t + s], nd[4 * t + s]);
          store_group<VB>(p, (st * TILES + tb0 + t) * 32ull + gbase, v);
        }
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


// Instantiated shapes: (queries per lane, min CTAs per SM) for every depth; one
// next-hop width per translation unit (lookup_vb{1,2,4}.cu), so the ~150 kernels
// of each width compile in parallel. bench.py --sweep measures the shapes.
// The default-shape kernel of one depth: the staged-level count as a template
// constant when it is DEPTH or DEPTH - 1 (TAS), else read from the launch.
// TL = 2: two tiles per warp iteration through Phase A, Phase B one tile at a time
// (PBSEQ; 1024 threads, texture line paths, address input).
template <int D, int VB, int INPUT, int TEXL, int LEAFTEX, bool HALF, int TL = 1, int PLN = 0>
KernelFn pick_ta(int ta) {
  constexpr bool SEQ = TL > 1;
  if constexpr (PLN != 0) {
    // split-plane Phase A: trees of depth >= 3 with every internal level staged (then no
    // internal level is read from L2: TEXL 0) or all but the last (read through the
    // texture pipe: TEXL 1) — the stagings and pipes the 2- and 4-tile plans use
    if constexpr (D >= 3) {
      if constexpr (TEXL == 0) {
        if (ta == D) return lpm6_lookup_kernel<D, VB, TL, 1024, 1, false, INPUT, false, 0, LEAFTEX, HALF, D, SEQ, PLN>;
      } else {
        if (ta == D - 1)
          return lpm6_lookup_kernel<D, VB, TL, 1024, 1, false, INPUT, false, 1, LEAFTEX, HALF, D - 1, SEQ, PLN>;
      }
    }
    return nullptr;
  } else {
    if constexpr (LPM6_STATIC_TA != 0) {
      if (ta == D) return lpm6_lookup_kernel<D, VB, TL, 1024, 1, false, INPUT, false, TEXL, LEAFTEX, HALF, D, SEQ>;
      if constexpr (D >= 2)
        if (ta == D - 1)
          return lpm6_lookup_kernel<D, VB, TL, 1024, 1, false, INPUT, false, TEXL, LEAFTEX, HALF, D - 1, SEQ>;
    }
    return lpm6_lookup_kernel<D, VB, TL, 1024, 1, false, INPUT, false, TEXL, LEAFTEX, HALF, 0, SEQ>;
  }
}

template <int VB, int INPUT, int TEXL, int LEAFTEX, bool HALF, int TL = 1, int PLN = 0>
KernelFn pick_depth_texl(int depth, int ta = 0) {
  switch (depth) {
    case 1: return pick_ta<1, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 2: return pick_ta<2, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 3: return pick_ta<3, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 4: return pick_ta<4, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 5: return pick_ta<5, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 6: return pick_ta<6, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    case 7: return pick_ta<7, VB, INPUT, TEXL, LEAFTEX, HALF, TL, PLN>(ta);
    default: return nullptr;
  }
}

// Leaf lines through the texture pipe (default shape, unchecked, address / key / packet input).
// texl: internal-level mode (0 LSU, 1 texture, 2 split); mode: leaf mode (1 texture,
// 2 split, 3 texture with the select extraction of 1-byte next hops). Instantiated:
// texl 0/1 with leaf modes 1 and 2, texl 2 with texture leaves, mode 3 for VB = 1.
template <int VB, int INPUT, bool HALF>
KernelFn pick_leaftex(int depth, int texl, int mode, int ta) {
  if (mode == 3) {  // texture leaves with the select extraction: 1-byte next hops only
    if constexpr (VB == 1 && !HALF)
      return texl == 1 ? pick_depth_texl<VB, INPUT, 1, 3, HALF>(depth, ta)
             : texl == 0 ? pick_depth_texl<VB, INPUT, 0, 3, HALF>(depth, ta) : nullptr;
    return nullptr;
  }
  if (texl == 2) return mode == 1 ? pick_depth_texl<VB, INPUT, 2, 1, HALF>(depth, ta) : nullptr;
  if (mode == 2)
    return texl ? pick_depth_texl<VB, INPUT, 1, 2, HALF>(depth, ta) : pick_depth_texl<VB, INPUT, 0, 2, HALF>(depth, ta);
  return texl ? pick_depth_texl<VB, INPUT, 1, 1, HALF>(depth, ta) : pick_depth_texl<VB, INPUT, 0, 1, HALF>(depth, ta);
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

template <int VB, int TILES, int THREADS, int MINB, bool CHECKED = false, int INPUT = kInAddr, bool HALF = false>
KernelFn pick_depth(int depth) {
  switch (depth) {
    case 0: return lpm6_lookup_kernel<0, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 1: return lpm6_lookup_kernel<1, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 2: return lpm6_lookup_kernel<2, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 3: return lpm6_lookup_kernel<3, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 4: return lpm6_lookup_kernel<4, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 5: return lpm6_lookup_kernel<5, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 6: return lpm6_lookup_kernel<6, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    case 7: return lpm6_lookup_kernel<7, VB, TILES, THREADS, MINB, CHECKED, INPUT, false, 0, 0, HALF>;
    default: return nullptr;
  }
}

// Split-plane kernels (PLANES = a.planes: 2, 3 or kAllPlanes): 2 or 4 tiles per warp, texture
// leaves (modes 1 and 3), address input.
template <int VB, bool HALF, int LT, int TL, int PLN>
KernelFn pick_planes_texl(const PickArgs& a) {
  return a.texl ? pick_depth_texl<VB, kInAddr, 1, LT, HALF, TL, PLN>(a.depth, a.ta)
                : pick_depth_texl<VB, kInAddr, 0, LT, HALF, TL, PLN>(a.depth, a.ta);
}
template <int VB, bool HALF, int LT, int TL>
KernelFn pick_planes_pu(const PickArgs& a) {
  switch (a.planes) {
    case 2: return pick_planes_texl<VB, HALF, LT, TL, 2>(a);
    case 3: return pick_planes_texl<VB, HALF, LT, TL, 3>(a);
    case kAllPlanes: return pick_planes_texl<VB, HALF, LT, TL, kAllPlanes>(a);
    default: return nullptr;
  }
}
template <int VB, bool HALF>
KernelFn pick_planes(const PickArgs& a) {
  if (a.leaftex == 1) return a.tiles == 4 ? pick_planes_pu<VB, HALF, 1, 4>(a) : pick_planes_pu<VB, HALF, 1, 2>(a);
  if constexpr (VB == 1 && !HALF)
    if (a.leaftex == 3) return a.tiles == 4 ? pick_planes_pu<VB, HALF, 3, 4>(a) : pick_planes_pu<VB, HALF, 3, 2>(a);
  return nullptr;
}

// The kernels of one leaf format. HALF (half-line leaves, 2-byte next hops only) is
// instantiated for the default shape: every input format, checked and unchecked,
// every line path; the other shapes exist for full leaf lines.
template <int VB, bool HALF>
KernelFn pick_kernel_fmt(const PickArgs& a) {
  const int depth = a.depth;
  const bool dflt = a.tiles == 1 && a.threads == 1024 && a.minb == 1;
  if (a.leaftex && (a.tiles == 2 || a.tiles == 4) && a.threads == 1024 && a.minb == 1) {
    // 2 or 4 tiles per warp through Phase A, Phase B one tile at a time (PBSEQ):
    // address input, texture leaves (modes 1 and 3), internal L2 levels on one pipe
    if (a.leafs || a.checked || a.input != kInAddr || a.texl > 1) return nullptr;
    if (a.planes) return pick_planes<VB, HALF>(a);  // split-plane Phase A: the same shapes
    if (a.leaftex == 1)
      return a.tiles == 4 ? (a.texl ? pick_depth_texl<VB, kInAddr, 1, 1, HALF, 4>(depth, a.ta)
                                    : pick_depth_texl<VB, kInAddr, 0, 1, HALF, 4>(depth, a.ta))
                          : (a.texl ? pick_depth_texl<VB, kInAddr, 1, 1, HALF, 2>(depth, a.ta)
                                    : pick_depth_texl<VB, kInAddr, 0, 1, HALF, 2>(depth, a.ta));
    if constexpr (VB == 1 && !HALF)
      if (a.leaftex == 3)
        return a.tiles == 4 ? (a.texl ? pick_depth_texl<VB, kInAddr, 1, 3, HALF, 4>(depth, a.ta)
                                      : pick_depth_texl<VB, kInAddr, 0, 3, HALF, 4>(depth, a.ta))
                            : (a.texl ? pick_depth_texl<VB, kInAddr, 1, 3, HALF, 2>(depth, a.ta)
                                      : pick_depth_texl<VB, kInAddr, 0, 3, HALF, 2>(depth, a.ta));
    return nullptr;
  }
  if (a.planes) return nullptr;  // split planes exist for 2 or 4 tiles per warp on the texture leaf paths only
  if (a.leaftex) {  // default shape, unchecked, no leaf image, depth >= 1
    if (a.leafs || a.checked || !dflt) return nullptr;
    switch (a.input) {
      case kInAddr: return pick_leaftex<VB, kInAddr, HALF>(depth, a.texl, a.leaftex, a.ta);
      case kInKey: return pick_leaftex<VB, kInKey, HALF>(depth, a.texl, a.leaftex, a.ta);
      case kInPacket: return pick_leaftex<VB, kInPacket, HALF>(depth, a.texl, a.leaftex, a.ta);
      default: return nullptr;
    }
  }
  if (a.texl) {  // internal L2 levels via the texture pipe: default shape, unchecked
    if (a.leafs || a.checked || !dflt) return nullptr;
    switch (a.input) {
      case kInAddr: return pick_depth_texl<VB, kInAddr, 1, 0, HALF>(depth);
      case kInKey: return pick_depth_texl<VB, kInKey, 1, 0, HALF>(depth);
      case kInPacket: return pick_depth_texl<VB, kInPacket, 1, 0, HALF>(depth);
      default: return nullptr;  // kInKeyOrd: LSU loads
    }
  }
  if (a.leafs) {  // leaf image: address input, default shape, depth <= kMaxLeafImageDepth
    if (HALF || a.input != kInAddr || !dflt) return nullptr;
    return a.checked ? pick_depth_leafs<VB, true>(depth) : pick_depth_leafs<VB, false>(depth);
  }
  if (a.input != kInAddr) {  // key / packet input: the default shape, unchecked and checked
    if (!dflt) return nullptr;
    if (a.input == kInKey)
      return a.checked ? pick_depth<VB, 1, 1024, 1, true, kInKey, HALF>(depth)
                       : pick_depth<VB, 1, 1024, 1, false, kInKey, HALF>(depth);
    if (a.input == kInPacket)
      return a.checked ? pick_depth<VB, 1, 1024, 1, true, kInPacket, HALF>(depth)
                       : pick_depth<VB, 1, 1024, 1, false, kInPacket, HALF>(depth);
    if (a.input == kInKeyOrd)
      return a.checked ? pick_depth<VB, 1, 1024, 1, true, kInKeyOrd, HALF>(depth)
                       : pick_depth<VB, 1, 1024, 1, false, kInKeyOrd, HALF>(depth);
    return nullptr;
  }
  if (a.checked) return dflt ? pick_depth<VB, 1, 1024, 1, true, kInAddr, HALF>(depth) : nullptr;
  if (dflt) return pick_depth<VB, 1, 1024, 1, false, kInAddr, HALF>(depth);
  if constexpr (!HALF) {
    if (a.tiles == 1 && a.threads == 256 && a.minb == 0) return pick_depth<VB, 1, 256, 0>(depth);
    if (a.tiles == 1 && a.threads == 256 && a.minb == 4) return pick_depth<VB, 1, 256, 4>(depth);
    if (a.tiles == 2 && a.threads == 256 && a.minb == 0) return pick_depth<VB, 2, 256, 0>(depth);
    if (a.tiles == 1 && a.threads == 512 && a.minb == 2) return pick_depth<VB, 1, 512, 2>(depth);
  }
  return nullptr;
}

// The kernel for one next-hop width (see pick_kernel in lookup_params.hpp).
template <int VB>
KernelFn pick_kernel_t(const PickArgs& a) {
  if (a.half) {
    if constexpr (VB == 2) return pick_kernel_fmt<VB, true>(a);
    return nullptr;
  }
  return pick_kernel_fmt<VB, false>(a);
}

}  // namespace
