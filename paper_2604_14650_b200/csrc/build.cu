// Device-side FIB build: rules -> elementary intervals -> B200 layout, all on
// the GPU. The result is bit-identical to the host build
// (intervals.cpp + layout.cpp), which is bit-identical to the reference's
// build_intervals (intervals.cpp:33-93); tests compare all three.
//
// The host build is a sequential sweep. Here the same intervals are computed
// data-parallel from their definition: the boundaries are the
// distinct rule starts and ends below 2^64 plus 0, and the next hop of the
// interval starting at x is the longest-prefix match of x over the rules (or
// the default) — exactly the stack top the reference's sweep holds after all
// events at x (intervals.cpp:58-73). Steps (one stream; CUB radix sort,
// unique, select-if, reduce):
//   1. validate + extract (top, len, next hop); the first offending rule in
//      input order decides the error, as in the host build;
//   2. sort the rules by (length, top) — a per-length sorted table with
//      duplicates adjacent;
//   3. candidates = {0} + starts + ends below 2^64, radix-sorted and uniqued;
//   4. per candidate: LPM by binary search in each present length, longest first;
//   5. merge adjacent equal next hops (the first of each run is kept);
//   6. plan the layout on the host from m and the widest next hop, then fill
//      internal separators, leaf lines and the shared-memory image in parallel.
#include <cub/cub.cuh>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>

#include "capi_internal.hpp"
#include "lpm6/layout.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// The build's temporaries come from a library-private stream-ordered memory pool
// per device whose release threshold keeps up to 2 GiB reserved between builds.
// (The device's default pool releases its memory at every synchronization, so
// each rebuild of a FibStore commit would map its ~10^8 bytes of temporaries
// again.) The pool is created once per device and lives as long as the process.
cudaMemPool_t build_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) throw Error(Errc::CudaError, "device index out of range");
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    ck(cudaMemPoolCreate(&pools[device], &props), "cudaMemPoolCreate (device build)");
    uint64_t keep = 2ull << 30;
    ck(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
  }
  return pools[device];
}

}  // namespace

// Line arrays of device-built FIBs come from a second private pool that keeps all of
// its memory: a FibStore commit allocates one and retires another every time, and
// cudaMalloc / cudaFree map and unmap device memory through the driver, which took
// 30-80 ms per call in a process holding tens of GB (measured, tools/gpu/run22.sh).
cudaMemPool_t lpm6::capi::fib_line_pool(int device) {
  static std::mutex mu;
  static cudaMemPool_t pools[64] = {};
  if (device < 0 || device >= 64) throw Error(Errc::CudaError, "device index out of range");
  std::lock_guard<std::mutex> lk(mu);
  if (!pools[device]) {
    cudaMemPoolProps props{};
    props.allocType = cudaMemAllocationTypePinned;
    props.location.type = cudaMemLocationTypeDevice;
    props.location.id = device;
    ck(cudaMemPoolCreate(&pools[device], &props), "cudaMemPoolCreate (FIB lines)");
    uint64_t keep = ~0ull;
    ck(cudaMemPoolSetAttribute(pools[device], cudaMemPoolAttrReleaseThreshold, &keep), "cudaMemPoolSetAttribute");
  }
  return pools[device];
}

namespace {

// Device buffer owned for the duration of one build (stream-ordered, build_pool).
struct DBuf {
  void* p = nullptr;
  cudaStream_t s = nullptr;
  DBuf() = default;
  DBuf(size_t bytes, cudaStream_t stream) : s(stream) {
    if (!bytes) return;
    int dev = 0;
    ck(cudaGetDevice(&dev), "cudaGetDevice");
    ck(cudaMallocFromPoolAsync(&p, bytes, build_pool(dev), s), "cudaMallocFromPoolAsync (device build)");
  }
  DBuf(const DBuf&) = delete;
  DBuf& operator=(const DBuf&) = delete;
  DBuf(DBuf&& o) noexcept : p(o.p), s(o.s) { o.p = nullptr; }
  DBuf& operator=(DBuf&& o) noexcept {
    std::swap(p, o.p);
    std::swap(s, o.s);
    return *this;
  }
  ~DBuf() {
    if (p) cudaFreeAsync(p, s);
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
  void* release() {
    void* q = p;
    p = nullptr;
    return q;
  }
};

using u64d = unsigned long long;

// Per-rule error codes in the host build's check order (intervals.cpp).
enum : unsigned { kErrLen = 1, kErrReserved = 2, kErrCanonical = 3 };

struct BuildStatus {
  u64d first_bad;      // (rule index << 8) | code, min over rules; ~0 = none
  unsigned duplicate;  // a (top, len) pair occurs twice
  unsigned sentinel;   // a boundary would equal the sentinel key
};

unsigned blocks_for(u64d n) {
  const u64d b = (n + 255) / 256;
  return static_cast<unsigned>(b < 1 ? 1 : (b > 8192 ? 8192 : b));
}

__global__ void extract_kernel(const lpm6cu_prefix* rules, u64d n, u64d* top, unsigned* len, unsigned* nh,
                               unsigned* idx, u64d* cand, BuildStatus* st) {
  for (u64d i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    const lpm6cu_prefix r = rules[i];
    unsigned code = 0;
    if (r.length < 0 || r.length > 64) {
      code = kErrLen;
    } else if (r.next_hop == 0xFFFFFFFFu) {
      code = kErrReserved;
    } else {
      const u64d keep = r.length == 0 ? 0ull : (~0ull << (64 - r.length));
      if (r.value_lo != 0 || (r.value_hi & ~keep) != 0) code = kErrCanonical;
    }
    if (code) atomicMin(&st->first_bad, (i << 8) | code);
    const unsigned L = code ? 0u : static_cast<unsigned>(r.length);
    const u64d start = r.value_hi;
    top[i] = start;
    len[i] = L;
    nh[i] = r.next_hop;
    idx[i] = static_cast<unsigned>(i);
    // end = start + 2^(64-L); it is dropped when it equals 2^64 (written as 0,
    // which is always a boundary anyway).
    const u64d width_m1 = L == 0 ? ~0ull : ((1ull << (64 - L)) - 1);
    const bool end_is_top = start + width_m1 < start || start + width_m1 == ~0ull;
    const u64d end = end_is_top ? 0ull : start + width_m1 + 1;
    cand[i] = start;
    cand[n + i] = end;
    if (!code && (start == ~0ull || (!end_is_top && end == ~0ull))) st->sentinel = 1;
  }
}

__global__ void gather_u32_kernel(const unsigned* src, const unsigned* idx, u64d n, unsigned* dst) {
  for (u64d i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) dst[i] = src[idx[i]];
}

__global__ void gather_rules_kernel(const u64d* top, const unsigned* nh, const unsigned* idx, u64d n, u64d* top_out,
                                    unsigned* nh_out) {
  for (u64d i = blockIdx.x * 256ull + threadIdx.x; i < n; i += gridDim.x * 256ull) {
    top_out[i] = top[idx[i]];
    nh_out[i] = nh[idx[i]];
  }
}

// Duplicates are adjacent after sorting by (len, top).
__global__ void dup_kernel(const u64d* top, const unsigned* len, u64d n, BuildStatus* st) {
  for (u64d i = blockIdx.x * 256ull + threadIdx.x + 1; i < n; i += gridDim.x * 256ull)
    if (top[i] == top[i - 1] && len[i] == len[i - 1]) st->duplicate = 1;
}

// len_start[L] = first sorted rule whose length is >= L, L = 0..65.
__global__ void len_start_kernel(const unsigned* len, u64d n, u64d* len_start) {
  const unsigned L = threadIdx.x;
  if (L > 65) return;
  u64d lo = 0, cnt = n;
  while (cnt > 0) {
    const u64d h = cnt / 2;
    if (len[lo + h] < L) {
      lo += h + 1;
      cnt -= h + 1;
    } else {
      cnt = h;
    }
  }
  len_start[L] = lo;
}

// Longest-prefix match of each candidate boundary over the per-length tables.
__global__ void lpm_kernel(const u64d* cand, const u64d* m_raw, const u64d* top, const unsigned* nh_sorted,
                           const u64d* len_start, unsigned default_nh, unsigned* out) {
  __shared__ u64d ls[66];
  if (threadIdx.x < 66) ls[threadIdx.x] = len_start[threadIdx.x];
  __syncthreads();
  const u64d m = *m_raw;
  for (u64d i = blockIdx.x * 256ull + threadIdx.x; i < m; i += gridDim.x * 256ull) {
    const u64d x = cand[i];
    unsigned v = default_nh;
    for (int L = 64; L >= 0; --L) {
      u64d lo = ls[L], cnt = ls[L + 1] - ls[L];
      if (cnt == 0) continue;
      const u64d key = L == 0 ? 0ull : (x & (~0ull << (64 - L)));
      while (cnt > 0) {  // lower_bound
        const u64d h = cnt / 2;
        if (top[lo + h] < key) {
          lo += h + 1;
          cnt -= h + 1;
        } else {
          cnt = h;
        }
      }
      if (lo < ls[L + 1] && top[lo] == key) {
        v = nh_sorted[lo];
        break;
      }
    }
    out[i] = v;
  }
}

__global__ void merge_flags_kernel(const unsigned* nh, const u64d* m_raw, int merge, unsigned char* flag) {
  const u64d m = *m_raw;
  for (u64d i = blockIdx.x * 256ull + threadIdx.x; i < m; i += gridDim.x * 256ull)
    flag[i] = (!merge || i == 0 || nh[i] != nh[i - 1]) ? 1 : 0;
}

struct Geo {
  unsigned depth, kl, vb, image_levels, leaf_words;
  u64d m, leaf_nodes, image_start;
  u64d level_start[kMaxLevels];
  u64d span[kMaxLevels];  // boundaries under one child of a level-l node
};

__global__ void internal_kernel(const Geo g, const u64d* bnd, u64d* lines) {
  const u64d words = g.level_start[g.depth];
  for (u64d w = blockIdx.x * 256ull + threadIdx.x; w < words; w += gridDim.x * 256ull) {
    unsigned l = 0;
    while (l + 1 < g.depth && w >= g.level_start[l + 1]) ++l;
    const u64d off = w - g.level_start[l];
    const u64d n = off >> 4;
    const unsigned j = static_cast<unsigned>(off & 15u);
    u64d v = ~0ull;
    if (j < kNodeKeys) {
      const u64d idx = (n * 16u + j + 1) * g.span[l];
      if (idx < g.m) v = bnd[idx];
    }
    lines[w] = v;
  }
}

__global__ void leaf_kernel(const Geo g, const u64d* bnd, const unsigned* nh, u64d* lines) {
  for (u64d n = blockIdx.x * 256ull + threadIdx.x; n < g.leaf_nodes; n += gridDim.x * 256ull) {
    u64d words[16];
#pragma unroll
    for (int w = 0; w < 16; ++w) words[w] = 0;
    for (unsigned j = 0; j < g.kl; ++j) {
      const u64d s = n * g.kl + j;
      words[j] = s < g.m ? bnd[s] : ~0ull;
      const u64d v = nh[s < g.m ? s : g.m - 1];
      const unsigned byte = 8 * g.kl + g.vb * j;  // little-endian value bytes after the keys
      for (unsigned b = 0; b < g.vb; ++b)
        words[(byte + b) >> 3] |= ((v >> (8 * b)) & 0xFFull) << (8 * ((byte + b) & 7u));
    }
    u64d* line = lines + g.level_start[g.depth] + n * g.leaf_words;  // 16, or 8 for half-line leaves
    for (unsigned w = 0; w < g.leaf_words; ++w) line[w] = words[w];
  }
}

// Leaf image of a small tree (layout.hpp): leaf line words at a 17-word stride.
__global__ void leaf_image_kernel(const Geo g, u64d dst_start, u64d* lines) {
  const u64d words = g.leaf_nodes * 16;
  for (u64d t = blockIdx.x * 256ull + threadIdx.x; t < words; t += gridDim.x * 256ull)
    lines[dst_start + (t >> 4) * kLeafImageStride + (t & 15u)] = lines[g.level_start[g.depth] + t];
}

__global__ void image_kernel(const Geo g, u64d* lines) {
  const u64d nodes = g.level_start[g.image_levels] >> 4;  // nodes of levels [0, image_levels)
  for (u64d t = blockIdx.x * 256ull + threadIdx.x; t < nodes * kNodeKeys; t += gridDim.x * 256ull) {
    const u64d node = t / kNodeKeys;  // global node index = word offset / 16
    const unsigned p = static_cast<unsigned>(t % kNodeKeys);
    lines[g.image_start + node * kNodeKeys + p] = lines[node * 16 + p];
  }
}

bool is_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

struct DeviceIntervals {
  DBuf bnd, nh;  // m merged boundaries / next hops on the device
  u64d m = 0;
  unsigned max_nh = 0;
};

// Steps 1-5. Throws the host build's error for invalid rule sets.
DeviceIntervals device_intervals(const lpm6cu_prefix* rules, u64d n, unsigned default_nh, bool merge,
                                 cudaStream_t s) {
  const u64d nn = n ? n : 1, nc = 2 * n + 1;
  DBuf rules_owned;
  const lpm6cu_prefix* d_rules = rules;
  if (n && !is_device_ptr(rules)) {
    rules_owned = DBuf(n * sizeof(lpm6cu_prefix), s);
    ck(cudaMemcpyAsync(rules_owned.p, rules, n * sizeof(lpm6cu_prefix), cudaMemcpyHostToDevice, s), "H2D rules");
    d_rules = rules_owned.as<lpm6cu_prefix>();
  }
  DBuf top(nn * 8, s), top2(nn * 8, s), len(nn * 4, s), len2(nn * 4, s), len3(nn * 4, s), nh(nn * 4, s),
      nh2(nn * 4, s);
  DBuf idx(nn * 4, s), idx2(nn * 4, s), idx3(nn * 4, s);
  DBuf cand(nc * 8, s), cand2(nc * 8, s), nh_raw(nc * 4, s), flags(nc, s), st(sizeof(BuildStatus), s),
      len_start(66 * 8, s);
  DBuf d_m_raw(8, s), d_m(8, s), d_max(4, s);
  DeviceIntervals out;
  out.bnd = DBuf(nc * 8, s);
  out.nh = DBuf(nc * 4, s);

  const BuildStatus init{~0ull, 0, 0};
  capi::BuildTrace tr("intervals");
  ck(cudaMemcpyAsync(st.p, &init, sizeof init, cudaMemcpyHostToDevice, s), "H2D status");
  if (n)
    extract_kernel<<<blocks_for(n), 256, 0, s>>>(d_rules, n, top.as<u64d>(), len.as<unsigned>(), nh.as<unsigned>(),
                                                  idx.as<unsigned>(), cand.as<u64d>(), st.as<BuildStatus>());
  ck(cudaMemsetAsync(cand.as<u64d>() + 2 * n, 0, 8, s), "origin candidate");  // boundary 0
  ck(cudaGetLastError(), "extract");

  // CUB temporary storage: the max over every call below.
  size_t tmp_bytes = 0, t = 0;
  const int in = static_cast<int>(nn), ic = static_cast<int>(nc);
  cub::DeviceRadixSort::SortPairs(nullptr, t, top.as<u64d>(), top2.as<u64d>(), idx.as<unsigned>(),
                                  idx2.as<unsigned>(), in, 0, 64, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceRadixSort::SortPairs(nullptr, t, len2.as<unsigned>(), len3.as<unsigned>(), idx2.as<unsigned>(),
                                  idx3.as<unsigned>(), in, 0, 7, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceRadixSort::SortKeys(nullptr, t, cand.as<u64d>(), cand2.as<u64d>(), ic, 0, 64, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceSelect::Unique(nullptr, t, cand2.as<u64d>(), cand.as<u64d>(), d_m_raw.as<u64d>(), ic, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceSelect::Flagged(nullptr, t, cand.as<u64d>(), flags.as<unsigned char>(), out.bnd.as<u64d>(),
                             d_m.as<u64d>(), ic, s);
  tmp_bytes = std::max(tmp_bytes, t);
  cub::DeviceReduce::Max(nullptr, t, nh_raw.as<unsigned>(), d_max.as<unsigned>(), ic, s);
  tmp_bytes = std::max(tmp_bytes, t);
  DBuf tmp(tmp_bytes, s);

  if (n) {
    // 2. rules by (len, top): sort by top, gather lengths, stable sort by length.
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, top.as<u64d>(), top2.as<u64d>(), idx.as<unsigned>(),
                                       idx2.as<unsigned>(), static_cast<int>(n), 0, 64, s),
       "sort rules by top");
    gather_u32_kernel<<<blocks_for(n), 256, 0, s>>>(len.as<unsigned>(), idx2.as<unsigned>(), n, len2.as<unsigned>());
    ck(cub::DeviceRadixSort::SortPairs(tmp.p, tmp_bytes, len2.as<unsigned>(), len3.as<unsigned>(),
                                       idx2.as<unsigned>(), idx3.as<unsigned>(), static_cast<int>(n), 0, 7, s),
       "sort rules by length");
    gather_rules_kernel<<<blocks_for(n), 256, 0, s>>>(top.as<u64d>(), nh.as<unsigned>(), idx3.as<unsigned>(), n,
                                                      top2.as<u64d>(), nh2.as<unsigned>());
    dup_kernel<<<blocks_for(n), 256, 0, s>>>(top2.as<u64d>(), len3.as<unsigned>(), n, st.as<BuildStatus>());
  }
  len_start_kernel<<<1, 96, 0, s>>>(len3.as<unsigned>(), n, len_start.as<u64d>());
  ck(cudaGetLastError(), "rule table");

  // 3. candidate boundaries
  ck(cub::DeviceRadixSort::SortKeys(tmp.p, tmp_bytes, cand.as<u64d>(), cand2.as<u64d>(), ic, 0, 64, s), "sort cand");
  ck(cub::DeviceSelect::Unique(tmp.p, tmp_bytes, cand2.as<u64d>(), cand.as<u64d>(), d_m_raw.as<u64d>(), ic, s),
     "unique cand");
  // 4. LPM per candidate
  ck(cudaMemsetAsync(nh_raw.p, 0, nc * 4, s), "memset");
  lpm_kernel<<<blocks_for(nc), 256, 0, s>>>(cand.as<u64d>(), d_m_raw.as<u64d>(), top2.as<u64d>(), nh2.as<unsigned>(),
                                            len_start.as<u64d>(), default_nh, nh_raw.as<unsigned>());
  // 5. merge
  ck(cudaMemsetAsync(flags.p, 0, nc, s), "memset");
  merge_flags_kernel<<<blocks_for(nc), 256, 0, s>>>(nh_raw.as<unsigned>(), d_m_raw.as<u64d>(), merge ? 1 : 0,
                                                    flags.as<unsigned char>());
  ck(cudaGetLastError(), "lpm/merge");
  ck(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, cand.as<u64d>(), flags.as<unsigned char>(), out.bnd.as<u64d>(),
                                d_m.as<u64d>(), ic, s),
     "select boundaries");
  ck(cub::DeviceSelect::Flagged(tmp.p, tmp_bytes, nh_raw.as<unsigned>(), flags.as<unsigned char>(),
                                out.nh.as<unsigned>(), d_m.as<u64d>(), ic, s),
     "select next hops");
  ck(cub::DeviceReduce::Max(tmp.p, tmp_bytes, nh_raw.as<unsigned>(), d_max.as<unsigned>(), ic, s), "max");

  BuildStatus hs;
  ck(cudaMemcpyAsync(&hs, st.p, sizeof hs, cudaMemcpyDeviceToHost, s), "D2H status");
  ck(cudaMemcpyAsync(&out.m, d_m.p, 8, cudaMemcpyDeviceToHost, s), "D2H m");
  ck(cudaMemcpyAsync(&out.max_nh, d_max.p, 4, cudaMemcpyDeviceToHost, s), "D2H max");
  tr.mark("enqueue");
  ck(cudaStreamSynchronize(s), "device build");
  tr.mark("sync");
  if (hs.first_bad != ~0ull) {
    const u64d i = hs.first_bad >> 8;
    switch (hs.first_bad & 0xFF) {
      case kErrLen:
        throw Error(Errc::UnsupportedPrefixLength, "unsupported prefix length (rule " + std::to_string(i) + ")");
      case kErrReserved:
        throw Error(Errc::ReservedNextHop, "rule " + std::to_string(i) + " uses the reserved next hop");
      default:
        throw Error(Errc::InvalidArgument, "non-canonical prefix (host bits set), rule " + std::to_string(i));
    }
  }
  if (hs.duplicate) throw Error(Errc::DuplicatePrefix, "duplicate prefix in the rule set");
  if (hs.sentinel)
    throw Error(Errc::SentinelCollision, "rule set produces a boundary at the sentinel key ffff:ffff:ffff:ffff::");
  return out;
}

}  // namespace

namespace lpm6::capi {

namespace {

// Step 6: lay out m device-resident intervals; returns the cudaMalloc'ed line array.
void* device_layout(const DeviceIntervals& iv, u32 vb, u32 leaf_format, uint32_t default_nh, cudaStream_t s,
                    lpm6cu_geometry* geom) {
  TreeLayout t = plan_layout(iv.m, vb, leaf_format);
  t.default_next_hop = default_nh;
  Geo g{};
  g.depth = t.depth;
  g.kl = t.leaf_keys;
  g.vb = t.value_bytes;
  g.image_levels = t.image_levels;
  g.leaf_words = t.leaf_words;
  g.m = t.num_keys;
  g.leaf_nodes = t.leaf_nodes;
  g.image_start = t.image_start;
  u64d span = t.leaf_keys;
  for (int l = static_cast<int>(t.depth) - 1; l >= 0; --l) {
    g.span[l] = span;
    span *= t.b;
  }
  for (int l = 0; l < kMaxLevels; ++l) g.level_start[l] = t.level_start[l];
  void* lines_p = nullptr;  // long-lived: owned by the FIB handle (fib_line_pool, freed by free_fib_lines)
  BuildTrace tr("layout");
  int dev = 0;
  ck(cudaGetDevice(&dev), "cudaGetDevice");
  ck(cudaMallocFromPoolAsync(&lines_p, t.total_words * 8, fib_line_pool(dev), s), "allocate lines");
  tr.mark("alloc");
  struct Owned {
    void* p;
    cudaStream_t s;
    ~Owned() {
      if (p) cudaFreeAsync(p, s);
    }
  } lines{lines_p, s};
  ck(cudaMemsetAsync(lines.p, 0xFF, t.total_words * 8, s), "memset lines");  // sentinel everywhere first
  if (t.depth > 0)
    internal_kernel<<<blocks_for(t.level_start[t.depth]), 256, 0, s>>>(g, iv.bnd.as<u64d>(),
                                                                        static_cast<u64d*>(lines.p));
  leaf_kernel<<<blocks_for(t.leaf_nodes), 256, 0, s>>>(g, iv.bnd.as<u64d>(), iv.nh.as<unsigned>(),
                                                       static_cast<u64d*>(lines.p));
  if (t.image_levels > 0)
    image_kernel<<<blocks_for((t.level_start[t.image_levels] >> 4) * kNodeKeys), 256, 0, s>>>(
        g, static_cast<u64d*>(lines.p));
  if (t.leaf_image)
    leaf_image_kernel<<<blocks_for(t.leaf_nodes * 16), 256, 0, s>>>(g, leaf_image_start(t),
                                                                   static_cast<u64d*>(lines.p));
  ck(cudaGetLastError(), "layout fill");
  ck(cudaStreamSynchronize(s), "layout fill");
  export_geometry(t, geom);
  void* result = lines.p;
  lines.p = nullptr;
  return result;
}

u32 value_bytes_for(const lpm6cu_build_opts* opts, unsigned max_nh) {
  u32 vb = opts ? opts->value_bytes : 0;
  const u32 need = max_nh <= 0xFFu ? 1 : (max_nh <= 0xFFFFu ? 2 : 4);
  if (vb == 0) vb = need;
  if (vb != 1 && vb != 2 && vb != 4) throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
  if (vb < need)
    throw Error(Errc::InvalidArgument, "next hop " + std::to_string(max_nh) + " does not fit in " +
                                           std::to_string(vb) + " byte(s)");
  return vb;
}

}  // namespace

// Steps 1-6: a device-resident line array (caller frees with cudaFree) + its geometry.
void* device_build_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh, const lpm6cu_build_opts* opts,
                        cudaStream_t s, lpm6cu_geometry* geom) {
  const bool merge = opts ? opts->merge_adjacent != 0 : true;
  BuildTrace tr("device build");
  DeviceIntervals iv = device_intervals(rules, n, default_nh, merge, s);
  tr.mark("intervals");
  void* lines = device_layout(iv, value_bytes_for(opts, iv.max_nh), opts ? opts->leaf_format : 0u, default_nh, s, geom);
  tr.mark("layout");
  return lines;
}

// Step 6 only, from host intervals already validated by the caller (a loaded
// snapshot): one host->device copy of the boundaries and next hops.
void* device_build_tree_from_intervals(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                                       uint32_t default_nh, const lpm6cu_build_opts* opts, cudaStream_t s,
                                       lpm6cu_geometry* geom) {
  DeviceIntervals iv;
  iv.m = m;
  iv.bnd = DBuf(m * 8, s);
  iv.nh = DBuf(m * 4, s);
  for (uint64_t i = 0; i < m; ++i) iv.max_nh = std::max(iv.max_nh, next_hops[i]);
  ck(cudaMemcpyAsync(iv.bnd.p, boundaries, m * 8, cudaMemcpyHostToDevice, s), "H2D boundaries");
  ck(cudaMemcpyAsync(iv.nh.p, next_hops, m * 4, cudaMemcpyHostToDevice, s), "H2D next hops");
  return device_layout(iv, value_bytes_for(opts, iv.max_nh), opts ? opts->leaf_format : 0u, default_nh, s, geom);
}

}  // namespace lpm6::capi

extern "C" int lpm6cu_build_intervals_device(int device, const lpm6cu_prefix* rules, uint64_t n,
                                             uint32_t default_nh, int merge, uint64_t* boundaries,
                                             uint32_t* next_hops, uint64_t capacity, uint64_t* m_out) {
  return guard([&] {
    if (n > 0 && !rules) throw Error(Errc::InvalidArgument, "rules is NULL");
    if (capacity < 2 * n + 1) throw Error(Errc::InvalidArgument, "capacity must be >= 2n+1");
    ck(cudaSetDevice(device), "cudaSetDevice");
    DeviceIntervals iv = device_intervals(rules, n, default_nh, merge != 0, nullptr);
    ck(cudaMemcpy(boundaries, iv.bnd.p, iv.m * 8, cudaMemcpyDeviceToHost), "D2H boundaries");
    ck(cudaMemcpy(next_hops, iv.nh.p, iv.m * 4, cudaMemcpyDeviceToHost), "D2H next hops");
    *m_out = iv.m;
  });
}
