// sm_100a batched LPM lookup kernels and the device half of the C ABI.
//
// One query = one predecessor search down the compact 16-key / 128-byte-node
// tree (layout.hpp). The kernel is the GPU form of the reference's
// search_batch + Listing 1:
//
//  * a group of G lanes (G = 4, 8 or 16) cooperates on one node: lane j holds
//    keys [j*16/G, (j+1)*16/G) of the node, so one warp-wide load instruction
//    fetches one full 128-byte line per query (256-bit LDG for G = 4);
//  * the node rank is computed branch-free: every lane compares its keys
//    against the broadcast query, then __ballot_sync/__popc (G = 8, 16) or a
//    two-step shuffle sum (G = 4) gives the count of keys <= query — the rank
//    of Listing 1's cmpge-mask + popcnt;
//  * each group carries G queries at once and the descent is fully unrolled
//    over the tree depth (template), so every level issues G independent node
//    loads per group before the first compare (the batching of P:812-847 as
//    memory-level parallelism);
//  * the top `smem_levels` levels are staged into shared memory once per CTA
//    with cp.async.bulk (TMA bulk copy) on an mbarrier; deeper levels are read
//    through L2 (the whole 1M-prefix tree fits in B200's L2);
//  * query addresses are read with coalesced 16-byte loads (one per lane,
//    L1::no_allocate, L2 evict_first) and next hops written with coalesced
//    streaming stores; lane L of a warp owns query L of the warp's 32-query tile;
//  * CTAs are persistent (grid = SMs x resident CTAs) and stride over tiles.
//
// Results are the reference's: key = min(addr >> 64, 0xFFFF...FFFE)
// (types.hpp:25), internal child = node * 17 + rank, leaf ordinal =
// leaf_node * 16 + rank - 1, next hop = values[ordinal].
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
constexpr int kK = 16;  // keys per node

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

template <int KPL>
__device__ __forceinline__ void ld_node_global(const unsigned long long* p, unsigned long long (&k)[KPL]) {
  if constexpr (KPL == 1) {
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(k[0]) : "l"(p));
  } else if constexpr (KPL == 2) {
    asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(k[0]), "=l"(k[1]) : "l"(p));
  } else {
    asm volatile("ld.global.nc.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(k[0]), "=l"(k[1]), "=l"(k[2]), "=l"(k[3])
                 : "l"(p));
  }
}

template <int KPL>
__device__ __forceinline__ void ld_node_shared(const unsigned long long* p, unsigned long long (&k)[KPL]) {
  const uint32_t a = smem_u32(p);
  if constexpr (KPL == 1) {
    asm volatile("ld.shared.u64 %0, [%1];" : "=l"(k[0]) : "r"(a));
  } else if constexpr (KPL == 2) {
    asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(k[0]), "=l"(k[1]) : "r"(a));
  } else {
    asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(k[0]), "=l"(k[1]) : "r"(a));
    asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];" : "=l"(k[2]), "=l"(k[3]) : "r"(a + 16));
  }
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
  const unsigned long long* keys;
  const unsigned char* values;
  unsigned long long level_start[LPM6CU_MAX_LEVELS];
  const uint4* addrs;
  unsigned char* out;
  unsigned long long n;
  unsigned int smem_levels;  // levels [0, smem_levels) read from shared memory
  unsigned int smem_bytes;   // = level_start[smem_levels] * 8
  unsigned int value_bytes;
};

// Count of node keys <= q across the G lanes of this group (Listing 1's
// popcnt(cmpge(q, node))). Every lane of the group gets the same value.
template <int G, int KPL>
__device__ __forceinline__ unsigned group_rank(unsigned long long q, const unsigned long long (&k)[KPL],
                                               unsigned gmask) {
  if constexpr (KPL <= 2) {
    unsigned r = 0;
#pragma unroll
    for (int t = 0; t < KPL; ++t) r += __popc(__ballot_sync(kFull, q >= k[t]) & gmask);
    return r;
  } else {
    unsigned c = 0;
#pragma unroll
    for (int t = 0; t < KPL; ++t) c += (q >= k[t]) ? 1u : 0u;
#pragma unroll
    for (int o = 1; o < G; o <<= 1) c += __shfl_xor_sync(kFull, c, o, G);
    return c;
  }
}

template <int G, int DEPTH>
__global__ void __launch_bounds__(256) lpm6_lookup_kernel(const LookupParams p) {
  constexpr int KPL = kK / G;  // keys per lane
  constexpr int Q = G;         // queries in flight per group: lane L owns query L of the tile
  extern __shared__ __align__(128) unsigned long long s_keys[];
  __shared__ __align__(8) uint64_t s_bar;

  if (p.smem_bytes > 0) {
    if (threadIdx.x == 0) {
      mbar_init(&s_bar, 1);
      mbar_arrive_expect_tx(&s_bar, p.smem_bytes);
      constexpr uint32_t kChunk = 32768;
      for (uint32_t off = 0; off < p.smem_bytes; off += kChunk) {
        const uint32_t sz = min(kChunk, p.smem_bytes - off);
        bulk_g2s(reinterpret_cast<char*>(s_keys) + off, reinterpret_cast<const char*>(p.keys) + off, sz,
                 &s_bar);
      }
    }
    __syncthreads();
    mbar_wait(&s_bar, 0);
  }

  const unsigned lane = threadIdx.x & 31u;
  const unsigned j = lane & (G - 1);
  const unsigned gmask = (G == 32 ? kFull : ((1u << G) - 1u)) << (lane & ~(G - 1u));
  const unsigned long long warp0 = (static_cast<unsigned long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const unsigned long long nwarps = (static_cast<unsigned long long>(gridDim.x) * blockDim.x) >> 5;
  const uint64_t pol_stream = policy_evict_first();
  const unsigned T = p.smem_levels;

  for (unsigned long long tile = warp0; tile * 32ull < p.n; tile += nwarps) {
    const unsigned long long qi = tile * 32ull + lane;
    unsigned long long key = 0;
    if (qi < p.n) {
      const uint4 a = ld_stream_v4(p.addrs + qi, pol_stream);
      key = (static_cast<unsigned long long>(a.w) << 32) | a.z;  // top 64 bits of the u128
    }
    key = key > kMaxQueryKey ? kMaxQueryKey : key;  // types.hpp:25

    unsigned long long qk[Q];
    unsigned node[Q];
#pragma unroll
    for (int s = 0; s < Q; ++s) {
      qk[s] = __shfl_sync(kFull, key, s, G);
      node[s] = 0;
    }

#pragma unroll
    for (int l = 0; l <= DEPTH; ++l) {
      unsigned long long kk[Q][KPL];
      if (static_cast<unsigned>(l) < T) {
        const unsigned long long* lvl = s_keys + p.level_start[l];
#pragma unroll
        for (int s = 0; s < Q; ++s) ld_node_shared<KPL>(lvl + node[s] * kK + j * KPL, kk[s]);
      } else {
        const unsigned long long* lvl = p.keys + p.level_start[l];
#pragma unroll
        for (int s = 0; s < Q; ++s) ld_node_global<KPL>(lvl + node[s] * kK + j * KPL, kk[s]);
      }
#pragma unroll
      for (int s = 0; s < Q; ++s) {
        const unsigned r = group_rank<G, KPL>(qk[s], kk[s], gmask);
        node[s] = (l < DEPTH) ? node[s] * (kK + 1) + r : node[s] * kK + r - 1;
      }
    }

    unsigned ord = node[0];
#pragma unroll
    for (int s = 1; s < Q; ++s) ord = (j == static_cast<unsigned>(s)) ? node[s] : ord;

    if (qi < p.n) {
      if (p.value_bytes == 1) {
        const unsigned char v = __ldg(p.values + ord);
        asm volatile("st.global.cs.u8 [%0], %1;" ::"l"(p.out + qi), "h"(static_cast<unsigned short>(v)));
      } else if (p.value_bytes == 2) {
        const unsigned short v = __ldg(reinterpret_cast<const unsigned short*>(p.values) + ord);
        asm volatile("st.global.cs.u16 [%0], %1;" ::"l"(p.out + 2 * qi), "h"(v));
      } else {
        const unsigned v = __ldg(reinterpret_cast<const unsigned*>(p.values) + ord);
        asm volatile("st.global.cs.u32 [%0], %1;" ::"l"(p.out + 4 * qi), "r"(v));
      }
    }
  }
}

using KernelFn = void (*)(const LookupParams);

template <int G>
KernelFn pick_depth(int depth) {
  switch (depth) {
    case 0: return lpm6_lookup_kernel<G, 0>;
    case 1: return lpm6_lookup_kernel<G, 1>;
    case 2: return lpm6_lookup_kernel<G, 2>;
    case 3: return lpm6_lookup_kernel<G, 3>;
    case 4: return lpm6_lookup_kernel<G, 4>;
    case 5: return lpm6_lookup_kernel<G, 5>;
    case 6: return lpm6_lookup_kernel<G, 6>;
    case 7: return lpm6_lookup_kernel<G, 7>;
    default: return nullptr;
  }
}

KernelFn pick_kernel(int g, int depth) {
  switch (g) {
    case 4: return pick_depth<4>(depth);
    case 8: return pick_depth<8>(depth);
    case 16: return pick_depth<16>(depth);
    default: return nullptr;
  }
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

struct lpm6cu_fib {
  int device = 0;
  lpm6cu_geometry g{};
  unsigned long long* d_keys = nullptr;
  unsigned char* d_values = nullptr;
  bool owns = true;
  lpm6cu_kernel_config cfg{};  // resolved
  int num_sms = 0;
  size_t max_smem_optin = 0;
  std::mutex host_mu;
  std::unique_ptr<HostPipeline> pipe;

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
    if (owns) {
      if (d_keys) cudaFree(d_keys);
      if (d_values) cudaFree(d_values);
    }
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

// Resolve automatic kernel settings against the device and the tree.
void resolve_config(lpm6cu_fib* f, const lpm6cu_kernel_config* req) {
  lpm6cu_kernel_config c{};
  if (req) c = *req;
  if (c.lanes_per_query == 0) c.lanes_per_query = 8;
  if (c.lanes_per_query != 4 && c.lanes_per_query != 8 && c.lanes_per_query != 16)
    throw Error(Errc::InvalidArgument, "lanes_per_query must be 4, 8 or 16");
  if (c.threads_per_cta == 0) c.threads_per_cta = 256;
  if (c.threads_per_cta != 256) throw Error(Errc::InvalidArgument, "threads_per_cta must be 256");
  const unsigned levels = f->g.depth + 1;
  const size_t budget = std::min<size_t>(f->max_smem_optin, 200 * 1024);
  if (req == nullptr || req->smem_levels == 0xFF) {
    // Auto: stage the deepest prefix of levels that fits 48 KiB (keeps >= 4 CTAs/SM).
    unsigned t = 0;
    for (unsigned cand = 1; cand <= levels; ++cand) {
      const unsigned long long bytes = (cand >= levels ? f->g.total_keys : f->g.level_start[cand]) * 8ull;
      if (bytes > 48 * 1024) break;
      t = cand;
    }
    c.smem_levels = t;
  }
  if (c.smem_levels > levels) c.smem_levels = levels;
  const unsigned long long staged =
      c.smem_levels == 0 ? 0
                         : (c.smem_levels >= levels ? f->g.total_keys : f->g.level_start[c.smem_levels]) * 8ull;
  if (staged > budget)
    throw Error(Errc::InvalidArgument, "smem_levels=" + std::to_string(c.smem_levels) + " needs " +
                                           std::to_string(staged) + " B of shared memory");
  f->cfg = c;
}

unsigned long long staged_bytes(const lpm6cu_fib* f) {
  const unsigned levels = f->g.depth + 1;
  const unsigned T = f->cfg.smem_levels;
  if (T == 0) return 0;
  return (T >= levels ? f->g.total_keys : f->g.level_start[T]) * 8ull;
}

void launch_lookup(const lpm6cu_fib* f, const void* d_addrs, unsigned long long n, void* d_out,
                   cudaStream_t stream) {
  if (n == 0) return;
  KernelFn fn = pick_kernel(static_cast<int>(f->cfg.lanes_per_query), static_cast<int>(f->g.depth));
  if (!fn) throw Error(Errc::InvalidArgument, "no kernel for depth " + std::to_string(f->g.depth));
  LookupParams p{};
  p.keys = f->d_keys;
  p.values = f->d_values;
  for (int l = 0; l < LPM6CU_MAX_LEVELS; ++l) p.level_start[l] = f->g.level_start[l];
  p.addrs = static_cast<const uint4*>(d_addrs);
  p.out = static_cast<unsigned char*>(d_out);
  p.n = n;
  p.smem_bytes = static_cast<unsigned>(staged_bytes(f));
  p.smem_levels = f->cfg.smem_levels;
  p.value_bytes = f->g.value_bytes;
  const int threads = static_cast<int>(f->cfg.threads_per_cta);
  const size_t smem = p.smem_bytes;
  if (smem > 48 * 1024)
    check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)),
               "cudaFuncSetAttribute");
  int per_sm = 0;
  check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, threads, smem), "occupancy");
  if (per_sm < 1) throw Error(Errc::CudaError, "lookup kernel cannot be resident with this configuration");
  if (f->cfg.ctas_per_sm > 0) per_sm = std::min<int>(per_sm, static_cast<int>(f->cfg.ctas_per_sm));
  const unsigned long long tiles = (n + 31) / 32;
  const unsigned long long warps_per_cta = threads / 32;
  unsigned long long grid = static_cast<unsigned long long>(f->num_sms) * per_sm;
  grid = std::min(grid, (tiles + warps_per_cta - 1) / warps_per_cta);
  fn<<<static_cast<unsigned>(grid), threads, smem, stream>>>(p);
  check_cuda(cudaGetLastError(), "lookup launch");
}

lpm6cu_fib* new_fib(int device, const lpm6cu_geometry* g) {
  if (!g) throw Error(Errc::InvalidArgument, "geometry is NULL");
  if (g->k != kK) throw Error(Errc::InvalidArgument, "the kernels take k = 16");
  if (g->depth > kMaxKernelDepth) throw Error(Errc::InvalidArgument, "tree depth above 7");
  if (g->value_bytes != 1 && g->value_bytes != 2 && g->value_bytes != 4)
    throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
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

int lpm6cu_fib_create(int device, const lpm6cu_geometry* g, const uint64_t* keys, const void* values,
                      lpm6cu_fib** out) {
  return guard([&] {
    if (!keys || !values || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, g));
    const size_t kbytes = g->total_keys * 8;
    const size_t vbytes = g->leaf_nodes * kK * g->value_bytes;
    check_cuda(cudaMalloc(&f->d_keys, kbytes), "cudaMalloc keys");
    check_cuda(cudaMalloc(&f->d_values, vbytes), "cudaMalloc values");
    check_cuda(cudaMemcpy(f->d_keys, keys, kbytes, cudaMemcpyHostToDevice), "copy keys");
    check_cuda(cudaMemcpy(f->d_values, values, vbytes, cudaMemcpyHostToDevice), "copy values");
    *out = f.release();
  });
}

int lpm6cu_fib_wrap_device(int device, const lpm6cu_geometry* g, const void* d_keys, const void* d_values,
                           lpm6cu_fib** out) {
  return guard([&] {
    if (!d_keys || !d_values || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    DeviceGuard dg(device);
    std::unique_ptr<lpm6cu_fib> f(new_fib(device, g));
    f->d_keys = static_cast<unsigned long long*>(const_cast<void*>(d_keys));
    f->d_values = static_cast<unsigned char*>(const_cast<void*>(d_values));
    f->owns = false;
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
    check_cuda(cudaMalloc(&f->d_keys, t.keys.size() * 8), "cudaMalloc keys");
    check_cuda(cudaMalloc(&f->d_values, t.values.size()), "cudaMalloc values");
    check_cuda(cudaMemcpy(f->d_keys, t.keys.data(), t.keys.size() * 8, cudaMemcpyHostToDevice), "copy keys");
    check_cuda(cudaMemcpy(f->d_values, t.values.data(), t.values.size(), cudaMemcpyHostToDevice), "copy values");
    *out = f.release();
  });
}

int lpm6cu_fib_geometry(const lpm6cu_fib* f, lpm6cu_geometry* g) {
  return guard([&] {
    if (!f || !g) throw Error(Errc::InvalidArgument, "NULL argument");
    *g = f->g;
  });
}

int lpm6cu_fib_device_arrays(const lpm6cu_fib* f, const void** k, const void** v) {
  return guard([&] {
    if (!f) throw Error(Errc::InvalidArgument, "NULL fib");
    if (k) *k = f->d_keys;
    if (v) *v = f->d_values;
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
