// Host half of the lookup: the FIB handle (lpm6cu_fib), kernel selection and
// launch, the host-buffer pipeline, the query generator and the C ABI of
// include/lpm6cu.h. The kernels are in lookup_kernel.cuh, instantiated per next-hop
// width in lookup_vb{1,2,4}.cu.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "capi_internal.hpp"
#include "lookup_params.hpp"
#include "lpm6/workload.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using namespace lpm6::kern;
using lpm6::capi::guard;

namespace {

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
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

// The staged image re-laid out for the split-plane Phase A (lookup_kernel.cuh PLANES):
// levels below `pu` as a plane of high words followed by a plane of low words, the
// others word for word. lvl_w[l] = first image word of level l (lvl_w[levels] = the end).
struct PlaneLevels {
  unsigned lvl_w[LPM6CU_MAX_LEVELS + 1];
  unsigned levels, pu;
};
__global__ void lpm6_planes_kernel(const unsigned long long* image, unsigned* out, const PlaneLevels pl) {
  const unsigned total = pl.lvl_w[pl.levels];
  for (unsigned w = blockIdx.x * blockDim.x + threadIdx.x; w < total; w += gridDim.x * blockDim.x) {
    unsigned l = 0;
    while (l + 1 < pl.levels && w >= pl.lvl_w[l + 1]) ++l;
    const unsigned long long k = image[w];
    if (l < pl.pu) {
      const unsigned w0 = pl.lvl_w[l], nw = pl.lvl_w[l + 1] - w0;
      out[2 * w0 + (w - w0)] = static_cast<unsigned>(k >> 32);
      out[2 * w0 + nw + (w - w0)] = static_cast<unsigned>(k);
    } else {
      out[2 * w] = static_cast<unsigned>(k);
      out[2 * w + 1] = static_cast<unsigned>(k >> 32);
    }
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
  bool pooled = false;  // d_lines from capi::fib_line_pool (device builds): cudaFreeAsync, no unmap
  bool quiesced = false;  // the owner knows no lookup can still read d_lines (FibStore reclaim)
  lpm6cu_kernel_config cfg{};  // resolved
  int num_sms = 0;
  size_t max_smem_optin = 0;
  std::mutex host_mu;
  std::unique_ptr<HostPipeline> pipe;
  std::mutex plan_mu;
  LaunchPlan plans[4][2];  // [input format][checked]
  unsigned long long root[16] = {};  // host copy of the root line (kernel parameter)
  cudaTextureObject_t tex = 0;       // texture object over the line array
  cudaStream_t zc_stream = nullptr;  // zero-copy host path (small pinned batches)
  cudaEvent_t zc_event = nullptr;
  bool root_ready = false;
  unsigned* d_planes = nullptr;  // the staged image as split planes (cfg.plane_levels >= 2), from fib_line_pool
  unsigned planes_pu = 0;        // the plane_levels d_planes was laid out for

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
    if (zc_stream) cudaStreamDestroy(zc_stream);
    if (zc_event) cudaEventDestroy(zc_event);
    if (owns && d_lines) {
      if (pooled) {
        // cudaFree would have waited for the whole device; keep that guarantee for a
        // plain destroy, and let an owner that already fenced its readers skip it.
        if (!quiesced) cudaDeviceSynchronize();
        cudaFreeAsync(d_lines, nullptr);
      } else {
        cudaFree(d_lines);
      }
    }
    if (d_err) cudaFree(d_err);
    if (d_planes) {
      if (!quiesced) cudaDeviceSynchronize();
      cudaFreeAsync(d_planes, nullptr);
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

// A non-blocking stream per device for the plane-image kernel: the legacy default stream
// would also wait for whatever the caller's blocking streams have queued (a store commit
// carries the kernel config to the new FIB while readers keep looking up).
cudaStream_t planes_stream(int device) {
  static std::mutex mu;
  static cudaStream_t streams[64] = {};
  std::lock_guard<std::mutex> lk(mu);
  if (device < 0 || device >= 64) return nullptr;
  if (!streams[device]) check_cuda(cudaStreamCreateWithFlags(&streams[device], cudaStreamNonBlocking), "planes stream");
  return streams[device];
}

// (Re)build the plane image for f->cfg.plane_levels (a no-op when it is current or not
// asked for). Synchronous: the tuning / configuration calls are not on the lookup path.
void ensure_planes(lpm6cu_fib* f) {
  const unsigned pu = f->cfg.plane_levels;
  if (pu < 2 || !f->d_lines || (f->d_planes && f->planes_pu == pu)) return;
  const unsigned levels = std::min<unsigned>(f->g.image_levels, f->g.depth);
  PlaneLevels pl{};
  pl.levels = levels;
  pl.pu = pu;
  for (unsigned l = 0; l <= levels; ++l)
    pl.lvl_w[l] = static_cast<unsigned>(f->g.level_start[l] / kLineWords * kNodeKeys);
  const size_t bytes = static_cast<size_t>(pl.lvl_w[levels]) * 8;
  if (bytes == 0) return;
  DeviceGuard dg(f->device);
  const cudaStream_t st = planes_stream(f->device);
  if (!f->d_planes)
    check_cuda(cudaMallocFromPoolAsync(reinterpret_cast<void**>(&f->d_planes), (bytes + 15) / 16 * 16,
                                       capi::fib_line_pool(f->device), st),
               "cudaMallocFromPoolAsync planes");
  lpm6_planes_kernel<<<32, 256, 0, st>>>(f->d_lines + f->g.image_start, f->d_planes, pl);
  check_cuda(cudaGetLastError(), "planes launch");
  check_cuda(cudaStreamSynchronize(st), "planes sync");
  f->planes_pu = pu;
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
  // 2 or 4 tiles per warp at 1024 threads: Phase A overlaps the tiles' probe chains, Phase B
  // takes one tile at a time (texture leaf paths 1 and 4; other plans run one tile)
  const bool two_tiles = (c.queries_per_lane == 2 || c.queries_per_lane == 4) && c.threads_per_cta == 1024 &&
                         c.min_ctas_per_sm == 1;
  if (!two_tiles && !pick_kernel(1, 0, static_cast<int>(c.queries_per_lane), static_cast<int>(c.threads_per_cta),
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
  if (c.line_path > 4) throw Error(Errc::InvalidArgument, "line_path must be 0..4");
  if (c.smem_levels > tmax) c.smem_levels = tmax;
  const unsigned long long staged = image_bytes_of(f->g, c.smem_levels);
  if (staged > budget)
    throw Error(Errc::InvalidArgument, "smem_levels=" + std::to_string(c.smem_levels) + " needs " +
                                           std::to_string(staged) + " B of shared memory");
  // Split-plane Phase A: levels 1 .. plane_levels - 1; 0 or 1 = none, clamped to the staged levels.
  if (c.plane_levels > LPM6CU_MAX_LEVELS) throw Error(Errc::InvalidArgument, "plane_levels above the level count");
  // The kernels exist for P = 2, 3 and every staged level (reported as smem_levels).
  if (c.plane_levels < 2 || c.smem_levels < 2 || c.smem_levels > depth) c.plane_levels = 0;
  if (c.plane_levels >= c.smem_levels) c.plane_levels = c.smem_levels;
  else if (c.plane_levels > 3) c.plane_levels = 3;
  f->cfg = c;
  f->invalidate_plans();
  ensure_planes(f);
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
  // The kernels store a 4-query group's next hops with one 4*vb-byte store, so the
  // result buffer must be 4*vb-byte aligned. A caller's pointer at any other byte
  // offset (a slice of a byte buffer) gets a stream-ordered aligned scratch buffer
  // and a device-to-device copy; the aligned fast path is unchanged.
  const unsigned long long vb_out = f->g.value_bytes;
  if (d_out && reinterpret_cast<uintptr_t>(d_out) % (4 * vb_out) != 0) {
    void* tmp = nullptr;
    check_cuda(cudaMallocAsync(&tmp, n * vb_out, stream), "cudaMallocAsync (unaligned result buffer)");
    try {
      launch_lookup(f, d_in, n, tmp, stream, input, pk, d_ord);
      check_cuda(cudaMemcpyAsync(d_out, tmp, n * vb_out, cudaMemcpyDefault, stream), "copy results");
    } catch (...) {
      cudaFreeAsync(tmp, stream);
      throw;
    }
    check_cuda(cudaFreeAsync(tmp, stream), "cudaFreeAsync");
    return;
  }
  const bool dflt = input != kInAddr;
  const unsigned tiles_cfg = dflt ? 1 : f->cfg.queries_per_lane;
  const unsigned threads_cta = dflt ? 1024 : f->cfg.threads_per_cta;
  const unsigned minb = dflt ? 1 : f->cfg.min_ctas_per_sm;
  // Leaf-image mode serves address input; key / packet input uses the internal image only.
  const bool leafs = leaf_image_mode(f) && input == kInAddr;
  // Texture pipe for internal L2 levels when the tree has any (smem_levels < depth).
  const unsigned smem_levels = leaf_image_mode(f) && !leafs ? f->g.depth : f->cfg.smem_levels;
  // texture line paths: the default shape, and 2 or 4 tiles per warp at 1024 threads (address input)
  const bool tex_shape = threads_cta == 1024 && minb == 1 && (tiles_cfg == 1 || input == kInAddr);
  const bool texl = f->tex && !leafs && input != kInKeyOrd && f->d_err == nullptr && smem_levels < f->g.depth &&
                    tex_shape && f->g.depth >= 2;
  // Line path plan (lpm6cu_kernel_config.line_path): 0 LSU leaves, 1 texture leaves,
  // 2 split leaves, 3 texture leaves + split internal L2 levels, 4 texture leaves
  // with the select extraction of 1-byte next hops (= 1 for wider next hops).
  const int plan_lp = static_cast<int>(f->cfg.line_path);
  // Packet input follows the line path only with half-line leaves: measured on the
  // bench's 64-byte frames, texture leaves take C2 from 53.9 to 58.0 G/s but C1 (full
  // 1-byte-next-hop leaf lines) from 56.5 down to 49.5 (tools/gpu/run24.sh).
  const bool path_input = input == kInAddr || input == kInKey ||
                          (input == kInPacket && f->g.leaf_words == kHalfLeafWords);
  const int leaftex = plan_lp != 0 && f->tex && !leafs && path_input &&
                              f->d_err == nullptr && tex_shape && f->g.depth >= 1
                          ? (plan_lp == 2 ? 2 : (plan_lp == 4 && f->g.value_bytes == 1) ? 3 : 1)
                          : 0;
  const int texl_mode = !texl ? 0 : (plan_lp == 3 && leaftex == 1) ? 2 : 1;
  // 2 or 4 tiles per warp at 1024 threads exist for texture leaves (paths 1 and 4) with
  // internal L2 levels on one pipe; any other plan of such a config runs one tile.
  const unsigned tiles = threads_cta == 1024 && tiles_cfg > 1 && !((leaftex == 1 || leaftex == 3) && texl_mode <= 1)
                             ? 1u
                             : tiles_cfg;
  const size_t smem = image_bytes_of(f->g, smem_levels);
  const int threads = static_cast<int>(threads_cta);
  // Split-plane Phase A: the 2- and 4-tile kernels of the texture leaf paths, when the
  // plane image is laid out for the configured level count.
  const bool planes_on = tiles > 1 && threads_cta == 1024 && f->cfg.plane_levels >= 2 && f->d_planes != nullptr &&
                         f->planes_pu == f->cfg.plane_levels && smem_levels >= 2 && f->g.depth >= 3 &&
                         (smem_levels == f->g.depth || smem_levels + 1 == f->g.depth);
  const unsigned pu = std::min<unsigned>(f->cfg.plane_levels, smem_levels);
  const int planes = !planes_on ? 0 : pu >= smem_levels ? kAllPlanes : pu >= 3 ? 3 : 2;
  LaunchPlan plan;
  {
    auto* mf = const_cast<lpm6cu_fib*>(f);
    std::lock_guard<std::mutex> lk(mf->plan_mu);
    LaunchPlan& slot = mf->plans[input][f->d_err != nullptr ? 1 : 0];
    if (!slot.valid) {
      KernelFn fn = pick_kernel(static_cast<int>(f->g.value_bytes), static_cast<int>(f->g.depth),
                                static_cast<int>(tiles), threads, static_cast<int>(minb), f->d_err != nullptr, input,
                                leafs, texl_mode, leaftex, f->g.leaf_words == kHalfLeafWords,
                                static_cast<int>(std::min<unsigned>(smem_levels, f->g.depth)), planes);
      if (!fn) throw Error(Errc::InvalidArgument, "no kernel instantiated for this configuration");
      // The attribute belongs to the kernel, which every FIB of this depth and
      // next-hop width shares: always set it to the device's opt-in maximum, never
      // to this FIB's own image size, so that no FIB can lower it under another.
      if (smem > 48 * 1024)
        check_cuda(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(f->max_smem_optin)),
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
  if (planes) {
    auto offb = [&](unsigned l) { return static_cast<unsigned>((f->g.level_start[l] / kLineWords) * kNodeKeys * 8); };
    p.image = reinterpret_cast<const unsigned long long*>(f->d_planes);
    for (unsigned l = 0; l < smem_levels; ++l)
      p.lo_delta[l] = static_cast<unsigned>((f->g.level_start[l + 1] - f->g.level_start[l]) / kLineWords * kNodeKeys * 4);
    if (pu < smem_levels) p.pl2pk = offb(pu) - 32u * offb(pu - 1);
  }
  for (int l = 0; l < LPM6CU_MAX_LEVELS; ++l) p.level_nodes[l] = f->g.level_nodes[l];
  p.err = f->d_err;
  std::memcpy(p.root, f->root, sizeof p.root);
  p.tex = f->tex;
  {
    auto off = [&](unsigned l) { return static_cast<unsigned>((f->g.level_start[l] / kLineWords) * kNodeKeys * 8); };
    const unsigned ta = p.smem_levels;
    p.img_step[0] = ta >= 2 ? off(1) : 0u;
    for (unsigned l = 1; l < ta; ++l) p.img_step[l] = l + 1 < ta ? off(l + 1) - 16u * off(l) : 0u - 16u * off(l);
  }
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
  const unsigned lw = g->leaf_words ? g->leaf_words : kLineWords;  // 0: a geometry from before leaf_words
  if (lw == kLineWords ? g->leaf_keys != leaf_keys_for(g->value_bytes)
                       : (lw != kHalfLeafWords || g->leaf_keys != kHalfLeafKeys || g->value_bytes != 2))
    throw Error(Errc::InvalidArgument, "leaf_keys / leaf_words mismatch");
  if (lw != kLineWords && g->leaf_image) throw Error(Errc::InvalidArgument, "a leaf image needs full leaf lines");
  if (g->depth > kMaxKernelDepth) throw Error(Errc::InvalidArgument, "tree depth above 7");
  if (g->value_bytes != 1 && g->value_bytes != 2 && g->value_bytes != 4)
    throw Error(Errc::InvalidArgument, "value_bytes must be 1, 2 or 4");
  // The geometry must describe a line array that holds what the kernels will read.
  if (g->image_levels > g->depth || g->level_start[g->depth] + g->leaf_nodes * lw > g->image_start)
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
  f->g.leaf_words = lw;
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
  // The root line (a half-line leaf when the whole tree is one leaf: fewer than 128 bytes).
  std::memset(f->root, 0xFF, sizeof f->root);
  const size_t root_bytes = std::min<size_t>(sizeof f->root, static_cast<size_t>(f->g.total_words) * 8);
  check_cuda(cudaMemcpy(f->root, f->d_lines, root_bytes, cudaMemcpyDeviceToHost), "read root line");
  f->root_ready = true;
}

// True for device (or managed) memory. Device memory must be on the FIB's own
// device: the kernel would fault on another GPU's allocation (no peer mapping is
// assumed), which poisons the whole CUDA context, so that is rejected here.
bool is_device_ptr(const void* p, int device) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice && a.device != device)
    throw Error(Errc::InvalidArgument, "buffer is on CUDA device " + std::to_string(a.device) +
                                           ", the FIB on device " + std::to_string(device));
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// Device address of page-locked, mapped host memory (cudaMallocHost /
// cudaHostAlloc / cudaHostRegister), or nullptr for pageable memory.
void* mapped_device_ptr(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

// Batches up to this many queries in pinned host memory are served zero-copy:
// the kernel reads the addresses and writes the next hops over PCIe itself, so
// a call is one launch and one sync instead of two copies around it. Measured
// call-to-result on the C1 FIB (tools/zc_latency.py): 256 queries 16 vs 28 us,
// 64K 39 vs 79 us, 1M 351 vs 390 us; from 2M on the copy pipeline is as fast
// or faster (673 vs 686 us).
constexpr unsigned long long kZeroCopyMax = 1ull << 20;

// Host buffers: chunked H2D / kernel / D2H on three streams ordered after `user`
// (or zero-copy for small pinned batches). input = kInAddr (16-byte addresses) or
// kInKey (8-byte keys: half the PCIe bytes).
void lookup_host(lpm6cu_fib* f, const void* addrs, unsigned long long n, void* out, cudaStream_t user,
                 int input = kInAddr) {
  const unsigned long long in_bytes = input == kInKey ? 8 : 16;
  std::lock_guard<std::mutex> lk(f->host_mu);
  const unsigned vb = f->g.value_bytes;
  if (n <= kZeroCopyMax) {
    void* da = mapped_device_ptr(addrs);
    void* dout = da ? mapped_device_ptr(out) : nullptr;
    if (da && dout) {
      if (!f->zc_stream) {
        check_cuda(cudaStreamCreateWithFlags(&f->zc_stream, cudaStreamNonBlocking), "stream");
        check_cuda(cudaEventCreateWithFlags(&f->zc_event, cudaEventDisableTiming), "event");
      }
      check_cuda(cudaEventRecord(f->zc_event, user), "event record");
      check_cuda(cudaStreamWaitEvent(f->zc_stream, f->zc_event, 0), "stream wait");
      launch_lookup(f, da, n, dout, f->zc_stream, input);
      check_cuda(cudaStreamSynchronize(f->zc_stream), "sync");
      return;
    }
  }
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
  // Small batches are cut into ~6 pieces (>= 64K queries) so their copies overlap too.
  const unsigned long long step =
      std::min(pp.chunk, (std::max<unsigned long long>(1ull << 16, (n + 5) / 6) + 63) & ~63ull);
  int s = 0;
  for (unsigned long long off = 0; off < n; off += step, s = (s + 1) % HostPipeline::kStreams) {
    const unsigned long long m = std::min(step, n - off);
    check_cuda(cudaMemcpyAsync(pp.d_in[s], src + off * in_bytes, m * in_bytes, cudaMemcpyHostToDevice, pp.streams[s]),
               "H2D");
    launch_lookup(f, pp.d_in[s], m, pp.d_out[s], pp.streams[s], input);
    check_cuda(cudaMemcpyAsync(dst + off * vb, pp.d_out[s], m * vb, cudaMemcpyDeviceToHost, pp.streams[s]), "D2H");
  }
  for (int i = 0; i < HostPipeline::kStreams; ++i) check_cuda(cudaStreamSynchronize(pp.streams[i]), "sync");
}

}  // namespace

void lpm6::capi::fib_destroy_quiesced(lpm6cu_fib* f) {
  if (!f) return;
  f->quiesced = true;
  delete f;
}

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
    if (!out) throw Error(Errc::InvalidArgument, "NULL out");
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
    capi::BuildTrace tr("fib_build_device");
    lpm6cu_geometry g;
    void* lines = capi::device_build_tree(rules, n, default_nh, opts, static_cast<cudaStream_t>(stream), &g);
    tr.mark("tree");
    std::unique_ptr<lpm6cu_fib> f;
    try {
      f.reset(new_fib(device, &g));
    } catch (...) {
      cudaFreeAsync(lines, static_cast<cudaStream_t>(stream));
      throw;
    }
    tr.mark("handle");
    f->d_lines = static_cast<unsigned long long*>(lines);
    f->pooled = true;
    load_root(f.get());
    tr.mark("root");
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

namespace {
// Line paths that differ from the others for this tree: 3 only with internal L2
// levels (it splits them), 4 only with 1-byte next hops (its extraction).
bool plan_applies(const lpm6cu_fib* f, unsigned path) {
  if (path == 3) return f->g.depth > f->cfg.smem_levels;
  if (path == 4) return f->g.value_bytes == 1;
  return path < 3;
}
}  // namespace

int lpm6cu_fib_tune_line_path(lpm6cu_fib* f, const void* d_addrs, uint64_t n, void* d_out, void* stream,
                              uint32_t reps, uint32_t* line_path) {
  return guard([&] {
    if (!f || !d_addrs || !d_out) throw Error(Errc::InvalidArgument, "NULL argument");
    if (n == 0) throw Error(Errc::InvalidArgument, "empty tuning batch");
    DeviceGuard dg(f->device);
    if (!is_device_ptr(d_addrs, f->device) || !is_device_ptr(d_out, f->device))
      throw Error(Errc::InvalidArgument, "lpm6cu_fib_tune_line_path takes device buffers");
    if (reinterpret_cast<uintptr_t>(d_addrs) % 16 != 0)
      throw Error(Errc::InvalidArgument, "addresses must be 16-byte aligned");
    const cudaStream_t st = static_cast<cudaStream_t>(stream);
    lpm6cu_kernel_config c = f->cfg;
    c.plane_levels = 0;  // the line paths and tile counts are timed on the packed image first
    const bool possible = f->tex && f->d_err == nullptr && !leaf_image_mode(f) && f->g.depth >= 1 &&
                          c.threads_per_cta == 1024 && c.min_ctas_per_sm == 1 &&
                          (c.queries_per_lane == 1 || c.queries_per_lane == 2 || c.queries_per_lane == 4);
    // Candidates: every applicable line path with one tile per warp, and the texture
    // leaf paths (1, 4) with 2 and 4 tiles (Phase A of the tiles overlapped).
    constexpr unsigned kTiles[3] = {1, 2, 4};
    auto tiles_apply = [&](unsigned path, unsigned ti) { return ti == 0 || path == 1 || path == 4; };
    unsigned best = 0, best_ti = 0;
    if (possible) {
      cudaEvent_t ev[2];
      check_cuda(cudaEventCreate(&ev[0]), "cudaEventCreate");
      if (cudaEventCreate(&ev[1]) != cudaSuccess) {
        cudaEventDestroy(ev[0]);
        throw Error(Errc::CudaError, "cudaEventCreate");
      }
      float ms[5][3] = {};
      try {
        const unsigned r = reps ? reps : 3;
        // Plan 3 differs from plan 1 only when the tree has internal L2 levels.
        // Two interleaved rounds, the faster of each plan's two timings kept, so a
        // clock ramp or a neighbour's burst during one plan's turn cannot pick it.
        for (unsigned round = 0; round < 2; ++round)
          for (unsigned path = 0; path < 5; ++path)
            for (unsigned ti = 0; ti < 3; ++ti) {
              if (!plan_applies(f, path) || !tiles_apply(path, ti)) continue;
              c.line_path = path;
              c.queries_per_lane = kTiles[ti];
              f->cfg = c;
              f->invalidate_plans();
              launch_lookup(f, d_addrs, n, d_out, st);  // untimed: resolves the plan, warms L2
              check_cuda(cudaEventRecord(ev[0], st), "cudaEventRecord");
              for (unsigned i = 0; i < r; ++i) launch_lookup(f, d_addrs, n, d_out, st);
              check_cuda(cudaEventRecord(ev[1], st), "cudaEventRecord");
              check_cuda(cudaEventSynchronize(ev[1]), "cudaEventSynchronize");
              float t = 0.f;
              check_cuda(cudaEventElapsedTime(&t, ev[0], ev[1]), "cudaEventElapsedTime");
              ms[path][ti] = round == 0 ? t : std::min(ms[path][ti], t);
            }
      } catch (...) {
        cudaEventDestroy(ev[0]);
        cudaEventDestroy(ev[1]);
        c.line_path = 0;
        c.queries_per_lane = 1;
        f->cfg = c;
        f->invalidate_plans();
        throw;
      }
      for (unsigned path = 0; path < 5; ++path)
        for (unsigned ti = 0; ti < 3; ++ti)
          if (plan_applies(f, path) && tiles_apply(path, ti) && ms[path][ti] < ms[best][best_ti]) {
            best = path;
            best_ti = ti;
          }
      // Split-plane Phase A: on each texture leaf path (1 and 4) with 2 and 4 tiles, plane
      // levels P = 2, 3 and every staged level; the fastest of all — packed or
      // planes — is kept (planes only when at least 0.5 % faster than the best packed plan).
      unsigned best_pu = 0;
      const unsigned ta = std::min<unsigned>(c.smem_levels, f->g.depth);
      if (f->g.depth >= 3 && ta >= 2 && (ta == f->g.depth || ta + 1 == f->g.depth)) {
        float best_ms = ms[best][best_ti] * 0.995f;
        unsigned cand[3] = {2u, 3u, ta};
        try {
          const unsigned r = reps ? reps : 3;
          for (unsigned path = 1; path <= 4; path += 3) {
            if (!plan_applies(f, path)) continue;
            for (unsigned ti = 1; ti < 3; ++ti)  // 2 and 4 tiles
            for (unsigned k = 0; k < 3; ++k) {
              c.line_path = path;
              c.queries_per_lane = kTiles[ti];
              const unsigned pu = cand[k];
              if (pu > ta || (k < 2 && pu == ta)) continue;  // 2 and 3 only below the staged levels
              c.plane_levels = pu;
              f->cfg = c;
              f->invalidate_plans();
              ensure_planes(f);
              float tmin = 0.f;
              for (unsigned round = 0; round < 2; ++round) {
                launch_lookup(f, d_addrs, n, d_out, st);
                check_cuda(cudaEventRecord(ev[0], st), "cudaEventRecord");
                for (unsigned i = 0; i < r; ++i) launch_lookup(f, d_addrs, n, d_out, st);
                check_cuda(cudaEventRecord(ev[1], st), "cudaEventRecord");
                check_cuda(cudaEventSynchronize(ev[1]), "cudaEventSynchronize");
                float t = 0.f;
                check_cuda(cudaEventElapsedTime(&t, ev[0], ev[1]), "cudaEventElapsedTime");
                tmin = round == 0 ? t : std::min(tmin, t);
              }
              if (tmin < best_ms) {
                best_ms = tmin;
                best_pu = pu;
                best = path;
                best_ti = ti;
              }
            }
          }
        } catch (...) {
          cudaEventDestroy(ev[0]);
          cudaEventDestroy(ev[1]);
          c.line_path = 0;
          c.queries_per_lane = 1;
          c.plane_levels = 0;
          f->cfg = c;
          f->invalidate_plans();
          throw;
        }
      }
      c.plane_levels = best_pu;
      cudaEventDestroy(ev[0]);
      cudaEventDestroy(ev[1]);
    }
    c.line_path = best;
    if (possible) c.queries_per_lane = kTiles[best_ti];
    f->cfg = c;
    f->invalidate_plans();
    ensure_planes(f);
    if (line_path) *line_path = best;
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
    const bool da = is_device_ptr(addrs, fib->device), dout = is_device_ptr(out, fib->device);
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

int lpm6cu_lookup_batch_device(const lpm6cu_fib* fib, const void* d_addrs, uint64_t n, void* d_out, void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!d_addrs || !d_out) throw Error(Errc::InvalidArgument, "NULL buffer");
    if (reinterpret_cast<uintptr_t>(d_addrs) % 16 != 0)
      throw Error(Errc::InvalidArgument, "addresses must be 16-byte aligned");
    int cur = -1;
    check_cuda(cudaGetDevice(&cur), "cudaGetDevice");
    if (cur == fib->device) {
      launch_lookup(fib, d_addrs, n, d_out, static_cast<cudaStream_t>(stream));
    } else {
      DeviceGuard dg(fib->device);
      launch_lookup(fib, d_addrs, n, d_out, static_cast<cudaStream_t>(stream));
    }
  });
}

int lpm6cu_lookup_keys(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, void* out, void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!keys || !out) throw Error(Errc::InvalidArgument, "NULL buffer");
    DeviceGuard dg(fib->device);
    const bool dk = is_device_ptr(keys, fib->device), dout = is_device_ptr(out, fib->device);
    if (dk != dout) throw Error(Errc::InvalidArgument, "keys and results must both be device or both be host memory");
    if (reinterpret_cast<uintptr_t>(keys) % 8 != 0) throw Error(Errc::InvalidArgument, "keys must be 8-byte aligned");
    if (dk)
      launch_lookup(fib, keys, n, out, static_cast<cudaStream_t>(stream), kInKey);
    else
      lookup_host(const_cast<lpm6cu_fib*>(fib), keys, n, out, static_cast<cudaStream_t>(stream), kInKey);
  });
}

int lpm6cu_search_batch(const lpm6cu_fib* fib, const uint64_t* keys, uint64_t n, uint32_t* ordinals, void* next_hops,
                        void* stream) {
  return guard([&] {
    if (!fib) throw Error(Errc::InvalidArgument, "NULL fib");
    if (n == 0) return;
    if (!keys || !ordinals) throw Error(Errc::InvalidArgument, "NULL buffer");
    DeviceGuard dg(fib->device);
    if (!is_device_ptr(keys, fib->device) || !is_device_ptr(ordinals, fib->device) ||
        (next_hops && !is_device_ptr(next_hops, fib->device)))
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
    if (!is_device_ptr(frames, fib->device) || !is_device_ptr(out, fib->device))
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
      cudaFreeAsync(lines, static_cast<cudaStream_t>(stream));
      throw;
    }
    f->d_lines = static_cast<unsigned long long*>(lines);
    f->pooled = true;
    load_root(f.get());
    *out = f.release();
  });
}

int lpm6cu_querygen_create(int device, int workload, const lpm6cu_prefix* rules, uint64_t nrules,
                           lpm6cu_querygen** out) {
  return guard([&] {
    if (!out || (nrules && !rules)) throw Error(Errc::InvalidArgument, "NULL argument");
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
