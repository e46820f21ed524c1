// C ABI of the reference file formats (PBT1 snapshots, PBTR key traces) and their
// loading straight into device memory (tree.hpp:90-96, S:250,
// S:475). Formats and validation live in lpm6/snapshot.cpp.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>

#include "capi_util.hpp"
#include "lpm6/snapshot.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

IntervalMap map_of(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m) {
  if (m && (!boundaries || !next_hops)) throw Error(Errc::InvalidArgument, "NULL argument");
  IntervalMap map;
  map.boundaries.assign(boundaries, boundaries + m);
  map.next_hops.assign(next_hops, next_hops + m);
  return map;
}

struct FileCloser {
  void operator()(FILE* f) const {
    if (f) std::fclose(f);
  }
};

struct PinnedBuf {
  void* p = nullptr;
  ~PinnedBuf() {
    if (p) cudaFreeHost(p);
  }
};

}  // namespace

extern "C" {

int lpm6_snapshot_encode(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, uint32_t k, void* buf,
                         uint64_t cap, uint64_t* size) {
  return guard([&] {
    if (!size) throw Error(Errc::InvalidArgument, "NULL size");
    const std::vector<unsigned char> img = save_snapshot(map_of(boundaries, next_hops, m), k);
    *size = img.size();
    if (!buf) return;
    if (cap < img.size()) throw Error(Errc::InvalidArgument, "buffer smaller than the snapshot");
    std::memcpy(buf, img.data(), img.size());
  });
}

int lpm6_snapshot_save(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m, uint32_t k,
                       const char* path) {
  return guard([&] {
    if (!path) throw Error(Errc::InvalidArgument, "NULL path");
    const std::vector<unsigned char> img = save_snapshot(map_of(boundaries, next_hops, m), k);
    write_file(path, img.data(), img.size());
  });
}

int lpm6_snapshot_decode(const void* buf, uint64_t size, uint64_t* boundaries, uint32_t* next_hops, uint64_t cap,
                         uint64_t* m, uint32_t* k) {
  return guard([&] {
    const LoadedSnapshot s = load_snapshot(buf, size);
    if (m) *m = s.map.size();
    if (k) *k = s.geometry.k;
    if (!boundaries && !next_hops) return;
    if (cap < s.map.size()) throw Error(Errc::InvalidArgument, "capacity below the snapshot's key count");
    if (boundaries) std::memcpy(boundaries, s.map.boundaries.data(), s.map.size() * 8);
    if (next_hops) std::memcpy(next_hops, s.map.next_hops.data(), s.map.size() * 4);
  });
}

int lpm6cu_fib_load_snapshot(int device, const char* path, uint32_t default_nh, const lpm6cu_build_opts* opts,
                             void* stream, lpm6cu_fib** out) {
  return guard([&] {
    if (!path || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    const std::vector<unsigned char> img = read_file(path);
    const LoadedSnapshot s = load_snapshot(img.data(), img.size(), default_nh);
    const int st = lpm6cu_fib_build_from_intervals(device, s.map.boundaries.data(), s.map.next_hops.data(),
                                                   s.map.size(), default_nh, opts, stream, out);
    if (st) throw Error(static_cast<Errc>(st - 1), lpm6cu_last_error());
  });
}

int lpm6_memory_footprint(const lpm6cu_geometry* g, lpm6cu_footprint* out) {
  return guard([&] {
    if (!g || !out) throw Error(Errc::InvalidArgument, "NULL argument");
    std::memset(out, 0, sizeof *out);
    out->internal_bytes = g->level_start[g->depth] * 8;
    out->leaf_bytes = g->leaf_nodes * (g->leaf_words ? g->leaf_words : 16) * 8;  // next hops are inside the leaves
    out->value_bytes = 0;
    out->image_bytes = (g->total_words - g->image_start) * 8;
    out->total_bytes = g->total_words * 8;
    out->bytes_per_interval = g->num_keys ? double(out->total_bytes) / double(g->num_keys) : 0.0;
    out->total_bytes_value8 = out->total_bytes;  // no separate value array to widen
    out->bytes_per_interval_value8 = out->bytes_per_interval;
  });
}

int lpm6_ref_memory_footprint(uint64_t m, uint32_t k, lpm6cu_footprint* out) {
  return guard([&] {
    if (!out) throw Error(Errc::InvalidArgument, "NULL argument");
    const RefGeometry g = plan_ref_geometry(m, k);
    std::memset(out, 0, sizeof *out);
    const uint64_t slots = g.allocated_leaf_nodes * k;
    out->leaf_bytes = slots * 8;
    out->internal_bytes = g.leaf_start * 8;
    out->value_bytes = slots * 4;
    out->total_bytes = out->leaf_bytes + out->internal_bytes + out->value_bytes;
    out->bytes_per_interval = m ? double(out->total_bytes) / double(m) : 0.0;
    out->total_bytes_value8 = out->leaf_bytes + out->internal_bytes + slots * 8;
    out->bytes_per_interval_value8 = m ? double(out->total_bytes_value8) / double(m) : 0.0;
  });
}

int lpm6_trace_save(const uint64_t* keys, uint64_t n, const char* path) {
  return guard([&] {
    if (!path || (n && !keys)) throw Error(Errc::InvalidArgument, "NULL argument");
    const std::vector<unsigned char> img = save_trace(keys, n);
    write_file(path, img.data(), img.size());
  });
}

int lpm6_trace_count(const void* buf, uint64_t size, uint64_t* n) {
  return guard([&] {
    if (!n) throw Error(Errc::InvalidArgument, "NULL n");
    *n = trace_key_count(buf, size);
  });
}

int lpm6cu_trace_load(int device, const char* path, uint64_t* d_keys, uint64_t cap, uint64_t* count, void* stream) {
  return guard([&] {
    if (!path || !count) throw Error(Errc::InvalidArgument, "NULL argument");
    std::unique_ptr<FILE, FileCloser> f(std::fopen(path, "rb"));
    if (!f) throw Error(Errc::Io, std::string("cannot open ") + path);
    unsigned char hdr[kTraceHeaderBytes];
    const size_t got = std::fread(hdr, 1, sizeof hdr, f.get());
    if (std::fseek(f.get(), 0, SEEK_END) != 0) throw Error(Errc::Io, std::string("cannot seek ") + path);
    const long fsize = std::ftell(f.get());
    if (fsize < 0) throw Error(Errc::Io, std::string("cannot size ") + path);
    const uint64_t n = trace_header_count(hdr, got, static_cast<uint64_t>(fsize));
    *count = n;
    if (!d_keys) return;
    if (cap < n) throw Error(Errc::InvalidArgument, "device buffer smaller than the trace");
    ck(cudaSetDevice(device), "cudaSetDevice");
    // File -> two pinned 32 MiB staging buffers -> device, the copy of one chunk
    // overlapping the read of the next.
    constexpr uint64_t kChunkKeys = 4u << 20;
    PinnedBuf stage[2];
    cudaEvent_t done[2] = {nullptr, nullptr};
    for (int i = 0; i < 2; ++i) {
      ck(cudaHostAlloc(&stage[i].p, kChunkKeys * 8, cudaHostAllocDefault), "cudaHostAlloc");
      ck(cudaEventCreateWithFlags(&done[i], cudaEventDisableTiming), "cudaEventCreate");
    }
    auto cleanup = [&] {
      for (cudaEvent_t e : done)
        if (e) cudaEventDestroy(e);
    };
    try {
      const cudaStream_t s = static_cast<cudaStream_t>(stream);
      if (std::fseek(f.get(), static_cast<long>(kTraceHeaderBytes), SEEK_SET) != 0)
        throw Error(Errc::Io, std::string("cannot seek ") + path);
      bool used[2] = {false, false};
      int b = 0;
      for (uint64_t off = 0; off < n; off += kChunkKeys, b ^= 1) {
        const uint64_t cnt = std::min(kChunkKeys, n - off);
        if (used[b]) ck(cudaEventSynchronize(done[b]), "staging reuse");
        if (std::fread(stage[b].p, 8, cnt, f.get()) != cnt) throw Error(Errc::Io, std::string("short read ") + path);
        ck(cudaMemcpyAsync(d_keys + off, stage[b].p, cnt * 8, cudaMemcpyHostToDevice, s), "H2D trace");
        ck(cudaEventRecord(done[b], s), "cudaEventRecord");
        used[b] = true;
      }
      ck(cudaStreamSynchronize(s), "trace load");
    } catch (...) {
      cleanup();
      throw;
    }
    cleanup();
  });
}

}  // extern "C"
