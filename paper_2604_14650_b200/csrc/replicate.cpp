// Single-process FIB replication over NCCL: the line array of one
// device FIB broadcast to the other GPUs of the node with one grouped
// ncclBroadcast (NVLink / NVSwitch), one communicator per device from
// ncclCommInitAll. This is the path for a C/C++ caller that drives all GPUs from
// one process; the torch.distributed path (one process per GPU,
// paper_2604_14650_b200/dispatch.py) broadcasts the same array.
//
// NCCL is loaded with dlopen on first use: the library has no link-time NCCL
// dependency, so it coexists with whatever libnccl.so.2 the host process (e.g.
// torch) already loaded.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "capi_util.hpp"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

struct NcclApi {
  ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  std::string load_error;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.load_error = std::string("cannot load libnccl.so.2: ") + (e ? e : "unknown");
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.comm_init_all = reinterpret_cast<decltype(api.comm_init_all)>(sym("ncclCommInitAll"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(sym("ncclCommDestroy"));
    api.broadcast = reinterpret_cast<decltype(api.broadcast)>(sym("ncclBroadcast"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(sym("ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(sym("ncclGroupEnd"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(sym("ncclGetErrorString"));
    if (!api.comm_init_all || !api.comm_destroy || !api.broadcast || !api.group_start || !api.group_end)
      api.load_error = "libnccl.so.2 lacks a required symbol";
  });
  if (!api.load_error.empty()) throw Error(Errc::NcclError, api.load_error);
  return api;
}

void ck_nccl(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw Error(Errc::NcclError,
                std::string(what) + ": " + (nccl().error_string ? nccl().error_string(r) : std::to_string(r)));
}

void ck(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

}  // namespace

extern "C" int lpm6cu_fib_replicate(const lpm6cu_fib* src, const int* devices, int ndev, lpm6cu_fib** out) {
  return guard([&] {
    if (!src || !devices || !out || ndev < 1) throw Error(Errc::InvalidArgument, "NULL argument or ndev < 1");
    lpm6cu_geometry g;
    const void* src_lines = nullptr;
    int st = lpm6cu_fib_geometry(src, &g);
    if (!st) st = lpm6cu_fib_device_lines(src, &src_lines);
    if (st) throw Error(static_cast<Errc>(st - 1), lpm6cu_last_error());
    int src_dev = -1;
    {
      cudaPointerAttributes a{};
      ck(cudaPointerGetAttributes(&a, src_lines), "cudaPointerGetAttributes");
      src_dev = a.device;
    }
    if (devices[0] != src_dev) throw Error(Errc::InvalidArgument, "devices[0] must be the source FIB's device");
    const NcclApi& api = nccl();
    const size_t bytes = g.total_words * 8;
    int prev = -1;
    cudaGetDevice(&prev);
    std::vector<void*> bufs(ndev, nullptr);
    std::vector<cudaStream_t> streams(ndev, nullptr);
    std::vector<ncclComm_t> comms(ndev, nullptr);
    auto cleanup = [&](bool free_bufs) {
      for (int i = 0; i < ndev; ++i) {
        cudaSetDevice(devices[i]);
        if (comms[i]) api.comm_destroy(comms[i]);
        if (streams[i]) cudaStreamDestroy(streams[i]);
        if (free_bufs && bufs[i]) cudaFree(bufs[i]);
      }
      if (prev >= 0) cudaSetDevice(prev);
    };
    try {
      for (int i = 0; i < ndev; ++i) {
        ck(cudaSetDevice(devices[i]), "cudaSetDevice");
        ck(cudaMalloc(&bufs[i], bytes), "cudaMalloc replica");
        ck(cudaStreamCreateWithFlags(&streams[i], cudaStreamNonBlocking), "cudaStreamCreate");
      }
      ck_nccl(api.comm_init_all(comms.data(), ndev, devices), "ncclCommInitAll");
      ck_nccl(api.group_start(), "ncclGroupStart");
      for (int i = 0; i < ndev; ++i)
        ck_nccl(api.broadcast(i == 0 ? src_lines : nullptr, bufs[i], bytes, ncclUint8, 0, comms[i], streams[i]),
                "ncclBroadcast");
      ck_nccl(api.group_end(), "ncclGroupEnd");
      for (int i = 0; i < ndev; ++i) {
        ck(cudaSetDevice(devices[i]), "cudaSetDevice");
        ck(cudaStreamSynchronize(streams[i]), "broadcast");
      }
    } catch (...) {
      cleanup(true);
      throw;
    }
    // Each replica becomes an owning FIB handle over its broadcast buffer.
    std::vector<lpm6cu_fib*> made(ndev, nullptr);
    for (int i = 0; i < ndev; ++i) {
      const int s2 = lpm6cu_fib_adopt_device(devices[i], &g, bufs[i], &made[i]);
      if (s2) {
        const std::string msg = lpm6cu_last_error();
        for (int j = 0; j < i; ++j) lpm6cu_fib_destroy(made[j]);
        for (int j = i; j < ndev; ++j)
          if (bufs[j]) {
            cudaSetDevice(devices[j]);
            cudaFree(bufs[j]);
          }
        cleanup(false);
        throw Error(static_cast<Errc>(s2 - 1), msg);
      }
      bufs[i] = nullptr;
    }
    cleanup(false);
    for (int i = 0; i < ndev; ++i) out[i] = made[i];
  });
}
