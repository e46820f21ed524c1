// Roofline probes: the L2 random-gather bandwidth and the shared-memory read
// bandwidth that bound the node loads of the lookup (the HBM term
// comes from MEASURED_PEAKS.json). They run on the same device as the lookup,
// with the tree-sized buffer the lookup's deeper levels live in.
#include <cuda_runtime.h>

#include <string>

#include "capi_util.hpp"
#include "lpm6/querygen.h"
#include "lpm6cu.h"

using namespace lpm6;
using lpm6::capi::guard;

namespace {

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) throw Error(Errc::CudaError, std::string(what) + ": " + cudaGetErrorString(e));
}

// Each group of LINE/32 lanes fetches one random line per iteration, lane j
// taking one 32-byte sector with a 256-bit load that bypasses L1 — the access
// shape of the lookup's node loads (4 lanes x 32 B per 128-byte node). The line
// index is a multiply-high range reduction of an LCG, so the probe is bound by the memory
// system, not by index arithmetic.
template <int LINE>
__global__ void __launch_bounds__(256) l2_gather_kernel(const unsigned long long* buf, unsigned long long lines,
                                                        int iters, unsigned long long* sink) {
  constexpr int LPL = LINE / 32;  // lanes per line
  const unsigned grp = (blockIdx.x * blockDim.x + threadIdx.x) / LPL;
  const unsigned j = threadIdx.x % LPL;
  unsigned long long acc = 0;
  unsigned long long h = mix64(grp);
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;  // LCG per group: uniform across its lanes
    const unsigned long long line = __umul64hi(h, lines);  // uniform in [0, lines)
    const unsigned long long* p = buf + line * (LINE / 8) + j * 4;
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u64 {%0,%1,%2,%3}, [%4];"
                 : "=l"(a), "=l"(b), "=l"(c), "=l"(d)
                 : "l"(p));
    acc ^= a + b + c + d;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

__global__ void __launch_bounds__(256) smem_read_kernel(int iters, unsigned long long* sink) {
  __shared__ __align__(16) unsigned long long s[4096];  // 32 KiB
  for (int i = threadIdx.x; i < 4096; i += blockDim.x) s[i] = i * 0x9E3779B97F4A7C15ull;
  __syncthreads();
  const unsigned lane = threadIdx.x & 31u;
  const unsigned warp = threadIdx.x >> 5;
  unsigned long long acc = 0;
  unsigned row = warp;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    // 32 lanes x 16 B = 512 B = 4 conflict-free 128-byte wavefronts.
    const unsigned long long* p = s + ((row & 63u) * 64 + lane * 2);
    unsigned long long a, b;
    asm volatile("ld.shared.v2.u64 {%0,%1}, [%2];"
                 : "=l"(a), "=l"(b)
                 : "r"(static_cast<unsigned>(__cvta_generic_to_shared(p))));
    acc += a ^ b;
    row += 7;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <class F>
double time_ms(F&& launch) {
  cudaEvent_t a, b;
  check(cudaEventCreate(&a), "event");
  check(cudaEventCreate(&b), "event");
  launch();  // warm-up
  check(cudaEventRecord(a), "record");
  launch();
  check(cudaEventRecord(b), "record");
  check(cudaEventSynchronize(b), "sync");
  float ms = 0;
  check(cudaEventElapsedTime(&ms, a, b), "elapsed");
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  check(cudaGetLastError(), "probe kernel");
  return ms;
}

}  // namespace

extern "C" {

int lpm6cu_probe_l2_gather(int device, uint64_t buffer_bytes, uint32_t line_bytes, double* gbps) {
  return guard([&] {
    if (!gbps) throw Error(Errc::InvalidArgument, "NULL gbps");
    if (line_bytes != 32 && line_bytes != 128) throw Error(Errc::InvalidArgument, "line_bytes must be 32 or 128");
    if (buffer_bytes < line_bytes) throw Error(Errc::InvalidArgument, "buffer smaller than a line");
    check(cudaSetDevice(device), "cudaSetDevice");
    int sms = 0;
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    unsigned long long* buf = nullptr;
    unsigned long long* sink = nullptr;
    check(cudaMalloc(&buf, buffer_bytes), "cudaMalloc");
    check(cudaMalloc(&sink, 8), "cudaMalloc");
    check(cudaMemset(buf, 0x5A, buffer_bytes), "memset");
    const unsigned long long lines = buffer_bytes / line_bytes;
    const int blocks = sms * 8, iters = 2048;
    double ms;
    if (line_bytes == 128)
      ms = time_ms([&] { l2_gather_kernel<128><<<blocks, 256>>>(buf, lines, iters, sink); });
    else
      ms = time_ms([&] { l2_gather_kernel<32><<<blocks, 256>>>(buf, lines, iters, sink); });
    const double groups = static_cast<double>(blocks) * 256 / (line_bytes / 32);
    *gbps = groups * iters * line_bytes / (ms * 1e-3) / 1e9;
    cudaFree(buf);
    cudaFree(sink);
  });
}

int lpm6cu_probe_smem(int device, double* gbps) {
  return guard([&] {
    if (!gbps) throw Error(Errc::InvalidArgument, "NULL gbps");
    check(cudaSetDevice(device), "cudaSetDevice");
    int sms = 0;
    check(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "attr");
    unsigned long long* sink = nullptr;
    check(cudaMalloc(&sink, 8), "cudaMalloc");
    const int blocks = sms * 4, iters = 16384;
    const double ms = time_ms([&] { smem_read_kernel<<<blocks, 256>>>(iters, sink); });
    *gbps = static_cast<double>(blocks) * 256 * 16 * iters / (ms * 1e-3) / 1e9;
    cudaFree(sink);
  });
}

}  // extern "C"
