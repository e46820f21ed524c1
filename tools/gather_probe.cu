// Microbenchmark: random gathers from an L2- or L1-resident buffer with the
// access shapes a node search can use. A "group" of LANES lanes reads BYTES
// bytes each from one random 128-byte line per iteration (contiguous, starting
// at a random sector when the group reads less than a line). Reports requested
// bytes/s, lines/s and sectors/s so the lookup's per-level cost can be read off.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/gather_probe tools/gather_probe.cu
//   tools/gather_probe
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <int BYTES>
__device__ __forceinline__ unsigned long long ld(const unsigned long long* p) {
  unsigned long long a = 0, b = 0, c = 0, d = 0;
  if constexpr (BYTES == 8) {
    asm volatile("ld.global.nc.u64 %0, [%1];" : "=l"(a) : "l"(p));
  } else if constexpr (BYTES == 16) {
    asm volatile("ld.global.nc.v2.u64 {%0,%1}, [%2];" : "=l"(a), "=l"(b) : "l"(p));
  } else {
    asm volatile("ld.global.nc.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
  }
  return a + b + c + d;
}

template <int LANES, int BYTES>
__global__ void __launch_bounds__(256) gather(const unsigned long long* buf, unsigned long long lines, int iters,
                                              unsigned long long* sink) {
  constexpr int GROUP_BYTES = LANES * BYTES;  // <= 128
  const unsigned grp = (blockIdx.x * blockDim.x + threadIdx.x) / LANES;
  const unsigned j = threadIdx.x % LANES;
  unsigned long long h = grp * 0x9E3779B97F4A7C15ull + 12345;
  unsigned long long acc = 0;
#pragma unroll 8
  for (int it = 0; it < iters; ++it) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    const unsigned long long line = __umul64hi(h, lines);
    const unsigned off = GROUP_BYTES >= 128 ? 0u : (static_cast<unsigned>(h >> 8) % (128 / GROUP_BYTES)) * GROUP_BYTES;
    const unsigned long long* p = buf + line * 16 + (off + j * BYTES) / 8;
    acc ^= ld<BYTES>(p);
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <int LANES, int BYTES>
void run(const unsigned long long* buf, unsigned long long bytes, unsigned long long* sink, int sms, const char* tag) {
  const unsigned long long lines = bytes / 128;
  const int blocks = sms * 8, iters = 1024;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  gather<LANES, BYTES><<<blocks, 256>>>(buf, lines, iters, sink);
  cudaEventRecord(a);
  gather<LANES, BYTES><<<blocks, 256>>>(buf, lines, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const double groups = double(blocks) * 256 / LANES;
  const double reqs = groups * iters / (ms * 1e-3);
  const int sectors = (LANES * BYTES + 31) / 32;
  printf("%-8s buf %8.2f MB lanes %2d x %2d B : %8.1f G groups/s  %8.1f GB/s  %8.1f G sectors/s  warp-instr/s %.1f G\n",
         tag, bytes / 1048576.0, LANES, BYTES, reqs / 1e9, reqs * LANES * BYTES / 1e9, reqs * sectors / 1e9,
         reqs / (32 / LANES) / 1e9);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long *buf, *sink;
  cudaMalloc(&buf, 64ull << 20);
  cudaMalloc(&sink, 8);
  cudaMemset(buf, 1, 64ull << 20);
  for (unsigned long long bytes : {48ull << 10, 4ull << 20, 32ull << 20}) {
    const char* tag = bytes < (1 << 20) ? "L1" : "L2";
    run<4, 32>(buf, bytes, sink, sms, tag);
    run<8, 16>(buf, bytes, sink, sms, tag);
    run<16, 8>(buf, bytes, sink, sms, tag);
    run<4, 8>(buf, bytes, sink, sms, tag);
    run<2, 16>(buf, bytes, sink, sms, tag);
    run<1, 32>(buf, bytes, sink, sms, tag);
    run<2, 32>(buf, bytes, sink, sms, tag);
    run<1, 16>(buf, bytes, sink, sms, tag);
    run<1, 8>(buf, bytes, sink, sms, tag);
  }
  printf("status %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
