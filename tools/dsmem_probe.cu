// Distributed shared memory probe: random 8-byte reads from the shared memory
// of the CTAs of a thread-block cluster (the access a cluster-sharded tree level
// would make), vs the same reads from the CTA's own shared memory.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/dsmem_probe tools/dsmem_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

__global__ void __launch_bounds__(1024, 1) probe(int words, int iters, int remote, unsigned long long* sink) {
  extern __shared__ unsigned long long s[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < words; i += blockDim.x) s[i] = i * 2654435761ull + blockIdx.x;
  cl.sync();
  const unsigned csize = cl.num_blocks();
  unsigned long long h = (blockIdx.x * 1024ull + threadIdx.x) * 0x9E3779B97F4A7C15ull + 1;
  unsigned long long acc = 0;
#pragma unroll 4
  for (int it = 0; it < iters; ++it) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    const unsigned idx = static_cast<unsigned>((h >> 33) % words);
    if (remote) {
      const unsigned r = static_cast<unsigned>(h >> 59) % csize;
      const unsigned long long* p = cl.map_shared_rank(s, r);
      acc += p[idx];
    } else {
      acc += s[idx];
    }
  }
  cl.sync();
  if (acc == 42) sink[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  const int smem = 200 * 1024, words = smem / 8, iters = 4096;
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(probe, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  for (int cs : {1, 2, 4, 8, 16}) {
    cudaLaunchConfig_t cfg = {};
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.blockDim = dim3(1024);
    cfg.dynamicSmemBytes = smem;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cfg.gridDim = dim3(cs);
    int maxc = 0;
    cudaError_t e = cudaOccupancyMaxActiveClusters(&maxc, probe, &cfg);
    if (e != cudaSuccess) {
      printf("cluster %2d: occupancy query failed: %s\n", cs, cudaGetErrorString(e));
      cudaGetLastError();
      continue;
    }
    cfg.gridDim = dim3(maxc * cs);
    for (int remote : {0, 1}) {
      if (cs == 1 && remote) continue;
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaLaunchKernelEx(&cfg, probe, words, iters, remote, sink);
      cudaEventRecord(a);
      cudaLaunchKernelEx(&cfg, probe, words, iters, remote, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      const double loads = double(maxc) * cs * 1024 * iters;
      printf("cluster %2d: %3d clusters (%3d SMs) %s: %7.1f G loads/s  %6.2f loads/clk/SM  (%s)\n", cs, maxc,
             maxc * cs, remote ? "remote" : "local ", loads / (ms * 1e-3) / 1e9,
             loads / (ms * 1e-3) / (maxc * cs) / 1.965e9, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
