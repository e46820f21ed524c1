// H2D copy shapes for the end-to-end path: full 16-byte addresses vs only the
// top 8 bytes (the lookup key) with a strided 2D copy, from pinned memory.
//   nvcc -O3 -o tools/h2d_probe tools/h2d_probe.cu && tools/h2d_probe
#include <cstdio>
#include <cuda_runtime.h>

int main() {
  const size_t n = 1ull << 23;  // 8M addresses = 128 MiB
  unsigned char *h, *d;
  cudaHostAlloc(&h, n * 16, cudaHostAllocDefault);
  cudaMalloc(&d, n * 16);
  for (size_t i = 0; i < n * 16; i += 4096) h[i] = 1;
  cudaStream_t s;
  cudaStreamCreate(&s);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(a, s);
    cudaMemcpyAsync(d, h, n * 16, cudaMemcpyHostToDevice, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("full 16B x %zu: %.3f ms  %.1f GB/s  %.2f G addr/s\n", n, ms, n * 16 / ms / 1e6, n / ms / 1e6);
    for (size_t w : {8, 16, 32, 64}) {
      // copy the top `w/2`.. bytes: rows of w bytes taken every 2w bytes would change layout;
      // here: width 8 of pitch 16 (the key only)
      if (w != 8) continue;
      cudaEventRecord(a, s);
      cudaMemcpy2DAsync(d, 8, h + 8, 16, 8, n, cudaMemcpyHostToDevice, s);
      cudaEventRecord(b, s);
      cudaEventSynchronize(b);
      cudaEventElapsedTime(&ms, a, b);
      printf("2D 8B of 16B x %zu: %.3f ms  %.1f GB/s useful  %.2f G addr/s\n", n, ms, n * 8 / ms / 1e6, n / ms / 1e6);
    }
    cudaEventRecord(a, s);
    cudaMemcpyAsync(h, d, n, cudaMemcpyDeviceToHost, s);
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    printf("D2H 1B x %zu: %.3f ms  %.1f GB/s\n", n, ms, n / ms / 1e6);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
