// Floor for a synchronous call: empty-kernel launch + stream sync, and the CUDA
// calls the zero-copy host path adds (pointer queries, event record + wait).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -o tools/launch_latency tools/launch_latency.cu
#include <chrono>
#include <cstdio>
#include <cuda_runtime.h>
__global__ void empty_kernel(int* p) { if (p && threadIdx.x == 1024) *p = 0; }
template <class F> double med_us(F f, int reps = 2000) {
  for (int i = 0; i < 50; ++i) f();
  auto t0 = std::chrono::steady_clock::now();
  for (int i = 0; i < reps; ++i) f();
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count() / reps;
}
int main() {
  cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  cudaEvent_t e; cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
  void* h; cudaMallocHost(&h, 1 << 20);
  printf("launch+sync       %.2f us\n", med_us([&] { empty_kernel<<<1, 32, 0, s>>>(nullptr); cudaStreamSynchronize(s); }));
  printf("launch+sync 148x1024 %.2f us\n", med_us([&] { empty_kernel<<<148, 1024, 0, s>>>(nullptr); cudaStreamSynchronize(s); }));
  printf("pointer attrs     %.2f us\n", med_us([&] { cudaPointerAttributes a; cudaPointerGetAttributes(&a, h); }));
  printf("event rec+wait    %.2f us\n", med_us([&] { cudaEventRecord(e, 0); cudaStreamWaitEvent(s, e, 0); }));
  return 0;
}
