// Microbenchmark: random 128-byte line fetches from an L2-resident buffer by the
// TMA bulk-copy engine (cp.async.bulk global -> shared, mbarrier completion)
// instead of LSU loads, each line then searched by its own thread with four
// 8-byte shared-memory probes. Question it answers: can the L2 levels of the
// lookup move off the L1 data pipe (which the LSU-load design saturates)?
//
// Each warp owns NBUF stages; a stage is 32 line slots (one per lane, 144-byte
// stride to skew banks) + one mbarrier. Every lane issues its own copy.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -o tools/tma_probe tools/tma_probe.cu
#include <cstdint>
#include <cstdio>
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

constexpr int kSlot = 144;  // bytes per lane slot (128 + 16 skew)

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)), "r"(count));
}
__device__ __forceinline__ void arrive_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          (unsigned)__cvta_generic_to_shared(dst)),
      "l"(src), "r"(bytes), "r"((unsigned)__cvta_generic_to_shared(bar))
      : "memory");
}
__device__ __forceinline__ void wait_parity(uint64_t* bar, unsigned parity) {
  asm volatile(
      "{\n.reg .pred p;\nW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W;\n}" ::"r"(
          (unsigned)__cvta_generic_to_shared(bar)),
      "r"(parity)
      : "memory");
}

template <int NBUF>
__global__ void tma_gather(const unsigned long long* buf, unsigned long long lines, int iters,
                           unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[32][NBUF];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * NBUF * 32 * kSlot;
  if (lane == 0)
    for (int s = 0; s < NBUF; ++s) mbar_init(&bars[warp][s], 32);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned long long h = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 7;
  auto next_line = [&]() {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    return __umul64hi(h, lines);
  };
  for (int s = 0; s < NBUF; ++s) {
    unsigned char* slot = wbase + (s * 32 + lane) * kSlot;
    arrive_tx(&bars[warp][s], 128);
    bulk_g2s(slot, buf + next_line() * 16, 128, &bars[warp][s]);
  }
  unsigned long long acc = 0;
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < NBUF; ++s) {
      wait_parity(&bars[warp][s], phase);
      const unsigned long long* w = reinterpret_cast<const unsigned long long*>(wbase + (s * 32 + lane) * kSlot);
      // four dependent probes, like a 16-way node search
      unsigned c = (w[7] <= acc) ? 8u : 0u;
      c |= (w[c | 3] <= acc) ? 4u : 0u;
      c |= (w[c | 1] <= acc) ? 2u : 0u;
      c |= (w[c] <= acc) ? 1u : 0u;
      acc += c + w[15];
      if (it + 1 < iters) {
        arrive_tx(&bars[warp][s], 128);
        bulk_g2s(wbase + (s * 32 + lane) * kSlot, buf + next_line() * 16, 128, &bars[warp][s]);
      }
    }
    phase ^= 1;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

// Tensor-TMA gather4: one instruction fetches 4 random lines (rows of the
// [lines x 16 u64] tensor) into 512 contiguous bytes. Lane 4g issues group g's
// copy into 512 contiguous bytes (TMA needs 128-byte aligned destinations).
constexpr int kGroupBytes = 512;
template <int NBUF>
__global__ void tma_gather4(const __grid_constant__ CUtensorMap tmap, unsigned long long lines, int iters,
                            unsigned long long* sink) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t bars[32][NBUF];
  const unsigned warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  unsigned char* wbase = smem + warp * NBUF * 8 * kGroupBytes;
  if (lane == 0)
    for (int s = 0; s < NBUF; ++s) mbar_init(&bars[warp][s], 8);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  unsigned long long h = (blockIdx.x * blockDim.x + threadIdx.x) * 0x9E3779B97F4A7C15ull + 7;
  auto next_line = [&]() {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    return static_cast<int>(__umul64hi(h, lines));
  };
  auto issue = [&](int s) {
    const int row = next_line();
    const int r0 = __shfl_sync(0xffffffffu, row, lane & ~3u), r1 = __shfl_sync(0xffffffffu, row, (lane & ~3u) | 1),
              r2 = __shfl_sync(0xffffffffu, row, (lane & ~3u) | 2), r3 = __shfl_sync(0xffffffffu, row, (lane & ~3u) | 3);
    if ((lane & 3) == 0) {
      uint64_t* bar = &bars[warp][s];
      unsigned char* dst = wbase + (s * 8 + (lane >> 2)) * kGroupBytes;
      arrive_tx(bar, 512);
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"((unsigned)__cvta_generic_to_shared(dst)),
          "l"(&tmap), "r"(0), "r"(r0), "r"(r1), "r"(r2), "r"(r3), "r"((unsigned)__cvta_generic_to_shared(bar))
          : "memory");
    }
  };
  for (int s = 0; s < NBUF; ++s) issue(s);
  unsigned long long acc = 0;
  unsigned phase = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int s = 0; s < NBUF; ++s) {
      wait_parity(&bars[warp][s], phase);
      const unsigned long long* w = reinterpret_cast<const unsigned long long*>(
          wbase + (s * 8 + (lane >> 2)) * kGroupBytes + (lane & 3) * 128);
      unsigned c = (w[7] <= acc) ? 8u : 0u;
      c |= (w[c | 3] <= acc) ? 4u : 0u;
      c |= (w[c | 1] <= acc) ? 2u : 0u;
      c |= (w[c] <= acc) ? 1u : 0u;
      acc += c + w[15];
      __syncwarp();
      if (it + 1 < iters) issue(s);
    }
    phase ^= 1;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <int NBUF>
void run_g4(const CUtensorMap& tmap, unsigned long long lines, unsigned long long* sink, int sms, int threads) {
  const int iters = 512;
  const size_t smem = size_t(threads / 32) * NBUF * 8 * kGroupBytes;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(tma_gather4<NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_gather4<NBUF>, threads, smem);
  if (per_sm < 1) return;
  const int blocks = sms * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma_gather4<NBUF><<<blocks, threads, smem>>>(tmap, lines, iters, sink);
  cudaEventRecord(a);
  tma_gather4<NBUF><<<blocks, threads, smem>>>(tmap, lines, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double n = double(blocks) * threads * iters * NBUF;
  printf("g4   NBUF=%d threads=%4d ctas/sm=%d smem=%6zu: %7.1f G lines/s %s\n", NBUF, threads, per_sm, smem,
         n / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

// LSU reference: 4 lanes per line, one 32-byte load each (the current Phase B shape).
__global__ void __launch_bounds__(1024) lsu_gather(const unsigned long long* buf, unsigned long long lines, int iters,
                                                   unsigned long long* sink) {
  const unsigned grp = (blockIdx.x * blockDim.x + threadIdx.x) / 4, j = threadIdx.x & 3;
  unsigned long long h = grp * 0x9E3779B97F4A7C15ull + 7, acc = 0;
  for (int it = 0; it < iters; ++it) {
    h = h * 6364136223846793005ull + 1442695040888963407ull;
    const unsigned long long* p = buf + __umul64hi(h, lines) * 16 + j * 4;
    unsigned long long a, b, c, d;
    asm volatile("ld.global.nc.L2::evict_last.v4.u64 {%0,%1,%2,%3}, [%4];" : "=l"(a), "=l"(b), "=l"(c), "=l"(d) : "l"(p));
    acc ^= a + b + c + d;
  }
  if (acc == 0x123456789ull) sink[0] = acc;
}

template <int NBUF>
void run_tma(const unsigned long long* buf, unsigned long long lines, unsigned long long* sink, int sms, int threads) {
  const int iters = 512;
  const size_t smem = size_t(threads / 32) * NBUF * 32 * kSlot;
  if (smem > 227 * 1024) return;
  cudaFuncSetAttribute(tma_gather<NBUF>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, tma_gather<NBUF>, threads, smem);
  if (per_sm < 1) {
    printf("tma NBUF=%d threads=%d: does not fit\n", NBUF, threads);
    return;
  }
  const int blocks = sms * per_sm;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  tma_gather<NBUF><<<blocks, threads, smem>>>(buf, lines, iters, sink);
  cudaEventRecord(a);
  tma_gather<NBUF><<<blocks, threads, smem>>>(buf, lines, iters, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  const cudaError_t e = cudaGetLastError();
  const double n = double(blocks) * threads * iters * NBUF;
  printf("tma  NBUF=%d threads=%4d ctas/sm=%d smem=%6zu: %7.1f G lines/s %s\n", NBUF, threads, per_sm, smem,
         n / (ms * 1e-3) / 1e9, e == cudaSuccess ? "" : cudaGetErrorString(e));
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  unsigned long long* sink;
  cudaMalloc(&sink, 8);
  for (unsigned long long mb : {4ull, 16ull}) {
    const unsigned long long bytes = mb << 20, lines = bytes / 128;
    unsigned long long* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 0x11, bytes);
    printf("buffer %llu MiB\n", mb);
    {
      cudaEvent_t a, b;
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      const int blocks = sms * 2, iters = 1024;
      lsu_gather<<<blocks, 1024>>>(buf, lines, iters, sink);
      cudaEventRecord(a);
      lsu_gather<<<blocks, 1024>>>(buf, lines, iters, sink);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms = 0;
      cudaEventElapsedTime(&ms, a, b);
      printf("lsu  4 lanes x 32 B            : %7.1f G lines/s\n", double(blocks) * 256 * iters / (ms * 1e-3) / 1e9);
    }
    run_tma<1>(buf, lines, sink, sms, 1024);
    run_tma<1>(buf, lines, sink, sms, 512);
    run_tma<2>(buf, lines, sink, sms, 512);
    run_tma<2>(buf, lines, sink, sms, 256);
    run_tma<4>(buf, lines, sink, sms, 256);
    run_tma<4>(buf, lines, sink, sms, 128);
    run_tma<8>(buf, lines, sink, sms, 128);
    {
      PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
      cudaDriverEntryPointQueryResult q;
      cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", reinterpret_cast<void**>(&encode), cudaEnableDefault, &q);
      CUtensorMap tmap;
      cuuint64_t dims[2] = {16, lines};
      cuuint64_t strides[1] = {128};
      cuuint32_t box[2] = {16, 1};
      cuuint32_t estr[2] = {1, 1};
      CUresult r = encode(&tmap, CU_TENSOR_MAP_DATA_TYPE_UINT64, 2, buf, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("cuTensorMapEncodeTiled failed: %d\n", (int)r);
      } else {
        run_g4<1>(tmap, lines, sink, sms, 1024);
        run_g4<2>(tmap, lines, sink, sms, 1024);
        run_g4<2>(tmap, lines, sink, sms, 512);
        run_g4<4>(tmap, lines, sink, sms, 512);
        run_g4<4>(tmap, lines, sink, sms, 256);
      }
    }
    cudaFree(buf);
  }
  return 0;
}
