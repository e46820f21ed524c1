// Serving-size latency through the C ABI from C++ (VERDICT r1 item 8): the C1 FIB,
// 256 .. 65,536 device-resident addresses; call-to-result (launch + stream sync)
// medians for lpm6cu_lookup_batch (pointer-kind checks) and
// lpm6cu_lookup_batch_device (launch only), and back-to-back call rates.
//   g++ -O2 -std=c++17 tools/latency_abi.cpp -Iinclude -I/usr/local/cuda/include \
//       -Lpaper_2604_14650_b200/lib -llpm6cu -L/usr/local/cuda/lib64 -lcudart \
//       -Wl,-rpath,$PWD/paper_2604_14650_b200/lib -o tools/latency_abi
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <vector>

#include "lpm6cu.h"

#define CK(x)                                                              \
  do {                                                                     \
    int st_ = (x);                                                         \
    if (st_) {                                                             \
      std::fprintf(stderr, "%s -> %d: %s\n", #x, st_, lpm6cu_last_error()); \
      return 1;                                                            \
    }                                                                      \
  } while (0)

static double now_us() {
  return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count();
}

int main() {
  uint64_t n_rules = 0;
  uint32_t dflt = 0;
  CK(lpm6_workload_fib(1, nullptr, 0, &n_rules, &dflt));
  std::vector<lpm6cu_prefix> rules(n_rules);
  CK(lpm6_workload_fib(1, rules.data(), n_rules, &n_rules, &dflt));
  lpm6cu_fib* fib = nullptr;
  CK(lpm6cu_fib_build(0, rules.data(), n_rules, dflt, nullptr, &fib));
  const uint64_t nmax = 65536;
  std::vector<uint64_t> h(2 * nmax);
  CK(lpm6_workload_queries_host(1, rules.data(), n_rules, 0, nmax, h.data(), 8));
  void *d_a = nullptr, *d_o = nullptr;
  cudaMalloc(&d_a, nmax * 16);
  cudaMalloc(&d_o, nmax * 4);
  cudaMemcpy(d_a, h.data(), nmax * 16, cudaMemcpyHostToDevice);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  std::printf("{\"fib\": \"C1\", \"rows\": [");
  bool first = true;
  for (uint64_t n : {256ull, 4096ull, 65536ull}) {
    for (int dev_entry = 0; dev_entry < 2; ++dev_entry) {
      auto call = [&]() {
        return dev_entry ? lpm6cu_lookup_batch_device(fib, d_a, n, d_o, s) : lpm6cu_lookup_batch(fib, d_a, n, d_o, s);
      };
      for (int i = 0; i < 50; ++i) CK(call());
      cudaStreamSynchronize(s);
      std::vector<double> lat;
      for (int i = 0; i < 2000; ++i) {
        const double t0 = now_us();
        CK(call());
        cudaStreamSynchronize(s);
        lat.push_back(now_us() - t0);
      }
      std::sort(lat.begin(), lat.end());
      const double t0 = now_us();
      for (int i = 0; i < 2000; ++i) CK(call());
      cudaStreamSynchronize(s);
      const double b2b = (now_us() - t0) / 2000;
      // the floor: an empty stream sync alone and an empty-kernel-free round trip
      std::printf("%s{\"batch\": %llu, \"entry\": \"%s\", \"us_call_to_result_median\": %.2f, \"p99\": %.2f, "
                  "\"us_per_call_back_to_back\": %.2f}",
                  first ? "" : ", ", static_cast<unsigned long long>(n),
                  dev_entry ? "lpm6cu_lookup_batch_device" : "lpm6cu_lookup_batch", lat[lat.size() / 2],
                  lat[lat.size() * 99 / 100], b2b);
      first = false;
    }
  }
  std::printf("]}\n");
  lpm6cu_fib_destroy(fib);
  return 0;
}
