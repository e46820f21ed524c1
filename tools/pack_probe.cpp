#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <thread>
#include <vector>
int main() {
  const size_t n = 1ull << 27;  // 2 GiB of addresses
  uint64_t* src = (uint64_t*)aligned_alloc(64, n * 16);
  uint64_t* dst = (uint64_t*)aligned_alloc(64, n * 8);
  for (size_t i = 0; i < 2 * n; ++i) src[i] = i * 0x9E3779B97F4A7C15ull;
  memset(dst, 0, n * 8);
  unsigned hw = std::thread::hardware_concurrency();
  for (unsigned T : {1u, 2u, 4u, 8u, hw}) {
    for (int rep = 0; rep < 2; ++rep) {
      auto t0 = std::chrono::steady_clock::now();
      std::vector<std::thread> th;
      for (unsigned t = 0; t < T; ++t)
        th.emplace_back([&, t] {
          size_t a = n * t / T, b = n * (t + 1) / T;
          for (size_t i = a; i < b; ++i) dst[i] = src[2 * i + 1];
        });
      for (auto& x : th) x.join();
      double s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (rep) printf("threads %2u: %.2f G addr/s (%.1f GB/s read+write)\n", T, n / s / 1e9, n * 24 / s / 1e9);
    }
  }
  printf("%llu\n", (unsigned long long)dst[12345]);
}
