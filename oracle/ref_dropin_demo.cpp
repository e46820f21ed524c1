// TEST INFRASTRUCTURE ONLY — the drop-in check, written the way a user of the
// reference would write it: a reference lpm6::FibTable (the reference's own
// fib.cpp, compiled in place) handed to lpm6::gpu::Fib (include/lpm6cu.hpp),
// results compared with the reference's own lookup_interval_oracle and
// lookup_linear_oracle (intervals.cpp:95-145).
//
//   oracle/_ref/ref_dropin_demo [n_rules] [n_queries] [--no-gpu-ok]
// exit 0 = every query matched (or, with --no-gpu-ok and no GPU, the library
// refused with CudaError); 3 = a mismatch (the reference CLI's verify code).
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "lpm6/fib.hpp"
#include "lpm6/intervals.hpp"
#include "lpm6cu.hpp"

int main(int argc, char** argv) {
  const uint64_t n_rules = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 20000;
  const uint64_t n_q = argc > 2 ? std::strtoull(argv[2], nullptr, 10) : 1u << 20;
  const bool no_gpu_ok = argc > 3 && std::strcmp(argv[3], "--no-gpu-ok") == 0;

  // The reference's synthetic FIB (fib.cpp:237-273) + a default route.
  lpm6::FibTable fib = lpm6::synth_fib(n_rules, lpm6::LengthDistribution::backbone_default(7));
  fib.insert(lpm6::Prefix{0, 0, 99});
  const lpm6::IntervalMap ref_map = lpm6::build_intervals(fib);

  // Our host build through the C ABI must equal the reference's build_intervals.
  std::vector<uint64_t> b(2 * fib.size() + 1);
  std::vector<uint32_t> nh(2 * fib.size() + 1);
  uint64_t m = 0;
  lpm6cu::check(lpm6_build_intervals(reinterpret_cast<const lpm6cu_prefix*>(fib.entries().data()), fib.size(),
                                     fib.default_next_hop(), 1, b.data(), nh.data(), b.size(), &m));
  if (m != ref_map.size() || std::memcmp(b.data(), ref_map.boundaries.data(), m * 8) != 0 ||
      std::memcmp(nh.data(), ref_map.next_hops.data(), m * 4) != 0) {
    std::printf("MISMATCH: build_intervals differs from the reference\n");
    return 3;
  }

  // Queries: every boundary and its neighbours, then in-prefix and uniform addresses.
  std::vector<lpm6::u128> addrs;
  addrs.reserve(n_q);
  std::mt19937_64 rng(11);
  for (uint64_t x : ref_map.boundaries) {
    for (uint64_t k : {x, x - 1, x + 1}) addrs.push_back((lpm6::u128(k) << 64) | rng());
    if (addrs.size() >= n_q / 2) break;
  }
  const auto& e = fib.entries();
  while (addrs.size() < n_q) {
    const lpm6::Prefix& p = e[rng() % e.size()];
    const lpm6::u128 host = (lpm6::u128(rng()) << 64) | rng();
    const lpm6::u128 mask = p.length == 0 ? 0 : ~lpm6::u128(0) << (128 - p.length);
    addrs.push_back((rng() & 3) ? (p.value | (host & ~mask)) : host);
  }

  try {
    lpm6::gpu::Fib gfib(0, fib);  // FibTable -> intervals -> B200 layout -> device
    std::vector<uint8_t> out(addrs.size() * gfib.value_bytes());
    gfib.lookup_batch(addrs.data(), addrs.size(), out.data());  // host buffers
    uint64_t bad = 0;
    for (size_t i = 0; i < addrs.size(); ++i) {
      uint32_t got = 0;
      std::memcpy(&got, out.data() + i * gfib.value_bytes(), gfib.value_bytes());
      const uint32_t want = lpm6::lookup_interval_oracle(ref_map, static_cast<uint64_t>(addrs[i] >> 64));
      if (got != want) {
        if (bad++ < 5) std::printf("mismatch at %zu: got %u want %u\n", i, got, want);
      } else if (i % 4096 == 0 && got != lpm6::lookup_linear_oracle(fib, addrs[i])) {
        if (bad++ < 5) std::printf("linear-oracle mismatch at %zu\n", i);
      }
    }
    std::printf("dropin: %zu rules, %zu intervals, %zu queries, %lu mismatches\n", fib.size(), ref_map.size(),
                addrs.size(), static_cast<unsigned long>(bad));
    return bad ? 3 : 0;
  } catch (const lpm6cu::Error& err) {
    std::printf("dropin: %s\n", err.what());
    return (no_gpu_ok && err.status() == LPM6CU_E_CUDA) ? 0 : 1;
  }
}
