// TEST INFRASTRUCTURE ONLY — the drop-in check, written the way a user of the
// reference would write it: a reference lpm6::FibTable (the reference's own
// fib.cpp, compiled in place) handed to lpm6::gpu::Fib (include/lpm6cu.hpp),
// results compared with the reference's own lookup_interval_oracle and
// lookup_linear_oracle (intervals.cpp:95-145).
//
// Then the same for the update engine: random route changes are applied to the
// reference FibTable with its own insert / erase / modify / insert_or_replace
// (fib.cpp:120-161) and staged into lpm6::gpu::FibStore; per-op outcomes must
// agree, and after each commit every lookup through the store's snapshot must
// equal lookup_interval_oracle(build_intervals(updated reference FibTable)).
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
    // single-address lookup(t, addr) on a few of them
    for (size_t i = 0; i < 64 && i < addrs.size(); ++i)
      if (gfib.lookup(addrs[i]) != lpm6::lookup_interval_oracle(ref_map, static_cast<uint64_t>(addrs[i] >> 64)) &&
          bad++ < 5)
        std::printf("single lookup mismatch at %zu\n", i);
    std::printf("dropin: %zu rules, %zu intervals, %zu queries, %lu mismatches\n", fib.size(), ref_map.size(),
                addrs.size(), static_cast<unsigned long>(bad));
    if (bad) return 3;

    // ---- update engine against the reference FibTable mutators ----
    lpm6::gpu::FibStore store(0, fib);
    lpm6::FibTable ref = fib;
    for (int round = 0; round < 3; ++round) {
      std::vector<lpm6_update_op> ops;
      std::vector<int> want_status;
      for (int i = 0; i < 2000; ++i) {
        lpm6_update_op op{};
        const auto& cur = ref.entries();
        lpm6::Prefix p;
        if (!cur.empty() && rng() % 3 != 0) {
          p = cur[rng() % cur.size()];
        } else {
          p.length = 16 + static_cast<int>(rng() % 49);
          const lpm6::u128 mask = ~lpm6::u128(0) << (128 - p.length);
          p.value = ((lpm6::u128(rng() | (1ull << 61)) << 64)) & mask;  // inside 2000::/3-ish, canonical
        }
        p.next_hop = 1 + static_cast<uint32_t>(rng() % 250);
        op.kind = static_cast<uint32_t>(rng() % 4);
        std::memcpy(&op.prefix, &p, sizeof p);
        int st = 0;
        try {
          switch (op.kind) {
            case LPM6_UPDATE_INSERT: ref.insert(p); break;
            case LPM6_UPDATE_DELETE: ref.erase(p.value, p.length); break;
            case LPM6_UPDATE_MODIFY: ref.modify(p.value, p.length, p.next_hop); break;
            default: ref.insert_or_replace(p); break;
          }
        } catch (const lpm6::Error& err) {
          st = static_cast<int>(err.code()) + 1;
        }
        ops.push_back(op);
        want_status.push_back(st);
      }
      std::vector<int32_t> got_status(ops.size());
      store.stage(ops.data(), ops.size(), got_status.data());
      for (size_t i = 0; i < ops.size(); ++i)
        if (got_status[i] != want_status[i]) {
          std::printf("store: op %zu status %d, reference %d\n", i, got_status[i], want_status[i]);
          return 3;
        }
      const uint64_t epoch = store.commit();
      const lpm6::IntervalMap map = lpm6::build_intervals(ref);
      auto snap = store.acquire();
      const lpm6::gpu::Fib sf = snap.fib();
      std::vector<uint8_t> o(addrs.size() * sf.value_bytes());
      sf.lookup_batch(addrs.data(), addrs.size(), o.data());
      uint64_t sbad = 0;
      for (size_t i = 0; i < addrs.size(); ++i) {
        uint32_t got = 0;
        std::memcpy(&got, o.data() + i * sf.value_bytes(), sf.value_bytes());
        if (got != lpm6::lookup_interval_oracle(map, static_cast<uint64_t>(addrs[i] >> 64)) && sbad++ < 5)
          std::printf("store mismatch at %zu\n", i);
      }
      std::printf("store: epoch %lu, %zu rules, %zu intervals, %lu mismatches\n", static_cast<unsigned long>(epoch),
                  ref.size(), map.size(), static_cast<unsigned long>(sbad));
      if (sbad || epoch != static_cast<uint64_t>(round) + 2) return 3;
    }
    return 0;
  } catch (const lpm6cu::Error& err) {
    std::printf("dropin: %s\n", err.what());
    return (no_gpu_ok && err.status() == LPM6CU_E_CUDA) ? 0 : 1;
  }
}
