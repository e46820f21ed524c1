// lpm6cu.hpp — header-only C++ wrapper over the C ABI (include/lpm6cu.h).
//
// lpm6::gpu::Fib is what a user of the reference's lpm6 library switches to:
//
//   lpm6::FibTable fib = lpm6::load_fib_file("rib.txt");      // reference, fib.hpp:119-121
//   lpm6::gpu::Fib gfib(/*device=*/0, fib);                     // build_intervals + layout + upload
//   gfib.lookup_batch(addrs, n, next_hops);                     // replaces search_batch / lookup
//
// Any FibTable-like type works as long as it has entries() (a contiguous range
// of lpm6::Prefix, fib.hpp:22-29: u128 value, int length, u32 next_hop) and
// default_next_hop(). Failures throw lpm6cu::Error (status = (int)Errc + 1); when
// the reference's lpm6/types.hpp is visible and LPM6CU_THROW_REFERENCE_ERROR is
// defined, they throw lpm6::Error with the same Errc instead (types.hpp:42-49).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <utility>

#include "lpm6cu.h"

namespace lpm6cu {

class Error : public std::runtime_error {
 public:
  Error(int status, const std::string& what) : std::runtime_error(what), status_(status) {}
  int status() const noexcept { return status_; }
  const char* code() const noexcept { return lpm6cu_status_name(status_); }

 private:
  int status_;
};

inline void check(int status) {
  if (status == LPM6CU_OK) return;
#ifdef LPM6CU_THROW_REFERENCE_ERROR
  if (status >= 1 && status <= 12)
    throw lpm6::Error(static_cast<lpm6::Errc>(status - 1), lpm6cu_last_error());
#endif
  throw Error(status, std::string(lpm6cu_status_name(status)) + ": " + lpm6cu_last_error());
}

}  // namespace lpm6cu

namespace lpm6::gpu {

class Fib {
 public:
  // From raw rules in lpm6::Prefix layout.
  Fib(int device, const lpm6cu_prefix* rules, uint64_t n, uint32_t default_next_hop,
      bool merge_adjacent = true, uint32_t value_bytes = 0) {
    lpm6cu_build_opts o{};
    o.merge_adjacent = merge_adjacent ? 1u : 0u;
    o.value_bytes = value_bytes;
    lpm6cu::check(lpm6cu_fib_build(device, rules, n, default_next_hop, &o, &h_));
  }

  // From a reference FibTable (or anything with entries() / default_next_hop()).
  template <class FibTable, class = decltype(std::declval<const FibTable&>().entries().data())>
  Fib(int device, const FibTable& fib, bool merge_adjacent = true, uint32_t value_bytes = 0)
      : Fib(device, reinterpret_cast<const lpm6cu_prefix*>(fib.entries().data()), fib.entries().size(),
            fib.default_next_hop(), merge_adjacent, value_bytes) {
    static_assert(sizeof(*fib.entries().data()) == sizeof(lpm6cu_prefix), "Prefix layout mismatch");
  }

  Fib(const Fib&) = delete;
  Fib& operator=(const Fib&) = delete;
  Fib(Fib&& o) noexcept : h_(std::exchange(o.h_, nullptr)) {}
  Fib& operator=(Fib&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
    }
    return *this;
  }
  ~Fib() { reset(); }

  lpm6cu_geometry geometry() const {
    lpm6cu_geometry g{};
    lpm6cu::check(lpm6cu_fib_geometry(h_, &g));
    return g;
  }
  uint32_t value_bytes() const { return geometry().value_bytes; }

  // n addresses (u128 little-endian, 16 bytes each) -> n next hops of value_bytes()
  // each. Host or device pointers; `stream` is a cudaStream_t (nullptr = default).
  void lookup_batch(const void* addrs, uint64_t n, void* out_next_hops, void* stream = nullptr) const {
    lpm6cu::check(lpm6cu_lookup_batch(h_, addrs, n, out_next_hops, stream));
  }

  lpm6cu_fib* handle() const { return h_; }

 private:
  void reset() {
    if (h_) lpm6cu_fib_destroy(h_);
    h_ = nullptr;
  }
  lpm6cu_fib* h_ = nullptr;
};

}  // namespace lpm6::gpu
