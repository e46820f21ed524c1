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

  // PBT1 snapshot file (the reference's save_snapshot_file output) -> device FIB.
  static Fib load_snapshot(int device, const std::string& path, uint32_t value_bytes = 0, void* stream = nullptr) {
    lpm6cu_build_opts o{};
    o.merge_adjacent = 1;
    o.value_bytes = value_bytes;
    Fib f;
    lpm6cu::check(lpm6cu_fib_load_snapshot(device, path.c_str(), 0, &o, stream, &f.h_));
    return f;
  }

  // Borrow a handle (a store snapshot's FIB): not destroyed by this object.
  static Fib borrow(const lpm6cu_fib* h) {
    Fib f;
    f.h_ = const_cast<lpm6cu_fib*>(h);
    f.owned_ = false;
    return f;
  }

  Fib(const Fib&) = delete;
  Fib& operator=(const Fib&) = delete;
  Fib(Fib&& o) noexcept : h_(std::exchange(o.h_, nullptr)), owned_(o.owned_) {}
  Fib& operator=(Fib&& o) noexcept {
    if (this != &o) {
      reset();
      h_ = std::exchange(o.h_, nullptr);
      owned_ = o.owned_;
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
  // Device buffers known to be on this FIB's GPU: the launch only (serving-size batches).
  void lookup_batch_device(const void* d_addrs, uint64_t n, void* d_out, void* stream = nullptr) const {
    lpm6cu::check(lpm6cu_lookup_batch_device(h_, d_addrs, n, d_out, stream));
  }

  // One address (the reference's lookup(t, addr)): a batch of one through
  // the host path — correct but latency-bound; batch where throughput matters.
  template <class U128>
  uint32_t lookup(const U128& addr) const {
    static_assert(sizeof(U128) == 16, "address must be a 16-byte little-endian u128");
    uint32_t out = 0;
    lpm6cu::check(lpm6cu_lookup_batch(h_, &addr, 1, &out, nullptr));
    return out & (value_bytes() == 4 ? 0xFFFFFFFFu : (1u << (8 * value_bytes())) - 1u);
  }

  // 8-byte keys (search_batch's input); device buffers.
  void lookup_keys(const uint64_t* d_keys, uint64_t n, void* d_out, void* stream = nullptr) const {
    lpm6cu::check(lpm6cu_lookup_keys(h_, d_keys, n, d_out, stream));
  }

  // search_batch: interval ordinals (+ next hops when d_next_hops != nullptr); device buffers.
  void search_batch(const uint64_t* d_keys, uint64_t n, uint32_t* d_ordinals, void* d_next_hops = nullptr,
                    void* stream = nullptr) const {
    lpm6cu::check(lpm6cu_search_batch(h_, d_keys, n, d_ordinals, d_next_hops, stream));
  }

  // Frames `stride` bytes apart, IPv6 destination at `dst_offset` (38 = Ethernet + IPv6); device buffers.
  void lookup_packets(const void* d_frames, uint64_t n, uint64_t stride, uint32_t dst_offset, void* d_out,
                      void* stream = nullptr) const {
    lpm6cu::check(lpm6cu_lookup_packets(h_, d_frames, n, stride, dst_offset, d_out, stream));
  }

  // Times the line paths (which L1TEX pipe carries the L2 lines, lpm6cu_kernel_config)
  // on a representative device batch and keeps the fastest; returns 0..3. Not
  // concurrent with lookups.
  uint32_t tune_line_path(const void* d_addrs, uint64_t n, void* d_out, void* stream = nullptr, uint32_t reps = 3) {
    uint32_t chosen = 0;
    lpm6cu::check(lpm6cu_fib_tune_line_path(h_, d_addrs, n, d_out, stream, reps, &chosen));
    return chosen;
  }

  lpm6cu_fib* handle() const { return h_; }

 private:
  Fib() = default;
  void reset() {
    if (h_ && owned_) lpm6cu_fib_destroy(h_);
    h_ = nullptr;
  }
  lpm6cu_fib* h_ = nullptr;
  bool owned_ = true;
};

// The reference's FibStore on the GPU: stage / commit / acquire / release.
class FibStore {
 public:
  template <class FibTable, class = decltype(std::declval<const FibTable&>().entries().data())>
  FibStore(int device, const FibTable& fib, uint32_t value_bytes = 0) {
    lpm6cu_build_opts o{};
    o.merge_adjacent = 1;
    o.value_bytes = value_bytes;
    lpm6cu::check(lpm6cu_store_create(device, reinterpret_cast<const lpm6cu_prefix*>(fib.entries().data()),
                                      fib.entries().size(), fib.default_next_hop(), &o, &h_));
  }
  FibStore(const FibStore&) = delete;
  FibStore& operator=(const FibStore&) = delete;
  ~FibStore() {
    if (h_) lpm6cu_store_destroy(h_);
  }

  // RAII pin: lookups through fib() see one epoch; the destructor releases on the
  // stream the snapshot was used on (set with use_on()).
  class Snapshot {
   public:
    explicit Snapshot(lpm6cu_store* st) { lpm6cu::check(lpm6cu_store_acquire(st, &s_)); }
    Snapshot(const Snapshot&) = delete;
    Snapshot& operator=(const Snapshot&) = delete;
    ~Snapshot() {
      if (s_) lpm6cu_store_release(s_, stream_);
    }
    uint64_t epoch() const {
      uint64_t e = 0;
      lpm6cu::check(lpm6cu_snapshot_info(s_, &e, nullptr, nullptr));
      return e;
    }
    Fib fib() const {
      const lpm6cu_fib* f = nullptr;
      lpm6cu::check(lpm6cu_snapshot_info(s_, nullptr, &f, nullptr));
      return Fib::borrow(f);
    }
    void use_on(void* stream) { stream_ = stream; }

   private:
    lpm6cu_snapshot* s_ = nullptr;
    void* stream_ = nullptr;
  };

  Snapshot acquire() const { return Snapshot(h_); }
  // Returns the ops staged; op_status (optional, n entries) gets 0 or a status per op.
  uint64_t stage(const lpm6_update_op* ops, uint64_t n, int32_t* op_status = nullptr) {
    uint64_t staged = 0;
    lpm6cu::check(lpm6cu_store_stage(h_, ops, n, &staged, op_status));
    return staged;
  }
  uint64_t commit() {
    uint64_t e = 0;
    lpm6cu::check(lpm6cu_store_commit(h_, &e));
    return e;
  }
  lpm6cu_store_stats stats() const {
    lpm6cu_store_stats s{};
    lpm6cu::check(lpm6cu_store_stats_get(h_, &s));
    return s;
  }

 private:
  lpm6cu_store* h_ = nullptr;
};

}  // namespace lpm6::gpu
