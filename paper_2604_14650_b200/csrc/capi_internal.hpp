// Helpers shared by the host and device halves of the C ABI.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_runtime.h>

#include "capi_util.hpp"
#include "lpm6/fib.hpp"
#include "lpm6/layout.hpp"
#include "lpm6cu.h"

namespace lpm6::capi {

// Host wall time of the phases of a device build, printed to stderr when the
// environment sets LPM6CU_TRACE_BUILD (diagnostics of sporadic slow commits).
class BuildTrace {
 public:
  explicit BuildTrace(const char* what) : what_(what), on_(std::getenv("LPM6CU_TRACE_BUILD") != nullptr) {}
  void mark(const char* phase) {
    if (!on_) return;
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[lpm6cu trace] %s: %s %.3f ms\n", what_, phase,
                 std::chrono::duration<double, std::milli>(now - t_).count());
    t_ = now;
  }

 private:
  const char* what_;
  bool on_;
  std::chrono::steady_clock::time_point t_ = std::chrono::steady_clock::now();
};

std::vector<Prefix> to_prefixes(const lpm6cu_prefix* rules, uint64_t n);
void export_geometry(const TreeLayout& t, lpm6cu_geometry* g);
Tree build_device_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                       const lpm6cu_build_opts* opts);

// The pool device-built line arrays come from (build.cu); release them with
// cudaFreeAsync once no lookup can still read them.
cudaMemPool_t fib_line_pool(int device);

// Destroy a FIB handle whose owner has already waited for every lookup that read it
// (FibStore: the snapshot's fences completed): frees without a device-wide sync.
void fib_destroy_quiesced(lpm6cu_fib* f);

// Device-side build (build.cu): returns a line array from fib_line_pool and its geometry.
void* device_build_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh, const lpm6cu_build_opts* opts,
                        cudaStream_t s, lpm6cu_geometry* geom);
// Layout only, from validated host intervals (build.cu).
void* device_build_tree_from_intervals(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                                       uint32_t default_nh, const lpm6cu_build_opts* opts, cudaStream_t s,
                                       lpm6cu_geometry* geom);

}  // namespace lpm6::capi
