// Helpers shared by the host and device halves of the C ABI.
#pragma once

#include <vector>

#include <cuda_runtime.h>

#include "capi_util.hpp"
#include "lpm6/fib.hpp"
#include "lpm6/layout.hpp"
#include "lpm6cu.h"

namespace lpm6::capi {

std::vector<Prefix> to_prefixes(const lpm6cu_prefix* rules, uint64_t n);
void export_geometry(const TreeLayout& t, lpm6cu_geometry* g);
Tree build_device_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh,
                       const lpm6cu_build_opts* opts);

// Device-side build (build.cu): returns a cudaMalloc'ed line array and its geometry.
void* device_build_tree(const lpm6cu_prefix* rules, uint64_t n, uint32_t default_nh, const lpm6cu_build_opts* opts,
                        cudaStream_t s, lpm6cu_geometry* geom);
// Layout only, from validated host intervals (build.cu).
void* device_build_tree_from_intervals(const uint64_t* boundaries, const uint32_t* next_hops, uint64_t m,
                                       uint32_t default_nh, const lpm6cu_build_opts* opts, cudaStream_t s,
                                       lpm6cu_geometry* geom);

}  // namespace lpm6::capi
