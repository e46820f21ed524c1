// Lookup kernels for 1-byte next hops (instantiated from lookup_kernel.cuh).
#include "lookup_kernel.cuh"

namespace lpm6::kern {
KernelFn pick_kernel_vb1(const PickArgs& a) { return pick_kernel_t<1>(a); }
}  // namespace lpm6::kern
