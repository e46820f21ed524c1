// Lookup kernels for 4-byte next hops (instantiated from lookup_kernel.cuh).
#include "lookup_kernel.cuh"

namespace lpm6::kern {
KernelFn pick_kernel_vb4(const PickArgs& a) { return pick_kernel_t<4>(a); }
}  // namespace lpm6::kern
