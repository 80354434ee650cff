// apo_update_fused12.cu -- the fused CEC2022 update (apo_fused.cuh), 12-warp instantiation (168
// registers, no spills); a separate TU so the library builds in parallel.
#include "apo_fused.cuh"

namespace apo {

const void* fused_kernel_12() { return (const void*)k_update_cec<13, 4, 12>; }

}  // namespace apo
