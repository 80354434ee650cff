// apo_update_dense.cu -- instantiates the fused update kernels with SEL=false
// (run_updates boundary: dense rank-ordered rows).
#include "apo_kernels.cuh"

namespace apo {

const void* pick_update_dense(int dim) {
    if (dim <= 32) return (const void*)k_update_group<false, 1>;
    if (dim <= 64) return (const void*)k_update_group<false, 2>;
    if (dim <= 128) return (const void*)k_update_group<false, 4>;
    if (dim <= kGroupMaxDim) return (const void*)k_update_group<false, 0>;
    return (const void*)k_update<false>;
}

}  // namespace apo
