// apo_update_sel.cu -- instantiates the fused update kernels with SEL=true
// (device-resident loop: slot-resident rows with per-slot buffer selectors).
#include "apo_kernels.cuh"

namespace apo {

const void* pick_update_sel(int dim) {
    if (dim <= 32) return (const void*)k_update_group<true, 1>;
    if (dim <= 64) return (const void*)k_update_group<true, 2>;
    if (dim <= 128) return (const void*)k_update_group<true, 4>;
    if (dim <= kGroupMaxDim) return (const void*)k_update_group<true, 0>;
    return (const void*)k_update<true>;
}

}  // namespace apo
