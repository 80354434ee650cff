// apo_batch.cu -- instantiates the persistent one-CTA-per-run batch kernel.
#include "apo_kernels.cuh"

namespace apo {

const void* pick_run_batch(int dim) {
    if (dim <= 32) return (const void*)k_run_batch<1>;
    if (dim <= 64) return (const void*)k_run_batch<2>;
    if (dim <= 128) return (const void*)k_run_batch<4>;
    if (dim <= kGroupMaxDim) return (const void*)k_run_batch<0>;
    return (const void*)k_run_batch<-1>;
}

}  // namespace apo
