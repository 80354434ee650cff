// apo_batch.cu -- picks the persistent one-CTA-per-run batch kernel (keyed or Philox build); each
// MAXC variant is instantiated in its own TU (apo_batch_m*.cu) so they build in parallel.
#include "apo_kernels.cuh"

namespace apo_philox {  // the same getters of the Philox builds (APO_PHILOX_VARIANT)
const void* batch_kernel_m1();
const void* batch_kernel_m2();
const void* batch_kernel_m4();
const void* batch_kernel_m0();
const void* batch_kernel_warp();
}  // namespace apo_philox

namespace apo_many {  // keyed, npairs > 1 (APO_MANY_PAIRS_VARIANT)
const void* batch_kernel_m1();
const void* batch_kernel_m2();
const void* batch_kernel_m4();
const void* batch_kernel_m0();
}  // namespace apo_many

namespace apo {

const void* batch_kernel_m1();
const void* batch_kernel_m2();
const void* batch_kernel_m4();
const void* batch_kernel_m0();
const void* batch_kernel_warp();

const void* pick_run_batch(int dim, int rng, bool many) {
    if (many && rng != RNG_PHILOX && dim <= kGroupMaxDim) {
        if (dim <= 32) return apo_many::batch_kernel_m1();
        if (dim <= 64) return apo_many::batch_kernel_m2();
        if (dim <= 128) return apo_many::batch_kernel_m4();
        return apo_many::batch_kernel_m0();
    }
    if (rng == RNG_PHILOX) {
        if (dim <= 32) return apo_philox::batch_kernel_m1();
        if (dim <= 64) return apo_philox::batch_kernel_m2();
        if (dim <= 128) return apo_philox::batch_kernel_m4();
        if (dim <= kGroupMaxDim) return apo_philox::batch_kernel_m0();
        return apo_philox::batch_kernel_warp();
    }
    if (dim <= 32) return batch_kernel_m1();
    if (dim <= 64) return batch_kernel_m2();
    if (dim <= 128) return batch_kernel_m4();
    if (dim <= kGroupMaxDim) return batch_kernel_m0();
    return batch_kernel_warp();
}

}  // namespace apo
