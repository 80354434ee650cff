// apo_batch_m0.cu -- k_run_batch<0> (see apo_batch.cu).
// Built twice (paper_2510_14982_b200/_lib.py): keyed-stream kernels (APO_RNG_KEYED_ONLY: no Philox call
// site in the hot loops, measured 1-9% faster) and, with APO_PHILOX_VARIANT, the same kernels for the
// Philox production stream under namespace apo_philox.
#ifdef APO_PHILOX_VARIANT
#define apo apo_philox
#else
#define APO_RNG_KEYED_ONLY 1
#endif
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m0() { return (const void*)k_run_batch<0>; }

}  // namespace apo
