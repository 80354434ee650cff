// apo_batch_m2.cu -- k_run_batch<2> (see apo_batch.cu).
// Built three times (paper_2510_14982_b200/_lib.py): keyed-stream kernels for npairs == 1
// (APO_RNG_KEYED_ONLY, NP = 1: no Philox call site, no many-pairs body -- each measured 1-9% faster),
// APO_MANY_PAIRS_VARIANT (keyed, npairs > 1, namespace apo_many) and APO_PHILOX_VARIANT (the Philox
// production stream, either pair case, namespace apo_philox).
#if defined(APO_PHILOX_VARIANT)
#define apo apo_philox
#define APO_BATCH_NP 0
#elif defined(APO_MANY_PAIRS_VARIANT)
#define apo apo_many
#define APO_RNG_KEYED_ONLY 1
#define APO_BATCH_NP 2
#else
#define APO_RNG_KEYED_ONLY 1
#define APO_BATCH_NP 1
#endif
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m2() { return (const void*)k_run_batch<2, APO_BATCH_NP>; }

}  // namespace apo
