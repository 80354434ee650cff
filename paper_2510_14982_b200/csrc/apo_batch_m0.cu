// apo_batch_m0.cu -- k_run_batch<0> (see apo_batch.cu).
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m0() { return (const void*)k_run_batch<0>; }

}  // namespace apo
