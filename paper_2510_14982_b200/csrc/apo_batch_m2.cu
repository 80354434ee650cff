// apo_batch_m2.cu -- k_run_batch<2> (see apo_batch.cu).
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m2() { return (const void*)k_run_batch<2>; }

}  // namespace apo
