// apo_batch_m4.cu -- k_run_batch<4> (see apo_batch.cu).
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m4() { return (const void*)k_run_batch<4>; }

}  // namespace apo
