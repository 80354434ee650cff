// apo_batch_m1.cu -- k_run_batch<1> (see apo_batch.cu).
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_m1() { return (const void*)k_run_batch<1>; }

}  // namespace apo
