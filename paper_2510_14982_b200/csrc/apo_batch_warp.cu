// apo_batch_warp.cu -- k_run_batch<-1> (see apo_batch.cu).
#include "apo_kernels.cuh"

namespace apo {

const void* batch_kernel_warp() { return (const void*)k_run_batch<-1>; }

}  // namespace apo
