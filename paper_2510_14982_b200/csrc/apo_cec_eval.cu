// apo_cec_eval.cu -- instantiates k_cec_eval (CEC2022 DMMA evaluation + greedy select).
#include "apo_kernels.cuh"

namespace apo {

template <bool SEL, bool FAST>
static const void* pick(int dim) {
    if (dim > kCecEvalMaxDim) return nullptr;
    switch (cec_nt(dim)) {
    case 2: return (const void*)k_cec_eval<SEL, 2, FAST>;
    case 4: return (const void*)k_cec_eval<SEL, 4, FAST>;
    case 7: return (const void*)k_cec_eval<SEL, 7, FAST>;
    default: return (const void*)k_cec_eval<SEL, 13, FAST>;
    }
}

// Every CEC2022 function takes the FAST form (one rotation staged in shared
// memory); the L1-only form stays in apo_kernels.cuh for experiments.
const void* pick_cec_eval(bool sel, int dim, bool fast) {
    (void)fast;
    return sel ? pick<true, true>(dim) : pick<false, true>(dim);
}

// Basic function b alone on each row of z (n <= rows' stride): variant 0 = the quad evaluator of the
// headline kernels (cec_basic_quad), 1 = the warp evaluator (batch kernel, GEMM finish).  Verification
// entry for the building blocks pinned to the reference (tests/test_cec_pinning.py).
__global__ void k_debug_cec_basic(int b, const double* z, long long rows, int n, const double* ew, double* out,
                                  int variant) {
    const int lane = threadIdx.x & 31;
    const long long w = (long long)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
    if (variant == 0) {
        const int q = lane >> 2, t = lane & 3;
        const long long r = w * 8 + q;
        const bool live = r < rows;
        const double v = cec_basic_quad(b, z + (live ? r : 0) * n, n, t, ew);
        if (live && t == 0) out[r] = v;
    } else if (w < rows) {
        const double v = cec_basic_warp(b, z + w * n, n, lane);
        if (lane == 0) out[w] = v;
    }
}

cudaError_t launch_debug_cec_basic(int b, const double* z, long long rows, int n, const double* ew, double* out,
                                   int variant, cudaStream_t st) {
    const long long warps = variant == 0 ? (rows + 7) / 8 : rows;
    const int grid = (int)((warps + 7) / 8);
    k_debug_cec_basic<<<grid > 0 ? grid : 1, 256, 0, st>>>(b, z, rows, n, ew, out, variant);
    return cudaGetLastError();
}

}  // namespace apo
