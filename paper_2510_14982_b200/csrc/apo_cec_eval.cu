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

}  // namespace apo
