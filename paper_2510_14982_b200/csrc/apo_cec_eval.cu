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

const void* pick_cec_eval(bool sel, int dim, bool fast) {
    if (fast) return sel ? pick<true, true>(dim) : pick<false, true>(dim);
    return sel ? pick<true, false>(dim) : pick<false, false>(dim);
}

}  // namespace apo
