// apo_cec_eval.cu -- instantiates k_cec_eval (CEC2022 DMMA evaluation + greedy select).
#include "apo_kernels.cuh"

namespace apo {

template <bool SEL>
static const void* pick(int dim) {
    if (dim > kCecEvalMaxDim) return nullptr;
    switch (cec_nt(dim)) {
    case 2: return (const void*)k_cec_eval<SEL, 2>;
    case 4: return (const void*)k_cec_eval<SEL, 4>;
    case 7: return (const void*)k_cec_eval<SEL, 7>;
    default: return (const void*)k_cec_eval<SEL, 13>;
    }
}

const void* pick_cec_eval(bool sel, int dim) { return sel ? pick<true>(dim) : pick<false>(dim); }

}  // namespace apo
