// apo_update_dense.cu -- instantiates the fused update kernels with SEL=false
// (run_updates boundary: dense rank-ordered rows).
// Built twice (paper_2510_14982_b200/_lib.py): keyed-stream kernels (APO_RNG_KEYED_ONLY: no Philox call
// site in the hot loops) and, with APO_PHILOX_VARIANT, the Philox build for sharded runs (apo_philox).
#ifdef APO_PHILOX_VARIANT
#define apo apo_philox
#else
#define APO_RNG_KEYED_ONLY 1
#endif
#include "apo_kernels.cuh"

namespace apo {

// cand_only: the CEC2022 split path (dim <= kCecEvalMaxDim).  Fused CEC2022
// (no split available) always takes the generic MAXC = 0 kernel so the
// register-resident variants carry no CEC code.
template <int NP>
const void* pick_update_dense_np(int dim, bool cand_only, bool cec) {
    if (cand_only) {
        if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_CAND, NP>;
        if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_CAND, NP>;
        if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_CAND, NP>;
        if (dim <= kGroupMaxDim) return (const void*)k_update_group<false, 0, KIND_CAND, NP>;
        return (const void*)k_update<false>;  // candidates-only through UpdArgs::cand_ok
    }
    if (dim > kGroupMaxDim) return (const void*)k_update<false>;
    if (cec) return (const void*)k_update_group<false, 0, KIND_ANY, NP>;
    if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_BASIC, NP>;
    if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_BASIC, NP>;
    if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_BASIC, NP>;
    return (const void*)k_update_group<false, 0, KIND_ANY, NP>;
}

const void* pick_update_dense(int dim, bool cand_only, bool cec, bool many) {  // many: npairs > 1
    return many ? pick_update_dense_np<2>(dim, cand_only, cec) : pick_update_dense_np<1>(dim, cand_only, cec);
}

}  // namespace apo
