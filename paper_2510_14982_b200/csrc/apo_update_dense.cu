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
const void* pick_update_dense(int dim, bool cand_only, bool cec) {
    if (cand_only) {
        if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_CAND>;
        if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_CAND>;
        if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_CAND>;
        if (dim <= kGroupMaxDim) return (const void*)k_update_group<false, 0, KIND_CAND>;
        return (const void*)k_update<false>;  // candidates-only through UpdArgs::cand_ok
    }
    if (dim > kGroupMaxDim) return (const void*)k_update<false>;
    if (cec) return (const void*)k_update_group<false, 0, KIND_ANY>;
    if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_BASIC>;
    if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_BASIC>;
    if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_BASIC>;
    return (const void*)k_update_group<false, 0, KIND_ANY>;
}

}  // namespace apo
