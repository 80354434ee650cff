// apo_update_scripted.cu -- the dense update kernels once more, built to read scripted draws
// (APO_RNG_TABLE_ENABLED: uniform() may look a draw up in an apo_draw_table), under their own
// namespace so their symbols stay apart from the keyed instantiations (apo_update_dense.cu).  Only
// apo_run_updates_scripted / apo_select_dr_scripted launch them; every other entry runs kernels with
// no table code at all (even a never-taken table branch measured +1.5-9% on the C4 update).
#define APO_RNG_TABLE_ENABLED 1
#define apo apo_scripted
#include "apo_kernels.cuh"
#undef apo

namespace apo_scripted {

// The same choice as pick_update_dense (apo_update_dense.cu).
template <int NP>
const void* pick_np(int dim, bool cand_only, bool cec) {
    if (cand_only) {
        if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_CAND, NP>;
        if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_CAND, NP>;
        if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_CAND, NP>;
        if (dim <= kGroupMaxDim) return (const void*)k_update_group<false, 0, KIND_CAND, NP>;
        return (const void*)k_update<false>;
    }
    if (dim > kGroupMaxDim) return (const void*)k_update<false>;
    if (cec) return (const void*)k_update_group<false, 0, KIND_ANY, NP>;
    if (dim <= 32) return (const void*)k_update_group<false, 1, KIND_BASIC, NP>;
    if (dim <= 64) return (const void*)k_update_group<false, 2, KIND_BASIC, NP>;
    if (dim <= 128) return (const void*)k_update_group<false, 4, KIND_BASIC, NP>;
    return (const void*)k_update_group<false, 0, KIND_ANY, NP>;
}

const void* pick(int dim, bool cand_only, bool cec, bool many) {  // many: npairs > 1
    return many ? pick_np<2>(dim, cand_only, cec) : pick_np<1>(dim, cand_only, cec);
}

// The coordinator's set from scripted draws: the reference's partial Fisher-Yates over ranks 1..ps
// (core.py:271-278 -> rng.py:137-156, counters 1..count) run by one thread.
__global__ void k_dr_scripted(int ps, int count, Key base, int* __restrict__ perm, uint8_t* __restrict__ in_dr) {
    if (threadIdx.x != 0 || blockIdx.x != 0) return;
    for (int k = 0; k < ps; k++) {
        perm[k] = k;
        in_dr[k] = 0;
    }
    for (int j = 0; j < count; j++) {
        int r = j + (int)(uniform(base, 1ull + (uint64_t)j) * (double)(ps - j));
        if (r > ps - 1) r = ps - 1;
        const int a = perm[j];
        perm[j] = perm[r];
        perm[r] = a;
        in_dr[perm[j]] = 1;
    }
}

}  // namespace apo_scripted

namespace apo {

const void* pick_update_scripted(int dim, bool cand_only, bool cec, bool many) {
    return apo_scripted::pick(dim, cand_only, cec, many);
}

cudaError_t launch_dr_scripted(uint64_t table, int ps, int count, int* perm, uint8_t* in_dr, cudaStream_t st) {
    const apo_scripted::Key base = apo_scripted::stream_key(apo_scripted::RNG_TABLE, table, 0, apo_scripted::kCoordinator);
    apo_scripted::k_dr_scripted<<<1, 32, 0, st>>>(ps, count, base, perm, in_dr);
    return cudaGetLastError();
}

}  // namespace apo
