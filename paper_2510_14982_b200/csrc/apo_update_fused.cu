// apo_update_fused.cu -- the fused CEC2022 update (apo_fused.cuh): 16-warp instantiation + launch.
#include <cstdlib>

#include "apo_fused.cuh"

namespace apo {

const void* fused_kernel_12();  // apo_update_fused12.cu

// Instantiated for the C4 shape class (65 <= D <= 104, one pair); other shapes keep the split path.
// APO_FUSED_WARPS: 16 warps (128 registers, some spills) or 12 (up to 168 registers).
static const void* pick_fused(int dim, int warps) {
    if (cec_nt(dim) != 13 || dim <= 64) return nullptr;
    return warps >= 16 ? (const void*)k_update_cec<13, 4, 16> : fused_kernel_12();
}

static const int kNcomp[12] = {1, 1, 1, 1, 1, 1, 1, 1, 5, 3, 5, 6};
static const int kFirstRot[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0};  // first rflag = 1 (kCecSpec)

// Shape of the fused launch for this objective: warps per CTA (0: does not fit), shared memory bytes
// and whether the shift vectors are staged too.
int fused_cec_shape(const UpdArgs& a, int optin, size_t* smem, int* stage_shift) {
    if (a.P.npairs > 1 || !pick_fused(a.P.dim, 16)) return 0;
    const int dim = a.P.dim, nt = cec_nt(dim), ncomp = kNcomp[a.O.cec.fn - 1];
    const int avail = optin - 1024;  // block_finish's static shared memory
    for (int ss = 1; ss >= 0; ss--) {
        const size_t head =
            (fused_rot_bytes(dim, nt) + (ss ? 8 * (size_t)((ncomp * dim + 1) & ~1) : 0) + 15) & ~(size_t)15;
        if (head >= (size_t)avail) continue;
        int w = (int)(((size_t)avail - head) / fused_warp_bytes(dim));
        const int env_w = getenv("APO_FUSED_WARPS") ? atoi(getenv("APO_FUSED_WARPS")) : 16;
        if (w > env_w) w = env_w;
        w = w >= 16 ? 16 : w >= 12 ? 12 : 0;  // the instantiated CTA shapes
        if (w > 0) {
            *smem = head + (size_t)w * fused_warp_bytes(dim);
            *stage_shift = ss;
            return w;
        }
    }
    return 0;
}

// Launch on `st` (rank range [a.rank_lo, a.rank_hi), SEL rows); counter: one zeroed-here u32.
cudaError_t launch_update_cec_fused(const UpdArgs& a, cudaStream_t st, unsigned* counter, int optin, int num_sms) {
    int stage_shift = 0;
    size_t smem = 0;
    const int warps = fused_cec_shape(a, optin, &smem, &stage_shift);
    if (warps < 1) return cudaErrorInvalidConfiguration;
    const void* fn = pick_fused(a.P.dim, warps);
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int bsm_comp = kFirstRot[a.O.cec.fn - 1], ncomp = kNcomp[a.O.cec.fn - 1];
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    const long long groups = ((long long)(a.rank_hi - a.rank_lo) + 31) / 32;
    const long long need = (groups + warps - 1) / warps;
    const int grid = (int)(need < num_sms ? need : num_sms);
    UpdArgs aa = a;
    void* args[] = {(void*)&aa, (void*)&bsm_comp, (void*)&ncomp, (void*)&stage_shift, (void*)&counter};
    return cudaLaunchKernel(fn, dim3(grid), dim3(32 * warps), args, smem, st);
}

}  // namespace apo
