// apo_update_fused_ws.cu -- the warp-specialised fused CEC2022 update (apo_fused.cuh k_update_cec_ws):
// instantiation + launch.  Own TU so the library builds in parallel.
#include <cstdlib>

#include "apo_fused.cuh"

namespace apo {

static const int kNcompWs[12] = {1, 1, 1, 1, 1, 1, 1, 1, 5, 3, 5, 6};
static const int kFirstRotWs[12] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 1, 0, 0};  // first rflag = 1 (kCecSpec)

// Ring depth (X tiles) that fits next to M^T and the producers' scratch; 0 = does not fit.
int ws_shape(const UpdArgs& a, int optin, int np, size_t* smem, int* stage_shift) {
    const int dim = a.P.dim, nt = cec_nt(dim), ncomp = kNcompWs[a.O.cec.fn - 1];
    if (a.P.npairs > 1 || nt != 13 || dim <= 64 || (a.P.ld & 1)) return 0;
    const size_t avail = (size_t)optin - 1024;  // block_finish's static shared memory
    for (int ss = 1; ss >= 0; ss--) {
        for (int q = 12; q >= 2; q--) {
            const WsLayout L = ws_layout(dim, nt, ncomp, ss != 0, np, q);
            if (L.total <= avail) {
                *smem = L.total;
                *stage_shift = ss;
                return q;
            }
        }
    }
    return 0;
}

int ws_producers() {
    const int env = getenv("APO_WS_PRODUCERS") ? atoi(getenv("APO_WS_PRODUCERS")) : 8;
    return env < 1 ? 1 : env > 15 ? 15 : env;
}

cudaError_t launch_update_cec_ws(const UpdArgs& a, cudaStream_t st, unsigned* counter, int optin, int num_sms) {
    const int np = ws_producers();
    size_t smem = 0;
    int stage_shift = 0;
    int q = ws_shape(a, optin, np, &smem, &stage_shift);
    if (q < 2) return cudaErrorInvalidConfiguration;
    const void* fn = (const void*)k_update_cec_ws<13, 4>;
    cudaError_t e = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
    int bsm_comp = kFirstRotWs[a.O.cec.fn - 1], ncomp = kNcompWs[a.O.cec.fn - 1], npv = np;
    e = cudaMemsetAsync(counter, 0, sizeof(unsigned), st);
    if (e != cudaSuccess) return e;
    UpdArgs aa = a;
    void* args[] = {(void*)&aa, (void*)&bsm_comp, (void*)&ncomp, (void*)&stage_shift, (void*)&npv, (void*)&q,
                    (void*)&counter};
    return cudaLaunchKernel(fn, dim3(num_sms), dim3(512), args, smem, st);
}

}  // namespace apo
