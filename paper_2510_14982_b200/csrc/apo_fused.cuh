// apo_fused.cuh -- CEC2022 (D <= 104) on the HBM-resident population as ONE kernel per
// iteration: candidate generation (the group path of apo_group.cuh, numba_backend.py:141-257) and the
// DMMA evaluation + greedy select (k_cec_eval's quad evaluator, numba_backend.py:259-290) share a warp.
//
// The split path (k_update_group<KIND_CAND> then k_cec_eval) writes every candidate row to HBM and
// reads it back in the second kernel (~1.7 GB per iteration at ps = 10^6, D = 100).  Here a warp
// generates 8 candidates into a shared-memory tile (and, speculatively, into the slot's alternate
// buffer, where an accepted row must end up), then rotates the tile with mma.sync.m8n8k4.f64 against
// the CTA's shared-memory copy of M^T, evaluates the basic functions per lane quad and flips the
// slot selectors of accepted rows.  Warps of one SM interleave the issue-bound candidate phase with
// the DMMA-bound rotation, so the two overlap instead of running back to back.
//
// Shared memory per CTA: [rotation `bsm_comp` (n4 x (8 NT + 4)) | shift vectors (staged when they fit)]
// + per warp [group header (draw scalars, row keys, mask bits) | union(phase-A permutations, 8-row X tile)].
// Arithmetic: the candidate half is bit-exact with the oracle (this TU keeps --fmad=false); the
// evaluation is k_cec_eval's code compiled without FMA contraction (closer to the oracle than the
// split path, which contracts), so the two paths agree to ~1e-15 relative, not bit for bit.
#pragma once
#include "apo_kernels.cuh"

namespace apo {

__host__ __device__ inline size_t fused_warp_bytes(int dim) {
    const size_t perm = 32 * (size_t)((dim + 3) & ~3);
    const size_t xt = 8 * (size_t)kCecRows * (size_t)cec_stride(dim);
    return group_head_bytes(dim) + (((perm > xt ? perm : xt) + 15) & ~(size_t)15);
}
__host__ __device__ inline size_t fused_rot_bytes(int dim, int nt) {
    return 8 * (size_t)((dim + 3) & ~3) * (size_t)cec_bsm_stride(nt);
}

template <int NT, int MAXC, int WARPS>
__global__ void __launch_bounds__(32 * WARPS, 1) k_update_cec(UpdArgs A, int bsm_comp, int ncomp, int stage_shift,
                                                      unsigned* counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    const IterParams& P = A.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int dim = P.dim, n4 = (dim + 3) & ~3, cs = cec_stride(dim);
    // the staged rotation (+ shift vectors when they fit): one copy per persistent CTA
    double* bsm = reinterpret_cast<double*>(smem);
    CecData C = A.O.cec;
    {
        const int bs = cec_bsm_stride(NT), w8 = 8 * NT;
        const double* rsrc = C.rot_pad + (size_t)bsm_comp * n4 * w8;
        for (int e = threadIdx.x; e < n4 * w8; e += blockDim.x) {
            const int i = e / w8, j = e - i * w8;
            bsm[i * bs + j] = rsrc[e];
        }
        if (stage_shift) {
            double* osm = bsm + (size_t)n4 * bs;
            for (int i = threadIdx.x; i < ncomp * dim; i += blockDim.x) osm[i] = C.shift[i];
            C.shift = osm;
        }
    }
    const size_t head = fused_rot_bytes(dim, NT) + (stage_shift ? 8 * (size_t)((ncomp * dim + 1) & ~1) : 0);
    unsigned char* wbase = smem + ((head + 15) & ~(size_t)15) + (size_t)warp * fused_warp_bytes(dim);
    const GroupScratch g = group_scratch(wbase, dim, false, 0);
    double* X = reinterpret_cast<double*>(wbase + group_head_bytes(dim));  // aliases the permutations
    __syncthreads();
    const SelSlots R{A.pos0, A.pos1, A.sel, A.fit, A.order, P.ld};
    const double* ew = A.O.table_len >= dim ? A.O.table : nullptr;  // ELLIPS weights (host libm)
    const int q = lane >> 2, t = lane & 3;
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    const int ngroups = (A.rank_hi - A.rank_lo + 31) / 32;
    auto claim = [&]() -> int {
        unsigned v = 0;
        if (lane == 0) v = atomicAdd(counter, 1u);
        return (int)__shfl_sync(kFull, v, 0);
    };
    for (int grp = claim(); grp < ngroups; grp = claim()) {
        const int i0 = A.rank_lo + grp * 32 + 1;
        const int n = min(32, A.rank_hi - (i0 - 1));
        if (lane < n) {  // phase A: lane = protozoon (draws, partner/pairs, exp weight, mask chain)
            const int r0 = i0 - 1 + lane;
            const bool dr = ((A.in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0;
            group_phase_a(P, R, i0 + lane, dr, dr ? A.p_dr[r0] : 0.0, g, lane);
        }
        __syncwarp();
        for (int h = 0; h < n; h += kCecRows) {
            const int nb = min(kCecRows, n - h);
            unsigned okmask = 0;
            for (int m = 0; m < nb; m++) {  // phase B: warp = protozoon, candidate -> alt buffer + X row m
                const int p = h + m;
                double* dst = R.alt_key(g.slot[4 * p]);
                const bool ok = group_candidate<MAXC, false, true, SelSlots, true>(P, A.O, R, i0 + p, p, dst,
                                                                                   X + (size_t)m * cs, nullptr, g,
                                                                                   lane, nullptr);
                okmask |= (ok ? 1u : 0u) << m;
            }
            if (n4 > dim)  // zero pads: the rotation runs over n4 inputs (dead rows are never read back)
                for (int e = lane; e < kCecRows * (n4 - dim); e += 32) {
                    const int r = e / (n4 - dim);
                    X[(size_t)r * cs + dim + (e - r * (n4 - dim))] = 0.0;
                }
            __syncwarp();
            const bool live = q < nb;
            const int own_key = live ? g.slot[4 * (h + q)] : 0;
            const double* src = live ? R.alt_key(own_key) : nullptr;  // compositions re-read the candidate
            bool ok = false;
            double fit_i = 0.0;
            if (live && t == 0) {
                ok = ((okmask >> q) & 1u) != 0;
                fit_i = A.fit[own_key >> 1];
            }
            const double nf = cec_eval_quad<NT>(C, X, src, cs, dim, lane, ew, bsm, bsm_comp);
            if (live && t == 0) {  // greedy select (numba_backend.py:270-290)
                const int own = own_key >> 1;
                double kept = fit_i;
                bool acc = false, warned = false;
                if (ok && isfinite(nf)) {
                    acc = nf < fit_i;
                    if (acc) kept = nf;
                } else {
                    warned = true;
                }
                A.out_fit[own] = kept;
                const uint8_t cur = (uint8_t)(own_key & 1);
                A.sel_next[own] = acc ? (uint8_t)(cur ^ 1) : cur;
                const unsigned long long k = sort_key(kept);
                my_min = k < my_min ? k : my_min;
                my_warn += warned ? 1u : 0u;
            }
            __syncwarp();
        }
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}


}  // namespace apo
