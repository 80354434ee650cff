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


// ---------------------------------------------------------------------------
// Warp-specialised form (APO_CEC_FUSED=2).  The one-warp-does-both kernel above cannot give the
// candidate half its TMA row ring (shared memory goes to M^T and the X tiles) and exposes the random
// row gathers.  Here warps [0, NP) PRODUCE candidates exactly like k_update_group<KIND_CAND> (phase A
// lane-per-protozoon, rows of each member TMA-staged through a 2-stage mbarrier ring) into a CTA ring
// of Q X tiles (8 candidates each; also written to the slot's alternate buffer), and warps [NP, W)
// CONSUME full tiles: DMMA rotation against the CTA's shared M^T, basic functions per lane quad,
// greedy select.  full[q]/empty[q] mbarriers (32 arrivals: every lane releases its own writes) order
// the hand-off; producers and consumers claim ring slots in order through shared counters, and a
// producer that runs out of groups publishes an empty tile (nb = 0) that retires one consumer.
struct WsMeta {
    int nb;
    unsigned okmask;
    int keys[kCecRows];  // SelSlots keys (slot * 2 + selector) of the tile's rows
};

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

struct WsLayout {
    size_t rot, bars, meta, tiles, prod, total;
    int q;
};

__host__ __device__ inline WsLayout ws_layout(int dim, int nt, int ncomp, bool stage_shift, int np, int q) {
    WsLayout L;
    size_t o = fused_rot_bytes(dim, nt) + (stage_shift ? 8 * (size_t)((ncomp * dim + 1) & ~1) : 0);
    L.rot = 0;
    o = (o + 15) & ~(size_t)15;
    L.bars = o;  // full[q], empty[q], then 4 u32 counters (slot claims: producers, consumers; producers done)
    o += 16 * (size_t)q + 16;
    L.meta = o;
    o += sizeof(WsMeta) * (size_t)q;
    o = (o + 15) & ~(size_t)15;
    L.tiles = o;
    o += 8 * (size_t)kCecRows * (size_t)cec_stride(dim) * (size_t)q;
    L.prod = o;
    o += group_scratch_bytes(dim, true, 0) * (size_t)np;
    L.total = o;
    L.q = q;
    return L;
}

template <int NT, int MAXC>
__global__ void __launch_bounds__(512, 1) k_update_cec_ws(UpdArgs A, int bsm_comp, int ncomp, int stage_shift,
                                                          int np, int q_tiles, unsigned* counter) {
    extern __shared__ __align__(16) unsigned char smem[];
    const IterParams& P = A.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int dim = P.dim, n4 = (dim + 3) & ~3, cs = cec_stride(dim);
    const WsLayout L = ws_layout(dim, NT, ncomp, stage_shift != 0, np, q_tiles);
    const int Q = q_tiles;
    double* bsm = reinterpret_cast<double*>(smem + L.rot);
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + L.bars);
    uint64_t* empty = full + Q;
    unsigned* ctr = reinterpret_cast<unsigned*>(empty + Q);  // [0] producer slot claims, [1] consumer claims
    WsMeta* meta = reinterpret_cast<WsMeta*>(smem + L.meta);
    double* tiles = reinterpret_cast<double*>(smem + L.tiles);
    const size_t tile_elems = (size_t)kCecRows * cs;
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
        if (threadIdx.x < Q) {
            mbar_init(&full[threadIdx.x], 32);
            mbar_init(&empty[threadIdx.x], 32);
        }
        if (threadIdx.x == 0) ctr[0] = ctr[1] = ctr[2] = 0;
        // tile pads [dim, n4) are never written by a candidate: zero them once
        for (int e = threadIdx.x; e < Q * kCecRows * (n4 - dim); e += blockDim.x) {
            const int r = e / (n4 - dim);
            tiles[(size_t)r * cs + dim + (e - r * (n4 - dim))] = 0.0;
        }
        mbar_fence_init();
    }
    __syncthreads();
    const SelSlots R{A.pos0, A.pos1, A.sel, A.fit, A.order, P.ld};
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    if (warp < np) {
        // ------------------------------------------------------------- producer
        const GroupScratch g = group_scratch(smem + L.prod + (size_t)warp * group_scratch_bytes(dim, true, 0), dim,
                                             true, 0);
        if (lane < kStages) mbar_init(&g.bar[lane], 1);
        mbar_fence_init();
        __syncwarp();
        unsigned ring_phase = 0;
        const int ngroups = (A.rank_hi - A.rank_lo + 31) / 32;
        auto issue = [&](int p) {  // TMA the rows member p reads into ring stage p % kStages
            if (lane == 0) {
                const int op = g.op[p];
                const int nrows = op == OP_AUTOTROPH ? 4 : op == OP_HETEROTROPH ? 3 : op == OP_REPRODUCTION ? 1 : 0;
                const int st = p % kStages;
                double* dst = g.ring + (size_t)st * 4 * g.rld;
                const unsigned bytes = (unsigned)(8 * P.ld);
                fence_proxy_async();
                mbar_expect_tx(&g.bar[st], bytes * (unsigned)nrows);
                const int* sl = g.slot + 4 * p;
                if (nrows >= 1) bulk_g2s(dst, R.at_key(sl[0]), bytes, &g.bar[st]);
                if (nrows == 4) bulk_g2s(dst + g.rld, R.at_key(sl[1]), bytes, &g.bar[st]);
                if (nrows >= 3) {
                    bulk_g2s(dst + 2 * g.rld, R.at_key(sl[2]), bytes, &g.bar[st]);
                    bulk_g2s(dst + 3 * g.rld, R.at_key(sl[3]), bytes, &g.bar[st]);
                }
            }
        };
        auto take_slot = [&]() -> unsigned {
            unsigned v = 0;
            if (lane == 0) v = atomicAdd(&ctr[0], 1u);
            v = __shfl_sync(kFull, v, 0);
            const unsigned s = v % (unsigned)Q;
            mbar_wait(&empty[s], ((v / (unsigned)Q) & 1u) ^ 1u);
            return v;
        };
        for (;;) {
            unsigned gv = 0;
            if (lane == 0) gv = atomicAdd(counter, 1u);
            const int grp = (int)__shfl_sync(kFull, gv, 0);
            if (grp >= ngroups) break;
            const int i0 = A.rank_lo + grp * 32 + 1;
            const int n = min(32, A.rank_hi - (i0 - 1));
            if (lane < n) {
                const int r0 = i0 - 1 + lane;
                const bool dr = ((A.in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0;
                group_phase_a(P, R, i0 + lane, dr, dr ? A.p_dr[r0] : 0.0, g, lane);
            }
            __syncwarp();
            for (int p = 0; p < kStages && p < n; p++) issue(p);
            for (int h = 0; h < n; h += kCecRows) {
                const int nb = min(kCecRows, n - h);
                const unsigned v = take_slot();
                const unsigned s = v % (unsigned)Q;
                double* X = tiles + (size_t)s * tile_elems;
                unsigned okmask = 0;
                for (int m = 0; m < nb; m++) {
                    const int p = h + m;
                    const int st = p % kStages;
                    mbar_wait(&g.bar[st], (ring_phase >> st) & 1u);
                    ring_phase ^= 1u << st;
                    const double* staged = g.ring + (size_t)st * 4 * g.rld;
                    double* dst = R.alt_key(g.slot[4 * p]);
                    const bool ok = group_candidate<MAXC, false, true, SelSlots, true>(
                        P, A.O, R, i0 + p, p, dst, X + (size_t)m * cs, nullptr, g, lane, staged);
                    okmask |= (ok ? 1u : 0u) << m;
                    __syncwarp();
                    if (p + kStages < n) issue(p + kStages);
                }
                if (lane < nb) meta[s].keys[lane] = g.slot[4 * (h + lane)];
                if (lane == 0) {
                    meta[s].nb = nb;
                    meta[s].okmask = okmask;
                }
                mbar_arrive(&full[s]);  // every lane: releases its own candidate / meta writes
            }
            __syncwarp();  // the next group's phase A rewrites the header and permutations
        }
        // the last producer to finish retires every consumer with an empty tile (claimed after all real
        // tiles: every other producer's slot claims precede its increment of ctr[2])
        __threadfence_block();
        unsigned done = 0;
        if (lane == 0) done = atomicAdd(&ctr[2], 1u);
        done = __shfl_sync(kFull, done, 0);
        if (done == (unsigned)np - 1) {
            const int nconsumers = (int)(blockDim.x >> 5) - np;
            for (int c = 0; c < nconsumers; c++) {
                const unsigned v = take_slot();
                const unsigned s = v % (unsigned)Q;
                if (lane == 0) meta[s].nb = 0;
                mbar_arrive(&full[s]);
            }
        }
    } else {
        // ------------------------------------------------------------- consumer
        const double* ew = A.O.table_len >= dim ? A.O.table : nullptr;  // ELLIPS weights (host libm)
        const int qd = lane >> 2, t = lane & 3;
        for (;;) {
            unsigned v = 0;
            if (lane == 0) v = atomicAdd(&ctr[1], 1u);
            v = __shfl_sync(kFull, v, 0);
            const unsigned s = v % (unsigned)Q;
            mbar_wait(&full[s], (v / (unsigned)Q) & 1u);
            const int nb = meta[s].nb;
            if (nb == 0) {
                mbar_arrive(&empty[s]);
                break;
            }
            const unsigned okmask = meta[s].okmask;
            const bool live = qd < nb;
            const int own_key = live ? meta[s].keys[qd] : 0;
            const double* src = live ? R.alt_key(own_key) : nullptr;  // compositions re-read the candidate
            double fit_i = 0.0;
            if (live && t == 0) fit_i = A.fit[own_key >> 1];
            double* X = tiles + (size_t)s * tile_elems;
            const double nf = cec_eval_quad<NT>(C, X, src, cs, dim, lane, ew, bsm, bsm_comp);
            if (live && t == 0) {  // greedy select (numba_backend.py:270-290)
                const int own = own_key >> 1;
                double kept = fit_i;
                bool acc = false, warned = false;
                if (((okmask >> qd) & 1u) && isfinite(nf)) {
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
            mbar_arrive(&empty[s]);  // the rotation rewrote X in place: done with the tile
        }
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

}  // namespace apo
