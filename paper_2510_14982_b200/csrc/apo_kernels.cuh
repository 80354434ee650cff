// apo_kernels.cuh -- kernel templates shared by the translation units of libapo_b200.so.
//
// The update and batch kernels are instantiated in their own TUs
// (apo_update_sel.cu, apo_update_dense.cu, apo_batch.cu) so the library
// builds in parallel; apo_kernels.cu holds the small kernels and the C ABI
// and reaches the templates through the pick_* getters below.
#pragma once
#include <cstdint>
#ifdef APO_BATCH_CLOCK
#include <cstdio>
#endif
#include "apo_group.cuh"
#include "apo_update.cuh"

namespace apo {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;

// ---------------------------------------------------------------------------
// Update launch arguments.  SEL mode (device-resident loop): rows live in
// pos0/pos1 selected per slot by sel[], ranks map to slots through order[],
// candidates go to the alternate buffer and sel_next/out_fit (by slot)
// record what is kept.  Dense mode (run_updates boundary): rank-ordered rows
// in pos -> out_pos, out_fit/out_acc/out_warn by rank.
struct UpdArgs {
    IterParams P;
    ObjDesc O;
    const double* pos0;
    const double* pos1;
    const uint8_t* sel;
    uint8_t* sel_next;
    const double* pos;
    double* out_pos;
    const double* fit;
    const int* order;
    double* out_fit;
    const uint8_t* in_dr_bytes;
    const unsigned* in_dr_bits;
    const double* p_dr;
    uint8_t* out_acc;
    uint8_t* out_warn;
    unsigned long long* warn_count;
    unsigned long long* trace_key;
    int cec_bufs;      // CEC2022 scratch rows (cec_bufs_for(code))
    uint8_t* cand_ok;  // non-null: candidates only (k_cec_eval finishes the update)
    int rank_lo, rank_hi;  // 0-based rank range to update; [0, ps) unless sharded
    int gsize;             // group path: consecutive ranks per warp (1..32; fewer spread small populations)
};

__device__ __forceinline__ void block_finish(unsigned long long my_min, unsigned my_warn,
                                             unsigned long long* warn_count, unsigned long long* trace_key) {
    __shared__ unsigned long long red_min[32];
    __shared__ unsigned red_warn[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long m2 = __shfl_xor_sync(kFull, my_min, o);
        my_min = m2 < my_min ? m2 : my_min;
        my_warn += __shfl_xor_sync(kFull, my_warn, o);
    }
    if (lane == 0) {
        red_min[warp] = my_min;
        red_warn[warp] = my_warn;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned long long m = ~0ull;
        unsigned w = 0;
        for (int k = 0; k < nwarps; k++) {
            m = red_min[k] < m ? red_min[k] : m;
            w += red_warn[k];
        }
        if (trace_key && m != ~0ull) atomicMin(trace_key, m);
        if (warn_count && w) atomicAdd(warn_count, (unsigned long long)w);
    }
}

// Warp-per-protozoon path (dim > 256).
template <bool SEL>
__global__ void __launch_bounds__(kThreads) k_update(UpdArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const IterParams& P = A.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const WarpScratch s = warp_scratch(smem + (size_t)warp * warp_scratch_bytes(P.dim), P.dim);
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    for (int r0 = A.rank_lo + blockIdx.x * nwarps + warp; r0 < A.rank_hi; r0 += gridDim.x * nwarps) {
        const bool dr = A.in_dr_bits ? ((A.in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0 : A.in_dr_bytes[r0] != 0;
        const double pdr = dr ? A.p_dr[r0] : 0.0;
        UpdateResult res;
        const bool co = A.cand_ok != nullptr;  // candidates only (CEC2022 large-D GEMM path)
        if constexpr (SEL) {
            const SelSlots R{A.pos0, A.pos1, A.sel, A.fit, A.order, P.ld};
            const int slot = A.order[r0];
            res = update_protozoon(P, A.O, R, r0 + 1, dr, pdr, R.alt(slot), s, lane, co);
            if (lane == 0) {
                if (co) {
                    A.cand_ok[slot] = res.accepted ? 1 : 0;
                } else {
                    A.out_fit[slot] = res.fitness;
                    A.sel_next[slot] = A.sel[slot] ^ 1;  // the full kept row went to the alternate buffer
                }
            }
        } else {
            const DenseRows R{A.pos, A.fit, P.ld};
            res = update_protozoon(P, A.O, R, r0 + 1, dr, pdr, A.out_pos + (size_t)r0 * P.ld, s, lane, co);
            if (lane == 0) {
                if (co) {
                    A.cand_ok[r0] = res.accepted ? 1 : 0;
                } else {
                    A.out_fit[r0] = res.fitness;
                    if (A.out_acc) A.out_acc[r0] = res.accepted ? 1 : 0;
                    if (A.out_warn) A.out_warn[r0] = res.warned ? 1 : 0;
                }
            }
        }
        if (co) continue;
        if (lane == 0) {
            const unsigned long long k = sort_key(res.fitness);
            my_min = k < my_min ? k : my_min;
            my_warn += res.warned ? 1u : 0u;
        }
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

// Group path (dim <= 256): one warp per 32 consecutive ranks, see apo_group.cuh.
#ifndef APO_GROUP_MIN_BLOCKS
#define APO_GROUP_MIN_BLOCKS 2
#endif
// KIND: KIND_ANY (every objective), KIND_BASIC (no CEC2022 code), KIND_CAND
// (candidates only: the CEC2022 split, k_cec_eval finishes the update).
template <bool SEL, int MAXC, int KIND, int NP>
__global__ void __launch_bounds__(kThreads, APO_GROUP_MIN_BLOCKS) k_update_group(UpdArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const IterParams& P = A.P;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    // SEL rows have an even stride (16-byte aligned) -> TMA-staged rows
    constexpr bool kStage = SEL && MAXC > 0 && 32 * MAXC <= APO_STAGE_MAX_DIM;
    const GroupScratch g = group_scratch(smem + (size_t)warp * group_scratch_bytes(P.dim, kStage, A.cec_bufs), P.dim,
                                         kStage, A.cec_bufs);
    unsigned ring_phase = 0;
    if (kStage) {
        if (lane < kStages) mbar_init(&g.bar[lane], 1);
        mbar_fence_init();
        __syncwarp();
    }
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    const int G = A.gsize;
    const int ngroups = (A.rank_hi - A.rank_lo + G - 1) / G;
    for (int grp = blockIdx.x * nwarps + warp; grp < ngroups; grp += gridDim.x * nwarps) {
        const int i0 = A.rank_lo + grp * G + 1;
        const int n = min(G, A.rank_hi - (i0 - 1));
        if constexpr (SEL) {
            const SelSlots R{A.pos0, A.pos1, A.sel, A.fit, A.order, P.ld};
            update_group<MAXC, OUT_SEL, KIND, NP>(P, A.O, R, i0, n, A.in_dr_bytes, A.in_dr_bits, A.p_dr, nullptr, A.out_fit,
                                        true, nullptr, nullptr, A.sel_next, g, lane, my_min, my_warn, &ring_phase,
                                        A.cand_ok);
        } else if (A.order) {  // sharded: rows addressed through the rank->row order, outputs by rank
            const OrderedSlots R{A.pos, A.fit, A.order, P.ld};
            update_group<MAXC, OUT_FIXUP, KIND, NP>(P, A.O, R, i0, n, A.in_dr_bytes, A.in_dr_bits, A.p_dr, A.out_pos,
                                          A.out_fit, false, A.out_acc, A.out_warn, nullptr, g, lane, my_min,
                                          my_warn, nullptr, A.cand_ok);
        } else {
            const DenseSlots R{A.pos, A.fit, P.ld};
            update_group<MAXC, OUT_FIXUP, KIND, NP>(P, A.O, R, i0, n, A.in_dr_bytes, A.in_dr_bits, A.p_dr, A.out_pos,
                                          A.out_fit, false, A.out_acc, A.out_warn, nullptr, g, lane, my_min,
                                          my_warn, nullptr, A.cand_ok);
        }
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

// ---------------------------------------------------------------------------
// Persistent batched runs: one CTA = one independent run, resident in SMEM.
struct BatchArgs {
    const uint64_t* seeds;
    const ObjDesc* objs;
    int ps, dim, ld, max_iterations, n_iters, npairs;
    double pf_max, lower, upper, span, eps;
    const double* sched;  // [max_iterations][3]
    const double* p_dr;   // [ps]
    double* best_fit;
    double* best_pos;
    double* trace;
    double* final_pos;
    double* final_fit;
    long long* warnings;
    int cec_bufs;   // max over the batch's objectives of cec_bufs_for(code)
    int tab_smem;   // doubles of threshold prefix table staged in shared memory (0 = none)
    int rng;        // RngMode
    int nruns;
    // persistent mode (run_counter non-null): CTAs claim runs run_order[0], [1], ... (costliest first) until
    // none is left, so an SM that drew cheap runs takes more; else CTA b does run b
    const int* run_order;
    unsigned* run_counter;
    int lpp;        // npairs == 1: lane-per-protozoon groups at dim <= kLppMaxDim (update_group_lpp)
    int lpp_group;  // protozoa per warp on that path
    int group;      // minimum protozoa per warp on the warp-per-protozoon path (0: spread over all warps)
};

struct BatchLayout {
    size_t pos0, pos1, fit0, fit1, keys, order, rankof, newrank, chead, cprev, crj, cbits, tab, warps, total;
};

__host__ __device__ inline size_t batch_warp_bytes(int dim, int cec_bufs) {
    const size_t ws = warp_scratch_bytes(dim);  // init + warp path
    if (dim > kGroupMaxDim) return ws;
    const size_t gs = group_scratch_bytes(dim, false, cec_bufs);
    return gs > ws ? gs : ws;
}

__host__ __device__ inline BatchLayout batch_layout(int ps, int dim, int ld, int nwarps, int cec_bufs,
                                                int tab_smem = 0) {
    BatchLayout L;
    size_t o = 0;
    auto take = [&](size_t bytes) {
        size_t at = o;
        o += (bytes + 15) & ~(size_t)15;
        return at;
    };
    L.pos0 = take(8 * (size_t)ps * ld);
    L.pos1 = take(8 * (size_t)ps * ld);
    L.fit0 = take(8 * (size_t)ps);
    L.fit1 = take(8 * (size_t)ps);
    L.keys = take(8 * (size_t)ps);
    L.order = take(4 * (size_t)ps);
    L.rankof = take(4 * (size_t)ps);
    L.newrank = take(4 * (size_t)ps);
    L.chead = take(4 * (size_t)ps);
    L.cprev = take(4 * (size_t)ps);
    L.crj = take(4 * (size_t)ps);
    L.cbits = take(4 * (size_t)((ps + 31) / 32));
    L.tab = take(8 * (size_t)tab_smem);
    L.warps = take(batch_warp_bytes(dim, cec_bufs) * (size_t)nwarps);
    L.total = o;
    return L;
}

// MAXC >= 0: group path (apo_group.cuh); MAXC < 0: warp-per-protozoon (dim > 256).
// A run is latency-bound (one CTA walks ps protozoa per iteration behind __syncthreads), so more warps
// per run pay: with more runs than SMs the launch is one persistent kBatchPersistThreads CTA per SM
// that claims runs costliest first, else each run gets a kBatchWideThreads CTA; callers sharing the GPU
// can ask for kThreads CTAs (96 registers: 2 CTAs/SM).  apo_run_batch_shaped picks the shape.
constexpr int kBatchWideThreads = 512;
constexpr int kBatchPersistThreads = 640;
constexpr int kBatchMaxThreads = 640;  // 96 registers: 5 warps per SM sub-partition (16K registers each)
#ifndef APO_BATCH_MAXNREG
#define APO_BATCH_MAXNREG 96
#endif
// NP as in update_group: 1 / 2 = built for npairs == 1 / > 1 only (the keyed builds), 0 = either.
template <int MAXC, int NP = 0>
__global__ void __maxnreg__(APO_BATCH_MAXNREG) k_run_batch(BatchArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ unsigned long long red_min[32];
    __shared__ unsigned red_warn[32];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int ps = A.ps, dim = A.dim, ld = A.ld;
    const BatchLayout L = batch_layout(ps, dim, ld, nwarps, A.cec_bufs, A.tab_smem);
    double* pos[2] = {reinterpret_cast<double*>(smem + L.pos0), reinterpret_cast<double*>(smem + L.pos1)};
    double* fit[2] = {reinterpret_cast<double*>(smem + L.fit0), reinterpret_cast<double*>(smem + L.fit1)};
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(smem + L.keys);
    int* order = reinterpret_cast<int*>(smem + L.order);
    int* rankof = reinterpret_cast<int*>(smem + L.rankof);
    int* newrank = reinterpret_cast<int*>(smem + L.newrank);
    WarpScratch cs;
    cs.head = reinterpret_cast<int*>(smem + L.chead);
    cs.prev = reinterpret_cast<int*>(smem + L.cprev);
    cs.rj = reinterpret_cast<int*>(smem + L.crj);
    cs.bits = reinterpret_cast<unsigned*>(smem + L.cbits);
    unsigned char* wbase = smem + L.warps + (size_t)warp * batch_warp_bytes(dim, A.cec_bufs);
    const GroupScratch g = group_scratch(wbase, dim, false, A.cec_bufs);
    const WarpScratch ws = MAXC >= 0 ? g.ws : warp_scratch(wbase, dim);
    __shared__ int s_run;
    for (int claim = 0;; claim++) {
    if (threadIdx.x == 0) {
        int k = A.nruns;
        if (A.run_counter) k = (int)atomicAdd(A.run_counter, 1u);
        else if (claim == 0) k = blockIdx.x;
        s_run = k < A.nruns ? (A.run_order ? A.run_order[k] : k) : -1;
    }
    __syncthreads();
    const int run = s_run;
    if (run < 0) break;
    const uint64_t seed = A.seeds[run];
    ObjDesc O = A.objs[run];
    if (A.tab_smem > 0 && (O.code == OBJ_OTSU_ML || O.code == OBJ_KAPUR_ML)) {
        // the 256-bin prefix tables live in shared memory for the whole run
        double* tab = reinterpret_cast<double*>(smem + L.tab);
        for (int k = threadIdx.x; k < O.table_len && k < A.tab_smem; k += blockDim.x) tab[k] = O.table[k];
        O.table = tab;
        __syncthreads();
    }
    double* trace = A.trace ? A.trace + (size_t)run * (A.n_iters + 1) : nullptr;

    // initialisation (engine.py:116-139); the init scratch aliases this warp's group scratch
    unsigned long long my_min = ~0ull;
    const WarpScratch iws = warp_scratch(wbase, dim);
    for (int r0 = warp; r0 < ps; r0 += nwarps) {
        const Key base = stream_key(A.rng, seed, 0, (uint64_t)(r0 + 1));
        double* row = pos[0] + (size_t)r0 * ld;
        for (int d = lane; d < dim; d += 32) row[d] = A.lower + uniform(base, (uint64_t)d) * A.span;
        __syncwarp();
        for (int d = lane; d < dim; d += 32) iws.cand[d] = row[d];
        __syncwarp();
        const double f = eval_warp(O, iws.cand, iws.terms, dim, lane, iws.aux);
        if (lane == 0) {
            fit[0][r0] = f;
            keys[r0] = sort_key(f);
            order[r0] = r0;
            rankof[r0] = r0;
            my_min = sort_key(f) < my_min ? sort_key(f) : my_min;
        }
    }
    if (lane == 0) red_min[warp] = my_min;
    __syncthreads();
    if (threadIdx.x == 0 && trace) {
        unsigned long long m = ~0ull;
        for (int k = 0; k < nwarps; k++) m = red_min[k] < m ? red_min[k] : m;
        trace[0] = key_to_double(m);
    }
    unsigned warn_total = 0;
    int cur = 0;
#ifdef APO_BATCH_CLOCK
    long long clk_sum[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    long long clk_prev = clock64();
#define CLK(k)                                       \
    do {                                             \
        const long long now_ = clock64();            \
        clk_sum[k] += now_ - clk_prev;               \
        clk_prev = now_;                             \
    } while (0)
#else
#define CLK(k) \
    do {       \
    } while (0)
#endif
    for (int t = 0; t < A.n_iters; t++) {
        // 1. stable sort by fitness, ties by previous rank (core.py:504-513): each rank is a count of
        //    smaller keys, S lanes per element (S a power of two, the counts folded by shuffles); the
        //    coordinator draws (2.) run meanwhile on the last warp when the sort leaves it idle
        const uint64_t key_it = (uint64_t)t + 1;
        const int dr_warp = nwarps - 1;
#ifndef APO_BATCH_OVERLAP
#define APO_BATCH_OVERLAP 1
#endif
        const bool dr_overlap = APO_BATCH_OVERLAP && ps <= 32 * dr_warp;
        auto coordinator = [&]() {  // core.py:263-278
            const Key cbase = stream_key(A.rng, seed, key_it, kCoordinator);
            const double pf = A.pf_max * uniform(cbase, 0);
            const int count = (int)ceil((double)ps * pf);
            build_mask(ps, count, cbase, 1, cs, lane);
        };
#ifdef APO_BATCH_CLOCK
        const long long own_s0 = clock64();
        if (dr_overlap && warp == dr_warp) coordinator();
        if (dr_overlap && warp == dr_warp) clk_sum[6] += clock64() - own_s0;
#else
        if (dr_overlap && warp == dr_warp) coordinator();
#endif
        const int span = dr_overlap ? 32 * dr_warp : (int)blockDim.x;
        int lgS = 0;
        while (APO_BATCH_OVERLAP && lgS < 3 && (2 << lgS) * ps <= span) lgS++;
        const int S = 1 << lgS;
        for (int base_t = 0; base_t < ps * S; base_t += span) {
            const int tt = base_t + (int)threadIdx.x;
            int cnt = 0;
            const int sl = tt >> lgS;
            const bool act = (int)threadIdx.x < span && sl < ps;
            if (act) {
                // branch-free count of (key, previous rank) pairs below this one (both loads always issued)
                const unsigned long long k = keys[sl];
                const int pr = rankof[sl];
#pragma unroll 4
                for (int q = tt & (S - 1); q < ps; q += S) {
                    const unsigned long long kq = keys[q];
                    const int rq = rankof[q];
                    cnt += (int)((kq < k) | ((kq == k) & (rq < pr)));
                }
            }
            if ((int)threadIdx.x < span) {  // whole warps: span is a multiple of 32 and S divides 32
                for (int o = 1; o < S; o <<= 1) cnt += __shfl_xor_sync(kFull, cnt, o);
                if (act && (tt & (S - 1)) == 0) newrank[sl] = cnt;
            }
        }
#ifdef APO_BATCH_CLOCK
        if (!(dr_overlap && warp == dr_warp)) clk_sum[7] += clock64() - own_s0;
#endif
        __syncthreads();
        CLK(0);
        for (int sl = threadIdx.x; sl < ps; sl += blockDim.x) {
            order[newrank[sl]] = sl;
            rankof[sl] = newrank[sl];
        }
        if (!dr_overlap && warp == 0) coordinator();
        __syncthreads();
        CLK(1);
        // 3. fused updates
        IterParams P;
        P.seed = seed;
        P.key_iteration = key_it;
        P.ps = ps;
        P.dim = dim;
        P.npairs = A.npairs;
        P.ld = ld;
        P.lower = A.lower;
        P.upper = A.upper;
        P.span = A.span;
        P.eps = A.eps;
        P.p_ah = A.sched[3 * t];
        P.f_mult = A.sched[3 * t + 1];
        P.decay = A.sched[3 * t + 2];
        P.rng = A.rng;
        set_iteration_base(P);
        const int nxt = cur ^ 1;
        my_min = ~0ull;
        unsigned my_warn = 0;
        if constexpr (MAXC >= 0) {
            const OrderedSlots R{pos[cur], fit[cur], order, ld};
            const bool lpp = MAXC == 1 && NP != 2 && A.lpp && O.code < OBJ_CEC_BASE && dim <= kLppMaxDim;
            const int G = lpp ? min(32, max(A.lpp_group, (ps + nwarps - 1) / nwarps))
                              : min(32, max(A.group, (ps + nwarps - 1) / nwarps));
#ifdef APO_BATCH_CLOCK
            const long long own0 = clock64();
#endif
            for (int q = warp; q * G < ps; q += nwarps) {
                const int i0 = q * G + 1;
                if (MAXC == 1 && lpp)
                    update_group_lpp(P, O, R, i0, min(G, ps - q * G), cs.bits, A.p_dr, pos[nxt], fit[nxt], g, lane,
                                     my_min, my_warn);
                else
                    update_group<MAXC, OUT_FIXUP, KIND_ANY, NP>(P, O, R, i0, min(G, ps - q * G), nullptr, cs.bits, A.p_dr,
                                                            pos[nxt], fit[nxt], true, nullptr, nullptr, nullptr, g,
                                                            lane, my_min, my_warn);
            }
#ifdef APO_BATCH_CLOCK
            clk_sum[5] += clock64() - own0;
#endif
            __syncthreads();
            CLK(2);
            for (int sl = threadIdx.x; sl < ps; sl += blockDim.x) keys[sl] = sort_key(fit[nxt][sl]);
        } else {
            const OrderedRows R{pos[cur], fit[cur], order, ld};
            for (int r0 = warp; r0 < ps; r0 += nwarps) {
                const bool dr = ((cs.bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0;
                const int slot = order[r0];
                const UpdateResult res = update_protozoon(P, O, R, r0 + 1, dr, dr ? A.p_dr[r0] : 0.0,
                                                          pos[nxt] + (size_t)slot * ld, ws, lane);
                if (lane == 0) {
                    fit[nxt][slot] = res.fitness;
                    const unsigned long long k = sort_key(res.fitness);
                    keys[slot] = k;
                    my_min = k < my_min ? k : my_min;
                    my_warn += res.warned ? 1u : 0u;
                }
            }
        }
        for (int o = 16; o > 0; o >>= 1) {
            const unsigned long long m2 = __shfl_xor_sync(kFull, my_min, o);
            my_min = m2 < my_min ? m2 : my_min;
            my_warn += __shfl_xor_sync(kFull, my_warn, o);
        }
        if (lane == 0) {
            red_min[warp] = my_min;
            red_warn[warp] = my_warn;
        }
        __syncthreads();
        CLK(3);
        if (threadIdx.x == 0) {
            unsigned long long m = ~0ull;
            for (int k = 0; k < nwarps; k++) {
                m = red_min[k] < m ? red_min[k] : m;
                warn_total += red_warn[k];
            }
            if (trace) trace[t + 1] = key_to_double(m);
        }
        cur = nxt;
        __syncthreads();
        CLK(4);
    }
#ifdef APO_BATCH_CLOCK
    if (threadIdx.x == 0 || threadIdx.x == 32 * (nwarps - 1))
        printf("batch clock run %d thread %d: sort %lld order+dr %lld update %lld reduce %lld tail %lld own-update %lld own-coord %lld own-sort %lld (cycles/iter)\n",
               run, (int)threadIdx.x, clk_sum[0] / A.n_iters, clk_sum[1] / A.n_iters, clk_sum[2] / A.n_iters,
               clk_sum[3] / A.n_iters, clk_sum[4] / A.n_iters, clk_sum[5] / A.n_iters, clk_sum[6] / A.n_iters,
               clk_sum[7] / A.n_iters);
    if (threadIdx.x == 0)
        printf("lpp warp 0 (cycles/iter): phaseA %llu cand+fold %llu select %llu\n", g_lpp_clk[0] / A.n_iters,
               g_lpp_clk[1] / A.n_iters, g_lpp_clk[3] / A.n_iters);
#endif
#undef CLK
    // outputs in reference row order (row r = order[r])
    if (threadIdx.x == 0) {
        int best = 0;
        for (int r = 1; r < ps; r++)
            if (fit[cur][order[r]] < fit[cur][order[best]]) best = r;
        red_warn[0] = (unsigned)best;
        A.best_fit[run] = fit[cur][order[best]];
        if (A.warnings) A.warnings[run] = warn_total;
    }
    __syncthreads();
    const int bslot = order[red_warn[0]];
    if (A.best_pos)
        for (int d = threadIdx.x; d < dim; d += blockDim.x) A.best_pos[(size_t)run * dim + d] = pos[cur][(size_t)bslot * ld + d];
    if (A.final_pos)
        for (int e = threadIdx.x; e < ps * dim; e += blockDim.x) {
            const int r = e / dim, d = e - r * dim;
            A.final_pos[(size_t)run * ps * dim + e] = pos[cur][(size_t)order[r] * ld + d];
        }
    if (A.final_fit)
        for (int r = threadIdx.x; r < ps; r += blockDim.x) A.final_fit[(size_t)run * ps + r] = fit[cur][order[r]];
    __syncthreads();  // shared memory is reused by the next claimed run
    }
}


// ---------------------------------------------------------------------------
// CEC2022 on an HBM-resident population: k_update_group writes every
// candidate (+ a finiteness flag) and k_cec_eval then evaluates them in
// 8-row DMMA tiles (one tile per warp), applies the greedy select
// (numba_backend.py:270-290) and folds the best-so-far / warning count.
// Rows are indexed by slot (SEL: the candidate is in the slot's alternate
// buffer) or by rank (dense: the candidate is out_pos[r]; rejected rows are
// rewritten with the old row).
constexpr int kCecEvalMaxDim = 104;  // 13 register-resident n-tiles
// n-tiles per rotation in k_cec_eval (rot_pad rows are 8 * cec_nt(n) wide)
__host__ __device__ inline int cec_nt(int n) { return cec_nt_dev(n); }
struct CecEvalArgs {
    int n_rows, dim, ld, bufs;
    int row0;          // first row (dense: rank) of the range
    const int* order;  // dense + sharded: old row/fitness of rank r at order[r] (nullable)
    ObjDesc O;
    const double* pos0;  // SEL
    const double* pos1;
    const uint8_t* sel;
    uint8_t* sel_next;
    const double* pos;  // dense: old rows (rank order)
    double* out_pos;    // dense: candidates in, kept rows out
    uint8_t* out_acc;
    uint8_t* out_warn;
    const double* fit;
    double* out_fit;
    const uint8_t* cand_ok;
    unsigned long long* warn_count;
    unsigned long long* trace_key;
    unsigned* tile_counter;  // zeroed before the launch: warps claim 8-row tiles dynamically
    int prefetch;            // FAST: double-buffer X with cp.async (else one X tile per warp, more warps)
    int bsm_comp;            // FAST: the component whose rotation is staged in shared memory
    int ncomp;               // shift vectors to stage
    int init;                // iteration 0: evaluate the rows of pos0 (slot order) into out_fit, no select
};

// FAST (F1-F8: one rotation): the CTA stages that rotation in shared memory
// once (persistent CTAs) and every warp double-buffers its X tile with
// cp.async, so the next tile's candidate rows stream in while this one is
// evaluated.  Otherwise (compositions: up to 6 rotations) B is read through
// L1 and each warp has one X tile plus W.
__host__ __device__ inline int cec_bsm_stride(int nt) { return 8 * nt + 4; }
__host__ __device__ inline size_t cec_eval_warp_bytes(int dim, int bufs, bool prefetch) {
    return 8 * (size_t)((prefetch ? 2 : 1) + bufs) * kCecRows * (size_t)cec_stride(dim);  // bufs = W buffers
}
__host__ __device__ inline size_t cec_bsm_bytes(int dim, int nt, int ncomp) {  // rotation + shift vectors
    return 8 * (size_t)((dim + 3) & ~3) * (size_t)cec_bsm_stride(nt) + 8 * (size_t)ncomp * (size_t)((dim + 1) & ~1);
}

__device__ __forceinline__ void cp_async8(double* dst, const double* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_prev() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

template <bool SEL, int NT, bool FAST>
__global__ void __launch_bounds__(512, 1) k_cec_eval(CecEvalArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int q = lane >> 2, t = lane & 3;  // quad q owns row q of the tile
    const int dim = A.dim, cs = cec_stride(dim), n4 = (dim + 3) & ~3;
    const bool pf = FAST && A.prefetch;
    double* base = reinterpret_cast<double*>(smem + (size_t)warp * cec_eval_warp_bytes(dim, A.bufs, pf));
    double* bsm = nullptr;
    CecData C = A.O.cec;
    if constexpr (FAST) {
        bsm = reinterpret_cast<double*>(smem + (size_t)nwarps * cec_eval_warp_bytes(dim, A.bufs, pf));
        const int bs = cec_bsm_stride(NT), w8 = 8 * NT;
        const double* rsrc = C.rot_pad + (size_t)A.bsm_comp * n4 * w8;
        for (int e = threadIdx.x; e < n4 * w8; e += blockDim.x) {
            const int i = e / w8, j = e - i * w8;
            bsm[i * bs + j] = rsrc[e];
        }
        double* osm = bsm + (size_t)n4 * bs;  // the shift vectors too (read once per element per tile)
        for (int i = threadIdx.x; i < A.ncomp * dim; i += blockDim.x) osm[i] = C.shift[i];
        C.shift = osm;
        __syncthreads();
    }
    const double* ew = A.O.table_len >= dim ? A.O.table : nullptr;  // ELLIPS weights (host libm)
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    const int ntiles = (A.n_rows + kCecRows - 1) / kCecRows;
    const int stride = gridDim.x * nwarps;
    auto row_of = [&](int tile) { return A.row0 + tile * kCecRows + q; };
    auto live_in = [&](int tile) { return tile < ntiles && row_of(tile) < A.row0 + A.n_rows; };
    // row q of `tile` -> X tile `buf` (cp.async); pads and dead rows are zero
    auto issue = [&](int tile, int buf, uint8_t selq) {
        double* xrow = base + (size_t)buf * kCecRows * cs + (size_t)q * cs;
        const bool live = live_in(tile);
        const double* src = nullptr;
        if (live) {
            const int r = row_of(tile);
            if constexpr (SEL) src = (selq || A.init ? A.pos0 : A.pos1) + (size_t)r * A.ld;  // the alternate buffer
            else src = A.out_pos + (size_t)r * A.ld;
        }
        for (int i = t; i < n4; i += 4) {
            if (live && i < dim) cp_async8(xrow + i, src + i);
            else xrow[i] = 0.0;
        }
    };
    auto sel_of = [&](int tile) -> uint8_t {
        if constexpr (SEL) return (live_in(tile) && !A.init) ? A.sel[row_of(tile)] : (uint8_t)0;
        return 0;
    };
    // dynamic tile claims (lane 0 + broadcast) keep the warps of an SM finishing together
    auto claim = [&]() -> int {
        unsigned v = 0;
        if (lane == 0) v = atomicAdd(A.tile_counter, 1u);
        return (int)__shfl_sync(kFull, v, 0);
    };
    // split form: the atomic is issued at the top of a tile and its value consumed at the bottom
    auto claim_issue = [&]() -> unsigned { return lane == 0 ? atomicAdd(A.tile_counter, 1u) : 0u; };
    auto claim_take = [&](unsigned v) -> int { return (int)__shfl_sync(kFull, v, 0); };
    (void)stride;
    int tile = claim();
    int tile_nxt = 0;
    uint8_t sel_cur = sel_of(tile), sel_nxt = 0;
    if (pf) {
        if (tile < ntiles) issue(tile, 0, sel_cur);
        cp_async_commit();
    }
    tile_nxt = tile < ntiles ? claim() : ntiles;
    sel_nxt = sel_of(tile_nxt);
    int buf = 0;
    while (tile < ntiles) {
        const int r0 = A.row0 + tile * kCecRows;
        const int nb = min(kCecRows, A.row0 + A.n_rows - r0);
        const int r = r0 + q;
        const bool live = q < nb;
        // per-row scalars for the select, loaded early so their latency hides behind the evaluation
        bool ok = false;
        double fit_i = 0.0;
        if (live && t == 0 && !A.init) {
            ok = A.cand_ok[r] != 0;
            fit_i = A.fit[(!SEL && A.order) ? A.order[r] : r];
        }
        const uint8_t cur = sel_cur;
        int tile_next;
        if (pf) {
            tile_next = tile_nxt;
            if (tile_next < ntiles) issue(tile_next, buf ^ 1, sel_nxt);
            cp_async_commit();
            sel_cur = sel_nxt;
            tile_nxt = tile_next < ntiles ? claim() : ntiles;
            sel_nxt = sel_of(tile_nxt);
            cp_async_wait_prev();
        } else {
            issue(tile, 0, cur);
            cp_async_commit();
            tile_next = tile_nxt;  // claimed one tile ahead
            sel_cur = sel_nxt;
#ifndef APO_CEC_L2_PREFETCH
#define APO_CEC_L2_PREFETCH 1
#endif
            if (APO_CEC_L2_PREFETCH && SEL && !A.init && lane < kCecRows && tile_next < ntiles) {
                // the next tile's candidate rows into L2 while this one evaluates (one bulk prefetch per
                // row; SEL rows have an even stride, so 8 * ld bytes is a multiple of 16)
                const int rn = A.row0 + tile_next * kCecRows + lane;
                if (rn < A.row0 + A.n_rows) {
                    const double* src = (A.sel[rn] ? A.pos0 : A.pos1) + (size_t)rn * A.ld;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"((unsigned)(8 * A.ld))
                                 : "memory");
                }
            }
            cp_async_wait_all();
        }
        // the claim after next: issued now, read after the evaluation (its latency hides behind it)
        const unsigned pending = (!pf && tile_next < ntiles) ? claim_issue() : 0u;
        __syncwarp();
        const double* qsrc = nullptr;  // this quad's candidate row (compositions re-read it per component)
        if (live) qsrc = SEL ? (cur || A.init ? A.pos0 : A.pos1) + (size_t)r * A.ld : A.out_pos + (size_t)r * A.ld;
        const double nf = cec_eval_quad<NT>(C, base + (size_t)buf * kCecRows * cs, qsrc, cs, dim, lane, ew, bsm,
                                            A.bsm_comp);
        bool acc = false;
        if (A.init) {  // iteration 0 (engine.py:116-139): the fitness of every initial row
            if (live && t == 0) {
                A.out_fit[r] = nf;
                const unsigned long long k = sort_key(nf);
                my_min = k < my_min ? k : my_min;
            }
        } else if (live && t == 0) {
            double kept = fit_i;
            bool warned = false;
            if (ok && isfinite(nf)) {
                acc = nf < fit_i;
                if (acc) kept = nf;
            } else {
                warned = true;
            }
            A.out_fit[r] = kept;
            if constexpr (SEL) {
                A.sel_next[r] = acc ? (uint8_t)(cur ^ 1) : cur;
            } else {
                if (A.out_acc) A.out_acc[r] = acc ? 1 : 0;
                if (A.out_warn) A.out_warn[r] = warned ? 1 : 0;
            }
            const unsigned long long k = sort_key(kept);
            my_min = k < my_min ? k : my_min;
            my_warn += warned ? 1u : 0u;
        }
        if constexpr (!SEL) {
            unsigned rej = __ballot_sync(kFull, live && t == 0 && !acc);
            while (rej) {
                const int qq = (__ffs(rej) - 1) >> 2;
                rej &= rej - 1;
                const int old_row = A.order ? A.order[r0 + qq] : r0 + qq;
                const double* x = A.pos + (size_t)old_row * A.ld;
                double* dst = A.out_pos + (size_t)(r0 + qq) * A.ld;
                for (int d = lane; d < dim; d += 32) dst[d] = x[d];
            }
        }
        __syncwarp();
        if (pf) buf ^= 1;
        if (!pf) {
            tile_nxt = tile_next < ntiles ? claim_take(pending) : ntiles;
            sel_nxt = sel_of(tile_nxt);
        }
        tile = tile_next;
    }
    cp_async_wait_all();
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

// ---------------------------------------------------------------------------
// The reference's six objectives on an HBM-resident population, split like CEC2022: k_update_group
// <KIND_CAND> writes candidates (+ a finiteness flag), then k_basic_eval evaluates them LANE PER
// PROTOZOON -- the reference's sequential left-to-right loop (numba_backend.py:93-131) run by one lane
// over its own candidate, bit for bit -- and applies the greedy select (numba_backend.py:270-290).
// The fused group kernel instead folds each protozoon's terms with 1 of 32 lanes while the warp waits;
// here a warp transposes 32 candidate rows through shared memory in 32 x 32 blocks (coalesced row
// reads, conflict-free column reads: stride 33) and all 32 lanes fold at once.
struct BasicEvalArgs {
    int n_rows, dim, ld;
    int row0;          // first row (dense: rank) of the range
    const int* order;  // dense + order: old row/fitness of rank r at order[r] (nullable)
    ObjDesc O;
    const double* pos0;  // SEL: candidate of slot r in its alternate buffer
    const double* pos1;
    const uint8_t* sel;
    uint8_t* sel_next;
    const double* pos;  // dense: old rows
    double* out_pos;    // dense: candidates in, kept rows out
    uint8_t* out_acc;
    uint8_t* out_warn;
    const double* fit;
    double* out_fit;
    const uint8_t* cand_ok;
    unsigned long long* warn_count;
    unsigned long long* trace_key;
};

__host__ __device__ inline bool basic_split_code(int code) { return code >= OBJ_SPHERE && code <= OBJ_GRIEWANK; }


// Greedy select of row r (numba_backend.py:270-290), rejected rows restored in dense mode.
template <bool SEL>
__device__ __forceinline__ void basic_select(const BasicEvalArgs& A, int g0, int nb, int lane, uint8_t cur, double nf,
                                             unsigned long long& my_min, unsigned& my_warn) {
    const int r = g0 + lane;
    const bool live = lane < nb;
    bool acc = false;
    if (live) {
        const double fit_i = A.fit[(!SEL && A.order) ? A.order[r] : r];
        double kept = fit_i;
        bool warned = false;
        if (A.cand_ok[r] && isfinite(nf)) {
            acc = nf < fit_i;
            if (acc) kept = nf;
        } else {
            warned = true;
        }
        A.out_fit[r] = kept;
        if constexpr (SEL) {
            A.sel_next[r] = acc ? (uint8_t)(cur ^ 1) : cur;
        } else {
            if (A.out_acc) A.out_acc[r] = acc ? 1 : 0;
            if (A.out_warn) A.out_warn[r] = warned ? 1 : 0;
        }
        const unsigned long long k = sort_key(kept);
        my_min = k < my_min ? k : my_min;
        my_warn += warned ? 1u : 0u;
    }
    if constexpr (!SEL) {
        unsigned rej = __ballot_sync(kFull, live && !acc);
        while (rej) {
            const int j = __ffs(rej) - 1;
            rej &= rej - 1;
            const int old_row = A.order ? A.order[g0 + j] : g0 + j;
            const double* x = A.pos + (size_t)old_row * A.ld;
            double* dst = A.out_pos + (size_t)(g0 + j) * A.ld;
            for (int d = lane; d < A.dim; d += 32) dst[d] = x[d];
        }
    }
}

// Even row strides: no staging at all -- each lane streams its own candidate row with 16-byte loads
// (a warp instruction touches 32 rows, the second half of each 32-byte sector follows from L1) and folds
// it in registers; small enough to run 48 warps per SM, so the row streams of many warps overlap.
constexpr int kBasicDirectWarps = 8;
#ifndef APO_BASIC_UNROLL
#define APO_BASIC_UNROLL 4
#endif
constexpr int kBasicUnroll = APO_BASIC_UNROLL;  // 16-byte loads in flight per lane
template <bool SEL>
__global__ void __launch_bounds__(32 * kBasicDirectWarps) k_basic_eval_direct(BasicEvalArgs A) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    const int dim = A.dim, code = A.O.code;
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    const int ngroups = (A.n_rows + 31) / 32;
    for (int grp = blockIdx.x * nwarps + warp; grp < ngroups; grp += gridDim.x * nwarps) {
        const int g0 = A.row0 + grp * 32;
        const int nb = min(32, A.row0 + A.n_rows - g0);
        const int r = g0 + lane;
        const bool live = lane < nb;
        uint8_t cur = 0;
        if constexpr (SEL) cur = live ? A.sel[r] : 0;
        BasicFold f;
        if (live) {
            const double* row = SEL ? (cur ? A.pos0 : A.pos1) + (size_t)r * A.ld : A.out_pos + (size_t)r * A.ld;
            const double2* row2 = reinterpret_cast<const double2*>(row);
            const int h = dim >> 1;
#pragma unroll kBasicUnroll
            for (int k = 0; k < h; k++) {
                const double2 v = __ldcs(row2 + k);  // streamed once: evict-first
                f.add(code, A.O.table, 2 * k, v.x);
                f.add(code, A.O.table, 2 * k + 1, v.y);
            }
            if (dim & 1) f.add(code, A.O.table, dim - 1, __ldcs(row + dim - 1));
        }
        basic_select<SEL>(A, g0, nb, lane, cur, f.value(code, dim), my_min, my_warn);
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

// Any row stride: 32 x 32 blocks moved with 8-byte cp.async (coalesced), double-buffered.
constexpr int kBasicEvalWarps = 4;
constexpr size_t kBasicEvalWarpBytes = 2 * 32 * 33 * 8 + 32 * 8;  // two 32 x 33 blocks + 32 row pointers
constexpr size_t kBasicEvalSmem = (size_t)kBasicEvalWarps * kBasicEvalWarpBytes;

template <bool SEL>
__global__ void __launch_bounds__(32 * kBasicEvalWarps) k_basic_eval(BasicEvalArgs A) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
    unsigned char* wbase = smem + (size_t)warp * kBasicEvalWarpBytes;
    double(*T)[32][33] = reinterpret_cast<double(*)[32][33]>(wbase);  // [2 buffers][row][column]
    const double** rows = reinterpret_cast<const double**>(wbase + 2 * 32 * 33 * 8);
    const int dim = A.dim, code = A.O.code;
    const int nblk = (dim + 31) / 32;
    unsigned long long my_min = ~0ull;
    unsigned my_warn = 0;
    const int ngroups = (A.n_rows + 31) / 32;
    for (int grp = blockIdx.x * nwarps + warp; grp < ngroups; grp += gridDim.x * nwarps) {
        const int g0 = A.row0 + grp * 32;
        const int nb = min(32, A.row0 + A.n_rows - g0);
        const int r = g0 + lane;  // this lane's row
        const bool live = lane < nb;
        uint8_t cur = 0;
        if constexpr (SEL) cur = live ? A.sel[r] : 0;
        if (live) {
            if constexpr (SEL) rows[lane] = (cur ? A.pos0 : A.pos1) + (size_t)r * A.ld;  // the alternate buffer
            else rows[lane] = A.out_pos + (size_t)r * A.ld;
        }
        __syncwarp();
        auto issue = [&](int b) {
            const int d = 32 * b + lane;
            if (d < dim)
                for (int jr = 0; jr < nb; jr++) cp_async8(&T[b & 1][jr][lane], rows[jr] + d);
            cp_async_commit();
        };
        issue(0);
        BasicFold f;
        for (int b = 0; b < nblk; b++) {
            if (b + 1 < nblk) {
                issue(b + 1);
                cp_async_wait_prev();
            } else {
                cp_async_wait_all();
            }
            __syncwarp();
            const int d0 = 32 * b, w = min(32, dim - d0);
            if (live) {
                const double* trow = T[b & 1][lane];
                for (int k = 0; k < w; k++) f.add(code, A.O.table, d0 + k, trow[k]);
            }
            __syncwarp();  // T[b & 1] is refilled by issue(b + 2)
        }
        basic_select<SEL>(A, g0, nb, lane, cur, f.value(code, dim), my_min, my_warn);
    }
    block_finish(my_min, my_warn, A.warn_count, A.trace_key);
}

// CEC2022 at D > kCecEvalMaxDim: transform -> DMMA GEMM -> finish (apo_cec_gemm.cu).
struct CecGemmArgs {
    int n_rows, row0, dim, ld, kp, np, comp;
    ObjDesc O;
    const double* pos0;  // SEL (sel != nullptr): candidate of slot r in its alternate buffer
    const double* pos1;
    const uint8_t* sel;
    uint8_t* sel_next;
    const double* pos;  // dense: old rows (through order if non-null)
    double* out_pos;    // dense: candidates in, kept rows out
    const int* order;
    uint8_t* out_acc;
    uint8_t* out_warn;
    const double* fit;
    double* out_fit;
    const uint8_t* cand_ok;
    unsigned long long* warn_count;
    unsigned long long* trace_key;
    double* Y;  // scratch (set by cec_gemm_finish)
    double* Z;
};
int cec_gemm_finish(const CecGemmArgs& A, cudaStream_t st, int num_sms);
__host__ __device__ inline int gemm_kp(int dim) { return (dim + 15) & ~15; }
__host__ __device__ inline int gemm_np(int dim) { return (dim + 63) & ~63; }

// Kernel getters (defined in the instantiating TUs).
const void* pick_update_sel(int dim, bool cand_only, bool cec, bool many);
const void* pick_update_dense(int dim, bool cand_only, bool cec, bool many);
const void* pick_update_scripted(int dim, bool cand_only, bool cec, bool many);  // apo_update_scripted.cu
cudaError_t launch_dr_scripted(uint64_t table, int ps, int count, int* perm, uint8_t* in_dr, cudaStream_t st);
const void* pick_run_batch(int dim, int rng, bool many);
// apo_prologue.cu: stable sort + Dr set as one launch for small populations (else the CUB prologue)
bool prologue_small_fits(long long ps);
cudaError_t launch_prologue_small(int ps, const double* fit, const int* order_in, int* order_out, int count,
                                  Key cbase, unsigned* dr_bits, unsigned long long* scratch_keys, int* scratch_rank,
                                  int num_sms, cudaStream_t st);
const void* pick_cec_eval(bool sel, int dim, bool fast);
cudaError_t launch_debug_cec_basic(int b, const double* z, long long rows, int n, const double* ew, double* out,
                                   int variant, cudaStream_t st);
// apo_update_fused.cu: CEC2022 (D <= 104, SEL rows) candidates + DMMA evaluation + select in one kernel
int fused_cec_shape(const UpdArgs& a, int optin, size_t* smem, int* stage_shift);
cudaError_t launch_update_cec_fused(const UpdArgs& a, cudaStream_t st, unsigned* counter, int optin, int num_sms);

}  // namespace apo
