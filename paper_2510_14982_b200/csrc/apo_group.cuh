// apo_group.cuh -- the fused APO update for a group of 32 consecutive ranks per warp.
//
// Same arithmetic as update_protozoon (apo_update.cuh, numba_backend.py:141-290),
// re-mapped to cut the warp-instruction count:
//   phase A, lane = protozoon: decision (slot 0), op-specific scalar draws,
//            partner / neighbour pair 0 + its exp weight, and the partial
//            Fisher-Yates mask chain run sequentially per lane on a private
//            uint8 permutation in shared memory (D <= 256) -- 32 chains per
//            warp instruction instead of one;
//   phase B, warp = protozoon: rows loaded into registers (MAXC chunks of 32
//            dims, all loads issued up front), per-dimension vector draws,
//            candidate, clamp, fitness (eval_warp), greedy select and the kept
//            row written straight from registers.
#pragma once
#include <type_traits>

#include "apo_update.cuh"

namespace apo {

constexpr int kGroupMaxDim = 256;  // uint8 permutations

// ---------------------------------------------------------------------------
// TMA bulk copies (cp.async.bulk, SASS UBLKCP) + mbarrier completion.
__device__ __forceinline__ unsigned smem_u32(const void* p) {
    return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_fence_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(dst)),
        "l"(src), "r"(bytes), "r"(smem_u32(bar))
        : "memory");
}
// The same two on 32-bit shared-memory addresses computed once per kernel (the ring's hot path).
__device__ __forceinline__ void mbar_expect_tx_s(unsigned bar, unsigned bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
}
__device__ __forceinline__ void bulk_g2s_s(unsigned dst, const void* src, unsigned bytes, unsigned bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
        "l"(src), "r"(bytes), "r"(bar)
        : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
    asm volatile(
        "{\n\t.reg .pred P1;\n"
        "APO_WAIT_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n\t"
        "@!P1 bra APO_WAIT_%=;\n}" ::"r"(smem_u32(bar)),
        "r"(parity)
        : "memory");
}
__device__ __forceinline__ void fence_proxy_async() {
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}

// Row staging ring: kStages protozoa x 4 rows, per warp (HBM-resident paths).
#ifndef APO_STAGES
#define APO_STAGES 2
#endif
constexpr int kStages = APO_STAGES;
#ifndef APO_STAGE_MAX_DIM
#define APO_STAGE_MAX_DIM 128
#endif


// Terms batch: protozoa whose per-dimension fitness terms are staged in shared
// memory before 1 lane each folds them sequentially.
#ifndef APO_LOAD_CHUNKS
#define APO_LOAD_CHUNKS 2
#endif
#ifndef APO_GROUP_BATCH_SMALL_D
#define APO_GROUP_BATCH_SMALL_D 16
#endif
#ifndef APO_GROUP_BATCH_LARGE_D
#define APO_GROUP_BATCH_LARGE_D 4
#endif
__host__ __device__ inline int group_batch(int dim) {
    return dim <= 64 ? APO_GROUP_BATCH_SMALL_D : APO_GROUP_BATCH_LARGE_D;
}
__host__ __device__ inline int group_tstride(int dim) { return dim | 1; }  // odd: conflict-free lane rows

// Per-warp shared scratch of the group path.
struct GroupScratch {
    unsigned char* perm;  // [32][dp]
    unsigned* bits;       // [32][words]
    double* f;            // [32] forage factor (auto/hetero) or scale (repro)
    double* sgn;          // [32] heterotroph sign
    double* w;            // [32] pair-0 weight
    int* slot;            // [32][4] own, partner, km, kp slots
    int* op;              // [32]
    double* T;            // [batch][tstride] fitness terms
    double* ring;         // [kStages][4][rld] staged rows (nullptr if not staging)
    uint64_t* bar;        // [kStages] mbarriers of the ring
    const double** rsrc;  // [32][4] global source of each ring row (staging; set before the first issue)
    unsigned* rmask;      // [32] ring rows a member reads: bit r = row r (own, partner, km, kp)
    WarpScratch ws;       // only ws.pk / ws.pw (pair cache for npairs > 1) are used
    int dp, words, tstride, cstride, batch, rld;
};

__host__ __device__ inline int ring_ld(int dim) { return (dim + 1) & ~1; }
__host__ __device__ inline size_t ring_bytes(int dim, bool stage) {
    // rows, mbarriers (16 B each), then the per-member row sources and masks
    return stage ? (size_t)kStages * 4 * 8 * (size_t)ring_ld(dim) + 16 * kStages + 32 * 4 * 8 + 32 * 4 : 0;
}

// Layout: [header: scalars, slots, ops, pair cache, mask bits][union: phase-A
// permutations (32 x dp bytes) | phase-B terms (batch x tstride doubles)].
// The permutations are dead once phase A ends, so the terms reuse them.
__host__ __device__ inline size_t group_head_bytes(int dim) {
    const size_t words = (size_t)(dim + 31) / 32;
    size_t b = 32 * 8 * 3 + 32 * 4 * 4 + 32 * 4 + 32 * words * 4;
    b += 8 * 3 * kMaxCachedPairs;
    return (b + 15) & ~(size_t)15;
}

// CEC2022 objectives evaluate kCecRows candidates at once (one DMMA m-tile):
// rows X (candidates), Z (rotation output) and, for compositions, W (the
// per-component shifted copy), each kCecRows x cec_stride doubles.  The
// stride is a multiple of 4 that is not a multiple of 8, so the A-fragment
// loads of a DMMA (rows g = lane/4, columns t = lane%4) are bank-conflict
// free.  cec_bufs = 0 (not CEC), 2 (F1-F8) or 3 (F9-F12).
constexpr int kCecRows = 8;
constexpr int kCecQuadMaxDim = 104;  // rot_pad exists for dim <= 104 (objectives.py, include/apo_b200.h)
__host__ __device__ inline int cec_nt_dev(int n) { return n <= 16 ? 2 : n <= 32 ? 4 : n <= 56 ? 7 : 13; }
__host__ __device__ inline int cec_stride(int dim) {
    const int s = (dim + 3) & ~3;
    return (s & 7) ? s : s + 4;
}
__host__ __device__ inline int cec_bufs_for(int code) {
    return code <= 100 ? 0 : (code - 100 >= 9 ? 3 : 2);
}

__host__ __device__ inline size_t group_union_bytes(int dim, int cec_bufs = 0) {
    const size_t perm = 32 * (size_t)((dim + 3) & ~3);
    size_t terms = 8 * (size_t)group_batch(dim) * (size_t)group_tstride(dim);
    const size_t cec = 8 * (size_t)cec_bufs * kCecRows * (size_t)cec_stride(dim);
    if (cec > terms) terms = cec;
    return ((perm > terms ? perm : terms) + 15) / 16 * 16;
}

__host__ __device__ inline size_t group_scratch_bytes(int dim, bool stage = false, int cec_bufs = 0) {
    return group_head_bytes(dim) + group_union_bytes(dim, cec_bufs) + ring_bytes(dim, stage);
}

__device__ inline GroupScratch group_scratch(unsigned char* base, int dim, bool stage = false, int cec_bufs = 0) {
    GroupScratch g;
    g.dp = (dim + 3) & ~3;
    g.words = (dim + 31) / 32;
    g.tstride = group_tstride(dim);
    g.cstride = cec_stride(dim);
    g.batch = group_batch(dim);
    g.f = reinterpret_cast<double*>(base);
    g.sgn = g.f + 32;
    g.w = g.sgn + 32;
    g.ws.pw = g.w + 32;
    g.slot = reinterpret_cast<int*>(g.ws.pw + kMaxCachedPairs);
    g.op = g.slot + 128;
    g.ws.pk = g.op + 32;
    g.bits = reinterpret_cast<unsigned*>(g.ws.pk + 2 * kMaxCachedPairs);
    g.perm = base + group_head_bytes(dim);
    g.T = reinterpret_cast<double*>(base + group_head_bytes(dim));
    g.rld = ring_ld(dim);
    if (stage) {
        g.ring = reinterpret_cast<double*>(base + group_head_bytes(dim) + group_union_bytes(dim, cec_bufs));
        g.bar = reinterpret_cast<uint64_t*>(g.ring + (size_t)kStages * 4 * g.rld);
        g.rsrc = reinterpret_cast<const double**>(g.bar + 2 * kStages);
        g.rmask = reinterpret_cast<unsigned*>(g.rsrc + 32 * 4);
    } else {
        g.ring = nullptr;
        g.bar = nullptr;
        g.rsrc = nullptr;
        g.rmask = nullptr;
    }
    g.ws.cand = g.ws.terms = nullptr;
    g.ws.head = g.ws.prev = g.ws.rj = nullptr;
    g.ws.bits = nullptr;
    return g;
}

struct DenseSlots {
    const double* pos;
    const double* fit;
    int ld;
    __device__ __forceinline__ int slot(int rank1) const { return rank1 - 1; }
    __device__ __forceinline__ int key(int rank1) const { return rank1 - 1; }
    __device__ __forceinline__ int slot_of(int key) const { return key; }
    __device__ __forceinline__ const double* at_key(int key) const { return pos + (size_t)key * ld; }
    __device__ __forceinline__ const double* at(int slot) const { return pos + (size_t)slot * ld; }
    __device__ __forceinline__ double fit_at(int slot) const { return fit[slot]; }
    __device__ __forceinline__ const double* row(int rank1) const { return at(rank1 - 1); }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[rank1 - 1]; }
};

struct OrderedSlots {
    const double* pos;
    const double* fit;
    const int* order;
    int ld;
    __device__ __forceinline__ int slot(int rank1) const { return order[rank1 - 1]; }
    __device__ __forceinline__ int key(int rank1) const { return order[rank1 - 1]; }
    __device__ __forceinline__ int slot_of(int key) const { return key; }
    __device__ __forceinline__ const double* at_key(int key) const { return pos + (size_t)key * ld; }
    __device__ __forceinline__ const double* at(int slot) const { return pos + (size_t)slot * ld; }
    __device__ __forceinline__ double fit_at(int slot) const { return fit[slot]; }
    __device__ __forceinline__ const double* row(int rank1) const { return at(order[rank1 - 1]); }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[order[rank1 - 1]]; }
};

// HBM-resident population with two row buffers per slot: sel[slot] says which
// buffer holds the current row.  A candidate is written to the other buffer;
// acceptance just flips the slot's selector for the next iteration, so a
// rejected candidate costs no row copy.
struct SelSlots {
    const double* pos0;
    const double* pos1;
    const uint8_t* sel;
    const double* fit;
    const int* order;
    int ld;
    __device__ __forceinline__ int slot(int rank1) const { return order[rank1 - 1]; }
    // key = slot*2 + selector: resolved once in phase A so phase B row loads
    // do not wait on the selector load.
    __device__ __forceinline__ int key(int rank1) const {
        const int s = order[rank1 - 1];
        return (s << 1) | (int)sel[s];
    }
    __device__ __forceinline__ int slot_of(int key) const { return key >> 1; }
    __device__ __forceinline__ const double* at_key(int key) const {
        return ((key & 1) ? pos1 : pos0) + (size_t)(key >> 1) * ld;
    }
    __device__ __forceinline__ double* alt_key(int key) const {
        return const_cast<double*>(((key & 1) ? pos0 : pos1) + (size_t)(key >> 1) * ld);
    }
    __device__ __forceinline__ const double* at(int slot) const {
        return (sel[slot] ? pos1 : pos0) + (size_t)slot * ld;
    }
    __device__ __forceinline__ double* alt(int slot) const {
        return const_cast<double*>((sel[slot] ? pos0 : pos1) + (size_t)slot * ld);
    }
    __device__ __forceinline__ double fit_at(int slot) const { return fit[slot]; }
    __device__ __forceinline__ const double* row(int rank1) const { return at(order[rank1 - 1]); }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[order[rank1 - 1]]; }
};

// Phase A for rank i (one lane).  Fills the lane's entries of g.
template <class Rows>
__device__ inline void group_phase_a(const IterParams& P, const Rows& R, int i, bool in_dr, double p_dr_i,
                                     const GroupScratch& g, int lane) {
    const int ps = P.ps, dim = P.dim;
    const Key base = iteration_key(P, (uint64_t)i);
    const double u_dec = uniform(base, kSlotDecision);
    int op;
    if (in_dr) op = (u_dec < p_dr_i) ? OP_DORMANCY : OP_REPRODUCTION;
    else op = (u_dec < P.p_ah) ? OP_AUTOTROPH : OP_HETEROTROPH;
    int* sl = g.slot + 4 * lane;  // row keys (see SelSlots::key)
    sl[0] = R.key(i);
    int count = 0;
    if (op == OP_REPRODUCTION) {
        const double sgn = uniform(base, kSlotSign) < 0.5 ? 1.0 : -1.0;
        const double mag = uniform(base, kSlotMagnitude);
        count = (int)ceil((double)dim * uniform(base, kSlotMaskSize));
        g.f[lane] = sgn * mag;
    } else if (op != OP_DORMANCY) {
        int km, kp;
        if (op == OP_AUTOTROPH) {
            int partner = i;
            if (ps > 1) {
                int j0 = (int)(uniform(base, kSlotPartner) * (double)(ps - 1));
                if (j0 > ps - 2) j0 = ps - 2;
                if (j0 >= i - 1) j0 += 1;
                partner = j0 + 1;
            }
            sl[1] = R.key(partner);
            if (i == 1) {
                km = 1;
            } else {
                km = 1 + (int)(uniform(base, kPairsBase) * (double)(i - 1));
                if (km > i - 1) km = i - 1;
            }
            if (i == ps) {
                kp = ps;
            } else {
                kp = i + 1 + (int)(uniform(base, kPairsBase + 1) * (double)(ps - i));
                if (kp > ps) kp = ps;
            }
        } else {
            g.sgn[lane] = uniform(base, kSlotSign) < 0.5 ? 1.0 : -1.0;
            km = i - 1 < 1 ? 1 : i - 1;
            kp = i + 1 > ps ? ps : i + 1;
        }
        g.f[lane] = uniform(base, kSlotForage) * P.f_mult;
        count = (int)ceil((double)((long long)dim * i) / (double)ps);
        const int skm = R.key(km), skp = R.key(kp);
        sl[2] = skm;
        sl[3] = skp;
        g.w[lane] = rank_weight(R.fit_at(R.slot_of(skm)), R.fit_at(R.slot_of(skp)), P.eps);
    }
    g.op[lane] = op;
    // mask: sequential partial Fisher-Yates on this lane's permutation
    // (numba_backend.py:74-90), then scatter the first `count` values.
    unsigned* bits = g.bits + (size_t)lane * g.words;
    for (int w = 0; w < g.words; w++) bits[w] = 0u;
    if (op != OP_DORMANCY && count > 0) {
        unsigned char* perm = g.perm + (size_t)lane * g.dp;
        // identity, four entries per 32-bit store (rows are 4-byte aligned, dim <= 256); bytes past dim
        // are never read
        unsigned* perm4 = reinterpret_cast<unsigned*>(perm);
        for (int w = 0; w < (dim + 3) >> 2; w++) perm4[w] = 0x03020100u + 0x04040404u * (unsigned)w;
        for (int j = 0; j < count; j++) {
            int r = j + (int)(uniform(base, kMaskBase + (uint64_t)j) * (double)(dim - j));
            if (r > dim - 1) r = dim - 1;
            const unsigned char a = perm[j], b = perm[r];
            perm[j] = b;
            perm[r] = a;
            bits[b >> 5] |= 1u << (b & 31);
        }
    }
}

__device__ __forceinline__ double gmask(const GroupScratch& g, int p, int d) {
    return ((g.bits[p * g.words + (d >> 5)] >> (d & 31)) & 1u) ? 1.0 : 0.0;
}

// Pairs k >= 1 when npairs > 1 (warp-parallel, cached in g.ws.pk / g.ws.pw).
template <class Rows>
__device__ inline void group_extra_pairs(const IterParams& P, const Rows& R, int i, int op, const Key& base,
                                         const GroupScratch& g, int lane) {
    const int ps = P.ps;
    if (lane >= 1 && lane < kMaxCachedPairs && lane < P.npairs) {
        const int k = lane;
        int km, kp;
        if (op == OP_AUTOTROPH) {
            if (i == 1) {
                km = 1;
            } else {
                km = 1 + (int)(uniform(base, kPairsBase + 2ull * k) * (double)(i - 1));
                if (km > i - 1) km = i - 1;
            }
            if (i == ps) {
                kp = ps;
            } else {
                kp = i + 1 + (int)(uniform(base, kPairsBase + 2ull * k + 1) * (double)(ps - i));
                if (kp > ps) kp = ps;
            }
        } else {
            km = i - (k + 1);
            if (km < 1) km = 1;
            kp = i + (k + 1);
            if (kp > ps) kp = ps;
        }
        g.ws.pk[2 * k] = R.key(km);
        g.ws.pk[2 * k + 1] = R.key(kp);
        g.ws.pw[k] = rank_weight(R.fitness(km), R.fitness(kp), P.eps);
    }
    __syncwarp();
}

// acc for pairs k >= 1 at dimension d (pair 0 is added by the caller first,
// so the accumulation order matches the reference: acc = 0; acc += w_k*(...)).
template <class Rows>
__device__ __forceinline__ double extra_pairs_acc(const IterParams& P, const Rows& R, int i, int op, const Key& base,
                                                  const GroupScratch& g, double acc, int d) {
    for (int k = 1; k < P.npairs; k++) {
        int skm, skp;
        double w;
        if (k < kMaxCachedPairs) {
            skm = g.ws.pk[2 * k];
            skp = g.ws.pk[2 * k + 1];
            w = g.ws.pw[k];
        } else {
            const int ps = P.ps;
            int km, kp;
            if (op == OP_AUTOTROPH) {
                if (i == 1) {
                    km = 1;
                } else {
                    km = 1 + (int)(uniform(base, kPairsBase + 2ull * k) * (double)(i - 1));
                    if (km > i - 1) km = i - 1;
                }
                if (i == ps) {
                    kp = ps;
                } else {
                    kp = i + 1 + (int)(uniform(base, kPairsBase + 2ull * k + 1) * (double)(ps - i));
                    if (kp > ps) kp = ps;
                }
            } else {
                km = i - (k + 1);
                if (km < 1) km = 1;
                kp = i + (k + 1);
                if (kp > ps) kp = ps;
            }
            skm = R.key(km);
            skp = R.key(kp);
            w = rank_weight(R.fit_at(R.slot_of(skm)), R.fit_at(R.slot_of(skp)), P.eps);
        }
        acc = acc + w * (R.at_key(skm)[d] - R.at_key(skp)[d]);
    }
    return acc;
}


__device__ __forceinline__ double clampv(double c, double lo, double hi) {
    if (c < lo) c = lo;
    else if (c > hi) c = hi;
    return c;
}

// hgbat/griewank stage two term rows per protozoon; CEC objectives stage the
// candidate itself (rows of stride cstride, see cec_stride).
__device__ __forceinline__ bool two_term_arrays(int code) {
    return code == OBJ_HGBAT || code == OBJ_GRIEWANK;
}

// Per-dimension fitness terms of candidate value c at dimension d (c_prev =
// candidate value at d-1, valid when d >= 1).  Row T1 (and T2 for the
// two-array objectives) belongs to one protozoon.  Each term is rounded
// exactly as the reference's accumulation loop rounds it
// (numba_backend.py:96-131).
__device__ __forceinline__ void write_terms(const ObjDesc& O, double* T1, double* T2, int d, double c, double c_prev) {
    switch (O.code) {
    case OBJ_SPHERE:
    case OBJ_BENT_CIGAR:
        T1[d] = c * c;
        break;
    case OBJ_ELLIPTIC:
        T1[d] = (O.table[d] * c) * c;
        break;
    case OBJ_HGBAT:
        T1[d] = c;
        T2[d] = c * c;
        break;
    case OBJ_ROSENBROCK:
        if (d >= 1) {
            const double a = c - c_prev * c_prev;
            const double b = c_prev - 1.0;
            T1[d - 1] = 100.0 * (a * a) + b * b;
        }
        break;
    case OBJ_GRIEWANK:
        T1[d] = c * c;
        T2[d] = cos_glibc(c / sqrt((double)d + 1.0));  // glibc-exact (numba_backend.py:130)
        break;
    default:
        if (O.code >= OBJ_CEC_BASE || O.code == OBJ_OTSU_ML || O.code == OBJ_KAPUR_ML) {
            T1[d] = c;
        } else if (d == 0) {
            long long idx = (long long)floor(c + 0.5);
            if (idx < 0) idx = 0;
            if (idx > O.table_len - 1) idx = O.table_len - 1;
            T1[0] = O.table[idx];
        }
        break;
    }
}

// Sequential left-to-right fold of one protozoon's terms (one lane).
__device__ inline double fold_terms(const ObjDesc& O, const double* T1, const double* T2, int dim) {
    double s = 0.0;
    switch (O.code) {
    case OBJ_SPHERE:
    case OBJ_ELLIPTIC:
#pragma unroll 4
        for (int d = 0; d < dim; d++) s += T1[d];
        return s;
    case OBJ_BENT_CIGAR:
#pragma unroll 4
        for (int d = 1; d < dim; d++) s += T1[d];
        return T1[0] + 1e6 * s;
    case OBJ_HGBAT: {
        double s1 = 0.0, s2 = 0.0;
#pragma unroll 4
        for (int d = 0; d < dim; d++) {
            s1 += T1[d];
            s2 += T2[d];
        }
        return sqrt(fabs(s2 * s2 - s1 * s1)) + (0.5 * s2 + s1) / (double)dim + 0.5;
    }
    case OBJ_ROSENBROCK:
#pragma unroll 4
        for (int d = 0; d < dim - 1; d++) s += T1[d];
        return s;
    case OBJ_GRIEWANK: {
        double p = 1.0;
#pragma unroll 4
        for (int d = 0; d < dim; d++) {
            s += T1[d];
            p *= T2[d];
        }
        return 1.0 + s / 4000.0 - p;
    }
    case OBJ_OTSU_ML:
    case OBJ_KAPUR_ML:
        return threshold_ml(O.code, T1, dim, O.table);
    default:
        return T1[0];
    }
}

enum OutMode : int {
    OUT_SEL = 0,    // speculative write to the slot's alternate buffer, flip sel_next on accept
    OUT_FIXUP = 1,  // write the candidate to the output row; rewrite rejected rows with the old row
};

// Candidate of member p (rank i) of the group, warp-cooperative: computes
// the clamped candidate, writes it to `cand_out`, stores its fitness terms in
// rows (T1, T2) and returns the finiteness vote.
// Objective classes an update kernel is compiled for (keeps CEC code out of kernels that never see it).
enum GroupKind : int { KIND_ANY = 0, KIND_BASIC = 1, KIND_CAND = 2 };

// XCOPY (with CO): the clamped candidate also goes to T1[d] (the fused CEC kernel's shared-memory tile).
// VOTE = false: returns this lane's finiteness only (the caller folds the warp's votes for a whole
// batch of members with one reduction instead of one vote per member).
template <int MAXC, bool MANY, bool CO, class Rows, bool XCOPY = false, bool VOTE = true>
__device__ inline bool group_candidate(const IterParams& P, const ObjDesc& O, const Rows& R, int i, int p,
                                       double* cand_out, double* T1, double* T2, const GroupScratch& g, int lane,
                                       const double* staged) {
    const int dim = P.dim;
    const int op = g.op[p];
    const int* sl = g.slot + 4 * p;
    const double* x = staged ? staged : R.at_key(sl[0]);
    const double f = g.f[p];
    const bool many = MANY && op >= OP_AUTOTROPH;
    Key base{};
    if (op != OP_AUTOTROPH || many) base = iteration_key(P, (uint64_t)i);
    if (many) group_extra_pairs(P, R, i, op, base, g, lane);
    const double* xj = staged ? staged + g.rld : R.at_key(sl[op == OP_AUTOTROPH ? 1 : 0]);
    const double* xm = staged ? staged + 2 * g.rld : R.at_key(sl[op >= OP_AUTOTROPH ? 2 : 0]);
    const double* xp = staged ? staged + 3 * g.rld : R.at_key(sl[op >= OP_AUTOTROPH ? 3 : 0]);
    const double w0 = g.w[p];
    const double sgn = g.sgn[p];
    const double npd = (double)P.npairs;
    const unsigned* mb = g.bits + p * g.words;
    bool ok = true;
    double carry = 0.0;  // candidate at d-1 for lane 0 of the next chunk

    auto mk = [&](int d) -> double { return ((mb[d >> 5] >> (d & 31)) & 1u) ? 1.0 : 0.0; };
    // AUTO: compile-time operation for the unrolled paths (-1: decided at run time from op)
    auto forage_t = [&](auto auto_tag, int d, double xd, double aj, double am, double ap) -> double {
        constexpr int AUTO = decltype(auto_tag)::value;
        double acc = 0.0;
        acc = acc + w0 * (am - ap);
        double ep = acc;
        if constexpr (MANY) {
            if (many) acc = extra_pairs_acc(P, R, i, op, base, g, acc, d);
            ep = acc / npd;
        }
        double direction;
        const bool is_auto = AUTO == 1 || (AUTO < 0 && op == OP_AUTOTROPH);
        if (is_auto) {
            direction = (aj - xd) + ep;
        } else {
            const double uv = uniform(base, kVectorBase + (uint64_t)d);
            direction = ((1.0 + (sgn * uv) * P.decay) * xd - xd) + ep;
        }
        return xd + (f * direction) * mk(d);
    };
    auto forage = [&](int d, double xd, double aj, double am, double ap) -> double {
        return forage_t(std::integral_constant<int, -1>{}, d, xd, aj, am, ap);
    };
    // every lane calls finish() once per chunk (the shuffles need the full warp)
    // CO (candidates only, CEC2022 on HBM): no fitness terms; only rosenbrock needs the d-1 neighbour
    const bool need_prev = !CO && O.code == OBJ_ROSENBROCK;
    auto finish = [&](int d, double c, bool valid) {
        c = clampv(c, P.lower, P.upper);
        double prev = 0.0;
        if (need_prev) {
            prev = __shfl_up_sync(kFull, c, 1);
            if (lane == 0) prev = carry;
            carry = __shfl_sync(kFull, c, 31);
        }
        if (valid) {
            ok = ok && isfinite(c);
            cand_out[d] = c;
            if constexpr (!CO) write_terms(O, T1, T2, d, c, prev);
            else if constexpr (XCOPY) T1[d] = c;
        }
    };

    // the two foraging operations (95% of protozoa), each with its own unrolled body: row loads issued
    // LC chunks at a time (up to 4 rows x LC chunks in flight) and the chunks' arithmetic interleaved
    auto unrolled = [&](auto auto_tag) {
        constexpr bool AUTO = decltype(auto_tag)::value == 1;
        constexpr int LC = (APO_LOAD_CHUNKS < MAXC ? APO_LOAD_CHUNKS : (MAXC > 0 ? MAXC : 1));
#pragma unroll
        for (int c0 = 0; c0 < (MAXC > 0 ? MAXC : 1); c0 += LC) {
            double xv[LC], aj[LC], am[LC], ap[LC];
#pragma unroll
            for (int u = 0; u < LC; u++) {
                const int d = lane + 32 * (c0 + u);
                if (d < dim) {
                    xv[u] = x[d];
                    aj[u] = AUTO ? xj[d] : 0.0;
                    am[u] = xm[d];
                    ap[u] = xp[d];
                }
            }
#pragma unroll
            for (int u = 0; u < LC; u++) {
                const int c = c0 + u;
                const int d = lane + 32 * c;
                if (32 * c < dim) finish(d, d < dim ? forage_t(auto_tag, d, xv[u], aj[u], am[u], ap[u]) : 0.0, d < dim);
            }
        }
    };
    // candidates-only kernels (no fitness code) afford a second unrolled body for the heterotroph; the
    // fused kernels keep one (register pressure: measured 50% slower with both)
    if (MAXC > 0 && op == OP_AUTOTROPH) {
        unrolled(std::integral_constant<int, 1>{});
    } else if (CO && MAXC > 0 && op == OP_HETEROTROPH) {
        unrolled(std::integral_constant<int, 0>{});
    } else {
        const int nch = (dim + 31) / 32;
        for (int c = 0; c < nch; c++) {
            const int d = lane + 32 * c;
            double cv = 0.0;
            if (d < dim) {
                const double xd = x[d];
                if (op == OP_DORMANCY) {
                    cv = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
                } else if (op == OP_REPRODUCTION) {
                    const double off = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
                    cv = xd + (f * off) * mk(d);
                } else {
                    cv = forage(d, xd, op == OP_AUTOTROPH ? xj[d] : 0.0, xm[d], xp[d]);
                }
            }
            finish(d, cv, d < dim);
        }
    }
    if constexpr (VOTE) return __all_sync(kFull, ok);
    return ok;
}

// One group of n <= 32 consecutive ranks [i0, i0+n) on one warp.
// MODE OUT_SEL:   rows via SelSlots; candidates go to R.alt(slot); sel_next and
//                 out_fit (by slot) record the kept state.
// MODE OUT_FIXUP: candidates go to out_rows (by slot if out_by_slot, else by
//                 rank); rejected rows are then rewritten with the old row.
// NP: 1 = built for npairs == 1 only, 2 = npairs > 1 only, 0 = either (decided per call).  The update
// kernels are instantiated per case: the unused candidate body costs registers even when never taken
// (C4 rosenbrock 1.371 -> 1.314 ms per iteration without it).
template <int MAXC, int MODE, int KIND, int NP = 0, class Rows>
__device__ inline void update_group(const IterParams& P, const ObjDesc& O, const Rows& R, int i0, int n,
                                    const uint8_t* in_dr_bytes, const unsigned* in_dr_bits, const double* p_dr,
                                    double* out_rows, double* out_fit, bool out_by_slot, uint8_t* out_acc,
                                    uint8_t* out_warn, uint8_t* sel_next, const GroupScratch& g, int lane,
                                    unsigned long long& my_min, unsigned& my_warn, unsigned* ring_phase = nullptr,
                                    uint8_t* cand_ok = nullptr) {
    if (lane < n) {
        const int r0 = i0 - 1 + lane;
        const bool dr = in_dr_bits ? ((in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0 : in_dr_bytes[r0] != 0;
        group_phase_a(P, R, i0 + lane, dr, dr ? p_dr[r0] : 0.0, g, lane);
    }
    __syncwarp();
    const bool staging = g.ring != nullptr;
    // TMA prefetch of member p's rows into ring stage p % kStages: lane r < 4 copies ring row r (own,
    // partner, km, kp) when the operation reads it, so the warp issues one address computation and one
    // bulk copy instead of four in sequence; lane 0 posts the byte count first.
    // The members' row sources and masks are resolved once, lane-parallel, before the first issue.
    unsigned ring_s = 0, bar_s = 0;
    auto issue = [&](int p) {
        if (lane < 4) {
            const unsigned m = g.rmask[p];
            const int st = p % kStages;
            const unsigned bytes = (unsigned)(8 * P.ld);
            const unsigned bar = bar_s + 8u * (unsigned)st;
            if (lane == 0) {
                fence_proxy_async();
                mbar_expect_tx_s(bar, bytes * (unsigned)__popc(m));
            }
            __syncwarp(0xFu);
            if ((m >> lane) & 1u) {
                fence_proxy_async();
                bulk_g2s_s(ring_s + 8u * (unsigned)((st * 4 + lane) * g.rld), g.rsrc[4 * p + lane], bytes, bar);
            }
        }
    };
    if (staging) {
        ring_s = smem_u32(g.ring);
        bar_s = smem_u32(g.bar);
        if (lane < n) {
            const int op = g.op[lane];
            const unsigned m = op == OP_AUTOTROPH ? 0xFu : op == OP_HETEROTROPH ? 0xDu : op == OP_REPRODUCTION ? 0x1u : 0u;
            g.rmask[lane] = m;
            for (int r = 0; r < 4; r++)
                if ((m >> r) & 1u) g.rsrc[4 * lane + r] = R.at_key(g.slot[4 * lane + r]);
        }
        __syncwarp();
        for (int p = 0; p < kStages && p < n; p++) issue(p);
    }
    const bool two = two_term_arrays(O.code);
    // KIND_BASIC kernels are never launched for CEC2022 objectives (the host routes those elsewhere)
    const bool cec = KIND == KIND_ANY && O.code >= OBJ_CEC_BASE;
    const int ts = cec ? g.cstride : g.tstride;
    // cand_ok != nullptr: candidates only (written + finiteness flag); the
    // fitness, greedy select and best-so-far run in k_cec_eval (CEC2022 on HBM).
    constexpr bool cand_only = KIND == KIND_CAND;  // cand_ok must then be non-null
    const int B = cand_only ? 32 : cec ? kCecRows : two ? g.batch / 2 : g.batch;
    double* T2base = g.T + (size_t)(g.batch / 2) * g.tstride;
    for (int h = 0; h < n; h += B) {
        const int nb = min(B, n - h);
        unsigned badbits = 0;  // bit q: a non-finite candidate element of member h+q in this lane
        for (int q = 0; q < nb; q++) {
            const int p = h + q, i = i0 + p;
            const int own_key = g.slot[4 * p];
            double* dst;
            if constexpr (MODE == OUT_SEL) dst = R.alt_key(own_key);
            else dst = out_rows + (size_t)(out_by_slot ? R.slot_of(own_key) : i - 1) * P.ld;
            double* T1 = cand_only ? g.T : g.T + (size_t)q * ts;
            double* T2 = two ? T2base + (size_t)q * g.tstride : nullptr;
            const double* staged = nullptr;
            if (staging) {
                const int st = p % kStages;
                mbar_wait(&g.bar[st], (*ring_phase >> st) & 1u);
                *ring_phase ^= 1u << st;
                staged = g.ring + (size_t)st * 4 * g.rld;
            }
            bool ok;
            if constexpr (NP == 1) {
                ok = group_candidate<MAXC, false, cand_only, Rows, false, false>(P, O, R, i, p, dst, T1, T2, g, lane,
                                                                             staged);
            } else if constexpr (NP == 2) {
                ok = group_candidate<MAXC, true, cand_only, Rows, false, false>(P, O, R, i, p, dst, T1, T2, g, lane,
                                                                            staged);
            } else {
                ok = P.npairs > 1 ? group_candidate<MAXC, true, cand_only, Rows, false, false>(P, O, R, i, p, dst, T1,
                                                                                              T2, g, lane, staged)
                                  : group_candidate<MAXC, false, cand_only, Rows, false, false>(P, O, R, i, p, dst, T1,
                                                                                               T2, g, lane, staged);
            }
            badbits |= (ok ? 0u : 1u) << q;
            if (staging) {
                __syncwarp();
                if (p + kStages < n) issue(p + kStages);
            }
        }
        __syncwarp();
        const unsigned okmask = ~__reduce_or_sync(kFull, badbits);
        if constexpr (cand_only) {
            if (lane < nb) {
                const int own_key = g.slot[4 * (h + lane)];
                cand_ok[MODE == OUT_SEL ? R.slot_of(own_key) : i0 - 1 + h + lane] = (uint8_t)((okmask >> lane) & 1u);
            }
            __syncwarp();
            continue;
        }
        bool acc = false, warned = false;
        double cec_f = 0.0;
        if constexpr (KIND == KIND_ANY) {
            if (cec) {  // the batch's staged candidates together (DMMA rotation, apo_cec.cuh)
                if (MAXC > 0 && O.cec.rot_pad && P.dim <= kCecQuadMaxDim) {
                    // quad-per-candidate evaluator (the k_cec_eval code): rows zero-padded to n4;
                    // compositions re-read candidate q from the row it was written to
                    const int q = lane >> 2, t4 = lane & 3, n4 = (P.dim + 3) & ~3;
                    for (int i = P.dim + t4; i < n4; i += 4) g.T[(size_t)q * ts + i] = 0.0;
                    const double* src = nullptr;
                    if (q < nb) {
                        const int own_key = g.slot[4 * (h + q)];
                        if constexpr (MODE == OUT_SEL) src = R.alt_key(own_key);
                        else src = out_rows + (size_t)(out_by_slot ? R.slot_of(own_key) : i0 - 1 + h + q) * P.ld;
                    }
                    __syncwarp();
                    const double* ew = O.table_len >= P.dim ? O.table : nullptr;
                    // the n-tile counts a register-resident variant can meet (MAXC bounds dim)
                    double fq = 0.0;
                    const int nt = cec_nt_dev(P.dim);
                    if constexpr (MAXC == 1) {
                        fq = nt == 2 ? cec_eval_quad<2, false>(O.cec, g.T, src, ts, P.dim, lane, ew)
                                     : cec_eval_quad<4, false>(O.cec, g.T, src, ts, P.dim, lane, ew);
                    } else if constexpr (MAXC == 2) {
                        fq = nt == 7 ? cec_eval_quad<7, false>(O.cec, g.T, src, ts, P.dim, lane, ew)
                                     : cec_eval_quad<13, false>(O.cec, g.T, src, ts, P.dim, lane, ew);
                    } else if constexpr (MAXC == 4) {
                        fq = cec_eval_quad<13, false>(O.cec, g.T, src, ts, P.dim, lane, ew);
                    }
                    cec_f = __shfl_sync(kFull, fq, (lane & 7) * 4);  // lane q < 8 <- quad q
                } else {
                    cec_f = cec_eval_batch(O.cec, g.T, g.T + (size_t)kCecRows * ts, g.T + (size_t)2 * kCecRows * ts,
                                           ts, nb, P.dim, lane);
                }
            }
        }
        if (lane < nb) {
            const int p = h + lane, i = i0 + p;
            const int own_key = g.slot[4 * p];
            const int own = R.slot_of(own_key);
            const double fit_i = R.fit_at(own);
            double kept = fit_i;
            if ((okmask >> lane) & 1u) {
                const double nf = cec
                                      ? cec_f
                                      : fold_terms(O, g.T + (size_t)lane * g.tstride,
                                                   two ? T2base + (size_t)lane * g.tstride : nullptr, P.dim);
                if (isfinite(nf)) {
                    acc = nf < fit_i;
                    if (acc) kept = nf;
                } else {
                    warned = true;
                }
            } else {
                warned = true;
            }
            out_fit[out_by_slot ? own : i - 1] = kept;
            if (out_acc) out_acc[i - 1] = acc ? 1 : 0;
            if (out_warn) out_warn[i - 1] = warned ? 1 : 0;
            if constexpr (MODE == OUT_SEL) {
                const uint8_t cur = (uint8_t)(own_key & 1);
                sel_next[own] = acc ? (uint8_t)(cur ^ 1) : cur;
            }
            const unsigned long long k = sort_key(kept);
            my_min = k < my_min ? k : my_min;
            my_warn += warned ? 1u : 0u;
        }
        if constexpr (MODE == OUT_FIXUP) {
            unsigned rej = __ballot_sync(kFull, lane < nb && !acc);
            while (rej) {
                const int q = __ffs(rej) - 1;
                rej &= rej - 1;
                const int p = h + q, i = i0 + p;
                const int own_key = g.slot[4 * p];
                const double* x = R.at_key(own_key);
                double* dst = out_rows + (size_t)(out_by_slot ? R.slot_of(own_key) : i - 1) * P.ld;
                for (int d = lane; d < P.dim; d += 32) dst[d] = x[d];
            }
        }
        __syncwarp();
    }
}

// The reference's loop (numba_backend.py:96-131) as a running state over a candidate's elements in order.
struct BasicFold {
    double s = 0.0, s2 = 0.0, p = 1.0, first = 0.0, prev = 0.0;
    __device__ __forceinline__ void add(int code, const double* table, int d, double c) {
        switch (code) {
        case OBJ_SPHERE: s += c * c; break;
        case OBJ_BENT_CIGAR:
            if (d == 0) first = c * c;
            else s += c * c;
            break;
        case OBJ_ELLIPTIC: s += (table[d] * c) * c; break;
        case OBJ_HGBAT:
            s += c;
            s2 += c * c;
            break;
        case OBJ_ROSENBROCK:
            if (d >= 1) {
                const double a = c - prev * prev;
                const double b = prev - 1.0;
                s += 100.0 * (a * a) + b * b;
            }
            prev = c;
            break;
        default:  // OBJ_GRIEWANK
            s += c * c;
            p *= cos_glibc(c / sqrt((double)d + 1.0));
            break;
        }
    }
    __device__ __forceinline__ double value(int code, int dim) const {
        switch (code) {
        case OBJ_SPHERE:
        case OBJ_ELLIPTIC:
        case OBJ_ROSENBROCK: return s;
        case OBJ_BENT_CIGAR: return first + 1e6 * s;
        case OBJ_HGBAT: return sqrt(fabs(s2 * s2 - s * s)) + (0.5 * s2 + s) / (double)dim + 0.5;
        default: return 1.0 + s / 4000.0 - p;
        }
    }
};

// Lane-per-protozoon update of a group (the batch kernel's reference objectives at dim <= kLppMaxDim,
// npairs == 1, rows in shared memory): phase A as above, then each lane builds its own candidate
// dimension by dimension (the same expressions as group_candidate, numba_backend.py:141-268), folds the
// reference's objective loop over it as it goes (BasicFold; thresholds and tables on the finished row)
// and applies the greedy select (numba_backend.py:270-290).  At D <= 8 a warp-per-protozoon pass
// leaves >= 24 of 32 lanes idle; one warp here carries 32 protozoa, which cuts the batch kernel's
// instruction count ~2.5x.  Each lane's D-step chain is serial, so this loses above D ~ 8 and for the
// CEC2022 functions (their quad-DMMA evaluation would serialise 4 passes per warp): measured in
// profiles/r02_batch_lpp.txt.  OUT_FIXUP by slot only.
constexpr int kLppMaxDim = 8;
#ifdef APO_BATCH_CLOCK
__device__ unsigned long long g_lpp_clk[4];
#define LPP_CLK(k)                                                                      \
    do {                                                                                \
        const long long now_ = clock64();                                               \
        if (threadIdx.x == 0) atomicAdd(&g_lpp_clk[k], (unsigned long long)(now_ - t_)); \
        t_ = now_;                                                                      \
    } while (0)
#else
#define LPP_CLK(k) \
    do {           \
    } while (0)
#endif
template <class Rows>
__device__ inline void update_group_lpp(const IterParams& P, const ObjDesc& O, const Rows& R, int i0, int n,
                                        const unsigned* in_dr_bits, const double* p_dr, double* out_rows,
                                        double* out_fit, const GroupScratch& g, int lane,
                                        unsigned long long& my_min, unsigned& my_warn) {
    const int dim = P.dim;
    const bool live = lane < n;
#ifdef APO_BATCH_CLOCK
    long long t_ = clock64();
#endif
    if (live) {
        const int r0 = i0 - 1 + lane;
        const bool dr = ((in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0;
        group_phase_a(P, R, i0 + lane, dr, dr ? p_dr[r0] : 0.0, g, lane);
    }
    LPP_CLK(0);
    bool ok = true;
    double nf = 0.0;
    int own_key = 0;
    double* dst = nullptr;
    const double* x = nullptr;
    if (live) {
        const int i = i0 + lane;
        const int op = g.op[lane];
        const int* sl = g.slot + 4 * lane;
        own_key = sl[0];
        x = R.at_key(own_key);
        const double* xj = R.at_key(sl[op == OP_AUTOTROPH ? 1 : 0]);
        const double* xm = R.at_key(sl[op >= OP_AUTOTROPH ? 2 : 0]);
        const double* xp = R.at_key(sl[op >= OP_AUTOTROPH ? 3 : 0]);
        dst = out_rows + (size_t)R.slot_of(own_key) * P.ld;
        Key base{};
        if (op != OP_AUTOTROPH) base = iteration_key(P, (uint64_t)i);
        const double f = g.f[lane], w0 = g.w[lane], sgn = g.sgn[lane];
        const unsigned* mb = g.bits + lane * g.words;
        const bool basic = O.code <= OBJ_GRIEWANK;
        BasicFold bf;
#pragma unroll 2
        for (int d = 0; d < dim; d++) {
            const double xd = x[d];
            const double m = ((mb[d >> 5] >> (d & 31)) & 1u) ? 1.0 : 0.0;
            double cv;
            if (op == OP_DORMANCY) {
                cv = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
            } else if (op == OP_REPRODUCTION) {
                const double off = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
                cv = xd + (f * off) * m;
            } else {
                double acc = 0.0;
                acc = acc + w0 * (xm[d] - xp[d]);
                const double ep = acc;
                double direction;
                if (op == OP_AUTOTROPH) {
                    direction = (xj[d] - xd) + ep;
                } else {
                    const double uv = uniform(base, kVectorBase + (uint64_t)d);
                    direction = ((1.0 + (sgn * uv) * P.decay) * xd - xd) + ep;
                }
                cv = xd + (f * direction) * m;
            }
            const double c = clampv(cv, P.lower, P.upper);
            ok = ok && isfinite(c);
            dst[d] = c;
            if (basic) bf.add(O.code, O.table, d, c);
        }
        if (basic) {
            nf = bf.value(O.code, dim);
        } else if (O.code == OBJ_OTSU_ML || O.code == OBJ_KAPUR_ML) {
            nf = threshold_ml(O.code, dst, dim, O.table);
        } else {  // OBJ_TABLE
            long long idx = (long long)floor(dst[0] + 0.5);
            if (idx < 0) idx = 0;
            if (idx > O.table_len - 1) idx = O.table_len - 1;
            nf = O.table[idx];
        }
    }
    LPP_CLK(1);
    if (live) {
        const int own = R.slot_of(own_key);
        const double fit_i = R.fit_at(own);
        double kept = fit_i;
        bool acc = false, warned = false;
        if (ok && isfinite(nf)) {
            acc = nf < fit_i;
            if (acc) kept = nf;
        } else {
            warned = true;
        }
        out_fit[own] = kept;
        if (!acc)
            for (int d = 0; d < dim; d++) dst[d] = x[d];
        const unsigned long long k = sort_key(kept);
        my_min = k < my_min ? k : my_min;
        my_warn += warned ? 1u : 0u;
    }
    __syncwarp();
    LPP_CLK(3);
}
#undef LPP_CLK

}  // namespace apo
