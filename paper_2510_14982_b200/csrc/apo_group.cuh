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
#include "apo_update.cuh"

namespace apo {

constexpr int kGroupMaxDim = 256;  // uint8 permutations

// Per-warp shared scratch of the group path.
struct GroupScratch {
    unsigned char* perm;  // [32][dp]
    unsigned* bits;       // [32][words]
    double* f;            // [32] forage factor (auto/hetero) or scale (repro)
    double* sgn;          // [32] heterotroph sign
    double* w;            // [32] pair-0 weight
    int* slot;            // [32][4] own, partner, km, kp slots
    int* op;              // [32]
    WarpScratch ws;       // cand/terms (+ pair cache for npairs > 1)
    int dp, words;
};

__host__ __device__ inline size_t group_scratch_bytes(int dim) {
    const size_t dp = (size_t)((dim + 3) & ~3);
    const size_t words = (size_t)(dim + 31) / 32;
    size_t b = 32 * dp + 32 * words * 4 + 32 * 8 * 3 + 32 * 4 * 4 + 32 * 4;
    b = (b + 15) & ~(size_t)15;
    return b + warp_scratch_bytes(dim);
}

__device__ inline GroupScratch group_scratch(unsigned char* base, int dim) {
    GroupScratch g;
    g.dp = (dim + 3) & ~3;
    g.words = (dim + 31) / 32;
    g.f = reinterpret_cast<double*>(base);
    g.sgn = g.f + 32;
    g.w = g.sgn + 32;
    g.slot = reinterpret_cast<int*>(g.w + 32);
    g.op = g.slot + 128;
    g.bits = reinterpret_cast<unsigned*>(g.op + 32);
    g.perm = reinterpret_cast<unsigned char*>(g.bits + 32 * g.words);
    size_t used = 32 * (size_t)g.dp + 32 * (size_t)g.words * 4 + 32 * 8 * 3 + 32 * 4 * 4 + 32 * 4;
    used = (used + 15) & ~(size_t)15;
    g.ws = warp_scratch(base + used, dim);
    return g;
}

struct DenseSlots {
    const double* pos;
    const double* fit;
    int ld;
    __device__ __forceinline__ int slot(int rank1) const { return rank1 - 1; }
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
    __device__ __forceinline__ const double* at(int slot) const { return pos + (size_t)slot * ld; }
    __device__ __forceinline__ double fit_at(int slot) const { return fit[slot]; }
    __device__ __forceinline__ const double* row(int rank1) const { return at(order[rank1 - 1]); }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[order[rank1 - 1]]; }
};

// Phase A for rank i (one lane).  Fills the lane's entries of g.
template <class Rows>
__device__ inline void group_phase_a(const IterParams& P, const Rows& R, int i, bool in_dr, double p_dr_i,
                                     const GroupScratch& g, int lane) {
    const int ps = P.ps, dim = P.dim;
    const uint64_t base = stream_base(P.seed, P.key_iteration, (uint64_t)i);
    const double u_dec = uniform(base, kSlotDecision);
    int op;
    if (in_dr) op = (u_dec < p_dr_i) ? OP_DORMANCY : OP_REPRODUCTION;
    else op = (u_dec < P.p_ah) ? OP_AUTOTROPH : OP_HETEROTROPH;
    int* sl = g.slot + 4 * lane;
    sl[0] = R.slot(i);
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
            sl[1] = R.slot(partner);
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
        const int skm = R.slot(km), skp = R.slot(kp);
        sl[2] = skm;
        sl[3] = skp;
        g.w[lane] = rank_weight(R.fit_at(skm), R.fit_at(skp), P.eps);
    }
    g.op[lane] = op;
    // mask: sequential partial Fisher-Yates on this lane's permutation
    // (numba_backend.py:74-90), then scatter the first `count` values.
    unsigned* bits = g.bits + (size_t)lane * g.words;
    for (int w = 0; w < g.words; w++) bits[w] = 0u;
    if (op != OP_DORMANCY && count > 0) {
        unsigned char* perm = g.perm + (size_t)lane * g.dp;
        for (int d = 0; d < dim; d++) perm[d] = (unsigned char)d;
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
__device__ inline void group_extra_pairs(const IterParams& P, const Rows& R, int i, int op, uint64_t base,
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
        g.ws.pk[2 * k] = R.slot(km);
        g.ws.pk[2 * k + 1] = R.slot(kp);
        g.ws.pw[k] = rank_weight(R.fitness(km), R.fitness(kp), P.eps);
    }
    __syncwarp();
}

// acc for pairs k >= 1 at dimension d (pair 0 is added by the caller first,
// so the accumulation order matches the reference: acc = 0; acc += w_k*(...)).
template <class Rows>
__device__ __forceinline__ double extra_pairs_acc(const IterParams& P, const Rows& R, int i, int op, uint64_t base,
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
            skm = R.slot(km);
            skp = R.slot(kp);
            w = rank_weight(R.fit_at(skm), R.fit_at(skp), P.eps);
        }
        acc = acc + w * (R.at(skm)[d] - R.at(skp)[d]);
    }
    return acc;
}

__device__ __forceinline__ double clampv(double c, double lo, double hi) {
    if (c < lo) c = lo;
    else if (c > hi) c = hi;
    return c;
}

// Phase B for member p (rank i) of the group: warp-cooperative.
// MAXC > 0: rows held in registers (dim <= 32*MAXC).  MAXC == 0: streaming.
template <int MAXC, class Rows>
__device__ inline UpdateResult group_phase_b(const IterParams& P, const ObjDesc& O, const Rows& R, int i, int p,
                                             double* out_rows, int out_ld, bool out_by_slot, const GroupScratch& g,
                                             int lane) {
    const int dim = P.dim;
    const int op = g.op[p];
    const int* sl = g.slot + 4 * p;
    const int own = sl[0];
    const double* x = R.at(own);
    const double fit_i = R.fit_at(own);
    const double f = g.f[p];
    const double w0 = g.w[p];
    const double sgn = g.sgn[p];
    const bool many = P.npairs > 1 && (op == OP_AUTOTROPH || op == OP_HETEROTROPH);
    uint64_t base = 0;
    if (op != OP_AUTOTROPH || many) base = stream_base(P.seed, P.key_iteration, (uint64_t)i);
    if (many) group_extra_pairs(P, R, i, op, base, g, lane);
    const double* xj = (op == OP_AUTOTROPH) ? R.at(sl[1]) : x;
    const double* xm = (op >= OP_AUTOTROPH) ? R.at(sl[2]) : x;
    const double* xp = (op >= OP_AUTOTROPH) ? R.at(sl[3]) : x;
    const double inv_np = (double)P.npairs;
    double* out_row = out_rows + (size_t)(out_by_slot ? own : i - 1) * out_ld;

    auto cand_at = [&](int d, double xd, double aj, double am, double ap) -> double {
        double c;
        if (op == OP_DORMANCY) {
            c = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
        } else if (op == OP_REPRODUCTION) {
            const double off = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
            c = xd + (f * off) * gmask(g, p, d);
        } else {
            double acc = 0.0;
            acc = acc + w0 * (am - ap);
            if (many) acc = extra_pairs_acc(P, R, i, op, base, g, acc, d);
            const double ep = P.npairs == 1 ? acc : acc / inv_np;
            double direction;
            if (op == OP_AUTOTROPH) {
                direction = (aj - xd) + ep;
            } else {
                const double uv = uniform(base, kVectorBase + (uint64_t)d);
                direction = ((1.0 + (sgn * uv) * P.decay) * xd - xd) + ep;
            }
            c = xd + (f * direction) * gmask(g, p, d);
        }
        return clampv(c, P.lower, P.upper);
    };

    UpdateResult res;
    res.accepted = false;
    res.warned = false;
    res.fitness = fit_i;
    bool ok = true;
    if constexpr (MAXC > 0) {
        double xv[MAXC], aj[MAXC], am[MAXC], ap[MAXC], cv[MAXC];
#pragma unroll
        for (int c = 0; c < MAXC; c++) {
            const int d = lane + 32 * c;
            if (d < dim) {
                xv[c] = x[d];
                if (op == OP_AUTOTROPH) aj[c] = xj[d];
                if (op >= OP_AUTOTROPH) {
                    am[c] = xm[d];
                    ap[c] = xp[d];
                }
            }
        }
#pragma unroll
        for (int c = 0; c < MAXC; c++) {
            const int d = lane + 32 * c;
            if (d < dim) {
                cv[c] = cand_at(d, xv[c], aj[c], am[c], ap[c]);
                ok = ok && isfinite(cv[c]);
                g.ws.cand[d] = cv[c];
            }
        }
        ok = __all_sync(kFull, ok);
        __syncwarp();
        if (ok) {
            const double nf = eval_warp(O, g.ws.cand, g.ws.terms, dim, lane);
            if (isfinite(nf)) {
                res.accepted = nf < fit_i;
                if (res.accepted) res.fitness = nf;
            } else {
                res.warned = true;
            }
        } else {
            res.warned = true;
        }
        if (res.accepted || out_row != x) {
#pragma unroll
            for (int c = 0; c < MAXC; c++) {
                const int d = lane + 32 * c;
                if (d < dim) out_row[d] = res.accepted ? cv[c] : xv[c];
            }
        }
    } else {
        for (int d = lane; d < dim; d += 32) {
            const double xd = x[d];
            const double c = cand_at(d, xd, op == OP_AUTOTROPH ? xj[d] : 0.0, op >= OP_AUTOTROPH ? xm[d] : 0.0,
                                     op >= OP_AUTOTROPH ? xp[d] : 0.0);
            ok = ok && isfinite(c);
            g.ws.cand[d] = c;
        }
        ok = __all_sync(kFull, ok);
        __syncwarp();
        if (ok) {
            const double nf = eval_warp(O, g.ws.cand, g.ws.terms, dim, lane);
            if (isfinite(nf)) {
                res.accepted = nf < fit_i;
                if (res.accepted) res.fitness = nf;
            } else {
                res.warned = true;
            }
        } else {
            res.warned = true;
        }
        if (res.accepted) {
            for (int d = lane; d < dim; d += 32) out_row[d] = g.ws.cand[d];
        } else if (out_row != x) {
            for (int d = lane; d < dim; d += 32) out_row[d] = x[d];
        }
    }
    __syncwarp();
    return res;
}

// One group of up to 32 ranks [i0, i0+n) on one warp.  in_dr via bits or
// bytes; results: fitness written to out_fit (by slot or rank), optional
// acc/warn bytes by rank; returns (min sort key, warned count) via refs.
template <int MAXC, class Rows>
__device__ inline void update_group(const IterParams& P, const ObjDesc& O, const Rows& R, int i0, int n,
                                    const uint8_t* in_dr_bytes, const unsigned* in_dr_bits, const double* p_dr,
                                    double* out_rows, double* out_fit, bool out_by_slot, uint8_t* out_acc,
                                    uint8_t* out_warn, const GroupScratch& g, int lane,
                                    unsigned long long& my_min, unsigned& my_warn) {
    if (lane < n) {
        const int r0 = i0 - 1 + lane;
        const bool dr = in_dr_bits ? ((in_dr_bits[r0 >> 5] >> (r0 & 31)) & 1u) != 0 : in_dr_bytes[r0] != 0;
        group_phase_a(P, R, i0 + lane, dr, dr ? p_dr[r0] : 0.0, g, lane);
    }
    __syncwarp();
    for (int p = 0; p < n; p++) {
        const int i = i0 + p;
        const UpdateResult res =
            group_phase_b<MAXC>(P, O, R, i, p, out_rows, P.ld, out_by_slot, g, lane);
        if (lane == 0) {
            out_fit[out_by_slot ? g.slot[4 * p] : i - 1] = res.fitness;
            if (out_acc) out_acc[i - 1] = res.accepted ? 1 : 0;
            if (out_warn) out_warn[i - 1] = res.warned ? 1 : 0;
            const unsigned long long k = sort_key(res.fitness);
            my_min = k < my_min ? k : my_min;
            my_warn += res.warned ? 1u : 0u;
        }
    }
    __syncwarp();
}

}  // namespace apo
