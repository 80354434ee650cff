// apo_update.cuh -- the fused per-protozoon APO update, one protozoon per warp.
//
// Reference: numba_backend.py:141-290 (_update_row), core.py:286-501.  One
// warp owns one protozoon (rank i, 1-based):
//   decide (slot 0) -> op-specific scalar draws -> mask (partial Fisher-Yates,
//   resolved warp-parallel, see build_mask) -> candidate row, lanes over
//   dimensions -> clamp + finiteness vote -> fitness (eval_warp) -> greedy
//   select -> write the kept row + fitness.
// Every floating-point expression keeps the reference's evaluation order and
// rounding (no contraction; the TU is built with --fmad=false), so oracle
// mode reproduces the reference bit for bit (griewank's cos excepted, see
// DESIGN.md).
#pragma once
#include "apo_device.cuh"
#include "apo_objective.cuh"

namespace apo {

constexpr unsigned kFull = 0xFFFFFFFFu;
constexpr int kMaxCachedPairs = 8;

enum Op : int { OP_DORMANCY = 0, OP_REPRODUCTION = 1, OP_AUTOTROPH = 2, OP_HETEROTROPH = 3 };

// Scalars of one iteration: numba_backend.py:358-366.
struct IterParams {
    uint64_t seed;
    uint64_t key_iteration;
    int ps;
    int dim;
    int npairs;
    int ld;  // row stride (doubles) of the source/target population
    double lower, upper, span, eps;
    double p_ah, f_mult, decay;
    int rng;  // RngMode: RNG_KEYED (reference fmix64, oracle mode) or RNG_PHILOX (production)
    // keyed mode: the (seed, iteration) part of every protozoon's stream base, mix64(mix64(H0^seed)^it)
    // (rng.py:79-99), hashed once per iteration instead of once per protozoon and call (set_iteration_base)
    uint64_t base_it;
    int has_base_it;
};

__host__ __device__ __forceinline__ void set_iteration_base(IterParams& P) {
    P.base_it = mix64(mix64(kH0 ^ P.seed) ^ P.key_iteration);
    P.has_base_it = 1;
}

// stream_key(P.rng, P.seed, P.key_iteration, individual), with the per-iteration hash reused
__host__ __device__ __forceinline__ Key iteration_key(const IterParams& P, uint64_t individual) {
    if (P.rng == RNG_KEYED && P.has_base_it) {
        Key k;
        k.mode = RNG_KEYED;
        k.a = mix64(P.base_it ^ individual);
        k.b = k.c = 0;
        return k;
    }
    return stream_key(P.rng, P.seed, P.key_iteration, individual);
}

// Per-warp shared-memory scratch (carved by warp_scratch()).
struct WarpScratch {
    double* cand;    // [dim] candidate, then the kept row
    double* terms;   // [dim] per-dimension fitness terms
    double* aux;     // [dim] second scratch row (CEC rotation output)
    int* head;       // [dim] latest mask step that hit a position
    int* prev;       // [dim] previous step hitting the same position
    int* rj;         // [dim] swap targets r_j of the partial Fisher-Yates
    unsigned* bits;  // [ceil(dim/32)] mask bitmap
    int* pk;         // [2*kMaxCachedPairs] (km, kp) per pair
    double* pw;      // [kMaxCachedPairs] pair weights
};

__host__ __device__ inline size_t warp_scratch_bytes(int dim) {
    const size_t d2 = (size_t)((dim + 1) & ~1);
    size_t words = (size_t)(dim + 31) / 32;
    size_t b = 24 * d2 + 12 * (size_t)dim + 4 * words + 8 * kMaxCachedPairs + 8 * kMaxCachedPairs;
    return (b + 15) & ~(size_t)15;
}

// cand and terms start 16-byte aligned (eval_warp reads them as double2).
__device__ inline WarpScratch warp_scratch(unsigned char* base, int dim) {
    WarpScratch s;
    const int d2 = (dim + 1) & ~1;
    s.cand = reinterpret_cast<double*>(base);
    s.terms = s.cand + d2;
    s.aux = s.terms + d2;
    s.pw = s.aux + d2;
    s.head = reinterpret_cast<int*>(s.pw + kMaxCachedPairs);
    s.prev = s.head + dim;
    s.rj = s.prev + dim;
    s.pk = s.rj + dim;
    s.bits = reinterpret_cast<unsigned*>(s.pk + 2 * kMaxCachedPairs);
    return s;
}

// ---------------------------------------------------------------------------
// Mask of `count` ones chosen by a partial Fisher-Yates over 1..n on counters
// ctr0.. (numba_backend.py:74-90, rng.py:137-156), resolved without the
// sequential swap chain:
//   step j swaps positions j and r_j = j + floor(u_j (n-j)) (r_j >= j), so the
//   value finally in slot j is the value position r_j held just before step j.
//   That value came from the latest earlier step j' with r_j' == r_j (it moved
//   there from slot j', which holds what it held before step j'), recursively;
//   with no earlier hit it is the untouched identity value.
// Steps are inserted 32 at a time; __match_any_sync orders same-target steps
// inside a round, so prev[j] is exactly "latest j' < j with r_j' == r_j".
// Result: bit p of s.bits set <=> value p+1 is among the first `count` slots,
// which is exactly mask[perm[j]-1] = 1 in the reference.
// If `sel` is non-null the selected 0-based values are also written there in
// slot order (the coordinator's Dr list needs them; the mask does not).
__device__ inline void build_mask(int n, int count, const Key& base, uint64_t ctr0, const WarpScratch& s, int lane) {
    const int words = (n + 31) >> 5;
    for (int p = lane; p < n; p += 32) s.head[p] = -1;
    for (int w = lane; w < words; w += 32) s.bits[w] = 0u;
    __syncwarp();
    for (int j0 = 0; j0 < count; j0 += 32) {
        const int j = j0 + lane;
        const bool act = j < count;
        int r = n + lane;  // unique dummy key for idle lanes
        if (act) {
            double u = uniform(base, ctr0 + (uint64_t)j);
            r = j + (int)(u * (double)(n - j));
            if (r > n - 1) r = n - 1;
            s.rj[j] = r;
        }
        const unsigned peers = __match_any_sync(kFull, r);
        int pj = -1;
        if (act) {
            const unsigned lower = peers & ((1u << lane) - 1u);
            pj = lower ? j0 + (31 - __clz(lower)) : s.head[r];
        }
        __syncwarp();
        if (act) {
            s.prev[j] = pj;
            const unsigned higher = lane == 31 ? 0u : (peers >> (lane + 1));
            if (higher == 0u) s.head[r] = j;
        }
        __syncwarp();
    }
    for (int j = lane; j < count; j += 32) {
        int p = s.rj[j], t = j;
        for (;;) {
            int q = s.head[p];
            while (q >= t) q = s.prev[q];
            if (q < 0) break;
            p = q;
            t = q;
        }
        atomicOr(&s.bits[p >> 5], 1u << (p & 31));
    }
    __syncwarp();
}

__device__ __forceinline__ double mask_at(const WarpScratch& s, int d) {
    return ((s.bits[d >> 5] >> (d & 31)) & 1u) ? 1.0 : 0.0;
}

// ---------------------------------------------------------------------------
// Row / fitness accessors: rank-ordered dense rows (the run_updates boundary)
// or slot-resident rows addressed through the rank->slot order (device loop).
struct DenseRows {
    const double* pos;
    const double* fit;
    int ld;
    __device__ __forceinline__ const double* row(int rank1) const { return pos + (size_t)(rank1 - 1) * ld; }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[rank1 - 1]; }
};

struct OrderedRows {
    const double* pos;
    const double* fit;
    const int* order;  // rank (0-based) -> slot
    int ld;
    __device__ __forceinline__ const double* row(int rank1) const {
        return pos + (size_t)order[rank1 - 1] * ld;
    }
    __device__ __forceinline__ double fitness(int rank1) const { return fit[order[rank1 - 1]]; }
};

struct UpdateResult {
    double fitness;  // kept fitness
    bool accepted;
    bool warned;
};

// One protozoon, one warp.  `out_row` receives the kept row.  All lanes of
// the warp must call this with identical arguments.
// cand_only: write the clamped candidate to out_row and return its finiteness
// in `accepted` (the fitness, greedy select and best-so-far run later: the
// CEC2022 large-D GEMM path, apo_gemm.cuh).
template <class Rows>
__device__ inline UpdateResult update_protozoon(const IterParams& P, const ObjDesc& O, const Rows& R, int i,
                                                bool in_dr, double p_dr_i, double* out_row, const WarpScratch& s,
                                                int lane, bool cand_only = false) {
    const int ps = P.ps, dim = P.dim;
    const double* x = R.row(i);
    const double fit_i = R.fitness(i);
    const Key base = iteration_key(P, (uint64_t)i);
    const double u_dec = uniform(base, kSlotDecision);

    int op;
    if (in_dr) op = (u_dec < p_dr_i) ? OP_DORMANCY : OP_REPRODUCTION;
    else op = (u_dec < P.p_ah) ? OP_AUTOTROPH : OP_HETEROTROPH;

    double sgn = 1.0, scale = 0.0, f = 0.0;
    int partner = i;
    const int npairs = P.npairs;
    if (op == OP_REPRODUCTION) {
        sgn = uniform(base, kSlotSign) < 0.5 ? 1.0 : -1.0;
        const double mag = uniform(base, kSlotMagnitude);
        const double usize = uniform(base, kSlotMaskSize);
        const int count = (int)ceil((double)dim * usize);
        build_mask(dim, count, base, kMaskBase, s, lane);
        scale = sgn * mag;
    } else if (op != OP_DORMANCY) {
        if (op == OP_AUTOTROPH) {
            if (ps > 1) {
                const double up = uniform(base, kSlotPartner);
                int j0 = (int)(up * (double)(ps - 1));
                if (j0 > ps - 2) j0 = ps - 2;
                if (j0 >= i - 1) j0 += 1;
                partner = j0 + 1;
            }
        } else {
            sgn = uniform(base, kSlotSign) < 0.5 ? 1.0 : -1.0;
        }
        f = uniform(base, kSlotForage) * P.f_mult;
        const int count = (int)ceil((double)((long long)dim * i) / (double)ps);
        build_mask(dim, count, base, kMaskBase, s, lane);
        // neighbour pairs + weights (core.py:359-410), cached for the chunk loop
        if (lane < kMaxCachedPairs && lane < npairs) {
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
            s.pk[2 * k] = km;
            s.pk[2 * k + 1] = kp;
            s.pw[k] = rank_weight(R.fitness(km), R.fitness(kp), P.eps);
        }
        __syncwarp();
    }

    // candidate, lanes over dimensions
    const double* xj = R.row(partner);
    bool ok = true;
    for (int d = lane; d < dim; d += 32) {
        const double xd = x[d];
        double c;
        if (op == OP_DORMANCY) {
            c = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
        } else if (op == OP_REPRODUCTION) {
            const double off = P.lower + uniform(base, kVectorBase + (uint64_t)d) * P.span;
            c = xd + (scale * off) * mask_at(s, d);
        } else {
            double acc = 0.0;
            for (int k = 0; k < npairs; k++) {
                int km, kp;
                double w;
                if (k < kMaxCachedPairs) {
                    km = s.pk[2 * k];
                    kp = s.pk[2 * k + 1];
                    w = s.pw[k];
                } else if (op == OP_AUTOTROPH) {
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
                    w = rank_weight(R.fitness(km), R.fitness(kp), P.eps);
                } else {
                    km = i - (k + 1);
                    if (km < 1) km = 1;
                    kp = i + (k + 1);
                    if (kp > ps) kp = ps;
                    w = rank_weight(R.fitness(km), R.fitness(kp), P.eps);
                }
                acc = acc + w * (R.row(km)[d] - R.row(kp)[d]);
            }
            const double ep = acc / (double)npairs;
            double direction;
            if (op == OP_AUTOTROPH) {
                direction = (xj[d] - xd) + ep;
            } else {
                const double uv = uniform(base, kVectorBase + (uint64_t)d);
                const double near_x = (1.0 + (sgn * uv) * P.decay) * xd;
                direction = (near_x - xd) + ep;
            }
            c = xd + (f * direction) * mask_at(s, d);
        }
        // clamp (numba_backend.py:259-268): NaN passes through, +-inf clamps
        if (c < P.lower) c = P.lower;
        else if (c > P.upper) c = P.upper;
        ok = ok && isfinite(c);
        s.cand[d] = c;
    }
    ok = __all_sync(kFull, ok);
    __syncwarp();

    UpdateResult res;
    res.accepted = false;
    res.warned = false;
    res.fitness = fit_i;
    if (cand_only) {
        for (int d = lane; d < dim; d += 32) out_row[d] = s.cand[d];
        res.accepted = ok;
        __syncwarp();
        return res;
    }
    if (ok) {
        const double nf = eval_warp(O, s.cand, s.terms, dim, lane, s.aux);
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
        for (int d = lane; d < dim; d += 32) out_row[d] = s.cand[d];
    } else if (out_row != x) {
        for (int d = lane; d < dim; d += 32) out_row[d] = x[d];
    }
    __syncwarp();
    return res;
}

}  // namespace apo
