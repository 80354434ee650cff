// apo_objective.cuh -- fitness evaluation, one candidate per warp.
//
// Basic functions: numba_backend.py:93-138 (== objectives.py:105-152).  The
// reference accumulates strictly left to right; in oracle mode lanes compute
// the per-dimension terms in parallel (each term is rounded exactly as in
// the reference) and lane 0 then accumulates them in order, so the sum is
// bit-identical.  Table lookup: objectives.py:213-219.
#pragma once
#include "apo_cec.cuh"
#include "apo_device.cuh"

namespace apo {

enum ObjCode : int {
    OBJ_SPHERE = 0,
    OBJ_BENT_CIGAR = 1,
    OBJ_ELLIPTIC = 2,
    OBJ_HGBAT = 3,
    OBJ_ROSENBROCK = 4,
    OBJ_GRIEWANK = 5,
    OBJ_TABLE = 6,
    OBJ_OTSU_ML = 7,   // multilevel Otsu over the prefix tables (apo_threshold_tables)
    OBJ_KAPUR_ML = 8,  // multilevel Kapur
};

constexpr int kThresholdTabLen = 515;
constexpr int kThresholdMaxK = 32;

// Objective descriptor; all pointers are device pointers.
struct ObjDesc {
    int code;
    int table_len;
    const double* table;  // elliptic weights (code 2) or value table (code 6)
    CecData cec;          // CEC2022 data (code OBJ_CEC_BASE + F)
    int flags;            // APO_OBJ_FMA_SMALL_D (include/apo_b200.h)
};

__device__ __forceinline__ double warp_bcast(double v, int src) { return __shfl_sync(0xFFFFFFFFu, v, src); }

// s = 0.0; for d in [from, to): s += t[d]  -- strictly left to right, with
// 16-byte shared loads (t must be 16-byte aligned).
__device__ __forceinline__ double seq_sum(const double* t, int from, int to) {
    double s = 0.0;
    int d = from;
    if ((d & 1) && d < to) s += t[d++];
#pragma unroll 4
    for (; d + 1 < to; d += 2) {
        const double2 v = *reinterpret_cast<const double2*>(t + d);
        s += v.x;
        s += v.y;
    }
    if (d < to) s += t[d];
    return s;
}

// Multilevel thresholding objective of k = dim thresholds x (one lane).
// Thresholds t_j = clamp(round_half_up(x_j), 0, 255) sorted ascending;
// classes [0,t_0], [t_0+1,t_1], ..., [t_{k-1}+1, 255]; empty classes add 0.
// tab: [N | C[0..256] | S[0..256]] with C = prefix counts and S = prefix
// v*count (Otsu) or prefix p ln p (Kapur).  Same expression order as
// oracle/threshold_oracle.c.  f = -(between-class variance) or -(entropy).
__host__ __device__ inline double threshold_ml(int code, const double* x, int k, const double* tab) {
    int t[kThresholdMaxK];
    for (int j = 0; j < k; j++) {
        const double r = floor(x[j] + 0.5);
        int v = !(r >= 0.0) ? 0 : r > 255.0 ? 255 : (int)r;
        int i = j;
        while (i > 0 && t[i - 1] > v) {
            t[i] = t[i - 1];
            i--;
        }
        t[i] = v;
    }
    const double N = tab[0];
    const double* C = tab + 1;
    const double* S = tab + 258;
    const double mu_t = S[256] / N;
    double f = 0.0;
    int lo = 0;
    for (int c = 0; c <= k; c++) {
        const int hi = c < k ? t[c] : 255;
        if (hi >= lo) {
            const double nc = C[hi + 1] - C[lo];
            if (nc > 0.0) {
                const double w = nc / N;
                if (code == OBJ_OTSU_ML) {
                    const double d = (S[hi + 1] - S[lo]) / nc - mu_t;
                    f += w * (d * d);
                } else {
                    f += log(w) - (S[hi + 1] - S[lo]) / w;
                }
            }
        }
        lo = hi + 1;
    }
    return -f;
}

// c: candidate [dim] (shared), t / aux: scratch [dim] (shared).  Returns the
// fitness on every lane.
__device__ inline double eval_warp(const ObjDesc& O, const double* c, double* t, int dim, int lane,
                                   double* aux = nullptr) {
    double f = 0.0;
    if (O.code >= OBJ_CEC_BASE) return cec_eval_warp(O.cec, c, t, aux, dim, lane);
    switch (O.code) {
    case OBJ_SPHERE:
        for (int d = lane; d < dim; d += 32) t[d] = c[d] * c[d];
        __syncwarp();
        if (lane == 0) f = seq_sum(t, 0, dim);
        break;
    case OBJ_BENT_CIGAR:
        for (int d = lane; d < dim; d += 32) t[d] = c[d] * c[d];
        __syncwarp();
        if (lane == 0) f = t[0] + 1e6 * seq_sum(t, 1, dim);
        break;
    case OBJ_ELLIPTIC:
        for (int d = lane; d < dim; d += 32) t[d] = (O.table[d] * c[d]) * c[d];
        __syncwarp();
        if (lane == 0) f = seq_sum(t, 0, dim);
        break;
    case OBJ_HGBAT:
        for (int d = lane; d < dim; d += 32) t[d] = c[d] * c[d];
        __syncwarp();
        if (lane == 0) {
            const double s1 = seq_sum(c, 0, dim);
            const double s2 = seq_sum(t, 0, dim);
            f = sqrt(fabs(s2 * s2 - s1 * s1)) + (0.5 * s2 + s1) / (double)dim + 0.5;
        }
        break;
    case OBJ_ROSENBROCK:
        for (int d = lane; d < dim - 1; d += 32) {
            const double a = c[d + 1] - c[d] * c[d];
            const double b = c[d] - 1.0;
            t[d] = 100.0 * (a * a) + b * b;
        }
        __syncwarp();
        if (lane == 0) f = seq_sum(t, 0, dim - 1);
        break;
    case OBJ_GRIEWANK:
        // glibc's cos (cos_glibc, apo_device.cuh): bit for bit with numba_backend.py:130
        for (int d = lane; d < dim; d += 32) t[d] = cos_glibc(c[d] / sqrt((double)d + 1.0));
        __syncwarp();
        if (lane == 0) {
            double s = 0.0, p = 1.0;
            for (int d = 0; d < dim; d++) {
                s += c[d] * c[d];
                p *= t[d];
            }
            f = 1.0 + s / 4000.0 - p;
        }
        break;
    case OBJ_OTSU_ML:
    case OBJ_KAPUR_ML:
        if (lane == 0) f = threshold_ml(O.code, c, dim, O.table);
        break;
    default: {  // OBJ_TABLE: table[round_half_up(x0)], clamped
        if (lane == 0) {
            long long idx = (long long)floor(c[0] + 0.5);
            if (idx < 0) idx = 0;
            if (idx > O.table_len - 1) idx = O.table_len - 1;
            f = O.table[idx];
        }
        break;
    }
    }
    f = warp_bcast(f, 0);
    __syncwarp();
    return f;
}

}  // namespace apo
