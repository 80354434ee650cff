// apo_cec.cuh -- CEC2022 F1-F12, one candidate per warp.
//
// Same definitions as the CPU restatement oracle/cec_oracle.c (parity
// UNPINNED: the reference package has no CEC2022 functions, SPEC.md:146,
// and the official code/data are unavailable offline; data are synthesised
// by cec2022.py).  Per candidate c (shared memory):
//   single:       z = M (scale * (c - o)) + offset, basic(z)
//   hybrid:       z = M (c - o), shuffled, split into segments, each segment
//                 scaled/offset and fed to its basic function, summed
//   composition:  per component k: z_k = [M_k] (scale_k (c - o_k)) + offset,
//                 fit_k = lam_k basic_k(z_k) + bias_k, combined with the
//                 cf_cal weights w_k = exp(-|c-o_k|^2/(2 D sigma_k^2))/|c-o_k|
// Rotations use transposed matrices (rot_t[k][i][j] = M_k[j][i]) so lane j's
// loads of row i are coalesced.  Reductions are warp trees (deterministic;
// agree with the oracle's sequential sums to ~1e-15 relative).
#pragma once
#include "apo_device.cuh"

namespace apo {

constexpr int OBJ_CEC_BASE = 100;  // code = 100 + F (1..12)

enum CecBasic : int {
    B_ZAKHAROV = 0, B_ROSENBROCK, B_ESCAFFER6, B_RASTRIGIN, B_STEP_RASTRIGIN, B_LEVY, B_BENT_CIGAR, B_DISCUS,
    B_ELLIPS, B_HGBAT, B_HAPPYCAT, B_KATSUURA, B_ACKLEY, B_SCHWEFEL, B_SCHAFFER_F7, B_GRIE_ROSEN, B_GRIEWANK
};

struct CecSpec {
    int kind;  // 0 single, 1 hybrid, 2 composition
    int ncomp;
    int basic[6];
    double p[6];
    int rflag[6];
    double lam[6];
    double sigma[6];
    double bias[6];
    double fstar;
};

__constant__ CecSpec kCecSpec[12] = {
    {0, 1, {B_ZAKHAROV}, {1}, {1}, {1}, {0}, {0}, 300.0},
    {0, 1, {B_ROSENBROCK}, {1}, {1}, {1}, {0}, {0}, 400.0},
    {0, 1, {B_ESCAFFER6}, {1}, {1}, {1}, {0}, {0}, 600.0},
    {0, 1, {B_STEP_RASTRIGIN}, {1}, {1}, {1}, {0}, {0}, 800.0},
    {0, 1, {B_LEVY}, {1}, {1}, {1}, {0}, {0}, 900.0},
    {1, 3, {B_BENT_CIGAR, B_HGBAT, B_RASTRIGIN}, {0.4, 0.4, 0.2}, {0}, {0}, {0}, {0}, 1800.0},
    {1, 6, {B_HGBAT, B_KATSUURA, B_ACKLEY, B_RASTRIGIN, B_SCHWEFEL, B_SCHAFFER_F7}, {0.1, 0.2, 0.2, 0.2, 0.1, 0.2},
     {0}, {0}, {0}, {0}, 2000.0},
    {1, 5, {B_KATSUURA, B_HAPPYCAT, B_GRIE_ROSEN, B_SCHWEFEL, B_ACKLEY}, {0.3, 0.2, 0.2, 0.1, 0.2}, {0}, {0}, {0},
     {0}, 2200.0},
    {2, 5, {B_ROSENBROCK, B_ELLIPS, B_BENT_CIGAR, B_DISCUS, B_ELLIPS}, {0}, {1, 0, 1, 1, 0},
     {1.0, 1e-6, 1e-26, 1e-6, 1e-6}, {10, 20, 30, 40, 50}, {0, 200, 300, 100, 400}, 2300.0},
    {2, 3, {B_SCHWEFEL, B_RASTRIGIN, B_HGBAT}, {0}, {0, 1, 0}, {1, 1, 1}, {20, 10, 10}, {0, 200, 100}, 2400.0},
    {2, 5, {B_ESCAFFER6, B_SCHWEFEL, B_GRIEWANK, B_ROSENBROCK, B_RASTRIGIN}, {0}, {1, 1, 1, 1, 1},
     {5e-4, 1, 10, 1, 10}, {20, 20, 30, 30, 20}, {0, 200, 300, 400, 200}, 2600.0},
    {2, 6, {B_HGBAT, B_RASTRIGIN, B_SCHWEFEL, B_BENT_CIGAR, B_ELLIPS, B_ESCAFFER6}, {0}, {1, 1, 1, 1, 1, 1},
     {10, 10, 2.5, 1e-26, 1e-6, 5e-4}, {10, 20, 30, 40, 50, 60}, {0, 300, 500, 100, 400, 200}, 2700.0},
};

constexpr double kPi = 3.1415926535897932384626433832795029;
constexpr double kE = 2.7182818284590452353602874713526625;

__device__ __forceinline__ double wsum(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}
__device__ __forceinline__ double wprod(double v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v *= __shfl_xor_sync(0xFFFFFFFFu, v, o);
    return v;
}

__device__ __forceinline__ double cec_scale(int b) {
    switch (b) {
    case B_ROSENBROCK: return 2.048 / 100.0;
    case B_RASTRIGIN:
    case B_STEP_RASTRIGIN: return 5.12 / 100.0;
    case B_HGBAT:
    case B_HAPPYCAT:
    case B_KATSUURA:
    case B_GRIE_ROSEN: return 5.0 / 100.0;
    case B_SCHWEFEL: return 1000.0 / 100.0;
    case B_GRIEWANK: return 600.0 / 100.0;
    default: return 1.0;
    }
}
__device__ __forceinline__ double cec_offset(int b) {
    switch (b) {
    case B_ROSENBROCK:
    case B_GRIE_ROSEN: return 1.0;
    case B_HGBAT:
    case B_HAPPYCAT: return -1.0;
    default: return 0.0;
    }
}

__device__ __forceinline__ double schaffer_g(double a, double b) {
    const double r2 = a * a + b * b;
    double t1 = sin(sqrt(r2));
    t1 = t1 * t1;
    const double t2 = 1.0 + 0.001 * r2;
    return 0.5 + (t1 - 0.5) / (t2 * t2);
}
__device__ __forceinline__ double grie_rosen_t(double a, double b) {
    const double t1 = a * a - b, t2 = a - 1.0;
    const double t = 100.0 * t1 * t1 + t2 * t2;
    return t * t / 4000.0 - cos(t) + 1.0;
}
// fmod(a, 500) for a >= 0, exactly, without a division: k = floor(a * 0.002) is the
// quotient or one off; a - k*500 is exact (Sterbenz: a and k*500 are within a factor
// of two, or k = 0) and the one-off cases are corrected by +/- 500 -- again exact,
// because the corrected value a - 500*floor(a/500) is representable.
__device__ __forceinline__ double fmod500(double a) {
    double m = a - floor(a * 0.002) * 500.0;
    if (m < 0.0) m += 500.0;
    else if (m >= 500.0) m -= 500.0;
    return m;
}

// sin(x) for 0 <= x <= 64 (the Schwefel argument sqrt(s) <= 22.4): x = k pi + r with
// pi in two parts, |r| <= pi/2, odd Taylor polynomial to degree 21 in FMAs.  Max abs
// error 2.2e-16 on [0, 24] against libm (checked on 2e4 points); larger x falls back.
__device__ __forceinline__ double sin_small(double x) {
    if (!(x <= 64.0)) return sin(x);
    const double k = rint(x * 0.31830988618379067154);
    const double r = fma(-k, 1.2246467991473532e-16, fma(-k, 3.141592653589793116, x));
    const double r2 = r * r;
    double p = 1.9572941063391263e-20;  // 1/21!
    p = fma(p, r2, -8.2206352466243295e-18);
    p = fma(p, r2, 2.8114572543455206e-15);
    p = fma(p, r2, -7.6471637318198164e-13);
    p = fma(p, r2, 1.6059043836821613e-10);
    p = fma(p, r2, -2.5052108385441720e-08);
    p = fma(p, r2, 2.7557319223985893e-06);
    p = fma(p, r2, -1.9841269841269841e-04);
    p = fma(p, r2, 8.3333333333333332e-03);
    p = fma(p, r2, -1.6666666666666666e-01);
    const double v = fma(r * r2, p, r);
    return ((long long)k & 1) ? -v : v;
}

// Schwefel term (CEC2022 schwefel_func), branch-free: with a = |z|,
//   |z| <= 500:  -z sin(sqrt|z|)
//   z  >  500:  -(500-m) sin(sqrt(500-m)) + ((z-500)/100)^2/n,  m = fmod(z, 500)
//   z  < -500:  -(-500+m) sin(sqrt(500-m)) + ((z+500)/100)^2/n, m = fmod(|z|, 500)
// are all -sign(z) s sin(sqrt s) (+ penalty) with s = a or 500 - m -- the same
// roundings as the three-way form (oracle/cec_oracle.c), without divergence.
__device__ __forceinline__ double schwefel_t(double zi, int n) {
    const double a = fabs(zi);
    const bool out = a > 500.0;
    const double s = out ? 500.0 - fmod500(a) : a;
    const double v = s * sin_small(sqrt(s));
    const double t = (zi > 0.0 ? zi - 500.0 : zi + 500.0) / 100.0;
    return (zi > 0.0 ? -v : v) + (out ? t * t / n : 0.0);
}

// Basic function b over z[0..n) (shared memory, already scaled + offset).
// Every lane returns the value.
__device__ inline double cec_basic_warp(int b, const double* z, int n, int lane) {
    double a = 0.0, c = 0.0;
    switch (b) {
    case B_ZAKHAROV:
        for (int i = lane; i < n; i += 32) {
            a += z[i] * z[i];
            c += 0.5 * (i + 1) * z[i];
        }
        a = wsum(a);
        c = wsum(c);
        return a + c * c + c * c * c * c;
    case B_ROSENBROCK:
        for (int i = lane; i < n - 1; i += 32) {
            const double t1 = z[i + 1] - z[i] * z[i], t2 = z[i] - 1.0;  // objectives.py:129-132
            a += 100.0 * (t1 * t1) + t2 * t2;
        }
        return wsum(a);
    case B_ESCAFFER6:
        for (int i = lane; i < n; i += 32) a += schaffer_g(z[i], z[i + 1 < n ? i + 1 : 0]);
        return wsum(a);
    case B_RASTRIGIN:
    case B_STEP_RASTRIGIN:
        for (int i = lane; i < n; i += 32) a += z[i] * z[i] - 10.0 * cos(2.0 * kPi * z[i]) + 10.0;
        return wsum(a);
    case B_LEVY: {
        for (int i = lane; i < n - 1; i += 32) {
            const double wi = 1.0 + z[i] / 4.0;
            const double s = sin(kPi * wi + 1.0);
            a += (wi - 1.0) * (wi - 1.0) * (1.0 + 10.0 * s * s);
        }
        a = wsum(a);
        const double w0 = 1.0 + z[0] / 4.0, wn = 1.0 + z[n - 1] / 4.0;
        const double s0 = sin(kPi * w0), sn = sin(2.0 * kPi * wn);
        return s0 * s0 + a + (wn - 1.0) * (wn - 1.0) * (1.0 + sn * sn);
    }
    case B_BENT_CIGAR:
        for (int i = lane; i < n; i += 32)
            if (i >= 1) a += z[i] * z[i];
        return z[0] * z[0] + 1e6 * wsum(a);
    case B_DISCUS:
        for (int i = lane; i < n; i += 32)
            if (i >= 1) a += z[i] * z[i];
        return 1e6 * z[0] * z[0] + wsum(a);
    case B_ELLIPS:
        for (int i = lane; i < n; i += 32) a += pow(10.0, 6.0 * i / (n > 1 ? n - 1 : 1)) * z[i] * z[i];
        return wsum(a);
    case B_HGBAT:
    case B_HAPPYCAT: {
        for (int i = lane; i < n; i += 32) {
            a += z[i] * z[i];
            c += z[i];
        }
        a = wsum(a);
        c = wsum(c);
        if (b == B_HGBAT) return sqrt(fabs(a * a - c * c)) + (0.5 * a + c) / n + 0.5;  // objectives.py:123-126
        return pow(fabs(a - n), 0.25) + (0.5 * a + c) / n + 0.5;
    }
    case B_KATSUURA: {
        const double t3 = pow((double)n, 1.2);
        double pr = 1.0;
        for (int i = lane; i < n; i += 32) {
            double t = 0.0;
            for (int j = 1; j <= 32; j++) {
                const double t1 = ldexp(1.0, j);
                const double t2 = t1 * z[i];
                t += fabs(t2 - floor(t2 + 0.5)) / t1;
            }
            pr *= pow(1.0 + (i + 1) * t, 10.0 / t3);
        }
        pr = wprod(pr);
        const double t1 = 10.0 / n / n;
        return pr * t1 - t1;
    }
    case B_ACKLEY: {
        for (int i = lane; i < n; i += 32) {
            a += z[i] * z[i];
            c += cos(2.0 * kPi * z[i]);
        }
        a = wsum(a);
        c = wsum(c);
        return kE - 20.0 * exp(-0.2 * sqrt(a / n)) - exp(c / n) + 20.0;
    }
    case B_SCHWEFEL:
        for (int i = lane; i < n; i += 32) a += schwefel_t(z[i] + 4.209687462275036e+002, n);
        return wsum(a) + 4.189828872724338e+002 * n;
    case B_SCHAFFER_F7: {
        for (int i = lane; i < n - 1; i += 32) {
            const double zi = sqrt(z[i] * z[i] + z[i + 1] * z[i + 1]);
            const double t = sin(50.0 * pow(zi, 0.2));
            a += sqrt(zi) + sqrt(zi) * t * t;
        }
        a = wsum(a);
        return n > 1 ? a * a / (n - 1) / (n - 1) : a * a;
    }
    case B_GRIE_ROSEN:
        for (int i = lane; i < n; i += 32) a += grie_rosen_t(z[i], z[i + 1 < n ? i + 1 : 0]);
        return wsum(a);
    default: {  // B_GRIEWANK
        double pr = 1.0;
        for (int i = lane; i < n; i += 32) {
            a += z[i] * z[i];
            pr *= cos_glibc(z[i] / sqrt(1.0 + i));  // the reference's griewank block (libm cos)
        }
        return 1.0 + wsum(a) / 4000.0 - wprod(pr);
    }
    }
}

// z[j] = sum_i rot_t[i][j] * y[i] + off (lane j); y, z shared.
__device__ __forceinline__ void cec_rotate(const double* __restrict__ rot_t, const double* y, double* z, int n,
                                           double off, int lane) {
    for (int j0 = 0; j0 < n; j0 += 32) {
        const int j = j0 + lane;
        double acc = 0.0;
        if (j < n) {
#pragma unroll 4
            for (int i = 0; i < n; i++) acc = fma(__ldg(rot_t + (size_t)i * n + j), y[i], acc);
            z[j] = acc + off;
        }
    }
}

struct CecData {
    int fn;                 // 1..12
    const double* shift;    // [ncomp][n]
    const double* rot_t;    // [ncomp][n][n]
    const int* shuffle;     // [n] (1-based)
    const double* rot_pad;  // [ncomp][n4][8 NT] zero-padded rot_t (k_cec_eval), nullable
    const double* rot_gemm;  // [Kp][Np] zero-padded rot_t of the rotated component (D > 104 GEMM path), nullable
};

// F_fn(c) for a candidate c[0..n) in shared memory; y, z: shared scratch [n].
__device__ inline double cec_eval_warp(const CecData& C, const double* c, double* y, double* z, int n, int lane) {
    const CecSpec& S = kCecSpec[C.fn - 1];
    double f = 0.0;
    if (S.kind == 0) {
        const int b = S.basic[0];
        const double sc = cec_scale(b);
        for (int i = lane; i < n; i += 32) {
            double xi = c[i];
            const double oi = C.shift[i];
            if (b == B_STEP_RASTRIGIN && fabs(xi - oi) > 0.5) xi = oi + floor(2.0 * (xi - oi) + 0.5) / 2.0;
            y[i] = (xi - oi) * sc;
        }
        __syncwarp();
        cec_rotate(C.rot_t, y, z, n, cec_offset(b), lane);
        __syncwarp();
        f = cec_basic_warp(b, z, n, lane);
    } else if (S.kind == 1) {
        for (int i = lane; i < n; i += 32) y[i] = c[i] - C.shift[i];
        __syncwarp();
        cec_rotate(C.rot_t, y, z, n, 0.0, lane);
        __syncwarp();
        // shuffle, then scale/offset each segment for its basic function
        int start = 0;
        int sizes[6];
        int tot = 0;
        for (int k = 0; k < S.ncomp - 1; k++) {
            sizes[k] = (int)ceil(S.p[k] * n);
            if (sizes[k] > n - tot) sizes[k] = n - tot;  // oracle: or_cec_segments
            tot += sizes[k];
        }
        sizes[S.ncomp - 1] = n - tot;
        for (int k = 0; k < S.ncomp; k++) {
            const int b = S.basic[k];
            const double sc = cec_scale(b), off = cec_offset(b);
            for (int i = lane; i < sizes[k]; i += 32) y[start + i] = z[C.shuffle[start + i] - 1] * sc + off;
            start += sizes[k];
        }
        __syncwarp();
        start = 0;
        for (int k = 0; k < S.ncomp; k++) {
            if (sizes[k] > 0) f += cec_basic_warp(S.basic[k], y + start, sizes[k], lane);
            start += sizes[k];
        }
    } else {
        double fit[6], w[6], wmax = 0.0, wsum_ = 0.0;
        int inf_at = -1;
        for (int k = 0; k < S.ncomp; k++) {
            const int b = S.basic[k];
            const double sc = cec_scale(b), off = cec_offset(b);
            const double* o = C.shift + (size_t)k * n;
            double d2 = 0.0;
            for (int i = lane; i < n; i += 32) {
                const double dv = c[i] - o[i];
                d2 += dv * dv;
                y[i] = dv * sc;
                if (!S.rflag[k]) z[i] = dv * sc + off;
            }
            d2 = wsum(d2);
            __syncwarp();
            if (S.rflag[k]) cec_rotate(C.rot_t + (size_t)k * n * n, y, z, n, off, lane);
            __syncwarp();
            fit[k] = S.lam[k] * cec_basic_warp(b, z, n, lane) + S.bias[k];
            __syncwarp();
            w[k] = d2 != 0.0 ? sqrt(1.0 / d2) * exp(-d2 / 2.0 / n / (S.sigma[k] * S.sigma[k]))
                             : __longlong_as_double(0x7ff0000000000000LL);
            if (d2 == 0.0 && inf_at < 0) inf_at = k;
            if (w[k] > wmax) wmax = w[k];
        }
        if (inf_at >= 0) {
            f = fit[inf_at];
        } else if (wmax == 0.0) {
            for (int k = 0; k < S.ncomp; k++) f += fit[k] / S.ncomp;
        } else {
            for (int k = 0; k < S.ncomp; k++) wsum_ += w[k];
            for (int k = 0; k < S.ncomp; k++) f += w[k] / wsum_ * fit[k];
        }
    }
    __syncwarp();
    return f + S.fstar;
}


// ---------------------------------------------------------------------------
// Batched evaluation: up to 8 candidates per warp, the rotation as one
// [8 x n] x [n x n] contraction.
//
// DMMA path (n >= APO_CEC_DMMA_MIN_DIM): mma.sync m8n8k4 f64 on the tensor
// cores.  A = Y (8 candidates x 4 input dims, shared memory), B = M^T
// (4 input dims x 8 output dims, read through L1 from the transposed
// rotation rot_t), C = Z (8 x 8).  Fragment layout (PTX ISA, m8n8k4 .f64):
// lane = 4 g + t holds A[g][t], B[t][g] and C[g][2t], C[g][2t+1].  Two
// n-tiles are in flight per k-step so consecutive mma's are independent.
// FMA path (small n): lane j of the warp owns output dim j for all 8 rows,
// so each loaded matrix element feeds 8 FMAs.
#ifndef APO_CEC_DMMA_MIN_DIM
#define APO_CEC_DMMA_MIN_DIM 16
#endif

__device__ __forceinline__ void dmma_m8n8k4(double& c0, double& c1, double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
                 : "+d"(c0), "+d"(c1)
                 : "d"(a), "d"(b));
}

// Z[q][j] = sum_i rot_t[i][j] * Y[q][i] + off, q < 8 (rows are independent:
// rows past the batch hold stale but harmless values).
__device__ inline void cec_rotate8(const double* __restrict__ rot_t, const double* Y, double* Z, int ys, int n,
                                   double off, int lane, bool dmma = true) {
    if (dmma && n >= APO_CEC_DMMA_MIN_DIM) {
        const int g = lane >> 2, t = lane & 3;
        const double* yrow = Y + (size_t)g * ys;
        for (int j0 = 0; j0 < n; j0 += 16) {
            const int ja = j0 + g, jb = j0 + 8 + g;
            const bool va = ja < n, vb = jb < n;
            double c0 = 0.0, c1 = 0.0, c2 = 0.0, c3 = 0.0;
#pragma unroll 2
            for (int i0 = 0; i0 < n; i0 += 4) {
                const int i = i0 + t;
                const bool vi = i < n;
                const double a = vi ? yrow[i] : 0.0;
                const double* brow = rot_t + (size_t)i * n;
                const double b0 = (vi && va) ? __ldg(brow + ja) : 0.0;
                const double b1 = (vi && vb) ? __ldg(brow + jb) : 0.0;
                dmma_m8n8k4(c0, c1, a, b0);
                dmma_m8n8k4(c2, c3, a, b1);
            }
            double* zrow = Z + (size_t)g * ys;
            const int ca = j0 + 2 * t, cb = j0 + 8 + 2 * t;
            if (ca < n) zrow[ca] = c0 + off;
            if (ca + 1 < n) zrow[ca + 1] = c1 + off;
            if (cb < n) zrow[cb] = c2 + off;
            if (cb + 1 < n) zrow[cb + 1] = c3 + off;
        }
    } else {
        for (int j = lane; j < n; j += 32) {
            double acc[8];
#pragma unroll
            for (int q = 0; q < 8; q++) acc[q] = 0.0;
            for (int i = 0; i < n; i++) {
                const double m = __ldg(rot_t + (size_t)i * n + j);
#pragma unroll
                for (int q = 0; q < 8; q++) acc[q] = fma(m, Y[(size_t)q * ys + i], acc[q]);
            }
#pragma unroll
            for (int q = 0; q < 8; q++) Z[(size_t)q * ys + j] = acc[q] + off;
        }
    }
}

// F_fn for candidates X[q][0..n), q < nb (stride xs).  Z, W: scratch rows of
// the same shape (W only for compositions).  X is overwritten.  Returns the
// fitness of candidate q on lane q.
__device__ inline double cec_eval_batch(const CecData& C, double* X, double* Z, double* W, int xs, int nb, int n,
                                        int lane) {
    const CecSpec& S = kCecSpec[C.fn - 1];
    const bool dmma = C.rot_pad != nullptr;  // objectives built without DMMA tables: FMA rotation
    double mine = 0.0;
    if (S.kind == 0) {
        const int b = S.basic[0];
        const double sc = cec_scale(b);
        for (int q = 0; q < nb; q++) {
            double* x = X + (size_t)q * xs;
            for (int i = lane; i < n; i += 32) {
                double xi = x[i];
                const double oi = C.shift[i];
                if (b == B_STEP_RASTRIGIN && fabs(xi - oi) > 0.5) xi = oi + floor(2.0 * (xi - oi) + 0.5) / 2.0;
                x[i] = (xi - oi) * sc;
            }
        }
        __syncwarp();
        cec_rotate8(C.rot_t, X, Z, xs, n, cec_offset(b), lane, dmma);
        __syncwarp();
        for (int q = 0; q < nb; q++) {
            const double v = cec_basic_warp(b, Z + (size_t)q * xs, n, lane);
            if (lane == q) mine = v;
        }
    } else if (S.kind == 1) {
        for (int q = 0; q < nb; q++) {
            double* x = X + (size_t)q * xs;
            for (int i = lane; i < n; i += 32) x[i] = x[i] - C.shift[i];
        }
        __syncwarp();
        cec_rotate8(C.rot_t, X, Z, xs, n, 0.0, lane, dmma);
        __syncwarp();
        int sizes[6];
        int tot = 0;
        for (int k = 0; k < S.ncomp - 1; k++) {
            sizes[k] = (int)ceil(S.p[k] * n);
            if (sizes[k] > n - tot) sizes[k] = n - tot;  // oracle: or_cec_segments
            tot += sizes[k];
        }
        sizes[S.ncomp - 1] = n - tot;
        for (int q = 0; q < nb; q++) {
            const double* z = Z + (size_t)q * xs;
            double* y = X + (size_t)q * xs;
            int start = 0;
            for (int k = 0; k < S.ncomp; k++) {
                const double sc = cec_scale(S.basic[k]), off = cec_offset(S.basic[k]);
                for (int i = lane; i < sizes[k]; i += 32) y[start + i] = z[C.shuffle[start + i] - 1] * sc + off;
                start += sizes[k];
            }
        }
        __syncwarp();
        for (int q = 0; q < nb; q++) {
            const double* y = X + (size_t)q * xs;
            double f = 0.0;
            int start = 0;
            for (int k = 0; k < S.ncomp; k++) {
                if (sizes[k] > 0) f += cec_basic_warp(S.basic[k], y + start, sizes[k], lane);
                start += sizes[k];
            }
            if (lane == q) mine = f;
        }
    } else {
        double fit[6], w[6];
        int inf_at = -1;
        for (int k = 0; k < S.ncomp; k++) {
            const int b = S.basic[k];
            const double sc = cec_scale(b), off = cec_offset(b);
            const double* o = C.shift + (size_t)k * n;
            double d2_mine = 0.0;
            for (int q = 0; q < nb; q++) {
                const double* x = X + (size_t)q * xs;
                double* y = W + (size_t)q * xs;
                double* z = Z + (size_t)q * xs;
                double d2 = 0.0;
                for (int i = lane; i < n; i += 32) {
                    const double dv = x[i] - o[i];
                    d2 += dv * dv;
                    y[i] = dv * sc;
                    if (!S.rflag[k]) z[i] = dv * sc + off;
                }
                d2 = wsum(d2);
                if (lane == q) d2_mine = d2;
            }
            __syncwarp();
            if (S.rflag[k]) cec_rotate8(C.rot_t + (size_t)k * n * n, W, Z, xs, n, off, lane, dmma);
            __syncwarp();
            double fk = 0.0;
            for (int q = 0; q < nb; q++) {
                const double v = S.lam[k] * cec_basic_warp(b, Z + (size_t)q * xs, n, lane) + S.bias[k];
                if (lane == q) fk = v;
            }
            __syncwarp();
            fit[k] = fk;
            w[k] = d2_mine != 0.0 ? sqrt(1.0 / d2_mine) * exp(-d2_mine / 2.0 / n / (S.sigma[k] * S.sigma[k]))
                                  : __longlong_as_double(0x7ff0000000000000LL);
            if (d2_mine == 0.0 && inf_at < 0) inf_at = k;
        }
        // combination (lane q holds candidate q's components)
        double wmax = 0.0, wsum_ = 0.0, f = 0.0;
        for (int k = 0; k < S.ncomp; k++)
            if (w[k] > wmax) wmax = w[k];
        if (inf_at >= 0) {
            f = fit[inf_at];
        } else if (wmax == 0.0) {
            for (int k = 0; k < S.ncomp; k++) f += fit[k] / S.ncomp;
        } else {
            for (int k = 0; k < S.ncomp; k++) wsum_ += w[k];
            for (int k = 0; k < S.ncomp; k++) f += w[k] / wsum_ * fit[k];
        }
        mine = f;
    }
    __syncwarp();
    return mine + S.fstar;
}


// ---------------------------------------------------------------------------
// k_cec_eval's evaluator: 8 candidates per warp, one QUAD of lanes per
// candidate (lane = 4 q + t).  This is the DMMA m8n8k4 fragment layout (A
// row g = lane/4, column t = lane%4), so the same quad that owns row q of the
// rotation input also evaluates candidate q: elements i = t, t+4, ... and two
// shuffles reduce a quad.  Rows are zero-padded to n4 = round_up(n, 4) and
// the rotation reads a zero-padded copy of M^T (rot_pad: [n4][8 NT] per
// component), so the inner loop carries no bounds checks.
__device__ __forceinline__ double qsum(double v) {
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    v += __shfl_xor_sync(0xFFFFFFFFu, v, 2);
    return v;
}
__device__ __forceinline__ double qprod(double v) {
    v *= __shfl_xor_sync(0xFFFFFFFFu, v, 1);
    v *= __shfl_xor_sync(0xFFFFFFFFu, v, 2);
    return v;
}

// Y[q][:] <- M Y[q][:] + off for the 8 rows of the warp, in place: all
// output tiles accumulate in registers (n <= 8 NT), A from shared memory,
// B through L1 from rot_pad.
template <int NT>
__device__ __forceinline__ void cec_rotate_quad(const double* __restrict__ rot_pad, double* Y, int ys, int n,
                                                double off, int lane, int bs = 8 * NT) {
    // B: rot_pad in global memory (row stride 8 NT, read through L1) or a shared-memory copy with
    // row stride bs = 8 NT + 4 (conflict-free: bs % 16 is 4 or 12)
    const int g = lane >> 2, t = lane & 3;
    const int n4 = (n + 3) & ~3;
    double acc[NT][2];
#pragma unroll
    for (int k = 0; k < NT; k++) acc[k][0] = acc[k][1] = 0.0;
    double* yrow = Y + (size_t)g * ys;
    const double* bp = rot_pad + (size_t)t * bs + g;
#pragma unroll 2
    for (int i0 = 0; i0 < n4; i0 += 4) {
        const double a = yrow[i0 + t];
        double b[NT];
#pragma unroll
        for (int k = 0; k < NT; k++) b[k] = bp[8 * k];
#pragma unroll
        for (int k = 0; k < NT; k++) dmma_m8n8k4(acc[k][0], acc[k][1], a, b[k]);
        bp += 4 * bs;
    }
    __syncwarp();
#pragma unroll
    for (int k = 0; k < NT; k++) {
        const int c = 8 * k + 2 * t;
        if (c < n) yrow[c] = acc[k][0] + off;
        if (c + 1 < n) yrow[c + 1] = acc[k][1] + off;
    }
    __syncwarp();
}

// Rotation by component k's matrix: the shared-memory copy when the CTA staged this component, else
// rot_pad through L1.  Two call sites on purpose: a pointer selected between the two would be generic
// and turn every B-fragment load into a generic LD instead of LDS.
template <int NT>
__device__ __forceinline__ void cec_rotate_comp(const CecData& C, const double* bsm, bool staged, int k, double* Y,
                                                int ys, int n, double off, int lane) {
    if (staged) {
        cec_rotate_quad<NT>(bsm, Y, ys, n, off, lane, 8 * NT + 4);
    } else {
        const int n4 = (n + 3) & ~3;
        cec_rotate_quad<NT>(C.rot_pad + (size_t)k * n4 * (8 * NT), Y, ys, n, off, lane, 8 * NT);
    }
}

// Basic function b over z[0..n) by the 4 lanes of a quad; every lane of the
// quad returns the value.  ew: host-computed ELLIPS weights (nullable).
// Z(i): element i of the basic function's input (a stored row, or an affine map of the candidate
// computed on the fly -- unrotated composition components need no scratch pass).
template <class Zf>
__device__ inline double cec_basic_quad_t(int b, const Zf& Z, int n, int t, const double* ew) {
    double a = 0.0, c = 0.0;
    switch (b) {
    case B_ZAKHAROV:
        for (int i = t; i < n; i += 4) {
            a += Z(i) * Z(i);
            c += 0.5 * (i + 1) * Z(i);
        }
        a = qsum(a);
        c = qsum(c);
        return a + c * c + c * c * c * c;
    case B_ROSENBROCK:
        for (int i = t; i < n - 1; i += 4) {
            const double t1 = Z(i + 1) - Z(i) * Z(i), t2 = Z(i) - 1.0;  // objectives.py:129-132
            a += 100.0 * (t1 * t1) + t2 * t2;
        }
        return qsum(a);
    case B_ESCAFFER6:
        for (int i = t; i < n; i += 4) a += schaffer_g(Z(i), Z(i + 1 < n ? i + 1 : 0));
        return qsum(a);
    case B_RASTRIGIN:
    case B_STEP_RASTRIGIN:
        for (int i = t; i < n; i += 4) a += Z(i) * Z(i) - 10.0 * cospi(2.0 * Z(i)) + 10.0;
        return qsum(a);
    case B_LEVY: {
        for (int i = t; i < n - 1; i += 4) {
            const double wi = 1.0 + Z(i) / 4.0;
            const double s = sin(kPi * wi + 1.0);
            a += (wi - 1.0) * (wi - 1.0) * (1.0 + 10.0 * s * s);
        }
        a = qsum(a);
        const double w0 = 1.0 + Z(0) / 4.0, wn = 1.0 + Z(n - 1) / 4.0;
        const double s0 = sin(kPi * w0), sn = sin(2.0 * kPi * wn);
        return s0 * s0 + a + (wn - 1.0) * (wn - 1.0) * (1.0 + sn * sn);
    }
    case B_BENT_CIGAR:
        for (int i = t; i < n; i += 4)
            if (i >= 1) a += Z(i) * Z(i);
        return Z(0) * Z(0) + 1e6 * qsum(a);
    case B_DISCUS:
        for (int i = t; i < n; i += 4)
            if (i >= 1) a += Z(i) * Z(i);
        return 1e6 * Z(0) * Z(0) + qsum(a);
    case B_ELLIPS:
        for (int i = t; i < n; i += 4)
            a += (ew ? ew[i] : pow(10.0, 6.0 * i / (n > 1 ? n - 1 : 1))) * Z(i) * Z(i);
        return qsum(a);
    case B_HGBAT:
    case B_HAPPYCAT: {
        for (int i = t; i < n; i += 4) {
            a += Z(i) * Z(i);
            c += Z(i);
        }
        a = qsum(a);
        c = qsum(c);
        if (b == B_HGBAT) return sqrt(fabs(a * a - c * c)) + (0.5 * a + c) / n + 0.5;
        return pow(fabs(a - n), 0.25) + (0.5 * a + c) / n + 0.5;
    }
    case B_KATSUURA: {
        const double t3 = pow((double)n, 1.2);
        double pr = 1.0;
        for (int i = t; i < n; i += 4) {
            double s = 0.0;
            double t1 = 1.0, inv = 1.0;
#pragma unroll 8
            for (int j = 1; j <= 32; j++) {
                t1 *= 2.0;  // 2^j and 2^-j are exact
                inv *= 0.5;
                const double t2 = t1 * Z(i);
                s += fabs(t2 - floor(t2 + 0.5)) * inv;
            }
            pr *= pow(1.0 + (i + 1) * s, 10.0 / t3);
        }
        pr = qprod(pr);
        const double t1 = 10.0 / n / n;
        return pr * t1 - t1;
    }
    case B_ACKLEY: {
        for (int i = t; i < n; i += 4) {
            a += Z(i) * Z(i);
            c += cospi(2.0 * Z(i));
        }
        a = qsum(a);
        c = qsum(c);
        return kE - 20.0 * exp(-0.2 * sqrt(a / n)) - exp(c / n) + 20.0;
    }
    case B_SCHWEFEL:
        for (int i = t; i < n; i += 4) a += schwefel_t(Z(i) + 4.209687462275036e+002, n);
        return qsum(a) + 4.189828872724338e+002 * n;
    case B_SCHAFFER_F7: {
        for (int i = t; i < n - 1; i += 4) {
            const double zi = sqrt(Z(i) * Z(i) + Z(i + 1) * Z(i + 1));
            const double s = sin(50.0 * pow(zi, 0.2));
            a += sqrt(zi) + sqrt(zi) * s * s;
        }
        a = qsum(a);
        return n > 1 ? a * a / (n - 1) / (n - 1) : a * a;
    }
    case B_GRIE_ROSEN:
        for (int i = t; i < n; i += 4) a += grie_rosen_t(Z(i), Z(i + 1 < n ? i + 1 : 0));
        return qsum(a);
    default: {  // B_GRIEWANK
        double pr = 1.0;
        for (int i = t; i < n; i += 4) {
            a += Z(i) * Z(i);
            pr *= cos_glibc(Z(i) / sqrt(1.0 + i));  // the reference's griewank block (libm cos)
        }
        return 1.0 + qsum(a) / 4000.0 - qprod(pr);
    }
    }
}

__device__ __forceinline__ double cec_basic_quad(int b, const double* z, int n, int t, const double* ew) {
    return cec_basic_quad_t(b, [z](int i) { return z[i]; }, n, t, ew);
}

// F_fn of the warp's 8 rows X[q] (stride xs, zero-padded to n4); W: second
// row buffer (hybrids, compositions).  X is overwritten except for
// compositions.  Every lane of quad q returns candidate q's fitness.
// DIRECT_UNROT: compositions evaluate unrotated components straight from the candidate (k_cec_eval);
// false keeps the register-lean one-component-at-a-time loop (the 3-CTA/SM batch kernel).
template <int NT, bool DIRECT_UNROT = true>
__device__ inline double cec_eval_quad(const CecData& C, double* X, const double* src, int xs, int n, int lane,
                                       const double* ew, const double* bsm = nullptr, int bsm_comp = 0) {
    // bsm: shared-memory copy (row stride 8 NT + 4) of rotation `bsm_comp`, the others via L1.
    // src: this quad's candidate row in global memory (nullptr for a dead row): compositions
    // re-read it for every component instead of keeping a second copy in shared memory.
    const bool staged0 = bsm && bsm_comp == 0;
    const CecSpec& S = kCecSpec[C.fn - 1];
    const int q = lane >> 2, t = lane & 3;
    const int n4 = (n + 3) & ~3;
    double* x = X + (size_t)q * xs;
    double f = 0.0;
    if (S.kind == 0) {
        const int b = S.basic[0];
        const double sc = cec_scale(b);
        for (int i = t; i < n; i += 4) {
            double xi = x[i];
            const double oi = C.shift[i];
            if (b == B_STEP_RASTRIGIN && fabs(xi - oi) > 0.5) xi = oi + floor(2.0 * (xi - oi) + 0.5) / 2.0;
            x[i] = (xi - oi) * sc;
        }
        __syncwarp();
        cec_rotate_comp<NT>(C, bsm, staged0, 0, X, xs, n, cec_offset(b), lane);
        f = cec_basic_quad(b, x, n, t, ew);
    } else if (S.kind == 1) {
        // rot_pad's output columns are pre-permuted by the shuffle (objectives.py), so the rotation
        // leaves z[shuffle[j]-1] in column j: the segments are contiguous, no gather
        for (int i = t; i < n; i += 4) x[i] = x[i] - C.shift[i];
        __syncwarp();
        cec_rotate_comp<NT>(C, bsm, staged0, 0, X, xs, n, 0.0, lane);
        int sizes[6];
        int tot = 0;
        for (int k = 0; k < S.ncomp - 1; k++) {
            sizes[k] = (int)ceil(S.p[k] * n);
            if (sizes[k] > n - tot) sizes[k] = n - tot;  // oracle: or_cec_segments
            tot += sizes[k];
        }
        sizes[S.ncomp - 1] = n - tot;
        int start = 0;
        for (int k = 0; k < S.ncomp; k++) {
            const double sc = cec_scale(S.basic[k]), off = cec_offset(S.basic[k]);
            const int end = start + sizes[k];
            for (int i = start + ((t - start) & 3); i < end; i += 4) x[i] = x[i] * sc + off;
            start = end;
        }
        __syncwarp();
        start = 0;
        for (int k = 0; k < S.ncomp; k++) {
            if (sizes[k] > 0) f += cec_basic_quad(S.basic[k], x + start, sizes[k], t, ew);
            start += sizes[k];
        }
    } else {
        double fit[6], wk[6];
        int inf_at = -1;
        if constexpr (DIRECT_UNROT) {
            unsigned zero_d2 = 0;
            bool x_intact = true;  // X still holds the candidate (a rotation overwrites it)
            // unrotated components first, evaluated straight from the candidate through an on-the-fly
            // affine map; rotated ones after (transform + DMMA rotation in place, re-reading the
            // candidate from L2 when an earlier rotation consumed it)
            for (int pass = 0; pass < 2; pass++) {
                for (int k = 0; k < S.ncomp; k++) {
                    const bool rot = S.rflag[k] != 0;
                    if (rot != (pass == 1)) continue;
                    const int b = S.basic[k];
                    const double sc = cec_scale(b), off = cec_offset(b);
                    const double* o = C.shift + (size_t)k * n;
                    double d2 = 0.0;
                    if (!rot) {
                        for (int i = t; i < n; i += 4) {
                            const double dv = x[i] - o[i];
                            d2 += dv * dv;
                        }
                        d2 = qsum(d2);
                        fit[k] = S.lam[k] * cec_basic_quad_t(b, [x, o, sc, off](int i) { return (x[i] - o[i]) * sc + off; },
                                                             n, t, ew) + S.bias[k];
                    } else {
                        if (!x_intact) {
                            for (int i = t; i < n; i += 4) x[i] = src ? src[i] : 0.0;
                            __syncwarp();
                        }
                        for (int i = t; i < n; i += 4) {
                            const double dv = x[i] - o[i];
                            d2 += dv * dv;
                            x[i] = dv * sc;
                        }
                        d2 = qsum(d2);
                        __syncwarp();
                        cec_rotate_comp<NT>(C, bsm, bsm && bsm_comp == k, k, X, xs, n, off, lane);
                        fit[k] = S.lam[k] * cec_basic_quad(b, x, n, t, ew) + S.bias[k];
                        x_intact = false;
                    }
                    __syncwarp();
                    wk[k] = d2 != 0.0 ? sqrt(1.0 / d2) * exp(-d2 / 2.0 / n / (S.sigma[k] * S.sigma[k]))
                                      : __longlong_as_double(0x7ff0000000000000LL);
                    if (d2 == 0.0) zero_d2 |= 1u << k;
                }
            }
            if (zero_d2) inf_at = __ffs(zero_d2) - 1;  // the first such component, as the oracle scans them
        } else {  // one component at a time, re-reading the candidate (register-lean: batch kernel)
            for (int k = 0; k < S.ncomp; k++) {
                const int b = S.basic[k];
                const double sc = cec_scale(b), off = cec_offset(b);
                const double* o = C.shift + (size_t)k * n;
                const bool rot = S.rflag[k] != 0;
                if (k > 0) {  // the candidate again (L2-resident: k_cec_eval just streamed it in)
                    for (int i = t; i < n; i += 4) x[i] = src ? src[i] : 0.0;
                    __syncwarp();
                }
                double d2 = 0.0;
                for (int i = t; i < n; i += 4) {
                    const double dv = x[i] - o[i];
                    d2 += dv * dv;
                    x[i] = rot ? dv * sc : dv * sc + off;
                }
                d2 = qsum(d2);
                __syncwarp();
                if (rot) {
                    cec_rotate_comp<NT>(C, bsm, bsm && bsm_comp == k, k, X, xs, n, off, lane);
                }
                fit[k] = S.lam[k] * cec_basic_quad(b, x, n, t, ew) + S.bias[k];
                __syncwarp();
                wk[k] = d2 != 0.0 ? sqrt(1.0 / d2) * exp(-d2 / 2.0 / n / (S.sigma[k] * S.sigma[k]))
                                  : __longlong_as_double(0x7ff0000000000000LL);
                if (d2 == 0.0 && inf_at < 0) inf_at = k;
            }
        }
        double wmax = 0.0, wsum_ = 0.0;
        for (int k = 0; k < S.ncomp; k++)
            if (wk[k] > wmax) wmax = wk[k];
        if (inf_at >= 0) {
            f = fit[inf_at];
        } else if (wmax == 0.0) {
            for (int k = 0; k < S.ncomp; k++) f += fit[k] / S.ncomp;
        } else {
            for (int k = 0; k < S.ncomp; k++) wsum_ += wk[k];
            for (int k = 0; k < S.ncomp; k++) f += wk[k] / wsum_ * fit[k];
        }
    }
    __syncwarp();
    return f + S.fstar;
}

}  // namespace apo
