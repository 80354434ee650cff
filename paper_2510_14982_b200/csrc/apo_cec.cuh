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
__device__ __forceinline__ double schwefel_t(double zi, int n) {
    if (zi > 500.0) {
        const double m = fmod(zi, 500.0);
        const double t = (zi - 500.0) / 100.0;
        return -(500.0 - m) * sin(sqrt(500.0 - m)) + t * t / n;
    }
    if (zi < -500.0) {
        const double m = fmod(fabs(zi), 500.0);
        const double t = (zi + 500.0) / 100.0;
        return -(-500.0 + m) * sin(sqrt(500.0 - m)) + t * t / n;
    }
    return -zi * sin(sqrt(fabs(zi)));
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
            const double t1 = z[i] * z[i] - z[i + 1], t2 = z[i] - 1.0;
            a += 100.0 * t1 * t1 + t2 * t2;
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
        if (b == B_HGBAT) return pow(fabs(a * a - c * c), 0.5) + (0.5 * a + c) / n + 0.5;
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
            pr *= cos(z[i] / sqrt(1.0 + i));
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
    int fn;                // 1..12
    const double* shift;   // [ncomp][n]
    const double* rot_t;   // [ncomp][n][n]
    const int* shuffle;    // [n] (1-based)
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

}  // namespace apo
