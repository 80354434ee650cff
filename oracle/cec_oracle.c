/*
 * cec_oracle.c -- CPU restatement of the CEC2022 F1-F12 benchmark suite.
 *
 * TEST INFRASTRUCTURE ONLY (see apo_oracle.c).  PARITY UNPINNED: the
 * reference package has no CEC2022 functions (non-goal) and the
 * official C code (cec22_test_func.cpp) and data files are not available
 * offline.  These definitions restate the CEC2017/2022 technical-report
 * conventions: sr_func (shift, scale, rotate), basic functions, hybrid
 * functions (shuffle + segment), composition functions (cf_cal weighting).
 * The shift/rotation/shuffle data are synthesised deterministically by
 * paper_2510_14982_b200/cec2022.py; this file only consumes them.
 *
 * Data layout (all row-major doubles):
 *   shift    [ncomp][D]
 *   rot      [ncomp][D][D]   z_i = sum_j rot[k][i][j] * y_j
 *   shuffle  [D]             1-based permutation (hybrids)
 * The CUDA evaluator (csrc/apo_cec.cuh) follows the same definitions;
 * tests/test_cec.py compares the two within 1e-9 relative.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define CEC_PI 3.1415926535897932384626433832795029
#define CEC_E 2.7182818284590452353602874713526625

/* y = scale * (x - o) (s) ; z = M y (r) */
static void sr_func(const double *x, double *z, int nx, const double *o, const double *M, double sh_rate, int s_flag,
                    int r_flag, double *tmp) {
    for (int i = 0; i < nx; i++) tmp[i] = (s_flag ? x[i] - o[i] : x[i]) * sh_rate;
    if (r_flag) {
        for (int i = 0; i < nx; i++) {
            double acc = 0.0;
            for (int j = 0; j < nx; j++) acc += M[(size_t)i * nx + j] * tmp[j];
            z[i] = acc;
        }
    } else {
        memcpy(z, tmp, sizeof(double) * (size_t)nx);
    }
}

/* Basic functions on an already shifted/scaled/rotated vector z (length n). */
double cec_zakharov(const double *z, int n) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < n; i++) {
        s1 += z[i] * z[i];
        s2 += 0.5 * (i + 1) * z[i];
    }
    return s1 + s2 * s2 + s2 * s2 * s2 * s2;
}

/* The five basic functions the reference also has are written in ITS rounding order
 * (objectives.py:112-142, numba_backend.py:93-131) so they are pinned to the reference's golden
 * values (tests/test_cec_pinning.py): rosenbrock as 100 (a a) + b b with a = z[i+1] - z[i]^2,
 * hgbat with sqrt, elliptic as (w z) z, griewank's product over cos(z / sqrt(i + 1)). */
double cec_rosenbrock(const double *z, int n) { /* z already +1 (objectives.py:129-132) */
    double f = 0.0;
    for (int i = 0; i < n - 1; i++) {
        double a = z[i + 1] - z[i] * z[i];
        double b = z[i] - 1.0;
        f += 100.0 * (a * a) + b * b;
    }
    return f;
}

static double schaffer_g(double a, double b) {
    double r2 = a * a + b * b;
    double t1 = sin(sqrt(r2));
    t1 = t1 * t1;
    double t2 = 1.0 + 0.001 * r2;
    return 0.5 + (t1 - 0.5) / (t2 * t2);
}

double cec_escaffer6(const double *z, int n) {
    double f = 0.0;
    for (int i = 0; i < n - 1; i++) f += schaffer_g(z[i], z[i + 1]);
    f += schaffer_g(z[n - 1], z[0]);
    return f;
}

double cec_rastrigin(const double *z, int n) {
    double f = 0.0;
    for (int i = 0; i < n; i++) f += z[i] * z[i] - 10.0 * cos(2.0 * CEC_PI * z[i]) + 10.0;
    return f;
}

double cec_levy(const double *z, int n) {
    double w0 = 1.0 + z[0] / 4.0, wn = 1.0 + z[n - 1] / 4.0;
    double s0 = sin(CEC_PI * w0);
    double sn = sin(2.0 * CEC_PI * wn);
    double f = s0 * s0 + (wn - 1.0) * (wn - 1.0) * (1.0 + sn * sn);
    for (int i = 0; i < n - 1; i++) {
        double wi = 1.0 + z[i] / 4.0;
        double s = sin(CEC_PI * wi + 1.0);
        f += (wi - 1.0) * (wi - 1.0) * (1.0 + 10.0 * s * s);
    }
    return f;
}

double cec_bent_cigar(const double *z, int n) {
    double s = 0.0;
    for (int i = 1; i < n; i++) s += z[i] * z[i];
    return z[0] * z[0] + 1e6 * s;
}

double cec_discus(const double *z, int n) {
    double s = 0.0;
    for (int i = 1; i < n; i++) s += z[i] * z[i];
    return 1e6 * z[0] * z[0] + s;
}

double cec_ellips(const double *z, int n) {
    double f = 0.0;
    for (int i = 0; i < n; i++) f += pow(10.0, 6.0 * i / (n > 1 ? n - 1 : 1)) * z[i] * z[i];
    return f;
}

double cec_hgbat(const double *z, int n) { /* z already -1 */
    double r2 = 0.0, sz = 0.0;
    for (int i = 0; i < n; i++) {
        r2 += z[i] * z[i];
        sz += z[i];
    }
    return sqrt(fabs(r2 * r2 - sz * sz)) + (0.5 * r2 + sz) / n + 0.5; /* objectives.py:123-126 */
}

double cec_happycat(const double *z, int n) { /* z already -1 */
    double r2 = 0.0, sz = 0.0;
    for (int i = 0; i < n; i++) {
        r2 += z[i] * z[i];
        sz += z[i];
    }
    return pow(fabs(r2 - n), 0.25) + (0.5 * r2 + sz) / n + 0.5;
}

double cec_katsuura(const double *z, int n) {
    double f = 1.0, t3 = pow((double)n, 1.2);
    for (int i = 0; i < n; i++) {
        double t = 0.0;
        for (int j = 1; j <= 32; j++) {
            double t1 = ldexp(1.0, j);
            double t2 = t1 * z[i];
            t += fabs(t2 - floor(t2 + 0.5)) / t1;
        }
        f *= pow(1.0 + (i + 1) * t, 10.0 / t3);
    }
    double t1 = 10.0 / n / n;
    return f * t1 - t1;
}

double cec_ackley(const double *z, int n) {
    double s1 = 0.0, s2 = 0.0;
    for (int i = 0; i < n; i++) {
        s1 += z[i] * z[i];
        s2 += cos(2.0 * CEC_PI * z[i]);
    }
    s1 = -0.2 * sqrt(s1 / n);
    s2 /= n;
    return CEC_E - 20.0 * exp(s1) - exp(s2) + 20.0;
}

static double schwefel_term(double zi, int n) {
    if (zi > 500.0) {
        double m = fmod(zi, 500.0);
        double t = (zi - 500.0) / 100.0;
        return -(500.0 - m) * sin(sqrt(500.0 - m)) + t * t / n;
    }
    if (zi < -500.0) {
        double m = fmod(fabs(zi), 500.0);
        double t = (zi + 500.0) / 100.0;
        return -(-500.0 + m) * sin(sqrt(500.0 - m)) + t * t / n;
    }
    return -zi * sin(sqrt(fabs(zi)));
}

double cec_schwefel(const double *z, int n) { /* z already scaled; +420.9687... applied here */
    double f = 0.0;
    for (int i = 0; i < n; i++) f += schwefel_term(z[i] + 4.209687462275036e+002, n);
    return f + 4.189828872724338e+002 * n;
}

double cec_schaffer_f7(const double *z, int n) {
    double f = 0.0;
    for (int i = 0; i < n - 1; i++) {
        double zi = sqrt(z[i] * z[i] + z[i + 1] * z[i + 1]);
        double t = sin(50.0 * pow(zi, 0.2));
        f += sqrt(zi) + sqrt(zi) * t * t;
    }
    return n > 1 ? f * f / (n - 1) / (n - 1) : f * f;
}

static double grie_rosen_term(double a, double b) {
    double t1 = a * a - b, t2 = a - 1.0;
    double t = 100.0 * t1 * t1 + t2 * t2;
    return t * t / 4000.0 - cos(t) + 1.0;
}

double cec_grie_rosen(const double *z, int n) { /* z already +1 */
    double f = 0.0;
    for (int i = 0; i < n - 1; i++) f += grie_rosen_term(z[i], z[i + 1]);
    return f + grie_rosen_term(z[n - 1], z[0]);
}

double cec_griewank(const double *z, int n) {
    double s = 0.0, p = 1.0;
    for (int i = 0; i < n; i++) {
        s += z[i] * z[i];
        p *= cos(z[i] / sqrt(1.0 + i));
    }
    return 1.0 + s / 4000.0 - p;
}

/* Basic-function ids shared with csrc/apo_cec.cuh and cec2022.py */
enum {
    B_ZAKHAROV = 0, B_ROSENBROCK, B_ESCAFFER6, B_RASTRIGIN, B_STEP_RASTRIGIN, B_LEVY, B_BENT_CIGAR, B_DISCUS,
    B_ELLIPS, B_HGBAT, B_HAPPYCAT, B_KATSUURA, B_ACKLEY, B_SCHWEFEL, B_SCHAFFER_F7, B_GRIE_ROSEN, B_GRIEWANK
};

/* scale applied by sr_func and the post-shift each basic function applies */
double cec_basic_scale(int b) {
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

double cec_basic_offset(int b) {
    switch (b) {
    case B_ROSENBROCK:
    case B_GRIE_ROSEN: return 1.0;
    case B_HGBAT:
    case B_HAPPYCAT: return -1.0;
    default: return 0.0;
    }
}

double cec_basic_eval(int b, const double *z, int n) {
    switch (b) {
    case B_ZAKHAROV: return cec_zakharov(z, n);
    case B_ROSENBROCK: return cec_rosenbrock(z, n);
    case B_ESCAFFER6: return cec_escaffer6(z, n);
    case B_RASTRIGIN:
    case B_STEP_RASTRIGIN: return cec_rastrigin(z, n);
    case B_LEVY: return cec_levy(z, n);
    case B_BENT_CIGAR: return cec_bent_cigar(z, n);
    case B_DISCUS: return cec_discus(z, n);
    case B_ELLIPS: return cec_ellips(z, n);
    case B_HGBAT: return cec_hgbat(z, n);
    case B_HAPPYCAT: return cec_happycat(z, n);
    case B_KATSUURA: return cec_katsuura(z, n);
    case B_ACKLEY: return cec_ackley(z, n);
    case B_SCHWEFEL: return cec_schwefel(z, n);
    case B_SCHAFFER_F7: return cec_schaffer_f7(z, n);
    case B_GRIE_ROSEN: return cec_grie_rosen(z, n);
    default: return cec_griewank(z, n);
    }
}

/* ------------------------------------------------------------------ spec */
typedef struct {
    int kind; /* 0 single, 1 hybrid, 2 composition */
    int ncomp;
    int basic[6];
    double p[6];     /* hybrid proportions */
    int rflag[6];    /* composition rotation flags */
    double lam[6];   /* composition scaling (fit *= lam) */
    double sigma[6]; /* composition delta */
    double bias[6];  /* composition biases */
    double fstar;
} cec_spec;

static const cec_spec SPECS[12] = {
    /* F1 */ {0, 1, {B_ZAKHAROV}, {1}, {1}, {1}, {0}, {0}, 300.0},
    /* F2 */ {0, 1, {B_ROSENBROCK}, {1}, {1}, {1}, {0}, {0}, 400.0},
    /* F3 */ {0, 1, {B_ESCAFFER6}, {1}, {1}, {1}, {0}, {0}, 600.0},
    /* F4 */ {0, 1, {B_STEP_RASTRIGIN}, {1}, {1}, {1}, {0}, {0}, 800.0},
    /* F5 */ {0, 1, {B_LEVY}, {1}, {1}, {1}, {0}, {0}, 900.0},
    /* F6 */ {1, 3, {B_BENT_CIGAR, B_HGBAT, B_RASTRIGIN}, {0.4, 0.4, 0.2}, {0}, {0}, {0}, {0}, 1800.0},
    /* F7 */
    {1, 6, {B_HGBAT, B_KATSUURA, B_ACKLEY, B_RASTRIGIN, B_SCHWEFEL, B_SCHAFFER_F7}, {0.1, 0.2, 0.2, 0.2, 0.1, 0.2},
     {0}, {0}, {0}, {0}, 2000.0},
    /* F8 */
    {1, 5, {B_KATSUURA, B_HAPPYCAT, B_GRIE_ROSEN, B_SCHWEFEL, B_ACKLEY}, {0.3, 0.2, 0.2, 0.1, 0.2}, {0}, {0}, {0},
     {0}, 2200.0},
    /* F9 */
    {2, 5, {B_ROSENBROCK, B_ELLIPS, B_BENT_CIGAR, B_DISCUS, B_ELLIPS}, {0}, {1, 0, 1, 1, 0},
     {1.0, 1e-6, 1e-26, 1e-6, 1e-6}, {10, 20, 30, 40, 50}, {0, 200, 300, 100, 400}, 2300.0},
    /* F10 */
    {2, 3, {B_SCHWEFEL, B_RASTRIGIN, B_HGBAT}, {0}, {0, 1, 0}, {1, 1, 1}, {20, 10, 10}, {0, 200, 100}, 2400.0},
    /* F11 */
    {2, 5, {B_ESCAFFER6, B_SCHWEFEL, B_GRIEWANK, B_ROSENBROCK, B_RASTRIGIN}, {0}, {1, 1, 1, 1, 1},
     {5e-4, 1, 10, 1, 10}, {20, 20, 30, 30, 20}, {0, 200, 300, 400, 200}, 2600.0},
    /* F12 */
    {2, 6, {B_HGBAT, B_RASTRIGIN, B_SCHWEFEL, B_BENT_CIGAR, B_ELLIPS, B_ESCAFFER6}, {0}, {1, 1, 1, 1, 1, 1},
     {10, 10, 2.5, 1e-26, 1e-6, 5e-4}, {10, 20, 30, 40, 50, 60}, {0, 300, 500, 100, 400, 200}, 2700.0},
};

/* Number of shift vectors / rotation matrices a function consumes. */
int or_cec_ncomp(int fn) { return SPECS[fn - 1].kind == 2 ? SPECS[fn - 1].ncomp : 1; }

/* Export the spec so the Python side and the CUDA tables stay in one place:
 * out[0]=kind, [1]=ncomp, [2]=fstar, then per component c (6 slots each):
 * basic, p, rflag, lam, sigma, bias. */
void or_cec_spec(int fn, double *out) {
    const cec_spec *S = &SPECS[fn - 1];
    out[0] = S->kind;
    out[1] = S->ncomp;
    out[2] = S->fstar;
    for (int c = 0; c < 6; c++) {
        out[3 + 6 * c + 0] = S->basic[c];
        out[3 + 6 * c + 1] = S->p[c];
        out[3 + 6 * c + 2] = S->rflag[c];
        out[3 + 6 * c + 3] = S->lam[c];
        out[3 + 6 * c + 4] = S->sigma[c];
        out[3 + 6 * c + 5] = S->bias[c];
    }
}

/* Hybrid segment sizes: ceil(p_i * n) for i < N-1, remainder last.  At
 * dimensions where the rounded-up sizes would exceed n (e.g. F7 at n = 12)
 * a segment is cut at n so every segment stays inside the candidate. */
void or_cec_segments(int fn, int n, int *sizes) {
    const cec_spec *S = &SPECS[fn - 1];
    int tot = 0;
    for (int c = 0; c < S->ncomp - 1; c++) {
        sizes[c] = (int)ceil(S->p[c] * n);
        if (sizes[c] > n - tot) sizes[c] = n - tot;
        tot += sizes[c];
    }
    sizes[S->ncomp - 1] = n - tot;
}

static void step_round(double *y, const double *x, const double *o, int n) {
    for (int i = 0; i < n; i++) {
        y[i] = x[i];
        if (fabs(x[i] - o[i]) > 0.5) y[i] = o[i] + floor(2.0 * (x[i] - o[i]) + 0.5) / 2.0;
    }
}

double or_cec_eval(int fn, const double *x, int n, const double *shift, const double *rot, const int *shuffle) {
    const cec_spec *S = &SPECS[fn - 1];
    double *z = malloc(sizeof(double) * (size_t)n * 3);
    double *tmp = z + n, *y = z + 2 * n;
    double f = 0.0;
    if (S->kind == 0) {
        int b = S->basic[0];
        const double *src = x;
        if (b == B_STEP_RASTRIGIN) {
            step_round(y, x, shift, n);
            src = y;
        }
        sr_func(src, z, n, shift, rot, cec_basic_scale(b), 1, 1, tmp);
        double off = cec_basic_offset(b);
        for (int i = 0; i < n; i++) z[i] += off;
        f = cec_basic_eval(b, z, n);
    } else if (S->kind == 1) {
        sr_func(x, z, n, shift, rot, 1.0, 1, 1, tmp);
        for (int i = 0; i < n; i++) y[i] = z[shuffle[i] - 1];
        int sizes[6], start = 0;
        or_cec_segments(fn, n, sizes);
        for (int c = 0; c < S->ncomp; c++) {
            int b = S->basic[c], m = sizes[c];
            double sc = cec_basic_scale(b), off = cec_basic_offset(b);
            for (int i = 0; i < m; i++) tmp[i] = y[start + i] * sc + off;
            if (m > 0) f += cec_basic_eval(b, tmp, m);
            start += m;
        }
    } else {
        double fit[6], w[6], wmax = 0.0, wsum = 0.0;
        for (int c = 0; c < S->ncomp; c++) {
            int b = S->basic[c];
            const double *o = shift + (size_t)c * n;
            sr_func(x, z, n, o, rot + (size_t)c * n * n, cec_basic_scale(b), 1, S->rflag[c], tmp);
            double off = cec_basic_offset(b);
            for (int i = 0; i < n; i++) z[i] += off;
            fit[c] = S->lam[c] * cec_basic_eval(b, z, n) + S->bias[c];
            double d2 = 0.0;
            for (int i = 0; i < n; i++) d2 += (x[i] - o[i]) * (x[i] - o[i]);
            w[c] = d2 != 0.0 ? sqrt(1.0 / d2) * exp(-d2 / 2.0 / n / (S->sigma[c] * S->sigma[c])) : INFINITY;
            if (w[c] > wmax) wmax = w[c];
        }
        int inf_at = -1;
        for (int c = 0; c < S->ncomp; c++) {
            if (isinf(w[c]) && inf_at < 0) inf_at = c;
            wsum += w[c];
        }
        if (inf_at >= 0) { /* x exactly at an optimum: that component alone */
            f = fit[inf_at];
        } else if (wmax == 0.0) {
            for (int c = 0; c < S->ncomp; c++) f += fit[c] / S->ncomp;
        } else {
            for (int c = 0; c < S->ncomp; c++) f += w[c] / wsum * fit[c];
        }
    }
    free(z);
    return f + S->fstar;
}

/* Basic function b (ids above) on each row of z: out[r] = g_b(z[r]) -- the building blocks alone. */
void or_cec_basic_batch(int b, const double *z, int64_t rows, int n, double *out) {
    for (int64_t r = 0; r < rows; r++) out[r] = cec_basic_eval(b, z + r * n, n);
}

/* Batch: out[r] = F_fn(x[r]) */
void or_cec_eval_batch(int fn, const double *x, int64_t rows, int n, const double *shift, const double *rot,
                       const int *shuffle, double *out, int nthreads) {
#pragma omp parallel for schedule(static) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < rows; r++) out[r] = or_cec_eval(fn, x + r * n, n, shift, rot, shuffle);
}
