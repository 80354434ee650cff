/*
 * apo_oracle.c -- CPU restatement of the reference APO iteration.
 *
 * TEST INFRASTRUCTURE ONLY.  This file is the checker for the CUDA path and
 * the CPU baseline timed by bench.py (`cpu_baseline`, `--impl reference`).
 * Nothing in the product package (paper_2510_14982_b200/) may link or call
 * it; tests/, __graft_entry__.smoke() and bench.py are the only users.
 *
 * Every function below restates a reference function (paths relative to
 * /root/reference/pkg/src/protozoa/) with the same floating-point
 * expression order, the same integer index math and glibc libm for the
 * transcendental calls, so results are bit-identical to the reference's
 * numba and numpy backends.  It must be compiled with -ffp-contract=off
 * (the reference never fuses a multiply-add).
 *
 * Parity pin: tests/test_oracle_golden.py checks this file against golden
 * vectors produced by the reference itself (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

/* ---------------------------------------------------------------------------
 * Keyed RNG: rng.py:79-111, numba_backend.py:52-71
 * ------------------------------------------------------------------------- */
#define H0 0x9E3779B97F4A7C15ULL
#define MUL1 0xFF51AFD7ED558CCDULL
#define MUL2 0xC4CEB9FE1A85EC53ULL
#define INV_2_53 (1.0 / 9007199254740992.0)

#define SLOT_DECISION 0ULL
#define SLOT_SIGN 1ULL
#define SLOT_MASK_SIZE 2ULL
#define SLOT_MAGNITUDE 3ULL
#define SLOT_FORAGE 4ULL
#define SLOT_PARTNER 5ULL
#define VECTOR_BASE 8ULL
#define MASK_BASE (1ULL << 32)
#define PAIRS_BASE (1ULL << 33)
#define COORD_INDEX 0xFFFFFFFFFFFFFFFFULL

double or_cec_eval(int fn, const double *x, int n, const double *shift, const double *rot, const int *shuffle);
int or_cec_ncomp(int fn);

/* CEC2022 objectives (code 100+F, cec_oracle.c): `table` packs
 * [shift ncomp*n][rot ncomp*n*n][shuffle n (as doubles)]. */
static double cec_packed(int fn, const double *x, int64_t n, const double *table) {
    int nc = or_cec_ncomp(fn);
    const double *shift = table, *rot = table + (size_t)nc * n, *sh = rot + (size_t)nc * n * n;
    int *shuffle = malloc(sizeof(int) * (size_t)n);
    for (int64_t i = 0; i < n; i++) shuffle[i] = (int)sh[i];
    double f = or_cec_eval(fn, x, (int)n, shift, rot, shuffle);
    free(shuffle);
    return f;
}

/* objective codes: objectives.py:34-42 */
enum { SPHERE = 0, BENT_CIGAR = 1, ELLIPTIC = 2, HGBAT = 3, ROSENBROCK = 4, GRIEWANK = 5, TABLE = 6 };

uint64_t or_mix(uint64_t z) { /* rng.py:79-86 */
    z ^= z >> 33;
    z *= MUL1;
    z ^= z >> 33;
    z *= MUL2;
    z ^= z >> 33;
    return z;
}

uint64_t or_stream_base(uint64_t seed, uint64_t iteration, uint64_t individual) { /* rng.py:89-97 */
    uint64_t h = or_mix(H0 ^ seed);
    h = or_mix(h ^ iteration);
    return or_mix(h ^ individual);
}

double or_u(uint64_t base, uint64_t counter) { /* rng.py:100-111 */
    return (double)(or_mix(base ^ counter) >> 11) * INV_2_53;
}

/* Partial Fisher-Yates over 1..n reading counters ctr0 .. ctr0+k-1: rng.py:137-156 */
void or_randperm(int64_t n, int64_t k, uint64_t base, uint64_t ctr0, int64_t *out, int64_t *scratch) {
    for (int64_t a = 0; a < n; a++) scratch[a] = a + 1;
    for (int64_t j = 0; j < k; j++) {
        double u = or_u(base, ctr0 + (uint64_t)j);
        int64_t r = j + (int64_t)(u * (double)(n - j));
        if (r > n - 1) r = n - 1;
        int64_t t = scratch[j];
        scratch[j] = scratch[r];
        scratch[r] = t;
    }
    for (int64_t j = 0; j < k; j++) out[j] = scratch[j];
}

/* ---------------------------------------------------------------------------
 * Objectives: numba_backend.py:93-138 (== objectives.py:105-152, 213-219)
 * ------------------------------------------------------------------------- */
double or_threshold_eval(int method, const double *x, int64_t k, const double *tab);

double or_eval(int64_t code, const double *x, int64_t n, const double *table, int64_t tlen) {
    double s, s1, s2, p;
    if (code > 100) return cec_packed((int)(code - 100), x, n, table);
    if (code == 7 || code == 8) return or_threshold_eval((int)(code - 7), x, n, table); /* multilevel Otsu / Kapur */
    switch (code) {
    case SPHERE:
        s = 0.0;
        for (int64_t d = 0; d < n; d++) s += x[d] * x[d];
        return s;
    case BENT_CIGAR:
        s = 0.0;
        for (int64_t d = 1; d < n; d++) s += x[d] * x[d];
        return x[0] * x[0] + 1e6 * s;
    case ELLIPTIC:
        s = 0.0;
        for (int64_t d = 0; d < n; d++) s += (table[d] * x[d]) * x[d];
        return s;
    case HGBAT:
        s1 = 0.0;
        s2 = 0.0;
        for (int64_t d = 0; d < n; d++) {
            s1 += x[d];
            s2 += x[d] * x[d];
        }
        return sqrt(fabs(s2 * s2 - s1 * s1)) + (0.5 * s2 + s1) / (double)n + 0.5;
    case ROSENBROCK:
        s = 0.0;
        for (int64_t d = 0; d < n - 1; d++) {
            double a = x[d + 1] - x[d] * x[d];
            double b = x[d] - 1.0;
            s += 100.0 * (a * a) + b * b;
        }
        return s;
    case GRIEWANK:
        s = 0.0;
        p = 1.0;
        for (int64_t d = 0; d < n; d++) {
            s += x[d] * x[d];
            p *= cos(x[d] / sqrt((double)d + 1.0));
        }
        return 1.0 + s / 4000.0 - p;
    default: { /* TABLE */
        int64_t idx = (int64_t)floor(x[0] + 0.5);
        if (idx < 0) idx = 0;
        if (idx > tlen - 1) idx = tlen - 1;
        return table[idx];
    }
    }
}

/* Elliptic weights: objectives.py:88-102 (Python float pow == C pow). */
void or_elliptic_weights(int64_t dim, double *w) {
    if (dim == 1) {
        w[0] = 1.0;
        return;
    }
    for (int64_t i = 0; i < dim; i++) w[i] = pow(10.0, 6.0 * (double)i / (double)(dim - 1));
}

/* ---------------------------------------------------------------------------
 * Per-individual update: numba_backend.py:74-90 (_fill_mask), :141-290 (_update_row)
 * ------------------------------------------------------------------------- */
static void fill_mask(double *mask, int64_t *perm, int64_t dim, int64_t count, uint64_t base) {
    for (int64_t d = 0; d < dim; d++) perm[d] = d + 1;
    for (int64_t j = 0; j < count; j++) {
        double u = or_u(base, MASK_BASE + (uint64_t)j);
        int64_t r = j + (int64_t)(u * (double)(dim - j));
        if (r > dim - 1) r = dim - 1;
        int64_t t = perm[j];
        perm[j] = perm[r];
        perm[r] = t;
    }
    for (int64_t d = 0; d < dim; d++) mask[d] = 0.0;
    for (int64_t j = 0; j < count; j++) mask[perm[j] - 1] = 1.0;
}

typedef struct {
    uint64_t seed, key_iteration;
    int64_t ps, dim, npairs;
    double lower, upper, span, eps, p_ah, f_mult, decay;
    int64_t code;
    const double *table;
    int64_t tlen;
} or_params;

static void update_row(int64_t i0, const double *pos, const double *fit, const uint8_t *in_dr, double *out_pos,
                       double *out_fit, uint8_t *out_acc, uint8_t *out_warn, const or_params *P, double *cand,
                       double *mask, int64_t *perm, double *acc) {
    const int64_t ps = P->ps, dim = P->dim, npairs = P->npairs;
    const int64_t i = i0 + 1;
    const double *x = pos + i0 * dim;
    uint64_t base = or_stream_base(P->seed, P->key_iteration, (uint64_t)i);
    double u_dec = or_u(base, SLOT_DECISION);

    if (in_dr[i0]) {
        double q = 1.0 - (double)i / (double)ps;
        double thr = 0.5 * (1.0 - cos(q * M_PI));
        if (u_dec < thr) { /* dormancy */
            for (int64_t d = 0; d < dim; d++) cand[d] = P->lower + or_u(base, VECTOR_BASE + (uint64_t)d) * P->span;
        } else { /* reproduction */
            double sgn = or_u(base, SLOT_SIGN) < 0.5 ? 1.0 : -1.0;
            double mag = or_u(base, SLOT_MAGNITUDE);
            double usize = or_u(base, SLOT_MASK_SIZE);
            int64_t count = (int64_t)ceil((double)dim * usize);
            fill_mask(mask, perm, dim, count, base);
            double scale = sgn * mag;
            for (int64_t d = 0; d < dim; d++) {
                double off = P->lower + or_u(base, VECTOR_BASE + (uint64_t)d) * P->span;
                cand[d] = x[d] + (scale * off) * mask[d];
            }
        }
    } else {
        for (int64_t d = 0; d < dim; d++) acc[d] = 0.0;
        if (u_dec < P->p_ah) { /* autotroph */
            int64_t j;
            if (ps == 1) {
                j = i;
            } else {
                double up = or_u(base, SLOT_PARTNER);
                int64_t j0 = (int64_t)(up * (double)(ps - 1));
                if (j0 > ps - 2) j0 = ps - 2;
                if (j0 >= i - 1) j0 += 1;
                j = j0 + 1;
            }
            double f = or_u(base, SLOT_FORAGE) * P->f_mult;
            int64_t count = (int64_t)ceil((double)(dim * i) / (double)ps);
            fill_mask(mask, perm, dim, count, base);
            for (int64_t k = 0; k < npairs; k++) {
                int64_t km, kp;
                if (i == 1) {
                    km = 1;
                } else {
                    double ukm = or_u(base, PAIRS_BASE + (uint64_t)(2 * k));
                    km = 1 + (int64_t)(ukm * (double)(i - 1));
                    if (km > i - 1) km = i - 1;
                }
                if (i == ps) {
                    kp = ps;
                } else {
                    double ukp = or_u(base, PAIRS_BASE + (uint64_t)(2 * k + 1));
                    kp = i + 1 + (int64_t)(ukp * (double)(ps - i));
                    if (kp > ps) kp = ps;
                }
                double w = exp(-fabs(fit[km - 1] / (fit[kp - 1] + P->eps)));
                const double *xm = pos + (km - 1) * dim, *xp = pos + (kp - 1) * dim;
                for (int64_t d = 0; d < dim; d++) acc[d] = acc[d] + w * (xm[d] - xp[d]);
            }
            const double *xj = pos + (j - 1) * dim;
            for (int64_t d = 0; d < dim; d++) {
                double epn = acc[d] / (double)npairs;
                double direction = (xj[d] - x[d]) + epn;
                cand[d] = x[d] + (f * direction) * mask[d];
            }
        } else { /* heterotroph */
            double sgn = or_u(base, SLOT_SIGN) < 0.5 ? 1.0 : -1.0;
            double f = or_u(base, SLOT_FORAGE) * P->f_mult;
            int64_t count = (int64_t)ceil((double)(dim * i) / (double)ps);
            fill_mask(mask, perm, dim, count, base);
            for (int64_t k = 1; k <= npairs; k++) {
                int64_t km = i - k, kp = i + k;
                if (km < 1) km = 1;
                if (kp > ps) kp = ps;
                double w = exp(-fabs(fit[km - 1] / (fit[kp - 1] + P->eps)));
                const double *xm = pos + (km - 1) * dim, *xp = pos + (kp - 1) * dim;
                for (int64_t d = 0; d < dim; d++) acc[d] = acc[d] + w * (xm[d] - xp[d]);
            }
            for (int64_t d = 0; d < dim; d++) {
                double uv = or_u(base, VECTOR_BASE + (uint64_t)d);
                double near = (1.0 + (sgn * uv) * P->decay) * x[d];
                double eph = acc[d] / (double)npairs;
                double direction = (near - x[d]) + eph;
                cand[d] = x[d] + (f * direction) * mask[d];
            }
        }
    }
    /* clamp + evaluate + greedy: numba_backend.py:259-290, core.py:487-501 */
    int ok = 1;
    for (int64_t d = 0; d < dim; d++) {
        double v = cand[d];
        if (v < P->lower) v = P->lower;
        else if (v > P->upper) v = P->upper;
        cand[d] = v;
        if (!isfinite(v)) ok = 0;
    }
    int accepted = 0, warned = 0;
    double new_fit = 0.0;
    if (ok) {
        new_fit = or_eval(P->code, cand, dim, P->table, P->tlen);
        if (isfinite(new_fit)) accepted = new_fit < fit[i0];
        else warned = 1;
    } else {
        warned = 1;
    }
    double *o = out_pos + i0 * dim;
    if (accepted) {
        memcpy(o, cand, sizeof(double) * (size_t)dim);
        out_fit[i0] = new_fit;
    } else {
        memcpy(o, x, sizeof(double) * (size_t)dim);
        out_fit[i0] = fit[i0];
    }
    out_acc[i0] = (uint8_t)accepted;
    out_warn[i0] = (uint8_t)warned;
}

/* run_updates: numba_backend.py:323-372.  Returns the warning count. */
int64_t or_run_updates(const double *pos, const double *fit, const uint8_t *in_dr, double *out_pos, double *out_fit,
                       uint8_t *out_acc, uint8_t *out_warn, int64_t ps, int64_t dim, uint64_t seed,
                       uint64_t key_iteration, int64_t npairs, double lower, double upper, double span, double eps,
                       double p_ah, double f_mult, double decay, int64_t code, const double *table, int64_t tlen,
                       int nthreads) {
    or_params P = {seed, key_iteration, ps, dim, npairs, lower, upper, span, eps, p_ah, f_mult, decay, code, table, tlen};
    if (nthreads < 1) nthreads = 1;
#pragma omp parallel num_threads(nthreads)
    {
        double *cand = malloc(sizeof(double) * (size_t)dim);
        double *mask = malloc(sizeof(double) * (size_t)dim);
        double *acc = malloc(sizeof(double) * (size_t)dim);
        int64_t *perm = malloc(sizeof(int64_t) * (size_t)dim);
#pragma omp for schedule(static)
        for (int64_t i0 = 0; i0 < ps; i0++)
            update_row(i0, pos, fit, in_dr, out_pos, out_fit, out_acc, out_warn, &P, cand, mask, perm, acc);
        free(cand);
        free(mask);
        free(acc);
        free(perm);
    }
    int64_t w = 0;
    for (int64_t i0 = 0; i0 < ps; i0++) w += out_warn[i0];
    return w;
}

/* ---------------------------------------------------------------------------
 * Engine pieces: core.py:263-278 (coordinator), core.py:504-513 (sort),
 * engine.py:116-139 (initialize), engine.py:142-212 (step / run)
 * ------------------------------------------------------------------------- */

/* numpy argsort(kind="stable") order: ascending, ties by index, -0.0 == +0.0,
 * NaN last (numpy sorts NaNs to the end). */
static int less_key(double a, double b) {
    if (isnan(b)) return !isnan(a);
    if (isnan(a)) return 0;
    return a < b;
}

static void merge_sort(int64_t *idx, int64_t *tmp, const double *key, int64_t n) {
    for (int64_t width = 1; width < n; width *= 2) {
        for (int64_t lo = 0; lo < n; lo += 2 * width) {
            int64_t mid = lo + width < n ? lo + width : n;
            int64_t hi = lo + 2 * width < n ? lo + 2 * width : n;
            int64_t a = lo, b = mid, o = lo;
            while (a < mid && b < hi) {
                if (less_key(key[idx[b]], key[idx[a]])) tmp[o++] = idx[b++];
                else tmp[o++] = idx[a++];
            }
            while (a < mid) tmp[o++] = idx[a++];
            while (b < hi) tmp[o++] = idx[b++];
        }
        memcpy(idx, tmp, sizeof(int64_t) * (size_t)n);
    }
}

void or_argsort_stable(const double *key, int64_t n, int64_t *order) {
    int64_t *tmp = malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
    for (int64_t a = 0; a < n; a++) order[a] = a;
    merge_sort(order, tmp, key, n);
    free(tmp);
}

/* pf and the Dr mask for one iteration: core.py:263-278, engine.py:157-162.
 * Returns the Dr count. */
int64_t or_select_dr(uint64_t seed, uint64_t key_iteration, int64_t ps, double pf_max, uint8_t *in_dr, int64_t *scratch,
                     int64_t *sel) {
    uint64_t base = or_stream_base(seed, key_iteration, COORD_INDEX);
    double pf = pf_max * or_u(base, 0);
    int64_t count = (int64_t)ceil((double)ps * pf);
    or_randperm(ps, count, base, 1, sel, scratch);
    memset(in_dr, 0, (size_t)ps);
    for (int64_t a = 0; a < count; a++) in_dr[sel[a] - 1] = 1;
    return count;
}

/* engine.py:116-139 */
void or_initialize(uint64_t seed, int64_t ps, int64_t dim, double lower, double span, int64_t code,
                   const double *table, int64_t tlen, double *pos, double *fit) {
    for (int64_t i = 1; i <= ps; i++) {
        uint64_t base = or_stream_base(seed, 0, (uint64_t)i);
        for (int64_t d = 0; d < dim; d++) pos[(i - 1) * dim + d] = lower + or_u(base, (uint64_t)d) * span;
    }
    for (int64_t r = 0; r < ps; r++) fit[r] = or_eval(code, pos + r * dim, dim, table, tlen);
}

/* One engine.step (engine.py:142-172): sort, coordinator draws, updates.
 * pos/fit are read; out_pos/out_fit receive the new population in
 * sorted-snapshot row order.  Returns the warning count. */
int64_t or_step(const double *pos, const double *fit, double *out_pos, double *out_fit, int64_t ps, int64_t dim,
                int64_t max_iterations, int64_t iteration, uint64_t seed, int64_t npairs, double pf_max, double lower,
                double upper, double eps, int64_t code, const double *table, int64_t tlen, int nthreads,
                uint8_t *out_in_dr) {
    int64_t *order = malloc(sizeof(int64_t) * (size_t)ps);
    double *spos = malloc(sizeof(double) * (size_t)(ps * dim));
    double *sfit = malloc(sizeof(double) * (size_t)ps);
    uint8_t *in_dr = malloc((size_t)ps);
    uint8_t *acc = malloc((size_t)ps), *warn = malloc((size_t)ps);
    int64_t *scratch = malloc(sizeof(int64_t) * (size_t)ps), *sel = malloc(sizeof(int64_t) * (size_t)ps);
    or_argsort_stable(fit, ps, order);
    for (int64_t r = 0; r < ps; r++) {
        memcpy(spos + r * dim, pos + order[r] * dim, sizeof(double) * (size_t)dim);
        sfit[r] = fit[order[r]];
    }
    uint64_t key_iteration = (uint64_t)iteration + 1;
    or_select_dr(seed, key_iteration, ps, pf_max, in_dr, scratch, sel);
    if (out_in_dr) memcpy(out_in_dr, in_dr, (size_t)ps);
    /* host scalars: numba_backend.py:357-366, core.py:220-250 */
    int64_t span_it = max_iterations - 1 > 1 ? max_iterations - 1 : 1;
    double ratio = (double)iteration / (double)span_it;
    double p_ah = 0.5 * (1.0 + cos(ratio * M_PI));
    double f_mult = 1.0 + cos(ratio * M_PI);
    double decay = 1.0 - ratio;
    int64_t w = or_run_updates(spos, sfit, in_dr, out_pos, out_fit, acc, warn, ps, dim, seed, key_iteration, npairs,
                               lower, upper, upper - lower, eps, p_ah, f_mult, decay, code, table, tlen, nthreads);
    free(order);
    free(spos);
    free(sfit);
    free(in_dr);
    free(acc);
    free(warn);
    free(scratch);
    free(sel);
    return w;
}

static double min_of(const double *f, int64_t n) { /* np.min (NaN propagates) */
    double m = f[0];
    for (int64_t a = 0; a < n; a++) {
        if (isnan(f[a])) return f[a];
        if (f[a] < m) m = f[a];
    }
    return m;
}

/* engine.run (engine.py:175-212) without timing.  trace must hold
 * max_iterations+1 entries.  On return pos/fit hold the final population
 * (sorted-snapshot order of the last step); out[0]=iterations_run,
 * out[1]=fe_count, out[2]=warnings, out[3]=argmin row. */
void or_run(int64_t ps, int64_t dim, int64_t max_iterations, int64_t max_fes, uint64_t seed, int64_t npairs,
            double pf_max, double lower, double upper, double eps, int64_t code, const double *table, int64_t tlen,
            int nthreads, double *pos, double *fit, double *trace, int64_t *out) {
    double *npos = malloc(sizeof(double) * (size_t)(ps * dim));
    double *nfit = malloc(sizeof(double) * (size_t)ps);
    or_initialize(seed, ps, dim, lower, upper - lower, code, table, tlen, pos, fit);
    int64_t fe = ps, warnings = 0, it = 0;
    trace[0] = min_of(fit, ps);
    for (int64_t t = 0; t < max_iterations; t++) {
        if (max_fes > 0 && fe >= max_fes) break;
        warnings += or_step(pos, fit, npos, nfit, ps, dim, max_iterations, t, seed, npairs, pf_max, lower, upper, eps,
                            code, table, tlen, nthreads, NULL);
        memcpy(pos, npos, sizeof(double) * (size_t)(ps * dim));
        memcpy(fit, nfit, sizeof(double) * (size_t)ps);
        fe += ps;
        it++;
        trace[it] = min_of(fit, ps);
    }
    int64_t best = 0;
    for (int64_t a = 1; a < ps; a++)
        if (fit[a] < fit[best]) best = a;
    out[0] = it;
    out[1] = fe;
    out[2] = warnings;
    out[3] = best;
    free(npos);
    free(nfit);
}

/* Many independent runs (seeds x objectives), one run per thread: the CPU
 * baseline for the batched suite. */
void or_run_many(int64_t nruns, const int64_t *codes, const uint64_t *seeds, const double *const *tables,
                 const int64_t *tlens, int64_t ps, int64_t dim, int64_t max_iterations, int64_t npairs, double pf_max,
                 double lower, double upper, double eps, int nthreads, double *best_fit, int64_t *fe_out) {
#pragma omp parallel for schedule(dynamic, 1) num_threads(nthreads > 0 ? nthreads : 1)
    for (int64_t r = 0; r < nruns; r++) {
        double *pos = malloc(sizeof(double) * (size_t)(ps * dim));
        double *fit = malloc(sizeof(double) * (size_t)ps);
        double *trace = malloc(sizeof(double) * (size_t)(max_iterations + 1));
        int64_t out[4];
        or_run(ps, dim, max_iterations, 0, seeds[r], npairs, pf_max, lower, upper, eps, codes[r], tables[r], tlens[r],
               1, pos, fit, trace, out);
        best_fit[r] = fit[out[3]];
        fe_out[r] = out[1];
        free(pos);
        free(fit);
        free(trace);
    }
}
