/*
 * threshold_oracle.c -- CPU restatement of multilevel Otsu / Kapur thresholding.
 *
 * TEST INFRASTRUCTURE ONLY (see apo_oracle.c).  PARITY UNPINNED: the
 * reference implements only single-threshold Otsu (imaging.py:203-240) and
 * lists multi-level thresholding as a non-goal.  The k = 1
 * special case is pinned to the reference through its own class convention
 * (class 0 holds intensities <= t, imaging.py:203-223) and rounding rule
 * (round_half_up, clamped, imaging.py:282-284 / objectives.py:213-219),
 * which this restatement generalises:
 *
 *   thresholds t_j = clamp(floor(x_j + 0.5), 0, 255), sorted ascending;
 *   classes [0, t_0], [t_0 + 1, t_1], ..., [t_{k-1} + 1, 255]; an empty
 *   class contributes 0;
 *   Otsu:  f = -sum_c (n_c / N) (s_c / n_c - S / N)^2   (between-class variance)
 *   Kapur: f = -sum_c [ ln(n_c / N) - (sum_{v in c} p_v ln p_v) / (n_c / N) ]
 *          with p_v = count_v / N and 0 ln 0 = 0 (total class entropy)
 *
 * Table layout (shared with the device, include/apo_b200.h):
 *   tab[0] = N; tab[1 + i] = sum_{v < i} count_v  (i = 0..256);
 *   tab[258 + i] = sum_{v < i} v count_v (Otsu) or sum_{v < i} p_v ln p_v (Kapur).
 */
#include <math.h>
#include <stdint.h>

#define OR_TAB_LEN 515

void or_threshold_tables(const int64_t *counts, int method, double *tab) {
    int64_t n = 0;
    for (int v = 0; v < 256; v++) n += counts[v];
    tab[0] = (double)n;
    int64_t c = 0;
    double s = 0.0;
    tab[1] = 0.0;
    tab[258] = 0.0;
    for (int v = 0; v < 256; v++) {
        c += counts[v];
        tab[2 + v] = (double)c;
        if (method == 0) {
            s += (double)v * (double)counts[v];
        } else if (counts[v] > 0) {
            const double p = (double)counts[v] / (double)n;
            s += p * log(p);
        }
        tab[259 + v] = s;
    }
}

static int round_clamp(double x) {
    double r = floor(x + 0.5);
    if (!(r >= 0.0)) return 0; /* also NaN */
    if (r > 255.0) return 255;
    return (int)r;
}

/* method 0 = Otsu, 1 = Kapur */
double or_threshold_eval(int method, const double *x, int64_t k, const double *tab) {
    int t[256];
    for (int64_t j = 0; j < k; j++) {
        int v = round_clamp(x[j]);
        int64_t i = j;
        while (i > 0 && t[i - 1] > v) { /* insertion sort */
            t[i] = t[i - 1];
            i--;
        }
        t[i] = v;
    }
    const double N = tab[0];
    const double *C = tab + 1, *S = tab + 258;
    const double mu_t = S[256] / N;
    double f = 0.0;
    int lo = 0;
    for (int64_t c = 0; c <= k; c++) {
        const int hi = c < k ? t[c] : 255; /* class [lo, hi] */
        if (hi >= lo) {
            const double nc = C[hi + 1] - C[lo];
            if (nc > 0.0) {
                const double w = nc / N;
                if (method == 0) {
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
