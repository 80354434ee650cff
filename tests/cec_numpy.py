"""A second, independent CEC2022 restatement in vectorised numpy -- TEST INFRASTRUCTURE ONLY.

Written from the CEC2022 technical-report definitions (sr_func: y = s (x - o), z = M y; hybrid
functions: z = M (x - o), shuffled, cut into segments of ceil(p_i D) dimensions, each basic function
applying its own scale/offset; composition functions: F = sum_k w_k/sum w (lambda_k g_k(z_k) + bias_k)
with w_k = d_k^-1/2 exp(-d_k / (2 D sigma_k^2)), d_k = |x - o_k|^2), NOT ported from
oracle/cec_oracle.c: rows are evaluated together, sums are numpy reductions (pairwise order), the
rotation is a matrix product.  tests/test_cec_pinning.py checks it against the C oracle at 1e-12, so
a transcription slip in either (segment bounds, shuffle direction, rotation transpose, Schwefel
branches, composition weights) shows up as a disagreement.  The shift/rotation/shuffle data come from
paper_2510_14982_b200/cec2022.py (the official data files are not available offline).
"""

import numpy as np

PI = np.pi


def bent_cigar(z):
    return z[:, 0] ** 2 + 1e6 * np.sum(z[:, 1:] ** 2, axis=1)


def discus(z):
    return 1e6 * z[:, 0] ** 2 + np.sum(z[:, 1:] ** 2, axis=1)


def ellips(z):
    n = z.shape[1]
    w = 10.0 ** (6.0 * np.arange(n) / max(n - 1, 1))
    return np.sum(w * z * z, axis=1)


def hgbat(z):  # z already shifted by -1
    n = z.shape[1]
    r2, s = np.sum(z * z, axis=1), np.sum(z, axis=1)
    return np.sqrt(np.abs(r2 ** 2 - s ** 2)) + (0.5 * r2 + s) / n + 0.5


def rastrigin(z):
    return np.sum(z * z - 10.0 * np.cos(2.0 * PI * z) + 10.0, axis=1)


def zakharov(z):
    i = np.arange(1, z.shape[1] + 1)
    s1, s2 = np.sum(z * z, axis=1), np.sum(0.5 * i * z, axis=1)
    return s1 + s2 ** 2 + s2 ** 4


def schwefel(z):
    n = z.shape[1]
    zz = z + 4.209687462275036e2
    m = np.mod(np.abs(zz), 500.0)
    g = np.where(np.abs(zz) <= 500.0, zz * np.sin(np.sqrt(np.abs(zz))), 0.0)
    g = np.where(zz > 500.0, (500.0 - m) * np.sin(np.sqrt(500.0 - m)) - (zz - 500.0) ** 2 / (10000.0 * n), g)
    g = np.where(zz < -500.0, (m - 500.0) * np.sin(np.sqrt(500.0 - m)) - (zz + 500.0) ** 2 / (10000.0 * n), g)
    return 4.189828872724338e2 * n - np.sum(g, axis=1)


def escaffer6(z):
    x, y = z, np.roll(z, -1, axis=1)
    r2 = x * x + y * y
    return np.sum(0.5 + (np.sin(np.sqrt(r2)) ** 2 - 0.5) / (1.0 + 0.001 * r2) ** 2, axis=1)


# (function, scale s, offset added after s * rotation) per basic function, as each CEC basic function
# applies it inside its own sr_func call
BASIC = {
    "bent_cigar": (bent_cigar, 1.0, 0.0),
    "discus": (discus, 1.0, 0.0),
    "ellips": (ellips, 1.0, 0.0),
    "hgbat": (hgbat, 0.05, -1.0),
    "rastrigin": (rastrigin, 0.0512, 0.0),
    "zakharov": (zakharov, 1.0, 0.0),
    "schwefel": (schwefel, 10.0, 0.0),
    "escaffer6": (escaffer6, 1.0, 0.0),
}

# CEC2022 parameter tables (technical report, Table of hybrid / composition functions)
HYBRID = {6: (["bent_cigar", "hgbat", "rastrigin"], [0.4, 0.4, 0.2], 1800.0)}
COMPOSITION = {
    # components: (basic, rotated, lambda, sigma, bias)
    10: ([("schwefel", False, 1.0, 20.0, 0.0), ("rastrigin", True, 1.0, 10.0, 200.0),
          ("hgbat", False, 1.0, 10.0, 100.0)], 2400.0),
    12: ([("hgbat", True, 10.0, 10.0, 0.0), ("rastrigin", True, 10.0, 20.0, 300.0),
          ("schwefel", True, 2.5, 30.0, 500.0), ("bent_cigar", True, 1e-26, 40.0, 100.0),
          ("ellips", True, 1e-6, 50.0, 400.0), ("escaffer6", True, 5e-4, 60.0, 200.0)], 2700.0),
}
SINGLE = {1: ("zakharov", 300.0), 4: ("step_rastrigin", 800.0)}


def evaluate(fn: int, x: np.ndarray, shift: np.ndarray, rot: np.ndarray, shuffle: np.ndarray) -> np.ndarray:
    """F_fn on every row of x ([rows, D]); rot[k] maps y to z = rot[k] @ y."""
    x = np.atleast_2d(np.asarray(x, dtype=np.float64))
    n = x.shape[1]
    if fn in SINGLE:
        name, fstar = SINGLE[fn]
        o = shift[0]
        if name == "step_rastrigin":  # non-continuous: coordinates farther than 1/2 from o snap to halves
            far = np.abs(x - o) > 0.5
            x = np.where(far, o + np.floor(2.0 * (x - o) + 0.5) / 2.0, x)
            name = "rastrigin"
        f, s, off = BASIC[name]
        z = (s * (x - o)) @ rot[0].T + off
        return f(z) + fstar
    if fn in HYBRID:
        names, p, fstar = HYBRID[fn]
        z = (x - shift[0]) @ rot[0].T
        y = z[:, np.asarray(shuffle) - 1]
        sizes = [int(np.ceil(pi * n)) for pi in p[:-1]]
        sizes.append(n - sum(sizes))
        total, start = np.zeros(x.shape[0]), 0
        for name, m in zip(names, sizes):
            f, s, off = BASIC[name]
            total = total + f(s * y[:, start:start + m] + off)
            start += m
        return total + fstar
    comps, fstar = COMPOSITION[fn]
    vals, ws = [], []
    for k, (name, rotated, lam, sigma, bias) in enumerate(comps):
        f, s, off = BASIC[name]
        d = x - shift[k]
        y = s * d
        z = (y @ rot[k].T if rotated else y) + off
        vals.append(lam * f(z) + bias)
        d2 = np.sum(d * d, axis=1)
        with np.errstate(divide="ignore", over="ignore"):
            ws.append(np.where(d2 != 0.0, np.sqrt(1.0 / d2) * np.exp(-d2 / (2.0 * n * sigma ** 2)), np.inf))
    vals, ws = np.array(vals), np.array(ws)
    out = np.empty(x.shape[0])
    for r in range(x.shape[0]):
        w = ws[:, r]
        if np.isinf(w).any():  # x at an optimum o_k: that component alone
            out[r] = vals[int(np.argmax(np.isinf(w))), r]
        elif w.max() == 0.0:
            out[r] = vals[:, r].mean()
        else:
            out[r] = np.sum(w / w.sum() * vals[:, r])
    return out + fstar
