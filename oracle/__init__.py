"""CPU oracle for the APO iteration -- TEST INFRASTRUCTURE ONLY.

A ctypes wrapper around ``liboracle_apo.so`` (built from apo_oracle.c and
friends by ``oracle/Makefile``).  The C code restates the reference's
numba kernel (/root/reference/pkg/src/protozoa/kernels/numba_backend.py)
and engine loop (engine.py) bit for bit.  Only ``tests/``,
``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline leg may import
this package; the product package never does.

Parity pin: tests/test_oracle_golden.py checks every entry point below
against vectors the reference itself produced (tests/golden/).  The
CEC2022 and multilevel-threshold restatements (cec_oracle.c,
threshold_oracle.c) have no reference counterpart: **parity unpinned** for
those.
"""

from __future__ import annotations

import ctypes as C
import math
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_apo.so")

COORDINATOR_INDEX = (1 << 64) - 1
CODES = {"sphere": 0, "bent_cigar": 1, "high_conditioned_elliptic": 2, "hgbat": 3, "rosenbrock": 4,
         "griewank": 5, "table": 6, "otsu_ml": 7, "kapur_ml": 8}

_lib = None


def build(force: bool = False) -> str:
    """Compile the oracle with its Makefile (gcc, -ffp-contract=off)."""
    if force or not os.path.exists(LIB_PATH) or any(
        os.path.getmtime(os.path.join(HERE, f)) > os.path.getmtime(LIB_PATH)
        for f in os.listdir(HERE) if f.endswith(".c")
    ):
        subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


_P = C.c_void_p
_I = C.c_int64
_U = C.c_uint64
_D = C.c_double


def _declare(L):
    L.or_mix.restype = _U
    L.or_mix.argtypes = [_U]
    L.or_stream_base.restype = _U
    L.or_stream_base.argtypes = [_U, _U, _U]
    L.or_u.restype = _D
    L.or_u.argtypes = [_U, _U]
    L.or_randperm.restype = None
    L.or_randperm.argtypes = [_I, _I, _U, _U, _P, _P]
    L.or_eval.restype = _D
    L.or_eval.argtypes = [_I, _P, _I, _P, _I]
    L.or_elliptic_weights.restype = None
    L.or_elliptic_weights.argtypes = [_I, _P]
    L.or_run_updates.restype = _I
    L.or_run_updates.argtypes = [_P, _P, _P, _P, _P, _P, _P, _I, _I, _U, _U, _I, _D, _D, _D, _D, _D, _D, _D, _I,
                                 _P, _I, C.c_int]
    L.or_argsort_stable.restype = None
    L.or_argsort_stable.argtypes = [_P, _I, _P]
    L.or_select_dr.restype = _I
    L.or_select_dr.argtypes = [_U, _U, _I, _D, _P, _P, _P]
    L.or_initialize.restype = None
    L.or_initialize.argtypes = [_U, _I, _I, _D, _D, _I, _P, _I, _P, _P]
    L.or_step.restype = _I
    L.or_step.argtypes = [_P, _P, _P, _P, _I, _I, _I, _I, _U, _I, _D, _D, _D, _D, _I, _P, _I, C.c_int, _P]
    L.or_run.restype = None
    L.or_run.argtypes = [_I, _I, _I, _I, _U, _I, _D, _D, _D, _D, _I, _P, _I, C.c_int, _P, _P, _P, _P]
    L.or_run_many.restype = None
    L.or_run_many.argtypes = [_I, _P, _P, _P, _P, _I, _I, _I, _I, _D, _D, _D, _D, C.c_int, _P, _P]
    for name, spec in _EXTRA_DECLS.items():
        if hasattr(L, name):
            fn = getattr(L, name)
            fn.restype, fn.argtypes = spec


_EXTRA_DECLS: dict = {
    "or_cec_eval_batch": (None, [C.c_int, _P, _I, C.c_int, _P, _P, _P, _P, C.c_int]),
    "or_cec_spec": (None, [C.c_int, _P]),
    "or_cec_basic_batch": (None, [C.c_int, _P, _I, C.c_int, _P]),
    "or_cec_ncomp": (C.c_int, [C.c_int]),
    "or_threshold_tables": (None, [_P, C.c_int, _P]),
    "or_threshold_eval": (C.c_double, [C.c_int, _P, _I, _P]),
}


def threshold_tables(counts, method: str) -> np.ndarray:
    """Prefix tables of a 256-bin histogram (threshold_oracle.c layout): method 'otsu' or 'kapur'."""
    c = np.ascontiguousarray(counts, dtype=np.int64)
    tab = np.zeros(515)
    lib().or_threshold_tables(_ptr(c), 0 if method == "otsu" else 1, _ptr(tab))
    return tab


def threshold_eval(method: str, x, tab) -> float:
    x = _f64(np.atleast_1d(x))
    return float(lib().or_threshold_eval(0 if method == "otsu" else 1, _ptr(x), x.size, _ptr(_f64(tab))))


def cec_eval(fn: int, x, nthreads: int = 1) -> np.ndarray:
    """CEC2022 F_fn on every row of x (CPU restatement, cec_oracle.c)."""
    from paper_2510_14982_b200.cec2022 import cec_data

    x = _f64(np.atleast_2d(x))
    rows, dim = x.shape
    shift, rot, shuffle = cec_data(fn, dim)
    sh = np.ascontiguousarray(shift)
    ro = np.ascontiguousarray(rot)
    su = np.ascontiguousarray(shuffle, dtype=np.int32)
    out = np.zeros(rows)
    lib().or_cec_eval_batch(fn, _ptr(x), rows, dim, _ptr(sh), _ptr(ro), _ptr(su), _ptr(out), nthreads)
    return out


CEC_BASIC = {"zakharov": 0, "rosenbrock": 1, "escaffer6": 2, "rastrigin": 3, "step_rastrigin": 4, "levy": 5,
             "bent_cigar": 6, "discus": 7, "ellips": 8, "hgbat": 9, "happycat": 10, "katsuura": 11, "ackley": 12,
             "schwefel": 13, "schaffer_f7": 14, "grie_rosen": 15, "griewank": 16}


def cec_basic(name: str, z) -> np.ndarray:
    """A CEC2022 basic function alone (cec_oracle.c cec_basic_eval) on every row of z, no shift/scale."""
    z = _f64(np.atleast_2d(z))
    out = np.zeros(z.shape[0])
    lib().or_cec_basic_batch(CEC_BASIC[name], _ptr(z), z.shape[0], z.shape[1], _ptr(out))
    return out


def cec_spec(fn: int) -> np.ndarray:
    out = np.zeros(3 + 36)
    lib().or_cec_spec(fn, _ptr(out))
    return out


def _ptr(a):
    return C.c_void_p(a.ctypes.data) if a is not None and a.size else C.c_void_p(0)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ---------------------------------------------------------------------------
# RNG (rng.py:79-156)


def stream_base(seed: int, iteration: int, individual: int) -> int:
    return int(lib().or_stream_base(seed, iteration, individual))


def draw_bits(seed, iteration, individual, counter) -> int:
    return int(lib().or_mix(stream_base(seed, iteration, individual) ^ (counter & ((1 << 64) - 1))))


def draw_uniform(seed, iteration, individual, counter) -> float:
    return float(lib().or_u(stream_base(seed, iteration, individual), counter & ((1 << 64) - 1)))


def randperm(n: int, k: int, seed: int, iteration: int, individual: int, counter: int) -> np.ndarray:
    out = np.zeros(max(k, 1), dtype=np.int64)
    scratch = np.zeros(max(n, 1), dtype=np.int64)
    lib().or_randperm(n, k, stream_base(seed, iteration, individual), counter, _ptr(out), _ptr(scratch))
    return out[:k]


# ---------------------------------------------------------------------------
# objectives


def elliptic_weights(dim: int) -> np.ndarray:
    w = np.zeros(dim)
    lib().or_elliptic_weights(dim, _ptr(w))
    return w


def cec_packed(fn: int, dim: int, data_seed: int = 2022):
    """Packed CEC2022 data [shift | rot | shuffle] for or_eval codes 100+F."""
    from paper_2510_14982_b200.cec2022 import cec_data  # data synthesis only (numpy)

    shift, rot, shuffle = cec_data(fn, dim, data_seed)
    return np.concatenate([shift.ravel(), rot.ravel(), shuffle.astype(np.float64)])


def objective_table(name: str, dim: int, table=None):
    """(code, table) the kernels read for a reference objective name."""
    if name.startswith("cec2022_f"):
        fn = int(name[len("cec2022_f"):])
        return 100 + fn, cec_packed(fn, dim)
    code = CODES[name]
    if code in (7, 8):
        return code, _f64(table)
    if code == 2:
        return code, elliptic_weights(dim)
    if code == 6:
        return code, _f64(table)
    return code, np.zeros(1)


def evaluate(name: str, x, table=None) -> float:
    x = _f64(x)
    code, tab = objective_table(name, x.size, table)
    return float(lib().or_eval(code, _ptr(x), x.size, _ptr(tab), tab.size))


# ---------------------------------------------------------------------------
# engine pieces


def schedules(iteration: int, max_iterations: int):
    """(p_ah, f_mult, decay) exactly as numba_backend.py:357-366 computes them."""
    span = max(max_iterations - 1, 1)
    ratio = iteration / span
    return 0.5 * (1.0 + math.cos(ratio * math.pi)), 1.0 + math.cos(ratio * math.pi), 1.0 - ratio


def run_updates(positions, fitness, in_dr, *, seed, iteration, max_iterations, name, lower, upper, npairs=1,
                eps=2.0 ** -52, table=None, key_iteration=None, nthreads=1):
    """numba_backend.run_updates (numba_backend.py:323-372) -> (pos, fit, acc, warn, nwarn)."""
    pos = _f64(positions)
    fit = _f64(fitness)
    ps, dim = pos.shape
    dr = np.ascontiguousarray(in_dr, dtype=np.uint8)
    code, tab = objective_table(name, dim, table)
    p_ah, f_mult, decay = schedules(iteration, max_iterations)
    out_pos = np.empty_like(pos)
    out_fit = np.empty(ps)
    acc = np.zeros(ps, dtype=np.uint8)
    warn = np.zeros(ps, dtype=np.uint8)
    kit = iteration + 1 if key_iteration is None else key_iteration
    nw = lib().or_run_updates(_ptr(pos), _ptr(fit), _ptr(dr), _ptr(out_pos), _ptr(out_fit), _ptr(acc), _ptr(warn),
                              ps, dim, seed, kit, npairs, lower, upper, upper - lower, eps, p_ah, f_mult, decay,
                              code, _ptr(tab), tab.size, nthreads)
    return out_pos, out_fit, acc.astype(bool), warn.astype(bool), int(nw)


def argsort_stable(key) -> np.ndarray:
    key = _f64(key)
    out = np.zeros(max(key.size, 1), dtype=np.int64)
    lib().or_argsort_stable(_ptr(key), key.size, _ptr(out))
    return out[:key.size]


def select_dr(seed: int, key_iteration: int, ps: int, pf_max: float) -> np.ndarray:
    in_dr = np.zeros(ps, dtype=np.uint8)
    scratch = np.zeros(ps, dtype=np.int64)
    sel = np.zeros(ps, dtype=np.int64)
    lib().or_select_dr(seed, key_iteration, ps, pf_max, _ptr(in_dr), _ptr(scratch), _ptr(sel))
    return in_dr.astype(bool)


def initialize(seed, ps, dim, lower, upper, name, table=None):
    code, tab = objective_table(name, dim, table)
    pos = np.zeros((ps, dim))
    fit = np.zeros(ps)
    lib().or_initialize(seed, ps, dim, lower, upper - lower, code, _ptr(tab), tab.size, _ptr(pos), _ptr(fit))
    return pos, fit


def step(positions, fitness, *, seed, iteration, max_iterations, name, lower, upper, npairs=1, pf_max=0.1,
         eps=2.0 ** -52, table=None, nthreads=1):
    pos = _f64(positions)
    fit = _f64(fitness)
    ps, dim = pos.shape
    code, tab = objective_table(name, dim, table)
    out_pos = np.empty_like(pos)
    out_fit = np.empty(ps)
    in_dr = np.zeros(ps, dtype=np.uint8)
    nw = lib().or_step(_ptr(pos), _ptr(fit), _ptr(out_pos), _ptr(out_fit), ps, dim, max_iterations, iteration, seed,
                       npairs, pf_max, lower, upper, eps, code, _ptr(tab), tab.size, nthreads, _ptr(in_dr))
    return out_pos, out_fit, int(nw), in_dr.astype(bool)


def run(*, ps, dim, max_iterations, seed, name, lower, upper, npairs=1, pf_max=0.1, eps=2.0 ** -52, max_fes=None,
        table=None, nthreads=1):
    """engine.run (engine.py:175-212): dict with trace, final population, counters, best."""
    code, tab = objective_table(name, dim, table)
    pos = np.zeros((ps, dim))
    fit = np.zeros(ps)
    trace = np.zeros(max_iterations + 1)
    out = np.zeros(4, dtype=np.int64)
    lib().or_run(ps, dim, max_iterations, 0 if max_fes is None else max_fes, seed, npairs, pf_max, lower, upper, eps,
                 code, _ptr(tab), tab.size, nthreads, _ptr(pos), _ptr(fit), _ptr(trace), _ptr(out))
    it = int(out[0])
    return dict(positions=pos, fitness=fit, trace=trace[:it + 1], iterations_run=it, fe_count=int(out[1]),
                warnings=int(out[2]), best_index=int(out[3]), best_fitness=float(fit[out[3]]),
                best_position=pos[out[3]].copy())


def run_many(names, seeds, *, ps, dim, max_iterations, lower, upper, npairs=1, pf_max=0.1, eps=2.0 ** -52,
             nthreads=None, tables=None):
    """Independent runs, one per thread -> (best fitness per run, fe per run)."""
    n = len(names)
    codes = np.zeros(n, dtype=np.int64)
    tabs = []
    for r, name in enumerate(names):
        codes[r], t = objective_table(name, dim, None if tables is None else tables[r])
        tabs.append(t)
    tab_ptrs = (C.c_void_p * n)(*[t.ctypes.data for t in tabs])
    tlens = np.array([t.size for t in tabs], dtype=np.int64)
    sd = np.array(seeds, dtype=np.uint64)
    best = np.zeros(n)
    fe = np.zeros(n, dtype=np.int64)
    lib().or_run_many(n, _ptr(codes), _ptr(sd), C.cast(tab_ptrs, C.c_void_p), _ptr(tlens), ps, dim, max_iterations,
                      npairs, pf_max, lower, upper, eps, nthreads or (os.cpu_count() or 1), _ptr(best), _ptr(fe))
    return best, fe
