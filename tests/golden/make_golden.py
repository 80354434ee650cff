"""Generate golden vectors by running the REFERENCE package itself.

Run in the build container (the reference is mounted read-only at
/root/reference; it does not exist on the GPU box, so the vectors are
committed as small .npz fixtures next to this script):

    NUMBA_CACHE_DIR=/tmp/numba_cache python tests/golden/make_golden.py

Everything here calls the reference's public API (`protozoa.run`,
`protozoa.step`, `protozoa.initialize`, `protozoa.rng`, `protozoa.core`,
`protozoa.imaging`) with its default numba backend, and records inputs and
outputs.  The oracle (oracle/apo_oracle.c) is pinned against these files by
tests/test_oracle_golden.py and the CUDA path by tests/test_gpu_parity.py.
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_cache_golden")
sys.path.insert(0, REF)

import protozoa as pz  # noqa: E402
from protozoa import core, engine, rng  # noqa: E402
from protozoa.kernels import get_backend  # noqa: E402


def kats():
    keys = [
        (0, 0, 0, 0),
        (1, 0, 0, 0),
        (42, 3, 17, 1000),
        (0xDEADBEEF, 1, rng.COORDINATOR_INDEX, 2**33 + 5),
        (2**64 - 1, 2**64 - 1, 2**64 - 1, 2**64 - 1),
        (0, 1, 1, 8),
        (7, 2, 5, 2**32),
    ]
    r = np.random.default_rng(7)
    for _ in range(64):
        keys.append(tuple(int(v) for v in r.integers(0, 2**63, size=4, dtype=np.uint64)))
    bits = [rng.draw_bits(rng.StreamKey(*k)) for k in keys]
    us = [rng.draw_uniform(rng.StreamKey(*k)) for k in keys]
    perms = []
    for (n, k, seed, it, ctr) in [(10, 4, 3, 1, 1), (100, 100, 9, 5, 0), (1000, 37, 1, 2, 7), (1, 1, 0, 0, 0)]:
        perms.append(dict(n=n, k=k, seed=seed, it=it, ctr=ctr,
                          out=rng.randperm(n, k, rng.StreamKey(seed, it, rng.COORDINATOR_INDEX, ctr)).tolist()))
    coord = []
    for (seed, it, ps, pf_max) in [(0, 1, 100, 0.1), (0, 1, 100, 0.05), (5, 17, 1000, 0.1), (123, 999, 50, 1.0)]:
        key = rng.StreamKey(seed, it, rng.COORDINATOR_INDEX)
        pf = core.proportion_fraction(key, pf_max)
        dr = core.select_dr_indices(ps, pf, key)
        coord.append(dict(seed=seed, it=it, ps=ps, pf_max=pf_max, pf=pf, dr=dr.tolist()))
    fixed_dr = core.select_dr_indices(100, 0.05, rng.StreamKey(0, 1, rng.COORDINATOR_INDEX)).tolist()
    return dict(
        keys=[[str(v) for v in k] for k in keys],
        bits=[str(b) for b in bits],
        u=[float(x).hex() for x in us],
        randperm=perms,
        coordinator=coord,
        select_dr_100_005=fixed_dr,
    )


def objective_vectors():
    out = {}
    r = np.random.default_rng(11)
    for name in pz.FUNCTION_NAMES:
        obj = pz.get_objective(name)
        pts, vals = [], []
        for dim in (2, 3, 10, 20, 100):
            for _ in range(8):
                x = r.uniform(-100, 100, size=dim)
                pts.append(x)
                vals.append(pz.evaluate(obj, x))
        out[name] = (pts, np.array(vals))
    return out


STEP_CASES = [
    # (name, objective, ps, dim, T, seed, npairs, pf_max, lower, upper, steps)
    ("sphere_small", "sphere", 12, 4, 15, 3, 1, 0.1, -50.0, 50.0, 6),
    ("griewank_ps1", "griewank", 1, 3, 5, 9, 1, 0.1, -30.0, 30.0, 4),
    ("bent_cigar_d10", "bent_cigar", 50, 10, 1000, 0, 1, 0.1, -100.0, 100.0, 4),
    ("elliptic_np3", "high_conditioned_elliptic", 40, 7, 50, 17, 3, 0.3, -100.0, 100.0, 5),
    ("hgbat_pf1", "hgbat", 33, 5, 20, 5, 2, 1.0, -10.0, 10.0, 5),
    ("rosenbrock_d20", "rosenbrock", 100, 20, 1000, 1, 1, 0.1, -100.0, 100.0, 4),
    ("griewank_d20", "griewank", 100, 20, 200, 2, 1, 0.1, -100.0, 100.0, 4),
    ("sphere_d1", "sphere", 17, 1, 9, 4, 1, 0.1, -5.0, 5.0, 5),
    ("sphere_last_iter", "sphere", 20, 6, 3, 8, 1, 0.1, -1.0, 2.0, 3),
]


def step_cases():
    out = {}
    for (name, objname, ps, dim, T, seed, npairs, pf_max, lo, hi, steps) in STEP_CASES:
        cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T,
                           neighbor_pairs=npairs, pf_max=pf_max, seed=seed)
        obj = pz.get_objective(objname)
        pop = pz.initialize(cfg, obj)
        rec = dict(init_pos=pop.positions.copy(), init_fit=pop.fitness.copy())
        snaps_pos, snaps_fit, in_drs, outs_pos, outs_fit, accs, warns = [], [], [], [], [], [], []
        bk = get_backend("numba")
        for t in range(steps):
            snap = core.sort_by_fitness(pop)
            coord = rng.StreamKey(cfg.seed, t + 1, rng.COORDINATOR_INDEX)
            pf = core.proportion_fraction(coord, cfg.pf_max)
            dr = core.select_dr_indices(cfg.ps, pf, coord)
            in_dr = np.zeros(cfg.ps, dtype=bool)
            if dr.size:
                in_dr[dr - 1] = True
            new_pos, new_fit, acc, warned = bk.run_updates(snap.positions, snap.fitness, in_dr, cfg, obj, t, t + 1,
                                                           parallel=False, workers=1)
            stepped = pz.step(pop, cfg, obj, t, pz.EngineMode.sequential())
            assert np.array_equal(stepped.positions, new_pos)
            snaps_pos.append(snap.positions)
            snaps_fit.append(snap.fitness)
            in_drs.append(in_dr)
            outs_pos.append(new_pos)
            outs_fit.append(new_fit)
            accs.append(acc)
            warns.append(warned)
            pop = stepped
        rec.update(snap_pos=np.array(snaps_pos), snap_fit=np.array(snaps_fit), in_dr=np.array(in_drs),
                   out_pos=np.array(outs_pos), out_fit=np.array(outs_fit), acc=np.array(accs),
                   warn=np.array(warns))
        rec["cfg"] = np.array([ps, dim, T, seed, npairs, steps], dtype=np.int64)
        rec["cfgf"] = np.array([pf_max, lo, hi, cfg.eps])
        out[name] = (objname, rec)
    return out


RUN_CASES = [
    # (name, objective, ps, dim, T, seed, lower, upper, max_fes)
    ("c1_sphere_d10", "sphere", 50, 10, 1000, 0, -100.0, 100.0, None),
    ("c1_bent_cigar_d10", "bent_cigar", 50, 10, 1000, 0, -100.0, 100.0, None),
    ("c2_rosenbrock_d20", "rosenbrock", 100, 20, 300, 3, -100.0, 100.0, None),
    ("c2_hgbat_d20", "hgbat", 100, 20, 300, 4, -100.0, 100.0, None),
    ("c2_elliptic_d20", "high_conditioned_elliptic", 100, 20, 300, 5, -100.0, 100.0, None),
    ("c2_griewank_d20", "griewank", 100, 20, 300, 6, -100.0, 100.0, None),
    ("budget_sphere", "sphere", 30, 5, 100, 1, -10.0, 10.0, 455),
]


def run_cases():
    out = {}
    for (name, objname, ps, dim, T, seed, lo, hi, max_fes) in RUN_CASES:
        cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T, seed=seed,
                           max_fes=max_fes)
        res = pz.run(cfg, objname)
        out[name] = (objname, dict(
            trace=res.trace, best_fitness=np.array(res.best_fitness), best_position=res.best_position,
            final_pos=res.population.positions, final_fit=res.population.fitness,
            counters=np.array([res.iterations_run, res.fe_count, res.warnings], dtype=np.int64),
            cfg=np.array([ps, dim, T, seed, -1 if max_fes is None else max_fes], dtype=np.int64),
            cfgf=np.array([lo, hi]),
        ))
    return out


def threshold_cases():
    r = np.random.default_rng(0)
    n = 256 * 256
    vals = np.concatenate([r.normal(70, 12, n // 2), r.normal(190, 14, n - n // 2)])
    img = pz.GrayImage(np.clip(np.round(vals), 0, 255).astype(np.uint8).reshape(256, 256))
    hist = pz.histogram(img)
    from protozoa.imaging import variance_table
    table = variance_table(hist)
    bt, bv = pz.brute_force_otsu(hist)
    res = pz.apo_threshold(img, ps=100, iterations=50, seed=0)
    return dict(pixels=img.pixels, counts=hist.counts, table=table, brute=np.array([bt, bv]),
                apo_t=np.array(res.threshold), apo_var=np.array(res.variance), apo_trace=res.run.trace)


def main():
    meta = kats()
    with open(os.path.join(HERE, "rng_kats.json"), "w") as fh:
        json.dump(meta, fh, indent=1)
    objs = objective_vectors()
    arrs = {}
    for name, (pts, vals) in objs.items():
        for k, p in enumerate(pts):
            arrs[f"{name}/x{k}"] = p
        arrs[f"{name}/f"] = vals
    np.savez_compressed(os.path.join(HERE, "objectives.npz"), **arrs)
    steps = step_cases()
    arrs = {}
    for name, (objname, rec) in steps.items():
        arrs[f"{name}/objective"] = np.array(objname)
        for k, v in rec.items():
            arrs[f"{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "steps.npz"), **arrs)
    runs = run_cases()
    arrs = {}
    for name, (objname, rec) in runs.items():
        arrs[f"{name}/objective"] = np.array(objname)
        for k, v in rec.items():
            arrs[f"{name}/{k}"] = v
    np.savez_compressed(os.path.join(HERE, "runs.npz"), **arrs)
    np.savez_compressed(os.path.join(HERE, "threshold.npz"), **threshold_cases())
    for f in sorted(os.listdir(HERE)):
        print(f, os.path.getsize(os.path.join(HERE, f)))


if __name__ == "__main__":
    main()
