"""Pin the CPU oracle (oracle/apo_oracle.c) to vectors the reference produced.

The golden files come from tests/golden/make_golden.py, which runs the
reference package (/root/reference/pkg/src/protozoa, numba backend).  Every
comparison here is bit-exact (np.array_equal / ==).
"""

import json
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN


@pytest.fixture(scope="module")
def kats():
    with open(os.path.join(GOLDEN, "rng_kats.json")) as fh:
        return json.load(fh)


def _groups(path):
    data = np.load(os.path.join(GOLDEN, path))
    groups = {}
    for key in data.files:
        name, field = key.split("/", 1)
        groups.setdefault(name, {})[field] = data[key]
    return groups


def test_rng_known_answers(kats):
    for key, bits, u in zip(kats["keys"], kats["bits"], kats["u"]):
        k = [int(v) for v in key]
        assert oracle.draw_bits(*k) == int(bits)
        assert oracle.draw_uniform(*k) == float.fromhex(u)


def test_survey_appendix_a_literals():
    # SURVEY.md Appendix A, printed from the reference (rng.py / core.py)
    assert oracle.draw_bits(0, 0, 0, 0) == 0x9065D5F9F9C1E615
    assert oracle.draw_uniform(0, 1, 1, 8) == 0.16433925735629307
    assert oracle.randperm(10, 4, 3, 1, oracle.COORDINATOR_INDEX, 1).tolist() == [7, 6, 4, 3]


def test_randperm_and_coordinator(kats):
    for p in kats["randperm"]:
        got = oracle.randperm(p["n"], p["k"], p["seed"], p["it"], oracle.COORDINATOR_INDEX, p["ctr"])
        assert got.tolist() == p["out"]
    for c in kats["coordinator"]:
        in_dr = oracle.select_dr(c["seed"], c["it"], c["ps"], c["pf_max"])
        want = np.zeros(c["ps"], dtype=bool)
        want[np.array(c["dr"], dtype=np.int64) - 1] = True
        assert np.array_equal(in_dr, want)


def test_objectives_bit_exact():
    data = np.load(os.path.join(GOLDEN, "objectives.npz"))
    names = sorted({k.split("/")[0] for k in data.files})
    assert len(names) == 6
    for name in names:
        vals = data[f"{name}/f"]
        for k, want in enumerate(vals):
            x = data[f"{name}/x{k}"]
            assert oracle.evaluate(name, x) == want, (name, k)


@pytest.mark.parametrize("case", sorted(_groups("steps.npz")))
def test_run_updates_teacher_forced(case):
    g = _groups("steps.npz")[case]
    ps, dim, T, seed, npairs, steps = (int(v) for v in g["cfg"])
    pf_max, lo, hi, eps = (float(v) for v in g["cfgf"])
    name = str(g["objective"])
    pos, fit = oracle.initialize(seed, ps, dim, lo, hi, name)
    assert np.array_equal(pos, g["init_pos"]) and np.array_equal(fit, g["init_fit"])
    for t in range(steps):
        order = oracle.argsort_stable(fit if t == 0 else g["out_fit"][t - 1])
        src_pos = pos if t == 0 else g["out_pos"][t - 1]
        src_fit = fit if t == 0 else g["out_fit"][t - 1]
        assert np.array_equal(src_pos[order], g["snap_pos"][t])
        assert np.array_equal(src_fit[order], g["snap_fit"][t])
        in_dr = oracle.select_dr(seed, t + 1, ps, pf_max)
        assert np.array_equal(in_dr, g["in_dr"][t])
        op, of, acc, warn, nw = oracle.run_updates(g["snap_pos"][t], g["snap_fit"][t], g["in_dr"][t], seed=seed,
                                                   iteration=t, max_iterations=T, name=name, lower=lo, upper=hi,
                                                   npairs=npairs, eps=eps)
        assert np.array_equal(op, g["out_pos"][t])
        assert np.array_equal(of, g["out_fit"][t])
        assert np.array_equal(acc, g["acc"][t])
        assert nw == int(g["warn"][t])
        op2, of2, nw2, _ = oracle.step(src_pos, src_fit, seed=seed, iteration=t, max_iterations=T, name=name,
                                       lower=lo, upper=hi, npairs=npairs, pf_max=pf_max, eps=eps, nthreads=3)
        assert np.array_equal(op2, g["out_pos"][t]) and np.array_equal(of2, g["out_fit"][t])


@pytest.mark.parametrize("case", sorted(_groups("runs.npz")))
def test_full_runs(case):
    g = _groups("runs.npz")[case]
    ps, dim, T, seed, max_fes = (int(v) for v in g["cfg"])
    lo, hi = (float(v) for v in g["cfgf"])
    res = oracle.run(ps=ps, dim=dim, max_iterations=T, seed=seed, name=str(g["objective"]), lower=lo, upper=hi,
                     max_fes=None if max_fes < 0 else max_fes, nthreads=2)
    assert np.array_equal(res["trace"], g["trace"])
    assert np.array_equal(res["positions"], g["final_pos"])
    assert np.array_equal(res["fitness"], g["final_fit"])
    assert res["best_fitness"] == float(g["best_fitness"])
    assert np.array_equal(res["best_position"], g["best_position"])
    assert [res["iterations_run"], res["fe_count"], res["warnings"]] == g["counters"].tolist()
