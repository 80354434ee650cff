"""CEC2022 F1-F12 (synthetic data): oracle known answers, GPU vs oracle.

PARITY UNPINNED against the reference (it has no CEC2022 functions,
SPEC.md:146).  What is pinned: F(o) = F* at the synthesised optimum (all 12
functions), and the CUDA evaluator against the C restatement
(oracle/cec_oracle.c) within 1e-9 relative (the GPU reduces with warp trees,
the oracle sequentially; transcendentals differ in the last ulp).
"""

import numpy as np
import pytest

import oracle
from paper_2510_14982_b200 import cec2022

RTOL = 1e-9


@pytest.mark.parametrize("fn", range(1, 13))
@pytest.mark.parametrize("dim", [10, 20, 100])
def test_oracle_optimum_is_fstar(fn, dim):
    o = cec2022.cec_data(fn, dim)[0][0]
    f = oracle.cec_eval(fn, o)[0]
    assert abs(f - cec2022.FSTAR[fn - 1]) < 1e-6


def test_data_is_deterministic_and_well_formed():
    for fn in (1, 6, 9, 12):
        a = cec2022.cec_data(fn, 20)
        cec2022.cec_data.cache_clear()
        b = cec2022.cec_data(fn, 20)
        for x, y in zip(a, b):
            assert np.array_equal(x, y)
        shift, rot, shuffle = a
        assert shift.shape == (cec2022.NCOMP[fn - 1], 20) and np.all(np.abs(shift) <= 80)
        for m in rot:
            np.testing.assert_allclose(m @ m.T, np.eye(20), atol=1e-12)
        assert sorted(shuffle.tolist()) == list(range(1, 21))


def test_names_resolve_and_stay_out_of_function_names():
    import paper_2510_14982_b200 as pz

    assert pz.get_objective("cec2022_f10").code == 110
    assert pz.get_objective("F6").code == 106
    assert len(pz.FUNCTION_NAMES) == 6 and "cec2022_f1" not in pz.FUNCTION_NAMES
    assert pz.get_objective("cec2022_f7").min_dim == 5


def test_oracle_values_are_finite_and_above_fstar_nearby():
    rnd = np.random.default_rng(0)
    for fn in range(1, 13):
        x = rnd.uniform(-100, 100, size=(16, 20))
        f = oracle.cec_eval(fn, x)
        assert np.all(np.isfinite(f)) and np.all(f >= cec2022.FSTAR[fn - 1] - 1e-6)


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("dim", [10, 20, 50, 100])
def test_device_eval_matches_oracle(dim):
    import paper_2510_14982_b200 as pz

    rnd = np.random.default_rng(dim)
    for fn in range(1, 13):
        x = rnd.uniform(-100, 100, size=(257, dim))
        x[0] = cec2022.cec_data(fn, dim)[0][0]  # the optimum
        got = pz.evaluate_batch(f"cec2022_f{fn}", x)
        want = oracle.cec_eval(fn, x, nthreads=8)
        np.testing.assert_allclose(got, want, rtol=RTOL, err_msg=f"F{fn} D={dim}")


@pytest.mark.gpu
@pytest.mark.parametrize("fn", [1, 4, 6, 7, 10, 12])
def test_teacher_forced_step_matches_oracle(fn):
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.kernels import get_backend

    name = f"cec2022_f{fn}"
    for ps, dim in ((100, 20), (3000, 50), (2000, 100), (300, 12), (700, 150), (260, 300)):
        cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=50, seed=fn)
        pos, fit = oracle.initialize(fn, ps, dim, -100.0, 100.0, name)
        order = oracle.argsort_stable(fit)
        sp, sf = pos[order], fit[order]
        in_dr = oracle.select_dr(fn, 4, ps, 0.1)
        want = oracle.run_updates(sp, sf, in_dr, seed=fn, iteration=3, max_iterations=50, name=name,
                                  lower=-100.0, upper=100.0, nthreads=8)
        got = get_backend("cuda").run_updates(sp, sf, in_dr, cfg, pz.get_objective(name), 3, 4)
        # candidates are identical; acceptance may only differ on exact ties (plateaus of the step
        # Rastrigin etc.), where the oracle's old fitness and the GPU's new one differ in the last ulp
        agree = got[2] == want[2]
        assert agree.mean() > 0.99
        np.testing.assert_allclose(got[0][agree], want[0][agree], rtol=RTOL, atol=1e-12)
        np.testing.assert_allclose(got[1][agree], want[1][agree], rtol=RTOL)
        for k in np.flatnonzero(~agree):
            cand = got[0][k] if got[2][k] else want[0][k]
            assert abs(oracle.cec_eval(fn, cand)[0] - sf[k]) <= 1e-9 * abs(sf[k])


@pytest.mark.gpu
def test_suite_batch_matches_oracle_runs():
    """C2 shape (small): F1-F12 x 2 seeds, batched kernel vs the oracle's run loop."""
    import paper_2510_14982_b200 as pz

    names = [f"cec2022_f{k}" for k in range(1, 13)] * 2
    seeds = list(range(len(names)))
    cfg = pz.ApoConfig(ps=60, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=40)
    res = pz.run_batch(cfg, names, seeds)
    want, _ = oracle.run_many(names, seeds, ps=60, dim=20, max_iterations=40, lower=-100.0, upper=100.0)
    # free-running: a last-ulp difference at an exact fitness tie can send one run down a
    # different (equally valid) trajectory, so 90% of the runs must agree tightly and all loosely; the
    # teacher-forced suites (test_headline_parity.py) pin every individual step at 1e-9
    rel = np.abs(res.best_fitness - want) / np.abs(want)
    print("runs within 1e-9:", int(np.sum(rel <= 1e-9)), "of", len(rel))
    assert np.mean(rel <= 1e-9) >= 0.9
    assert np.all(rel <= 1e-2)


@pytest.mark.gpu
@pytest.mark.parametrize("fn", [1, 4, 6, 10])
def test_fma_rotation_path_matches_oracle(fn):
    """BASELINE config 5's comparison path: the same objective without DMMA tables rotates with
    lane-per-output FMAs (fused update kernel); it must agree with the oracle like the DMMA path."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.kernels import get_backend

    name = f"cec2022_f{fn}"
    ps, dim = 1500, 50
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=50, seed=fn)
    pos, fit = oracle.initialize(fn, ps, dim, -100.0, 100.0, name)
    order = oracle.argsort_stable(fit)
    sp, sf = pos[order], fit[order]
    in_dr = oracle.select_dr(fn, 4, ps, 0.1)
    want = oracle.run_updates(sp, sf, in_dr, seed=fn, iteration=3, max_iterations=50, name=name,
                              lower=-100.0, upper=100.0, nthreads=8)
    for rot in ("fma", "dmma"):
        got = get_backend("cuda").run_updates(sp, sf, in_dr, cfg, pz.cec2022_objective(fn, rotation=rot), 3, 4)
        agree = got[2] == want[2]
        assert agree.mean() > 0.99, rot
        np.testing.assert_allclose(got[1][agree], want[1][agree], rtol=RTOL)


@pytest.mark.gpu
@pytest.mark.parametrize("fn", [1, 6, 10])
def test_large_dim_gemm_device_loop_matches_dense_path(fn):
    """D > 104: the device loop (slot layout, per-slot buffer selectors) through the DMMA GEMM path
    equals the dense reference-facing path step for step."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine

    name = f"cec2022_f{fn}"
    cfg = pz.ApoConfig(ps=500, dim=300, bounds=pz.Bounds(-100.0, 100.0, 300), max_iterations=6, seed=fn)
    run = engine.DeviceRun(cfg, pz.get_objective(name))
    run.initialize()
    run.iterate(6)
    pos, fit = run.population()
    run.close()
    pop = pz.initialize(cfg, name)
    for t in range(6):
        pop = pz.step(pop, cfg, name, t)
    np.testing.assert_allclose(fit, pop.fitness, rtol=1e-12)
    np.testing.assert_allclose(pos, pop.positions, rtol=1e-12)
