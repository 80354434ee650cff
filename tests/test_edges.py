"""Edge cases of the update path against the oracle (bit-exact): a one-protozoon population on every
path, non-finite fitness and rows in a step's input, the largest dimension the warp kernel takes.

The reference guards the same corners: ps = 1 has no partner but itself (core.py:300-313,
numba_backend.py:176-186), numpy's stable argsort puts NaN last (core.py:504-513) and non-finite
candidates count as warnings without being accepted (numba_backend.py:270-290)."""

import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


def _same(a, b):
    return np.array_equal(a, b, equal_nan=True)


@pytest.mark.parametrize("name,dim", [("sphere", 1), ("griewank", 5), ("rosenbrock", 40), ("hgbat", 300),
                                      ("cec2022_f6", 20)])
@pytest.mark.parametrize("path", ["batch", "device"])
def test_single_protozoon_runs(name, dim, path, monkeypatch):
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine

    if path == "device":
        monkeypatch.setattr(engine, "BATCH_PS_LIMIT", 0)
    cfg = pz.ApoConfig(ps=1, dim=dim, bounds=pz.Bounds(-10.0, 10.0, dim), max_iterations=30, seed=17)
    res = pz.run(cfg, name)
    want = oracle.run(ps=1, dim=dim, max_iterations=30, seed=17, name=name, lower=-10.0, upper=10.0)
    if name.startswith("cec2022"):  # CEC2022: 1e-9 (DMMA vs sequential sums), decisions identical
        np.testing.assert_allclose(res.trace, want["trace"], rtol=1e-9)
        np.testing.assert_allclose(res.population.positions, want["positions"], rtol=1e-9, atol=1e-12)
    else:
        assert np.array_equal(res.trace, want["trace"])
        assert np.array_equal(res.population.positions, want["positions"])
        assert np.array_equal(res.population.fitness, want["fitness"])
    assert res.warnings == want["warnings"]


@pytest.mark.parametrize("ps,dim", [(1, 3), (2, 1), (3, 300)])
def test_tiny_population_step(ps, dim):
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-4.0, 6.0, dim), max_iterations=9, seed=3, pf_max=1.0)
    pop = pz.initialize(cfg, "sphere")
    for t in range(4):
        got = pz.step(pop, cfg, "sphere", t)
        pos, fit, nw, _ = oracle.step(pop.positions, pop.fitness, seed=3, iteration=t, max_iterations=9,
                                      name="sphere", lower=-4.0, upper=6.0, pf_max=1.0)
        assert np.array_equal(got.positions, pos) and np.array_equal(got.fitness, fit)
        assert got.warnings - pop.warnings == nw
        pop = got


@pytest.mark.parametrize("name,dim", [("rosenbrock", 7), ("griewank", 40), ("sphere", 300)])
def test_non_finite_input_population(name, dim):
    """NaN / +-inf fitness values and NaN / inf rows in the step's input: the stable sort puts NaN last and
    -inf first, candidates built from non-finite rows are warnings, never accepted -- as the oracle does."""
    import paper_2510_14982_b200 as pz

    ps = 200
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-5.0, 5.0, dim), max_iterations=12, seed=8, pf_max=0.5)
    pop = pz.initialize(cfg, name)
    pos, fit = pop.positions.copy(), pop.fitness.copy()
    fit[[3, 50, 51]] = np.nan
    fit[[7, 120]] = np.inf
    fit[[9]] = -np.inf
    pos[11, 0] = np.nan
    pos[12, -1] = np.inf
    fit[[11, 12]] = 1.0  # finite fitness on non-finite rows: they sort into the middle and get partners
    bad = pz.Population(pos, fit, iteration=4, fe_count=5 * ps)
    for t in (4, 5):
        got = pz.step(bad, cfg, name, t)
        wpos, wfit, nw, _ = oracle.step(bad.positions, bad.fitness, seed=8, iteration=t, max_iterations=12,
                                        name=name, lower=-5.0, upper=5.0, pf_max=0.5)
        assert _same(got.positions, wpos) and _same(got.fitness, wfit)
        assert got.warnings - bad.warnings == nw and nw > 0
        bad = got


def test_largest_dimension_warp_kernel():
    """apo_max_dim() (one warp's shared-memory scratch fits a CTA), the warp-per-protozoon kernel's limit:
    one step bit-exact; one more is rejected loudly."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import _lib

    ps, dim = 40, int(_lib.load().apo_max_dim())
    assert 6000 <= dim <= 8192
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-1.0, 1.0, dim), max_iterations=5, seed=1)
    pop = pz.initialize(cfg, "griewank")
    got = pz.step(pop, cfg, "griewank", 2)
    pos, fit, nw, _ = oracle.step(pop.positions, pop.fitness, seed=1, iteration=2, max_iterations=5,
                                  name="griewank", lower=-1.0, upper=1.0)
    assert np.array_equal(got.positions, pos) and np.array_equal(got.fitness, fit) and got.warnings == nw
    d1 = dim + 1
    big = pz.ApoConfig(ps=4, dim=d1, bounds=pz.Bounds(-1.0, 1.0, d1), max_iterations=5, seed=1)
    with pytest.raises(Exception, match="dim"):
        pz.step(pz.Population(np.zeros((4, d1)), np.zeros(4), iteration=0, fe_count=4), big, "sphere", 0)
    with pytest.raises(Exception, match="dim"):
        pz.initialize(big, "sphere")


@pytest.mark.parametrize("npairs,dim", [(9, 10), (20, 40), (12, 300)])
def test_many_neighbour_pairs(npairs, dim, monkeypatch):
    """More neighbour pairs than the kernels cache (kMaxCachedPairs = 8): pairs k >= 8 are drawn on the
    fly per dimension (numba_backend.py:200-240); runs on the batch and device paths and a step, bit-exact."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine

    ps = 50
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-3.0, 7.0, dim), max_iterations=8, seed=21,
                       neighbor_pairs=npairs)
    want = oracle.run(ps=ps, dim=dim, max_iterations=8, seed=21, name="rosenbrock", lower=-3.0, upper=7.0,
                      npairs=npairs, nthreads=8)
    for limit in (engine.BATCH_PS_LIMIT, 0):
        monkeypatch.setattr(engine, "BATCH_PS_LIMIT", limit)
        res = pz.run(cfg, "rosenbrock")
        assert np.array_equal(res.trace, want["trace"]) and np.array_equal(res.population.positions, want["positions"])
    pop = pz.initialize(cfg, "rosenbrock")
    got = pz.step(pop, cfg, "rosenbrock", 3)
    pos, fit, nw, _ = oracle.step(pop.positions, pop.fitness, seed=21, iteration=3, max_iterations=8,
                                  name="rosenbrock", lower=-3.0, upper=7.0, npairs=npairs)
    assert np.array_equal(got.positions, pos) and np.array_equal(got.fitness, fit)
