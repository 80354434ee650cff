"""Checkpoint / resume of a run (the reference has none).

Every draw is keyed by (seed, iteration, individual, slot) (rng.py:1-19), so a
run resumed from a checkpointed Population must equal the uninterrupted run
bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu  # every test here needs the device


@pytest.mark.parametrize("name,ps,dim", [("rosenbrock", 500, 20), ("sphere", 3000, 64), ("cec2022_f6", 3000, 50)])
def test_resume_equals_uninterrupted_run(name, ps, dim, monkeypatch):
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine

    monkeypatch.setattr(engine, "BATCH_PS_LIMIT", 0)  # the device-resident loop
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=40, seed=5)
    full = pz.run(cfg, name)
    pop = pz.initialize(cfg, name)
    for t in range(17):  # checkpoint after 17 iterations of the same 40-iteration schedule
        pop = pz.step(pop, cfg, name, t)
    res = pz.resume(cfg, name, pop)
    assert res.iterations_run == 40 and res.fe_count == full.fe_count and res.warnings == full.warnings
    assert np.array_equal(res.population.positions, full.population.positions)
    assert np.array_equal(res.population.fitness, full.population.fitness)
    assert np.array_equal(res.trace, full.trace[17:])
    assert res.best_fitness == full.best_fitness and np.array_equal(res.best_position, full.best_position)


def test_resume_rejects_mismatched_population():
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=64, dim=8, bounds=pz.Bounds(-1.0, 1.0, 8), max_iterations=10)
    bad = pz.Population(np.zeros((32, 8)), np.zeros(32), iteration=2, fe_count=96)
    with pytest.raises(ValueError):
        pz.resume(cfg, "sphere", bad)


@pytest.mark.parametrize("name,ps,dim", [("rosenbrock", 600, 40), ("griewank", 300, 20)])
def test_resume_equals_oracle_run(name, ps, dim, monkeypatch):
    """A run checkpointed after 13 iterations (reference row order Population) and resumed on the device
    equals the oracle's uninterrupted run of the reference loop (engine.py:175-212) bit for bit."""
    import oracle
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine

    monkeypatch.setattr(engine, "BATCH_PS_LIMIT", 0)
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-30.0, 30.0, dim), max_iterations=30, seed=8)
    want = oracle.run(ps=ps, dim=dim, max_iterations=30, seed=8, name=name, lower=-30.0, upper=30.0)
    pop = pz.initialize(cfg, name)
    for t in range(13):
        pop = pz.step(pop, cfg, name, t)
    res = pz.resume(cfg, name, pop)
    assert np.array_equal(res.population.positions, want["positions"])
    assert np.array_equal(res.population.fitness, want["fitness"])
    assert np.array_equal(res.trace, want["trace"][13:]) and res.warnings == want["warnings"]
    assert res.best_fitness == want["best_fitness"]
