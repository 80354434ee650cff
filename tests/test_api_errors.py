"""Error behaviour of the reference-facing API (engine.py:92-97, 142-150; core.py:98-146) -- no GPU needed:
validation happens before any device work."""

import numpy as np
import pytest

import paper_2510_14982_b200 as pz


def _cfg(**kw):
    base = dict(ps=16, dim=4, bounds=pz.Bounds(-1.0, 1.0, 4), max_iterations=3)
    base.update(kw)
    return pz.ApoConfig(**base)


def test_config_reports_every_violation():
    with pytest.raises(pz.ConfigError) as err:
        pz.ApoConfig(ps=0, dim=4, bounds=pz.Bounds(-1.0, 1.0, 3), max_iterations=-1, pf_max=2.0, neighbor_pairs=0)
    text = str(err.value)
    for fragment in ("ps must be", "bounds cover", "max_iterations", "neighbor_pairs", "pf_max"):
        assert fragment in text


def test_external_objectives_are_rejected_like_the_numba_backend():
    f = pz.external_objective(lambda x: float(np.sum(x)))
    with pytest.raises(ValueError):
        pz.run(_cfg(), f)
    from paper_2510_14982_b200.kernels import get_backend

    with pytest.raises(ValueError):
        get_backend("cuda").run_updates(np.zeros((16, 4)), np.zeros(16), np.zeros(16, bool), _cfg(), f, 0, 1)


def test_unknown_backend_and_objective_names():
    from paper_2510_14982_b200.kernels import get_backend

    with pytest.raises(ValueError):
        get_backend("numba")
    with pytest.raises(ValueError):
        pz.get_objective("no_such_function")
    with pytest.raises(ValueError):
        pz.cec2022_objective(13)


def test_step_rejects_a_population_of_the_wrong_shape():
    pop = pz.Population(np.zeros((8, 4)), np.zeros(8))
    with pytest.raises(ValueError):
        pz.step(pop, _cfg(), "sphere", 0)


def test_multilevel_threshold_bounds():
    from paper_2510_14982_b200 import imaging

    with pytest.raises(ValueError):
        imaging.multilevel_objective(np.ones(256, dtype=np.int64), 33, "otsu")
    with pytest.raises(ValueError):
        imaging.threshold_tables_device(np.ones(256, dtype=np.int64), "triangle")
