"""Scripted draws (APO_RNG_TABLE): the reference's hand-traced worked example replayed on the GPU.

The reference pins one engine iteration with a ``ScriptedStream`` monkeypatched over its rng module
(/root/reference/pkg/tests/test_acceptance.py:34-175): four protozoa on the sphere, every draw solved by
hand so the step lands on round targets (keep, keep, accept, accept).  Here the same script is an
``rng.DrawTable`` the kernels read through ``engine.step(..., draws=table)``.  Checked three ways:
  * the reference test's own assertions (CPU-built expectations, GPU step);
  * the unmodified reference (baseline/_ref) replaying the same table through its numpy backend, bit-exact;
  * a table holding the keyed stream's own draws steps exactly like the keyed stream (every path:
    fused, basic split, CEC2022).
"""

import math
import os
import sys

import numpy as np
import pytest

from conftest import ROOT

from paper_2510_14982_b200 import core, rng
from paper_2510_14982_b200.rng import COORDINATOR_INDEX, DrawTable

REF_SITE = os.path.join(ROOT, "baseline", "_ref")

# test_acceptance.py:34-47 (the worked example's data)
START_POSITIONS = np.array([[4.8, 7.8, 9.4], [3.4, 8.4, 9.0], [1.4, 5.0, 8.0], [4.5, 1.2, 4.7]])
START_FITNESS = np.array([172.24, 163.12, 90.96, 43.78])
SORT_ORDER = [3, 2, 1, 0]
FINAL_POSITIONS = np.array([[4.5, 1.2, 4.7], [1.4, 5.0, 8.0], [2.9, 8.38, 9.11], [4.26, 6.32, 8.07]])


def worked_example() -> DrawTable:
    """The hand-solved draws of test_acceptance.py:83-134, written against this package's slot layout."""
    eps = 2.0 ** -52
    x = START_POSITIONS[SORT_ORDER]
    f = START_FITNESS[SORT_ORDER]
    w_best_worst = core.rank_weight(f[0], f[3], eps)
    w_mid_worst = core.rank_weight(f[1], f[3], eps)
    s = DrawTable(seed=0, iteration=2)
    s.scalars[(COORDINATOR_INDEX, core.COORD_SLOT_PF)] = 0.5  # pf = 0.05 -> ceil(4 * 0.05) = 1 rank
    s.perms[(COORDINATOR_INDEX, core.COORD_SLOT_DR_PERM, 4, 1)] = [2]
    bracket = (x[2][1] - x[0][1]) + w_best_worst * (x[0][1] - x[3][1])
    s.scalars[(1, core.SLOT_DECISION)] = 0.2  # rank 1: autotroph toward rank 3, second component only
    s.scalars[(1, core.SLOT_PARTNER)] = 0.5
    s.scalars[(1, core.SLOT_FORAGE)] = 0.57 / bracket
    s.scalars[(1, core.PAIRS_BASE + 1)] = 0.8
    s.perms[(1, core.MASK_BASE, 3, 1)] = [2]
    s.scalars[(2, core.SLOT_DECISION)] = 0.9  # rank 2: reproduction, overshoots the box
    s.scalars[(2, core.SLOT_SIGN)] = 0.1
    s.scalars[(2, core.SLOT_MASK_SIZE)] = 0.5
    s.scalars[(2, core.SLOT_MAGNITUDE)] = 0.9
    s.vectors[(2, core.VECTOR_BASE)] = [0.77, 8.53 / 9.0, 3.53 / 9.0]
    s.perms[(2, core.MASK_BASE, 3, 2)] = [2, 3]
    pair_diff = x[1] - x[3]
    delta = np.array([-0.5, -0.02, 0.11])
    s.scalars[(3, core.SLOT_DECISION)] = 0.9  # rank 3: heterotroph to [2.9, 8.38, 9.11]
    s.scalars[(3, core.SLOT_SIGN)] = 0.1
    s.scalars[(3, core.SLOT_FORAGE)] = 0.5
    s.vectors[(3, core.VECTOR_BASE)] = (2.0 * delta - w_mid_worst * pair_diff) / (0.5 * x[2])
    s.perms[(3, core.MASK_BASE, 3, 3)] = [1, 2, 3]
    s.scalars[(4, core.SLOT_DECISION)] = 0.2  # rank 4: autotroph toward rank 3, pulled by rank 1
    s.scalars[(4, core.SLOT_FORAGE)] = 0.3283
    s.scalars[(4, core.SLOT_PARTNER)] = 0.7
    s.scalars[(4, core.PAIRS_BASE)] = 0.1
    s.perms[(4, core.MASK_BASE, 3, 3)] = [1, 2, 3]
    return s


def keyed_counters(dim, npairs=1):
    return ([core.SLOT_DECISION, core.SLOT_SIGN, core.SLOT_MASK_SIZE, core.SLOT_MAGNITUDE, core.SLOT_FORAGE,
             core.SLOT_PARTNER] + [core.VECTOR_BASE + d for d in range(dim)] +
            [core.MASK_BASE + j for j in range(dim)] + [core.PAIRS_BASE + k for k in range(2 * npairs)])


def keyed_table(seed, key_iteration, ps, dim, npairs=1):
    t = DrawTable.from_stream(seed, key_iteration, range(1, ps + 1), keyed_counters(dim, npairs))
    coord = DrawTable.from_stream(seed, key_iteration, [COORDINATOR_INDEX], range(0, ps + 1))
    t.scalars.update(coord.scalars)
    return t


# ---------------------------------------------------------------------------- CPU


def test_scripted_permutations_invert_to_fisher_yates_draws():
    """perms -> uniforms: the partial Fisher-Yates of rng.randperm fed those uniforms yields the script."""
    rnd = np.random.default_rng(3)
    for _ in range(200):
        n = int(rnd.integers(1, 40))
        k = int(rnd.integers(0, n + 1))
        want = (rnd.permutation(n)[:k] + 1).tolist()
        t = DrawTable(1, 1)
        t.perms[(7, 100, n, k)] = want
        u = t.uniforms()
        arr = list(range(1, n + 1))
        for j in range(k):
            r = min(j + int(u[(7, 100 + j)] * (n - j)), n - 1)
            arr[j], arr[r] = arr[r], arr[j]
        assert arr[:k] == want


def test_draw_table_rejects_bad_scripts():
    t = DrawTable(0, 1)
    t.scalars[(1, 0)] = 0.25
    t.vectors[(1, 0)] = [0.5]  # the same draw scripted twice, differently
    with pytest.raises(ValueError, match="twice"):
        t.uniforms()
    t = DrawTable(0, 1)
    t.scalars[(1, 0)] = 1.0
    with pytest.raises(ValueError, match="outside"):
        t.uniforms()
    t = DrawTable(0, 1)
    t.perms[(1, 5, 3, 2)] = [1, 1]
    with pytest.raises(ValueError, match="distinct"):
        t.uniforms()


def test_table_from_stream_holds_the_keyed_draws():
    t = keyed_table(9, 4, 5, 3)
    ind, ctr, val = t.arrays()
    assert np.all(np.diff(ind.astype(object) * 2 ** 64 + ctr.astype(object)) > 0)  # sorted, unique
    for i, c, v in zip(ind[:50], ctr[:50], val[:50]):
        assert v == rng.draw_uniform(rng.StreamKey(9, 4, int(i), int(c)))


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_worked_example_replay_on_gpu():
    """test_acceptance.py:139-175's assertions, the step run by the CUDA kernels on the scripted table."""
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=4, dim=3, bounds=pz.Bounds(0.0, 10.0, 3), max_iterations=3, pf_max=0.1, seed=0)
    pop = pz.Population(START_POSITIONS.copy(), START_FITNESS.copy(), iteration=1, fe_count=4)
    out = pz.step(pop, cfg, "sphere", 1, draws=worked_example())
    ranked = START_POSITIONS[SORT_ORDER]
    changed = [not np.array_equal(out.positions[r], ranked[r]) for r in range(4)]
    assert changed == [False, False, True, True]  # keep, keep, accept, accept
    np.testing.assert_allclose(out.positions, FINAL_POSITIONS, atol=5e-3)
    assert out.fitness[0] == 43.78 and out.fitness[1] == 90.96
    assert abs(out.fitness[2] - 161.63) < 5e-3
    assert out.fitness[3] < 172.24
    assert out.iteration == 2 and out.fe_count == 8
    assert np.array_equal(pop.positions, START_POSITIONS)  # input untouched


@pytest.mark.gpu
def test_unscripted_draw_raises_lookup_error():
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=4, dim=3, bounds=pz.Bounds(0.0, 10.0, 3), max_iterations=3, pf_max=0.1, seed=0)
    pop = pz.Population(START_POSITIONS.copy(), START_FITNESS.copy(), iteration=1, fe_count=4)
    t = worked_example()
    del t.scalars[(3, core.SLOT_FORAGE)]
    with pytest.raises(LookupError, match=f"individual 3, counter {core.SLOT_FORAGE}"):
        pz.step(pop, cfg, "sphere", 1, draws=t)
    t = worked_example()
    del t.scalars[(COORDINATOR_INDEX, core.COORD_SLOT_PF)]
    with pytest.raises(LookupError, match="counter 0"):
        pz.step(pop, cfg, "sphere", 1, draws=t)
    with pytest.raises(ValueError, match="iteration"):
        pz.step(pop, cfg, "sphere", 0, draws=worked_example())


@pytest.mark.gpu
@pytest.mark.parametrize("name,ps,dim,npairs", [("rosenbrock", 64, 10, 1), ("griewank", 300, 40, 2),
                                                ("sphere", 2000, 3, 1), ("cec2022_f6", 500, 20, 1),
                                                ("hgbat", 97, 7, 3), ("sphere", 70, 300, 2)])
def test_keyed_stream_as_a_table_steps_like_the_stream(name, ps, dim, npairs):
    """A table holding the keyed stream's own draws reproduces the keyed step bit for bit: the table
    lookup is the only thing that changes between the two runs (fused, basic-split and CEC2022 paths)."""
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-30.0, 30.0, dim), max_iterations=20, seed=13,
                       neighbor_pairs=npairs)
    pop = pz.initialize(cfg, name)
    for t in (0, 5):
        want = pz.step(pop, cfg, name, t)
        got = pz.step(pop, cfg, name, t, draws=keyed_table(13, t + 1, ps, dim, npairs))
        assert np.array_equal(got.positions, want.positions) and np.array_equal(got.fitness, want.fitness)
        assert got.warnings == want.warnings
        pop = want


# ------------------------------------------------------ against the unmodified reference (baseline/_ref)


@pytest.fixture(scope="module")
def ref_protozoa():
    if not os.path.isdir(os.path.join(REF_SITE, "protozoa")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "numba_cache_scripted"))
    sys.path.insert(0, REF_SITE)
    try:
        import protozoa
    finally:
        sys.path.remove(REF_SITE)
    return protozoa


def scripted_reference(monkeypatch, table: DrawTable):
    """Point the reference's rng functions at `table`'s uniforms, consumed by the reference's own draw
    algorithms (rng.py:114-156): what its ScriptedStream monkeypatch does, from the same data."""
    from protozoa import rng as ref_rng

    u = table.uniforms()

    def at(key, offset=0):
        assert key.seed == table.seed and key.iteration == table.iteration, key
        slot = (key.individual_index, (key.draw_counter + offset) % 2 ** 64)
        if slot not in u:
            raise LookupError(f"unscripted draw at {slot}")
        return u[slot]

    def randperm(n, k, key):
        arr = np.arange(1, n + 1, dtype=np.int64)
        for j in range(k):
            r = min(j + int(at(key, j) * (n - j)), n - 1)
            arr[j], arr[r] = arr[r], arr[j]
        return arr[:k]

    monkeypatch.setattr(ref_rng, "draw_uniform", lambda key: at(key))
    monkeypatch.setattr(ref_rng, "draw_uniform_vector", lambda key, n: np.array([at(key, d) for d in range(n)]))
    monkeypatch.setattr(ref_rng, "randperm", randperm)


@pytest.mark.gpu
def test_worked_example_bit_exact_with_reference_numpy_backend(ref_protozoa, monkeypatch):
    import paper_2510_14982_b200 as pz

    protozoa = ref_protozoa
    table = worked_example()
    rcfg = protozoa.ApoConfig(ps=4, dim=3, bounds=protozoa.Bounds(0.0, 10.0, 3), max_iterations=3, pf_max=0.1,
                              seed=0)
    rpop = protozoa.Population(START_POSITIONS.copy(), START_FITNESS.copy(), iteration=1, fe_count=4)
    scripted_reference(monkeypatch, table)
    want = protozoa.step(rpop, rcfg, "sphere", 1, protozoa.EngineMode.sequential(), backend="numpy")
    cfg = pz.ApoConfig(ps=4, dim=3, bounds=pz.Bounds(0.0, 10.0, 3), max_iterations=3, pf_max=0.1, seed=0)
    got = pz.step(pz.Population(START_POSITIONS.copy(), START_FITNESS.copy(), iteration=1, fe_count=4), cfg,
                  "sphere", 1, draws=table)
    assert np.array_equal(got.positions, want.positions) and np.array_equal(got.fitness, want.fitness)


@pytest.mark.gpu
@pytest.mark.parametrize("name,ps,dim", [("rosenbrock", 12, 5), ("high_conditioned_elliptic", 40, 9),
                                         ("griewank", 25, 4)])
def test_random_scripts_bit_exact_with_reference_numpy_backend(ref_protozoa, monkeypatch, name, ps, dim):
    """Random scripts (every slot the reference may read, values from a seeded numpy generator, not the
    keyed stream) through both the reference's numpy backend and the CUDA kernels."""
    import paper_2510_14982_b200 as pz

    protozoa = ref_protozoa
    rnd = np.random.default_rng(ps * dim)
    table = DrawTable(seed=21, iteration=3)
    for ind in range(1, ps + 1):
        for c in keyed_counters(dim):
            table.scalars[(ind, c)] = float(rnd.random())
    table.scalars[(COORDINATOR_INDEX, core.COORD_SLOT_PF)] = float(rnd.random())
    for j in range(ps):
        table.scalars[(COORDINATOR_INDEX, core.COORD_SLOT_DR_PERM + j)] = float(rnd.random())
    lo, hi = -5.0, 5.0
    positions = rnd.uniform(lo, hi, size=(ps, dim))
    fitness = np.array([pz.evaluate(name, r) for r in positions])
    rcfg = protozoa.ApoConfig(ps=ps, dim=dim, bounds=protozoa.Bounds(lo, hi, dim), max_iterations=10, pf_max=0.5,
                              seed=21)
    scripted_reference(monkeypatch, table)
    want = protozoa.step(protozoa.Population(positions.copy(), fitness.copy(), iteration=2, fe_count=ps), rcfg, name,
                         2, protozoa.EngineMode.sequential(), backend="numpy")
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=10, pf_max=0.5, seed=21)
    got = pz.step(pz.Population(positions.copy(), fitness.copy(), iteration=2, fe_count=ps), cfg, name, 2,
                  draws=table)
    assert np.array_equal(got.positions, want.positions) and np.array_equal(got.fitness, want.fitness)
    assert got.warnings == want.warnings
    assert math.isfinite(got.fitness.min())
