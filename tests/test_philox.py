"""Production mode: the Philox4x32-10 stream (no reference counterpart).

North star: "in production Philox mode, best-fitness distributions over 30
seeds must be statistically indistinguishable from the reference".  The
reference stream (keyed fmix64) is bit-identical to the reference package
(tests/test_oracle_golden.py, test_gpu_parity.py), so the GPU in keyed mode
stands in for the reference distribution here.
"""

import numpy as np
import pytest

from paper_2510_14982_b200 import _lib

M = 0xFFFFFFFF


def philox_py(ctr, key):
    """Independent restatement of Philox4x32-10 (Salmon et al., SC'11, Random123)."""
    c = list(ctr)
    k0, k1 = key
    for _ in range(10):
        p0 = 0xD2511F53 * c[0]
        p1 = 0xCD9E8D57 * c[2]
        c = [((p1 >> 32) ^ c[1] ^ k0) & M, p1 & M, ((p0 >> 32) ^ c[3] ^ k1) & M, p0 & M]
        k0 = (k0 + 0x9E3779B9) & M
        k1 = (k1 + 0xBB67AE85) & M
    return c


def philox_lib(ctr, key):
    import ctypes as C

    lib = _lib.load()
    c = (C.c_uint32 * 4)(*ctr)
    k = (C.c_uint32 * 2)(*key)
    out = (C.c_uint32 * 4)()
    lib.apo_philox4x32_10(c, k, out)
    return list(out)


# Random123 known-answer vectors for philox4x32_10 (kat_vectors).
KATS = [
    ((0, 0, 0, 0), (0, 0), (0x6627E8D5, 0xE169C58D, 0xBC57AC4C, 0x9B00DBD8)),
    ((M, M, M, M), (M, M), (0x408F276D, 0x41C83B0E, 0xA20BC7C6, 0x6D5451FD)),
    ((0x243F6A88, 0x85A308D3, 0x13198A2E, 0x03707344), (0xA4093822, 0x299F31D0),
     (0xD16CFE09, 0x94FDCCEB, 0x5001E420, 0x24126EA1)),
]


@pytest.mark.parametrize("ctr,key,want", KATS)
def test_philox_known_answers(ctr, key, want):
    assert philox_py(ctr, key) == list(want)
    assert philox_lib(ctr, key) == list(want)


def test_philox_random_blocks_match_restatement():
    rnd = np.random.default_rng(0)
    for _ in range(200):
        ctr = tuple(int(v) for v in rnd.integers(0, 2 ** 32, 4))
        key = tuple(int(v) for v in rnd.integers(0, 2 ** 32, 2))
        assert philox_lib(ctr, key) == philox_py(ctr, key)


def test_keyed_stream_is_the_reference_stream():
    import oracle

    lib = _lib.load()
    for key in [(0, 0, 0, 0), (42, 3, 17, 1000), (7, 2, 5, 2 ** 32), (0xDEADBEEF, 1, 2 ** 64 - 1, 2 ** 33 + 5)]:
        assert lib.apo_rng_uniform(0, *key) == oracle.draw_uniform(*key)


def test_philox_stream_layout_and_statistics():
    lib = _lib.load()
    # the draw is the top 53 bits of output words 0..1 of block (slot lo, slot hi, individual, iteration)
    seed, it, ind, ctr = 0x1234_5678_9ABC_DEF0, 7, 33, 2 ** 32 + 9
    w = philox_py((ctr & M, ctr >> 32, ind, it), (seed & M, seed >> 32))
    assert lib.apo_rng_uniform(1, seed, it, ind, ctr) == (((w[0] << 32) | w[1]) >> 11) * 2.0 ** -53
    u = np.array([lib.apo_rng_uniform(1, 5, 1, i, c) for i in range(1, 101) for c in range(200)])
    assert abs(u.mean() - 0.5) < 0.01 and abs(u.var() - 1 / 12) < 0.005
    assert abs(np.corrcoef(u[:-1], u[1:])[0, 1]) < 0.02
    hist = np.bincount((u * 20).astype(int), minlength=20)
    chi2 = ((hist - u.size / 20) ** 2 / (u.size / 20)).sum()
    assert chi2 < 50.0  # 19 dof: p ~ 1e-4
    # streams of different protozoa / iterations / the coordinator differ
    assert lib.apo_rng_uniform(1, 5, 1, 1, 0) != lib.apo_rng_uniform(1, 5, 1, 2, 0)
    assert lib.apo_rng_uniform(1, 5, 1, 1, 0) != lib.apo_rng_uniform(1, 5, 2, 1, 0)
    assert lib.apo_rng_uniform(1, 5, 1, 2 ** 64 - 1, 0) != lib.apo_rng_uniform(1, 5, 1, 1, 0)


def test_config_rejects_unknown_rng():
    import paper_2510_14982_b200 as pz

    with pytest.raises(pz.ConfigError):
        pz.ApoConfig(ps=10, dim=2, bounds=pz.Bounds(-1.0, 1.0, 2), max_iterations=5, rng="mt19937")


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
def test_philox_runs_are_deterministic_and_differ_from_keyed():
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=100, rng="philox")
    a = pz.run_batch(cfg, ["cec2022_f1", "rosenbrock"], [3, 4])
    b = pz.run_batch(cfg, ["cec2022_f1", "rosenbrock"], [3, 4])
    assert np.array_equal(a.best_fitness, b.best_fitness) and np.array_equal(a.trace, b.trace)
    k = pz.run_batch(pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=100),
                     ["cec2022_f1", "rosenbrock"], [3, 4])
    assert not np.array_equal(a.trace, k.trace)
    assert np.all(np.diff(a.trace, axis=1) <= 0)  # best-so-far never increases
    # the device-resident loop (HBM path) also runs in Philox mode
    big = pz.ApoConfig(ps=4096, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=30, rng="philox")
    r1 = pz.run(big, "cec2022_f4")
    r2 = pz.run(big, "cec2022_f4")
    assert r1.best_fitness == r2.best_fitness and np.all(np.diff(r1.trace) <= 0)


@pytest.mark.gpu
@pytest.mark.parametrize("name,dim", [("sphere", 20), ("rosenbrock", 20), ("griewank", 20), ("cec2022_f1", 20),
                                      ("cec2022_f4", 20), ("cec2022_f6", 20), ("cec2022_f10", 20),
                                      ("cec2022_f12", 20)])
def test_philox_best_fitness_distribution_matches_reference_stream(name, dim):
    """30 seeds each; two-sided Mann-Whitney U on final best fitness, alpha = 0.001 per function."""
    from scipy.stats import mannwhitneyu

    import paper_2510_14982_b200 as pz

    base = dict(ps=100, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=500)
    seeds = list(range(30))
    keyed = pz.run_batch(pz.ApoConfig(**base), [name] * 30, seeds, want_trace=False).best_fitness
    philox = pz.run_batch(pz.ApoConfig(**base, rng="philox"), [name] * 30, [s + 1000 for s in seeds],
                          want_trace=False).best_fitness
    p = mannwhitneyu(keyed, philox, alternative="two-sided").pvalue
    assert p > 1e-3, f"{name}: keyed median {np.median(keyed):.6g} vs philox {np.median(philox):.6g}, p = {p:.2e}"


@pytest.mark.gpu
def test_philox_sharded_partitions_equal_device_loop():
    """Production mode keeps partition independence (every draw keyed by seed, iteration, rank, slot)."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import engine
    from paper_2510_14982_b200.shard import ShardedRun

    cfg = pz.ApoConfig(ps=1000, dim=30, bounds=pz.Bounds(-100.0, 100.0, 30), max_iterations=8, seed=3, rng="philox")
    sh = ShardedRun(cfg, "cec2022_f4", virtual_world=3)
    sh.initialize()
    sh.iterate(8)
    pos, fit = sh.population()
    sh.close()
    run = engine.DeviceRun(cfg, pz.get_objective("cec2022_f4"))
    run.initialize()
    run.iterate(8)
    pos1, fit1 = run.population()
    run.close()
    assert np.array_equal(fit, fit1) and np.array_equal(pos, pos1)
