"""CUDA path vs the oracle and the reference's golden vectors (needs a B200).

Tolerance: bit-exact (np.array_equal) everywhere, griewank included: its cos is
glibc 2.39's algorithm ported to the device (cos_glibc, apo_device.cuh), and
the rank weight's exp is glibc's too (exp_glibc).
"""

import math
import os

import numpy as np
import pytest

import oracle
from conftest import GOLDEN

pytestmark = pytest.mark.gpu

RTOL = 1e-9


@pytest.fixture(scope="module")
def pz():
    import torch

    import paper_2510_14982_b200 as pkg

    torch.cuda.set_device(0)
    return pkg


def _groups(path):
    data = np.load(os.path.join(GOLDEN, path))
    groups = {}
    for key in data.files:
        name, field = key.split("/", 1)
        groups.setdefault(name, {})[field] = data[key]
    return groups


def _same(a, b, name):
    assert np.array_equal(a, b), name


def test_device_cos_matches_libm(pz):
    """cos_glibc (griewank's cos) equals the host libm bit for bit over the griewank argument range and
    every branch of glibc's __cos (|x| < 2^-27, < 0.855, < 2.426, Cody-Waite reduced)."""
    import torch

    from paper_2510_14982_b200 import _lib

    rnd = np.random.default_rng(4)
    x = np.concatenate([rnd.uniform(-600, 600, 600_000), rnd.uniform(-2.5, 2.5, 300_000),
                        rnd.uniform(-1e-8, 1e-8, 10_000), rnd.uniform(-1e7, 1e7, 100_000),
                        np.array([0.0, -0.0, 0.855469, 2.426265, np.pi / 2, np.pi, 1e8])])
    xt = torch.as_tensor(x, device="cuda")
    out = torch.empty_like(xt)
    _lib.check(_lib.load().apo_debug_cos(_lib.ptr(xt), _lib.ptr(out), x.size, _lib.stream_handle()))
    want = np.array([math.cos(v) for v in x])
    assert np.array_equal(out.cpu().numpy().view(np.uint64), want.view(np.uint64))


def test_device_exp_matches_libm(pz):
    import torch

    from paper_2510_14982_b200 import _lib

    rnd = np.random.default_rng(3)
    x = np.concatenate([-rnd.random(400_000), -rnd.random(400_000) * 40, -rnd.random(200_000) * 800,
                        -np.exp(rnd.random(100_000) * 30 - 25), np.array([0.0, -0.0, -np.inf, -745.2, -708.4])])
    xt = torch.as_tensor(x, device="cuda")
    out = torch.empty_like(xt)
    _lib.check(_lib.load().apo_debug_exp(_lib.ptr(xt), _lib.ptr(out), x.size, _lib.stream_handle()))
    want = np.array([math.exp(v) for v in x])
    got = out.cpu().numpy()
    assert np.array_equal(got.view(np.uint64), want.view(np.uint64))


def test_initialize_matches_reference(pz):
    for name, g in _groups("steps.npz").items():
        ps, dim, T, seed, npairs, steps = (int(v) for v in g["cfg"])
        pf_max, lo, hi, eps = (float(v) for v in g["cfgf"])
        cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T, seed=seed)
        pop = pz.initialize(cfg, str(g["objective"]))
        assert np.array_equal(pop.positions, g["init_pos"])
        _same(pop.fitness, g["init_fit"], str(g["objective"]))


@pytest.mark.parametrize("case", sorted(_groups("steps.npz")))
def test_run_updates_teacher_forced_vs_reference(pz, case):
    from paper_2510_14982_b200.kernels import get_backend

    g = _groups("steps.npz")[case]
    ps, dim, T, seed, npairs, steps = (int(v) for v in g["cfg"])
    pf_max, lo, hi, eps = (float(v) for v in g["cfgf"])
    name = str(g["objective"])
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T, seed=seed,
                       neighbor_pairs=npairs, pf_max=pf_max, eps=eps)
    bk = get_backend("cuda")
    for t in range(steps):
        op, of, acc, nw = bk.run_updates(g["snap_pos"][t], g["snap_fit"][t], g["in_dr"][t], cfg,
                                         pz.get_objective(name), t, t + 1)
        _same(op, g["out_pos"][t], name)
        _same(of, g["out_fit"][t], name)
        assert np.array_equal(acc, g["acc"][t])
        assert nw == int(g["warn"][t])


@pytest.mark.parametrize("case", sorted(_groups("steps.npz")))
def test_step_vs_reference(pz, case):
    g = _groups("steps.npz")[case]
    ps, dim, T, seed, npairs, steps = (int(v) for v in g["cfg"])
    pf_max, lo, hi, eps = (float(v) for v in g["cfgf"])
    name = str(g["objective"])
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T, seed=seed,
                       neighbor_pairs=npairs, pf_max=pf_max, eps=eps)
    pop = pz.Population(g["init_pos"], g["init_fit"], fe_count=ps)
    for t in range(steps):
        before = pop.positions.copy()
        nxt = pz.step(pop, cfg, name, t)
        assert np.array_equal(pop.positions, before)  # input untouched
        _same(nxt.positions, g["out_pos"][t], name)
        _same(nxt.fitness, g["out_fit"][t], name)
        assert nxt.iteration == t + 1 and nxt.fe_count == pop.fe_count + ps
        pop = pz.Population(g["out_pos"][t], g["out_fit"][t], iteration=t + 1, fe_count=nxt.fe_count)


@pytest.mark.parametrize("case", sorted(_groups("runs.npz")))
@pytest.mark.parametrize("path", ["batch", "device"])
def test_full_runs_vs_reference(pz, case, path, monkeypatch):
    from paper_2510_14982_b200 import engine

    g = _groups("runs.npz")[case]
    ps, dim, T, seed, max_fes = (int(v) for v in g["cfg"])
    lo, hi = (float(v) for v in g["cfgf"])
    name = str(g["objective"])
    if path == "device":
        monkeypatch.setattr(engine, "BATCH_PS_LIMIT", 0)
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(lo, hi, dim), max_iterations=T, seed=seed,
                       max_fes=None if max_fes < 0 else max_fes)
    res = pz.run(cfg, name)
    assert [res.iterations_run, res.fe_count, res.warnings] == g["counters"].tolist()
    assert np.array_equal(res.trace, g["trace"])
    assert np.array_equal(res.population.positions, g["final_pos"])
    assert np.array_equal(res.population.fitness, g["final_fit"])
    assert res.best_fitness == float(g["best_fitness"])
    assert np.array_equal(res.best_position, g["best_position"])


@pytest.mark.parametrize("name", ["sphere", "bent_cigar", "high_conditioned_elliptic", "hgbat", "rosenbrock"])
def test_device_loop_vs_oracle_mid_size(pz, name, monkeypatch):
    """ps beyond the shared-memory kernel: the HBM-resident loop, bit-exact vs the oracle."""
    cfg = pz.ApoConfig(ps=3000, dim=37, bounds=pz.Bounds(-100.0, 100.0, 37), max_iterations=12, seed=11,
                       neighbor_pairs=2, pf_max=0.3)
    res = pz.run(cfg, name)
    want = oracle.run(ps=3000, dim=37, max_iterations=12, seed=11, name=name, lower=-100.0, upper=100.0,
                      npairs=2, pf_max=0.3, nthreads=8)
    assert np.array_equal(res.trace, want["trace"])
    assert np.array_equal(res.population.positions, want["positions"])
    assert np.array_equal(res.population.fitness, want["fitness"])
    assert res.best_fitness == want["best_fitness"]


@pytest.mark.parametrize("ps,pf_max", [(1000, 1.0), (2048, 0.5), (2049, 1.0), (5000, 1.0), (12289, 0.3),
                                        (24576, 0.1), (24577, 0.1)])
def test_device_loop_prologue_paths_vs_oracle(pz, ps, pf_max, monkeypatch):
    """The prologue (stable sort + Dr set) has three implementations by population size: counting in
    one launch (ps <= 2048), tile sort + merge (<= 24576, apo_prologue.cu), CUB radix sort beyond;
    all bit-exact, including Dr sets as large as the population (pf_max = 1)."""
    from paper_2510_14982_b200 import engine

    monkeypatch.setattr(engine, "BATCH_PS_LIMIT", 0)
    cfg = pz.ApoConfig(ps=ps, dim=3, bounds=pz.Bounds(-5.0, 5.0, 3), max_iterations=6, seed=ps, pf_max=pf_max)
    res = pz.run(cfg, "rosenbrock")
    want = oracle.run(ps=ps, dim=3, max_iterations=6, seed=ps, name="rosenbrock", lower=-5.0, upper=5.0,
                      pf_max=pf_max, nthreads=8)
    assert np.array_equal(res.trace, want["trace"])
    assert np.array_equal(res.population.positions, want["positions"])
    assert np.array_equal(res.population.fitness, want["fitness"])


def test_large_population_one_iteration_vs_oracle(pz):
    """C4 shape (ps=1M, D=100): one teacher-forced update, bit-exact."""
    import torch

    from paper_2510_14982_b200.kernels import get_backend

    ps, dim = 1_000_000, 100
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=100, seed=5)
    pos, fit = oracle.initialize(5, ps, dim, -100.0, 100.0, "rosenbrock")
    order = oracle.argsort_stable(fit)
    sp, sf = pos[order], fit[order]
    in_dr = oracle.select_dr(5, 8, ps, 0.1)
    want = oracle.run_updates(sp, sf, in_dr, seed=5, iteration=7, max_iterations=100, name="rosenbrock",
                              lower=-100.0, upper=100.0, nthreads=os.cpu_count() or 1)
    got = get_backend("cuda").run_updates(torch.as_tensor(sp, device="cuda"), torch.as_tensor(sf, device="cuda"),
                                          torch.as_tensor(in_dr, device="cuda"), cfg,
                                          pz.get_objective("rosenbrock"), 7, 8)
    assert np.array_equal(got[0].cpu().numpy(), want[0])
    assert np.array_equal(got[1].cpu().numpy(), want[1])
    assert np.array_equal(got[2].cpu().numpy(), want[2])


def test_sort_and_dr_vs_oracle(pz):
    import torch

    from paper_2510_14982_b200 import _lib

    lib = _lib.load()
    rnd = np.random.default_rng(0)
    for n in (1, 7, 1000, 100_000):
        f = np.round(rnd.normal(size=n), 2)  # many ties
        f[:: 7] = -0.0
        ft = torch.as_tensor(f, device="cuda")
        order = torch.empty(n, dtype=torch.int32, device="cuda")
        _lib.check(lib.apo_sort_order(_lib.ptr(ft), n, _lib.ptr(order), _lib.stream_handle()))
        assert np.array_equal(order.cpu().numpy(), oracle.argsort_stable(f))
    for (seed, it, ps, pf_max) in [(0, 1, 100, 0.1), (3, 9, 5000, 1.0), (9, 2, 1_000_000, 0.1), (1, 1, 1, 0.5)]:
        d = torch.empty(ps, dtype=torch.uint8, device="cuda")
        _lib.check(lib.apo_select_dr(seed, it, ps, pf_max, _lib.ptr(d), None, _lib.stream_handle()))
        assert np.array_equal(d.cpu().numpy().astype(bool), oracle.select_dr(seed, it, ps, pf_max))


def test_batch_matches_oracle_runs(pz):
    names = ["sphere", "bent_cigar", "high_conditioned_elliptic", "hgbat", "rosenbrock", "griewank"] * 4
    seeds = list(range(len(names)))
    cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=200)
    res = pz.run_batch(cfg, names, seeds)
    want, _ = oracle.run_many(names, seeds, ps=100, dim=20, max_iterations=200, lower=-100.0, upper=100.0)
    assert np.array_equal(res.best_fitness, want)


def test_persistent_batch_matches_oracle_runs(pz):
    """More runs than SMs: persistent CTAs claim runs costliest first (mixed objectives, so the claim
    order is not the run order); every result must land at its own index, bit-exact."""
    names = ["rosenbrock", "sphere", "hgbat", "bent_cigar", "high_conditioned_elliptic"] * 64
    seeds = [7 * k + 1 for k in range(len(names))]
    cfg = pz.ApoConfig(ps=24, dim=6, bounds=pz.Bounds(-30.0, 30.0, 6), max_iterations=40)
    res = pz.run_batch(cfg, names, seeds, want_trace=True)
    want, _ = oracle.run_many(names, seeds, ps=24, dim=6, max_iterations=40, lower=-30.0, upper=30.0)
    assert np.array_equal(res.best_fitness, want)
    assert np.array_equal(res.trace[:, -1], want)
    # CEC2022 mixes (cost-ordered claims across functions) agree with one-run-per-CTA launches
    cnames = [f"cec2022_f{k}" for k in range(1, 13)] * 15
    ccfg = pz.ApoConfig(ps=30, dim=10, bounds=pz.Bounds(-100.0, 100.0, 10), max_iterations=30)
    big = pz.run_batch(ccfg, cnames, list(range(len(cnames))))
    for k0 in range(0, len(cnames), 12):
        part = pz.run_batch(ccfg, cnames[k0:k0 + 12], list(range(k0, k0 + 12)))
        assert np.array_equal(part.best_fitness, big.best_fitness[k0:k0 + 12])
        assert np.array_equal(part.trace, big.trace[k0:k0 + 12])


@pytest.mark.parametrize("ps,dim", [(2, 1), (33, 3), (100, 5), (700, 4), (64, 8), (50, 9)])
def test_batch_lane_per_protozoon_groups_match_oracle(pz, ps, dim):
    """dim <= 8 (update_group_lpp: one lane per protozoon, 32 per warp, the fitness folded as the candidate
    is built) and dim = 9 (warp per protozoon) against the oracle's run loop, bit-exact; every reference
    objective, the default CTA and a 2-warp CTA (several groups per warp)."""
    names = ["sphere", "bent_cigar", "high_conditioned_elliptic", "hgbat", "rosenbrock", "griewank"]
    names = [n for n in names if pz.get_objective(n).min_dim <= dim]
    seeds = [11 * k + dim for k in range(len(names))]
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-20.0, 30.0, dim), max_iterations=25)
    want, _ = oracle.run_many(names, seeds, ps=ps, dim=dim, max_iterations=25, lower=-20.0, upper=30.0)
    for threads in (0, 64):
        res = pz.run_batch(cfg, names, seeds, want_trace=True, threads_per_run=threads)
        assert np.array_equal(res.best_fitness, want), threads
        assert np.array_equal(res.trace[:, -1], want), threads


def test_batch_launch_shapes_agree(pz):
    """apo_run_batch_shaped: any CTA size gives the same runs (rank counts, group sizes and the Dr warp
    depend on it, the results must not); out-of-range sizes are rejected."""
    names = [f"cec2022_f{k}" for k in (1, 6, 9, 12)] + ["rosenbrock", "griewank"]
    seeds = list(range(len(names)))
    cfg = pz.ApoConfig(ps=70, dim=12, bounds=pz.Bounds(-100.0, 100.0, 12), max_iterations=60)
    ref = pz.run_batch(cfg, names, seeds)
    for threads in (64, 256, 384, 640):
        got = pz.run_batch(cfg, names, seeds, threads_per_run=threads)
        assert np.array_equal(got.trace, ref.trace), threads
        assert np.array_equal(got.best_position, ref.best_position), threads
    for bad in (16, 672, 1024, 100):
        with pytest.raises(Exception, match="threads_per_run"):
            pz.run_batch(cfg, names, seeds, threads_per_run=bad)


def test_device_objective_cache_follows_objective_lifetime(pz):
    import copy
    import gc

    from paper_2510_14982_b200 import objectives

    assert pz.get_objective("cec2022_f5") is pz.get_objective("cec2022_f5")  # interned: tables built once
    base = len(objectives._DEV_CACHE)
    tmp = [copy.copy(pz.get_objective("high_conditioned_elliptic")) for _ in range(5)]
    for o in tmp:
        objectives.device_objective(o, 7)
    assert len(objectives._DEV_CACHE) == base + 5
    del tmp, o
    gc.collect()
    assert len(objectives._DEV_CACHE) == base


def test_histogram_and_threshold(pz):
    g = np.load(os.path.join(GOLDEN, "threshold.npz"))
    img = pz.GrayImage(g["pixels"])
    h = pz.histogram(img)
    assert np.array_equal(h.counts, g["counts"])
    rnd = np.random.default_rng(1)
    big = rnd.integers(0, 256, size=(4096, 4096), dtype=np.uint8)
    assert np.array_equal(pz.histogram(pz.GrayImage(big)).counts, np.bincount(big.ravel(), minlength=256))
    odd = big[:1001, :999].copy()
    assert np.array_equal(pz.histogram(pz.GrayImage(odd)).counts, np.bincount(odd.ravel(), minlength=256))
    res = pz.apo_threshold(img, ps=100, iterations=50, seed=0)
    assert res.threshold == int(g["apo_t"]) and res.variance == float(g["apo_var"])
    assert np.array_equal(res.run.trace, g["apo_trace"])


def _random_configs(n, seed=2026):
    """The reference's acceptance criterion 2 draws 200 random configurations (test_acceptance.py:
    183-205); here each one runs on the GPU and must equal the oracle run bit for bit."""
    rnd = np.random.default_rng(seed)
    names = ["sphere", "bent_cigar", "high_conditioned_elliptic", "hgbat", "rosenbrock", "griewank"]
    out = []
    for k in range(n):
        ps = int(rnd.choice([2, 3, 7, 33, 64, 100, 257, 700, 1500]))
        dim = int(rnd.choice([1, 2, 5, 17, 32, 33, 64, 100, 129, 300]))
        name = names[k % len(names)]
        if name in ("high_conditioned_elliptic", "rosenbrock") and dim < 2:
            dim = 2
        lo = float(rnd.uniform(-50, 0))
        hi = lo + float(rnd.uniform(0.5, 80))
        npairs = int(rnd.integers(1, min(ps - 1, 4) + 1)) if ps > 1 else 1
        out.append(dict(ps=ps, dim=dim, name=name, lo=lo, hi=hi, T=int(rnd.integers(1, 12)),
                        seed=int(rnd.integers(0, 2 ** 63)), npairs=npairs, pf_max=float(rnd.uniform(0.05, 1.0))))
    return out


@pytest.mark.parametrize("c", _random_configs(40), ids=lambda c: f"{c['name']}-{c['ps']}x{c['dim']}")
def test_random_configurations_bit_exact(pz, c, monkeypatch):
    from paper_2510_14982_b200 import engine

    want = oracle.run(ps=c["ps"], dim=c["dim"], max_iterations=c["T"], seed=c["seed"], name=c["name"],
                      lower=c["lo"], upper=c["hi"], npairs=c["npairs"], pf_max=c["pf_max"], nthreads=8)
    cfg = pz.ApoConfig(ps=c["ps"], dim=c["dim"], bounds=pz.Bounds(c["lo"], c["hi"], c["dim"]),
                       max_iterations=c["T"], seed=c["seed"], neighbor_pairs=c["npairs"], pf_max=c["pf_max"])
    for limit in (engine.BATCH_PS_LIMIT, 0):  # one-CTA batch kernel (when it fits) and the HBM device loop
        monkeypatch.setattr(engine, "BATCH_PS_LIMIT", limit)
        res = pz.run(cfg, c["name"])
        assert np.array_equal(res.trace, want["trace"])
        assert np.array_equal(res.population.positions, want["positions"])
        assert np.array_equal(res.population.fitness, want["fitness"])
        assert res.warnings == want["warnings"] and res.best_fitness == want["best_fitness"]


def test_run_buffers_recycled_and_released(pz):
    """Run buffers come from the stream-ordered pool: create/destroy repeatedly, populations stay
    right, and empty_cache() hands the pool back."""
    import torch

    cfg = pz.ApoConfig(ps=5000, dim=30, bounds=pz.Bounds(-100.0, 100.0, 30), max_iterations=5, seed=4)
    first = pz.run(cfg, "cec2022_f4")
    for _ in range(3):
        again = pz.run(cfg, "cec2022_f4")
        assert np.array_equal(again.population.positions, first.population.positions)
        assert np.array_equal(again.trace, first.trace)
    pz.empty_cache()
    torch.cuda.synchronize()
    assert np.array_equal(pz.run(cfg, "cec2022_f4").population.fitness, first.population.fitness)


@pytest.mark.parametrize("name,dim,bound", [("rosenbrock", 20, 100.0), ("cec2022_f6", 40, 100.0),
                                            ("cec2022_f1", 150, 100.0), ("griewank", 300, 100.0),
                                            ("cec2022_f1", 300, 100.0), ("sphere", 300, 1e200)])
def test_step_chunked_d2h_matches_single_launch(pz, name, dim, bound, monkeypatch):
    """step() at ps >= 2^16 updates in rank chunks (apo_run_updates_range) and copies each back while the
    next computes; identical to the one-launch update, for the group, CEC split, CEC GEMM and warp paths.
    The warp path (D > 256) must honour the rank range: F1 at D=300 is the GEMM path whose candidate rows
    would be overwritten by a later chunk, and sphere at +-1e200 overflows to inf, so every candidate
    warns and a chunk that re-ran the whole population would over-count."""
    from paper_2510_14982_b200 import engine

    cfg = pz.ApoConfig(ps=70_001, dim=dim, bounds=pz.Bounds(-bound, bound, dim), max_iterations=10, seed=9,
                       pf_max=0.3)
    pop = pz.initialize(cfg, name)
    chunked = pz.step(pop, cfg, name, 3)
    monkeypatch.setattr(engine, "STEP_CHUNK_MIN_PS", 1 << 40)
    whole = pz.step(pop, cfg, name, 3)
    assert np.array_equal(chunked.positions, whole.positions)
    assert np.array_equal(chunked.fitness, whole.fitness)
    assert chunked.warnings == whole.warnings
    if bound > 1e100:
        assert whole.warnings - pop.warnings == cfg.ps  # every candidate is inf: one warning each, no more


@pytest.mark.parametrize("name,dim", [("rosenbrock", 30), ("cec2022_f6", 100), ("cec2022_f10", 40),
                                      ("cec2022_f1", 150), ("hgbat", 200)])
def test_ordered_update_equals_gathered_snapshot(pz, name, dim):
    """apo_run_updates_ordered (rows read through the sort's rank -> row map, no gather) equals
    apo_run_updates_range on the gathered snapshot, bit for bit, on every update path (group, CEC
    split, CEC GEMM) and per rank chunk."""
    import torch

    from paper_2510_14982_b200 import _lib
    from paper_2510_14982_b200.core import iteration_scalars
    from paper_2510_14982_b200.kernels.cuda_backend import p_dr_device
    from paper_2510_14982_b200.objectives import device_objective

    ps = 5000
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=20, seed=13)
    pop = pz.initialize(cfg, name)
    dev = torch.device("cuda")
    pos = torch.as_tensor(pop.positions, device=dev)
    fit = torch.as_tensor(pop.fitness, device=dev)
    order = torch.empty(ps, dtype=torch.int32, device=dev)
    lib = _lib.load()
    _lib.check(lib.apo_sort_order(_lib.ptr(fit), ps, _lib.ptr(order), _lib.stream_handle()))
    in_dr = torch.as_tensor(oracle.select_dr(13, 5, ps, 0.1).astype(np.uint8), device=dev)
    dobj = device_objective(pz.get_objective(name), dim)
    p_ah, f_mult, decay = iteration_scalars(4, 20)
    pdr = p_dr_device(ps, dev)
    idx = order.long()
    snap_pos, snap_fit = pos.index_select(0, idx).contiguous(), fit.index_select(0, idx).contiguous()
    outs = []
    for ordered in (False, True):
        out_pos, out_fit = torch.empty_like(pos), torch.empty_like(fit)
        warn = torch.zeros(1, dtype=torch.int64, device=dev)
        for lo, hi in ((0, 1312), (1312, 4000), (4000, ps)):
            common = (ps, dim, 13, 5, 1, -100.0, 100.0, cfg.eps, p_ah, f_mult, decay, dobj.ref, _lib.ptr(pdr),
                      _lib.ptr(warn), lo, hi, _lib.stream_handle())
            if ordered:
                _lib.check(lib.apo_run_updates_ordered(_lib.ptr(pos), _lib.ptr(fit), _lib.ptr(order), _lib.ptr(in_dr),
                                                       _lib.ptr(out_pos), _lib.ptr(out_fit), None, None, *common))
            else:
                _lib.check(lib.apo_run_updates_range(_lib.ptr(snap_pos), _lib.ptr(snap_fit), _lib.ptr(in_dr),
                                                     _lib.ptr(out_pos), _lib.ptr(out_fit), None, None, *common))
        outs.append((out_pos.cpu().numpy(), out_fit.cpu().numpy(), int(warn.item())))
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
    assert outs[0][2] == outs[1][2]


@pytest.mark.parametrize("ps,dim", [(48, 6), (47, 6), (50, 7), (44, 6)])
def test_batch_shared_memory_just_under_48k(pz, ps, dim):
    """Batch launches whose dynamic shared memory lands just under 48 KB must still launch (the default
    limit covers static + dynamic; the attribute is now always set) and a failed launch must not poison
    the next call's error check."""
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-30.0, 30.0, dim), max_iterations=10, seed=8)
    res = pz.run(cfg, "rosenbrock")
    want = oracle.run(ps=ps, dim=dim, max_iterations=10, seed=8, name="rosenbrock", lower=-30.0, upper=30.0)
    assert np.array_equal(res.trace, want["trace"])
