"""Multilevel Otsu / Kapur thresholding (BASELINE config 3).

No reference counterpart beyond k = 1: the oracle restatement
(oracle/threshold_oracle.c) is pinned to the reference's single-threshold Otsu
table (tests/golden/threshold.npz, produced by the reference itself) and to
independent numpy formulas for k = 2; the CUDA path is then checked against
the oracle (Otsu bit-exact, Kapur to 1e-12: CUDA log vs glibc log).
"""

import itertools
import os

import numpy as np
import pytest

import oracle

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "threshold.npz")
KAPUR_RTOL = 1e-12


def otsu_np(counts, ts):
    """Independent restatement: sum_c w_c (mu_c - mu_T)^2 over classes [0,t0],[t0+1,t1],...,[t_{k-1}+1,255]."""
    counts = np.asarray(counts, dtype=np.float64)
    n = counts.sum()
    v = np.arange(256)
    mu_t = (v * counts).sum() / n
    edges = [0] + [t + 1 for t in sorted(ts)] + [256]
    out = 0.0
    for a, b in zip(edges[:-1], edges[1:]):
        nc = counts[a:b].sum()
        if nc > 0:
            out += nc / n * ((v[a:b] * counts[a:b]).sum() / nc - mu_t) ** 2
    return out


def kapur_np(counts, ts):
    counts = np.asarray(counts, dtype=np.float64)
    p = counts / counts.sum()
    edges = [0] + [t + 1 for t in sorted(ts)] + [256]
    h = 0.0
    for a, b in zip(edges[:-1], edges[1:]):
        w = p[a:b].sum()
        if w > 0:
            q = p[a:b][p[a:b] > 0] / w
            h += -(q * np.log(q)).sum()
    return h


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_oracle_k1_otsu_matches_reference_variance_table(golden):
    """k = 1 generalisation == the reference's between_class_variance table (its own output)."""
    tab = oracle.threshold_tables(golden["counts"], "otsu")
    got = np.array([-oracle.threshold_eval("otsu", [t], tab) for t in range(256)])
    np.testing.assert_allclose(got, golden["table"], rtol=1e-12, atol=1e-9)
    # rounding rule and clamping of the reference table objective (round half up, clamp to [0, 255])
    assert oracle.threshold_eval("otsu", [99.5], tab) == oracle.threshold_eval("otsu", [100.0], tab)
    assert oracle.threshold_eval("otsu", [-7.0], tab) == oracle.threshold_eval("otsu", [0.0], tab)
    assert oracle.threshold_eval("otsu", [300.0], tab) == oracle.threshold_eval("otsu", [255.0], tab)


@pytest.mark.parametrize("method", ["otsu", "kapur"])
def test_oracle_k2_matches_independent_formula(golden, method):
    counts = golden["counts"]
    tab = oracle.threshold_tables(counts, method)
    ref = otsu_np if method == "otsu" else kapur_np
    rnd = np.random.default_rng(1)
    for _ in range(200):
        ts = rnd.integers(0, 256, size=2)
        got = -oracle.threshold_eval(method, ts.astype(float), tab)
        np.testing.assert_allclose(got, ref(counts, ts), rtol=1e-10, atol=1e-10)
    # thresholds are order independent and duplicates give empty classes
    assert oracle.threshold_eval(method, [200.0, 40.0], tab) == oracle.threshold_eval(method, [40.0, 200.0], tab)
    np.testing.assert_allclose(-oracle.threshold_eval(method, [90.0, 90.0], tab), ref(counts, [90]), rtol=1e-12)


def test_oracle_brute_force_k2_optimum_is_a_global_max(golden):
    counts = golden["counts"]
    tab = oracle.threshold_tables(counts, "otsu")
    best = max((-oracle.threshold_eval("otsu", [a, b], tab), a, b)
               for a, b in itertools.combinations(range(0, 256, 3), 2))
    assert best[0] >= -oracle.threshold_eval("otsu", [float(golden["brute"][0])], tab) - 1e-9


# ---------------------------------------------------------------------------- GPU


def synthetic_image(size=1024, seed=0):
    """Trimodal 8-bit image (the bimodal pattern of test_imaging.py:259-262 plus a third mode)."""
    rnd = np.random.default_rng(seed)
    n = size * size
    comp = rnd.choice(3, size=n, p=[0.4, 0.35, 0.25])
    mu = np.array([60.0, 130.0, 200.0])[comp]
    sd = np.array([12.0, 10.0, 14.0])[comp]
    return np.clip(np.rint(rnd.normal(mu, sd)), 0, 255).astype(np.uint8).reshape(size, size)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["otsu", "kapur"])
def test_device_tables_match_oracle(method):
    from paper_2510_14982_b200 import imaging

    img = synthetic_image(512)
    counts = imaging.histogram_device(img).cpu().numpy()
    assert np.array_equal(counts, np.bincount(img.ravel(), minlength=256))
    got = imaging.threshold_tables_device(counts, method).cpu().numpy()
    want = oracle.threshold_tables(counts, method)
    if method == "otsu":
        assert np.array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=1e-14, atol=1e-16)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["otsu", "kapur"])
@pytest.mark.parametrize("k", [1, 2, 3, 5, 8])
def test_device_eval_matches_oracle(method, k):
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    obj = imaging.multilevel_objective(counts, k, method)
    rnd = np.random.default_rng(k)
    x = rnd.uniform(-20.0, 275.0, size=(301, k))
    x[0] = 127.5  # all thresholds equal: k-1 empty classes
    got = pz.evaluate_batch(obj, x)
    want = np.array([oracle.threshold_eval(method, r, obj.table) for r in x])
    if method == "otsu":
        assert np.array_equal(got, want)
    else:
        np.testing.assert_allclose(got, want, rtol=KAPUR_RTOL)


@pytest.mark.gpu
@pytest.mark.parametrize("method", ["otsu", "kapur"])
def test_batch_runs_match_oracle(method):
    """C3 shape (small): k = 2..5 thresholds x 4 seeds, batched kernel (table in SMEM) vs the oracle run loop."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    for k in (2, 3, 5):
        obj = imaging.multilevel_objective(counts, k, method)
        cfg = pz.ApoConfig(ps=50, dim=k, bounds=pz.Bounds(0.0, 255.0, k), max_iterations=60)
        seeds = list(range(4))
        res = pz.run_batch(cfg, [obj] * 4, seeds)
        name = f"{method}_ml"
        want, _ = oracle.run_many([name] * 4, seeds, ps=50, dim=k, max_iterations=60, lower=0.0, upper=255.0,
                                  tables=[obj.table] * 4)
        if method == "otsu":
            assert np.array_equal(res.best_fitness, want)
        else:
            np.testing.assert_allclose(res.best_fitness, want, rtol=1e-9)


@pytest.mark.gpu
def test_apo_multithreshold_finds_the_k2_optimum():
    import paper_2510_14982_b200 as pz

    img = synthetic_image(512)
    counts = np.bincount(img.ravel(), minlength=256)
    res = pz.apo_multithreshold(img, 2, "otsu", ps=100, iterations=200, seed=0)
    tab = oracle.threshold_tables(counts, "otsu")
    best = max(-oracle.threshold_eval("otsu", [a, b], tab) for a, b in itertools.combinations(range(256), 2))
    assert res.value >= best * (1 - 1e-9)
    assert len(res.thresholds) == 2 and res.thresholds[0] <= res.thresholds[1]


@pytest.mark.gpu
def test_concurrent_stream_batches_match_sequential():
    """run_batch on side streams with results dropped early must not let the caching allocator
    recycle in-flight buffers (regression: record_stream in engine.run_batch)."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    jobs = []
    for method in ("otsu", "kapur"):
        for k in (2, 3, 4):
            jobs.append((imaging.multilevel_objective(counts, k, method),
                         pz.ApoConfig(ps=64, dim=k, bounds=pz.Bounds(0.0, 255.0, k), max_iterations=200)))
    seq = [pz.run_batch(cfg, [obj] * 6, list(range(6)), want_trace=False).best_fitness for obj, cfg in jobs]
    streams = [torch.cuda.Stream() for _ in jobs]
    for (obj, cfg), st in zip(jobs, streams):  # results dropped while the kernels run
        pz.run_batch(cfg, [obj] * 6, list(range(6)), want_trace=False, device_out=True, stream=st)
    outs = [pz.run_batch(cfg, [obj] * 6, list(range(6)), want_trace=False, device_out=True, stream=st,
                         threads_per_run=256 if k % 2 else 0)
            for k, ((obj, cfg), st) in enumerate(zip(jobs, streams))]
    torch.cuda.synchronize()
    for o, s in zip(outs, seq):
        assert np.array_equal(o.best_fitness.cpu().numpy(), s)


@pytest.mark.gpu
def test_max_threshold_count_matches_oracle():
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    for method in ("otsu", "kapur"):
        obj = imaging.multilevel_objective(counts, 32, method)
        x = np.random.default_rng(5).uniform(0.0, 255.0, size=(64, 32))
        got = pz.evaluate_batch(obj, x)
        want = np.array([oracle.threshold_eval(method, r, obj.table) for r in x])
        np.testing.assert_allclose(got, want, rtol=KAPUR_RTOL)


@pytest.mark.gpu
def test_persistent_batch_mixed_tables_match_oracle():
    """More runs than SMs (persistent CTAs, costliest-first claims) with two different prefix tables:
    each claimed run re-stages its own table in shared memory."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    objs = {m: imaging.multilevel_objective(counts, 3, m) for m in ("otsu", "kapur")}
    methods = ["otsu", "kapur"] * 90
    seeds = list(range(len(methods)))
    cfg = pz.ApoConfig(ps=30, dim=3, bounds=pz.Bounds(0.0, 255.0, 3), max_iterations=30)
    res = pz.run_batch(cfg, [objs[m] for m in methods], seeds, want_trace=False)
    for m in ("otsu", "kapur"):
        idx = [i for i, x in enumerate(methods) if x == m]
        want, _ = oracle.run_many([f"{m}_ml"] * len(idx), [seeds[i] for i in idx], ps=30, dim=3,
                                  max_iterations=30, lower=0.0, upper=255.0, tables=[objs[m].table] * len(idx))
        if m == "otsu":
            assert np.array_equal(res.best_fitness[idx], want)
        else:
            np.testing.assert_allclose(res.best_fitness[idx], want, rtol=1e-9)


@pytest.mark.gpu
def test_side_stream_batch_with_a_dropped_objective():
    """The objective (and so its cached device table) is dropped while the kernel runs on a side stream."""
    import gc

    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    counts = np.bincount(synthetic_image(256).ravel(), minlength=256)
    cfg = pz.ApoConfig(ps=64, dim=4, bounds=pz.Bounds(0.0, 255.0, 4), max_iterations=300)
    want = pz.run_batch(cfg, [imaging.multilevel_objective(counts, 4, "otsu")] * 8, list(range(8)),
                        want_trace=False).best_fitness
    st = torch.cuda.Stream()
    out = pz.run_batch(cfg, [imaging.multilevel_objective(counts, 4, "otsu")] * 8, list(range(8)),
                       want_trace=False, device_out=True, stream=st)
    gc.collect()
    junk = [torch.full((4096,), -1.0e300, dtype=torch.float64, device="cuda") for _ in range(64)]  # reuse bait
    torch.cuda.synchronize()
    del junk
    assert np.array_equal(out.best_fitness.cpu().numpy(), want)
