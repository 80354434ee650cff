"""One population sharded by rank across processes (BASELINE config 4).

The reference's distributed-correctness contract is worker-count
independence (test_engine.py:209-217); here it becomes
partition independence: a sharded run equals the single-process run bit for
bit.  CPU: the ShardedRun orchestration (plan, in-place all-gather layout,
MIN/SUM reductions) over a world-size-2 gloo group, with the oracle as the
compute engine.  GPU: the CUDA range kernels with several virtual partitions
in one process against the single-GPU device loop and the oracle.
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2510_14982_b200.core import ApoConfig
from paper_2510_14982_b200.objectives import Bounds
from paper_2510_14982_b200.shard import ShardedRun, ShardPlan, decode_keys, encode_keys


def test_plan_partitions_whole_groups():
    for ps, world in [(1, 1), (100, 8), (1000, 8), (1_000_000, 8), (4096, 3), (33, 2)]:
        plan = ShardPlan(ps, world)
        assert plan.chunk % 32 == 0 and plan.ps_pad == plan.chunk * world >= ps
        covered = []
        for r in range(world):
            lo, hi = plan.range(r)
            assert lo == hi or lo == r * plan.chunk
            covered.extend(range(lo, hi))
        assert covered == list(range(ps))


@pytest.mark.parametrize("blocks", [2, 3, 4])
def test_block_plan_covers_every_rank_once(blocks):
    for ps, world in [(100, 8), (1000, 3), (1_000_000, 8), (4097, 2), (33, 2)]:
        plan = ShardPlan(ps, world, blocks)
        assert plan.chunk % 32 == 0 and plan.ps_pad == plan.chunk * world * blocks >= ps
        covered = []
        for s in range(blocks):  # block s of every rank is one contiguous span (in-place all-gather)
            span = [plan.block(r, s) for r in range(world)]
            for r, (lo, hi) in enumerate(span):
                assert lo == hi or lo == (s * world + r) * plan.chunk
            covered.extend(i for lo, hi in span for i in range(lo, hi))
        assert sorted(covered) == list(range(ps))


def test_key_encoding_round_trips_and_orders():
    x = np.array([-np.inf, -3.5, -1e-300, -0.0, 0.0, 1e-300, 2.0, np.inf, np.nan])
    k = encode_keys(x)
    back = decode_keys(k)
    assert np.array_equal(back[:-1], np.where(x[:-1] == 0, 0.0, x[:-1])) and np.isnan(back[-1])
    assert np.all(np.diff(k[:-1].astype(np.float64)) >= 0) and k[3] == k[4]


class OracleEngine:
    """Test-only stand-in for the device shard: the oracle iteration, replicated per process."""

    def __init__(self, cfg, obj, plan):
        self.cfg, self.plan, self.name = cfg, plan, obj.name
        self.cur = 0

    def initialize(self):
        c = self.cfg
        pos, fit = oracle.initialize(c.seed, c.ps, c.dim, c.bounds.lower, c.bounds.upper, self.name)
        self.pos = [torch.zeros(self.plan.ps_pad, c.dim, dtype=torch.float64) for _ in range(2)]
        self.fit = [torch.full((self.plan.ps_pad,), np.inf, dtype=torch.float64) for _ in range(2)]
        self.pos[0][:c.ps] = torch.from_numpy(pos)
        self.fit[0][:c.ps] = torch.from_numpy(fit)
        self.trace = [float(fit.min())]
        self.warn = 0
        self.cur, self.t = 0, 0

    def begin(self):
        c = self.cfg
        fit = self.fit[self.cur][:c.ps].numpy()
        self.order = oracle.argsort_stable(fit)
        self.in_dr = oracle.select_dr(c.seed, self.t + 1, c.ps, c.pf_max)
        self.trace.append(np.inf)

    def update_range(self, lo, hi):
        c = self.cfg
        sp = self.pos[self.cur][:c.ps].numpy()[self.order]
        sf = self.fit[self.cur][:c.ps].numpy()[self.order]
        out = oracle.run_updates(sp, sf, self.in_dr, seed=c.seed, iteration=self.t, max_iterations=c.max_iterations,
                                 name=self.name, lower=c.bounds.lower, upper=c.bounds.upper)
        nxt = self.cur ^ 1
        self.pos[nxt][lo:hi] = torch.from_numpy(out[0][lo:hi])
        self.fit[nxt][lo:hi] = torch.from_numpy(out[1][lo:hi])
        if hi > lo:
            self.trace[-1] = min(self.trace[-1], float(out[1][lo:hi].min()))
        self.warn += int(out[3][lo:hi].sum())

    def next_buffers(self):
        return self.pos[self.cur ^ 1], self.fit[self.cur ^ 1]

    def end(self):
        self.cur ^= 1
        self.t += 1

    def current(self):
        return self.pos[self.cur], self.fit[self.cur]

    def counters(self, n):
        return encode_keys(np.array(self.trace[:n + 1])), self.warn

    def close(self):
        pass


def _worker(rank, world, port, cfg, name, q, blocks=None):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        run = ShardedRun(cfg, name, engine=OracleEngine, blocks=blocks)
        run.initialize()
        run.iterate(cfg.max_iterations)
        pos, fit = run.population()
        trace, warn = run.trace_and_warnings()
        q.put((rank, pos, fit, trace, warn))
    finally:
        dist.destroy_process_group()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("name,ps,blocks", [("rosenbrock", 100, 1), ("griewank", 77, None), ("sphere", 200, 3)])
def test_gloo_world2_sharded_run_equals_single_process(name, ps, blocks):
    """blocks = 1: one all-gather per iteration; None (default 4, capped by ps) / 3: block-interleaved
    ranks with one asynchronous in-place all-gather per block."""
    cfg = ApoConfig(ps=ps, dim=6, bounds=Bounds(-5.0, 5.0, 6), max_iterations=12, seed=3)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, cfg, name, q, blocks)) for r in range(2)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = oracle.run(ps=ps, dim=6, max_iterations=12, seed=3, name=name, lower=-5.0, upper=5.0)
    for rank, pos, fit, trace, warn in got:
        assert np.array_equal(pos, want["positions"]) and np.array_equal(fit, want["fitness"]), rank
        assert np.array_equal(trace, want["trace"]) and warn == want["warnings"]


# ---------------------------------------------------------------------------- GPU


@pytest.mark.gpu
@pytest.mark.parametrize("name,ps,dim,world", [("rosenbrock", 1000, 20, 3), ("sphere", 4096, 100, 8),
                                               ("cec2022_f6", 2000, 50, 4), ("cec2022_f10", 777, 20, 5)])
def test_virtual_partitions_equal_single_gpu_and_oracle(name, ps, dim, world):
    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=15, seed=11)
    sh = ShardedRun(cfg, name, virtual_world=world, blocks=3)
    sh.initialize()
    sh.iterate(15)
    pos, fit = sh.population()
    trace, warn = sh.trace_and_warnings()
    sh.close()
    one = ShardedRun(cfg, name, virtual_world=1)
    one.initialize()
    one.iterate(15)
    pos1, fit1 = one.population()
    one.close()
    assert np.array_equal(pos, pos1) and np.array_equal(fit, fit1)
    ref = pz.run(cfg, name)  # device-resident loop (slot layout, SEL buffers)
    assert np.array_equal(trace, ref.trace) and warn == ref.warnings
    assert np.array_equal(fit, ref.population.fitness) and np.array_equal(pos, ref.population.positions)
    if not name.startswith("cec"):
        want = oracle.run(ps=ps, dim=dim, max_iterations=15, seed=11, name=name, lower=-100.0, upper=100.0)
        assert np.array_equal(pos, want["positions"]) and np.array_equal(trace, want["trace"])


# ---------------------------------------------------------------------------- independent runs


def oracle_batch(cfg, objs, seeds, want_trace=False):
    """Test-only stand-in for run_batch: the oracle run per (objective, seed), packed like BatchResult."""
    from paper_2510_14982_b200.engine import BatchResult

    outs = [oracle.run(ps=cfg.ps, dim=cfg.dim, max_iterations=cfg.max_iterations, seed=int(s), name=o.name,
                       lower=cfg.bounds.lower, upper=cfg.bounds.upper) for o, s in zip(objs, seeds)]
    return BatchResult(best_fitness=np.array([o["best_fitness"] for o in outs]),
                       best_position=np.stack([o["best_position"] for o in outs]),
                       trace=np.stack([o["trace"] for o in outs]) if want_trace else None,
                       warnings=np.array([o["warnings"] for o in outs], dtype=np.int64))


RUN_MANY_NAMES = ["sphere", "rosenbrock", "griewank", "hgbat", "bent_cigar"]
RUN_MANY_SEEDS = [0, 1, 2]


def _run_many_worker(rank, world, port, cfg, q):
    from paper_2510_14982_b200.engine import run_many

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        names = [n for n in RUN_MANY_NAMES for _ in RUN_MANY_SEEDS]
        seeds = [s for _ in RUN_MANY_NAMES for s in RUN_MANY_SEEDS]
        res = run_many(cfg, names, seeds, want_trace=True, batch_fn=oracle_batch)
        q.put((rank, res.best_fitness, res.best_position, res.trace, res.warnings, res.objectives, res.seeds))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_gloo_run_many_round_robin_equals_serial(world):
    """(objective, seed) runs round-robin over ranks, no collective while they run, one
    all-gather at the end; every rank ends with all runs in submission order, equal to the serial loop of
    the reference (engine.py:270-275) run by the oracle."""
    cfg = ApoConfig(ps=20, dim=5, bounds=Bounds(-10.0, 10.0, 5), max_iterations=15, seed=0)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run_many_worker, args=(r, world, port, cfg, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = [q.get(timeout=120) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    names = [n for n in RUN_MANY_NAMES for _ in RUN_MANY_SEEDS]
    seeds = [s for _ in RUN_MANY_NAMES for s in RUN_MANY_SEEDS]
    for rank, best, bpos, trace, warn, objs, sds in got:
        assert list(objs) == names and list(sds) == seeds
        for k, (n, s) in enumerate(zip(names, seeds)):
            want = oracle.run(ps=20, dim=5, max_iterations=15, seed=s, name=n, lower=-10.0, upper=10.0)
            assert best[k] == want["best_fitness"] and np.array_equal(bpos[k], want["best_position"]), (rank, k)
            assert np.array_equal(trace[k], want["trace"]) and warn[k] == want["warnings"]


@pytest.mark.gpu
def test_run_many_single_process_equals_oracle():
    """run_many at world size 1 is run_batch on the device: every run equals the oracle's serial run."""
    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.engine import run_many

    cfg = pz.ApoConfig(ps=20, dim=5, bounds=pz.Bounds(-10.0, 10.0, 5), max_iterations=15, seed=0)
    names = [n for n in RUN_MANY_NAMES for _ in RUN_MANY_SEEDS]
    seeds = [s for _ in RUN_MANY_NAMES for s in RUN_MANY_SEEDS]
    res = run_many(cfg, names, seeds, want_trace=True)
    want = oracle_batch(cfg, [pz.get_objective(n) for n in names], seeds, want_trace=True)
    assert np.array_equal(res.best_fitness, want.best_fitness)
    assert np.array_equal(res.best_position, want.best_position)
    assert np.array_equal(res.trace, want.trace) and np.array_equal(res.warnings, want.warnings)
