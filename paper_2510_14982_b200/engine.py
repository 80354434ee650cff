"""Run orchestration on the B200 (API parity with protozoa.engine).

``initialize`` / ``step`` / ``run`` / ``benchmark`` keep the reference's
signatures and results (engine.py:116-284).  What changes is where the loop
lives:

* ``step`` performs the reference's three phases on the device -- stable
  sort (C-ABI ``apo_sort_order``), coordinator draws (``apo_select_dr``) and
  the fused update (``run_updates`` of the cuda backend);
* ``run`` never returns to the host per iteration: small populations run in
  one persistent CTA with the population in shared memory
  (``apo_run_batch``), large ones in the device-resident loop
  (``apo_run_*``: key sort -> Dr -> one fused update launch per iteration);
* ``run_many`` batches independent (seed, objective) runs, one CTA each, and
  shards them across GPUs when torch.distributed is initialised (no
  collective; results gathered once at the end).
"""

from __future__ import annotations

import ctypes as C
import math
import time
from dataclasses import dataclass, field, replace
from statistics import fmean
from typing import Optional, Sequence

import numpy as np

from . import _lib, kernels
from .core import ApoConfig, ConfigError, Population, p_dr_table, schedule_table
from .objectives import EXTERNAL, Objective, device_objective, resolve_objective

SEQUENTIAL = "sequential"
PARALLEL = "parallel"

# Largest population routed to the single-CTA shared-memory kernel by run().
BATCH_PS_LIMIT = 256


@dataclass(frozen=True)
class EngineMode:
    """``sequential`` or ``parallel`` (engine.py:40-65).  On the device both
    modes run the same kernels; results never depend on the mode."""

    kind: str = SEQUENTIAL
    workers: object = None

    def __post_init__(self) -> None:
        if self.kind not in (SEQUENTIAL, PARALLEL):
            raise ValueError(f"kind must be {SEQUENTIAL!r} or {PARALLEL!r}, got {self.kind!r}")
        w = self.workers
        if w is not None and w != "auto" and not (isinstance(w, int) and w >= 1):
            raise ValueError(f"workers must be a positive integer or 'auto', got {w!r}")

    @staticmethod
    def sequential() -> "EngineMode":
        return EngineMode(SEQUENTIAL)

    @staticmethod
    def parallel(workers: object = "auto") -> "EngineMode":
        return EngineMode(PARALLEL, workers)


@dataclass
class RunResult:
    """Outcome of one run (engine.py:68-89)."""

    best_position: np.ndarray
    best_fitness: float
    trace: np.ndarray
    iterations_run: int
    fe_count: int
    warnings: int
    wall_clock_seconds: float
    mode: str
    workers: int
    backend: str
    config_echo: ApoConfig
    population: Population = field(repr=False, default=None)


def _resolve_backend(objective: Objective, backend: Optional[str]):
    if objective.code == EXTERNAL:
        raise ValueError("external objective functions need the reference's numpy backend; "
                         "the cuda backend evaluates objectives on the device")
    return kernels.get_backend(backend)


def resolve_workers(mode: EngineMode, backend) -> int:
    if mode.kind == SEQUENTIAL:
        return 1
    cap = max(1, int(backend.max_workers()))
    if mode.workers in (None, "auto"):
        return cap
    return min(int(mode.workers), cap)


def _check(cfg: ApoConfig, obj: Objective) -> None:
    bad = cfg.violations()
    if bad:
        raise ConfigError("invalid configuration:\n" + "\n".join(f"  - {b}" for b in bad))
    if cfg.dim < obj.min_dim:
        raise ConfigError(f"objective {obj.name!r} needs dim >= {obj.min_dim}, got dim = {cfg.dim}")


def _dev():
    import torch

    return torch.device("cuda", torch.cuda.current_device())


def _to_device(arr: np.ndarray, dev):
    """Host array -> device tensor; page-locked arrays (from _to_host) copy asynchronously at full PCIe rate."""
    import torch

    t = torch.from_numpy(np.ascontiguousarray(arr))
    return t.to(dev, non_blocking=t.is_pinned())


def _to_host(*tensors):
    """Device tensors -> numpy arrays backed by page-locked host memory (torch's caching host
    allocator), so a Population returned here can be fed back to step() without a staging copy."""
    import torch

    outs = []
    for t in tensors:
        h = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        h.copy_(t, non_blocking=True)
        outs.append(h)
    torch.cuda.current_stream().synchronize()
    return [h.numpy() for h in outs]


def initialize(cfg: ApoConfig, objective) -> Population:
    """Iteration-0 population on the device (engine.py:116-139); fe_count = ps."""
    import torch

    obj = resolve_objective(objective)
    _check(cfg, obj)
    if obj.code == EXTERNAL:
        raise ValueError("external objective functions cannot run on the cuda backend")
    lib = _lib.require_cuda()
    pos = torch.empty((cfg.ps, cfg.dim), dtype=torch.float64, device=_dev())
    fit = torch.empty(cfg.ps, dtype=torch.float64, device=pos.device)
    dobj = device_objective(obj, cfg.dim)
    _lib.check(lib.apo_initialize(cfg.seed, cfg.ps, cfg.dim, cfg.dim, cfg.bounds.lower, cfg.bounds.span, dobj.ref,
                                  _lib.ptr(pos), _lib.ptr(fit), _lib.stream_handle()), "apo_initialize")
    hp, hf = _to_host(pos, fit)
    return Population(hp, hf, iteration=0, fe_count=cfg.ps, warnings=0)


STEP_CHUNK_MIN_PS = 1 << 16  # step(): overlap the result's D2H with the update from this size on

_COPY_STREAMS: dict = {}


def _copy_stream(dev):
    """One long-lived side stream per device for step()'s copies: torch's caching allocator keeps blocks
    per stream, so a fresh stream each call would strand the 800 MB row buffer of the last call and
    allocate a new one (cudaMalloc/cudaFree spikes of 100-200 ms)."""
    import torch

    key = str(dev)
    st = _COPY_STREAMS.get(key)
    if st is None:
        st = _COPY_STREAMS[key] = torch.cuda.Stream(device=dev)
    return st


def step(pop: Population, cfg: ApoConfig, objective, iteration: int, mode: EngineMode = None,
         backend: Optional[str] = None, draws=None) -> Population:
    """One full iteration; returns the next population, input untouched (engine.py:142-172).

    draws: an rng.DrawTable -- every draw of the iteration is read from it instead of the keyed stream
    (the reference replays its hand-traced example this way, tests/test_acceptance.py:50-175); a draw the
    table lacks raises LookupError."""
    import torch

    mode = mode or EngineMode.sequential()
    obj = resolve_objective(objective)
    if pop.size != cfg.ps or pop.dim != cfg.dim:
        raise ValueError(f"population shape ({pop.size}, {pop.dim}) does not match config "
                         f"(ps={cfg.ps}, dim={cfg.dim})")
    if draws is not None:
        from .kernels import cuda_backend

        dev = _dev()
        new_pos, new_fit, _acc, warned = cuda_backend.scripted_step_device(
            _to_device(pop.positions, dev), _to_device(pop.fitness, dev), cfg, obj, iteration, draws)
        hp, hf = _to_host(new_pos, new_fit)
        return Population(hp, hf, iteration=iteration + 1, fe_count=pop.fe_count + cfg.ps,
                          warnings=pop.warnings + warned)
    bk = _resolve_backend(obj, backend)
    workers = resolve_workers(mode, bk)
    if cfg.rng != "keyed":
        raise ValueError("step() is the reference-facing per-iteration path and uses the reference's keyed "
                         "stream; Philox production mode runs through run()/run_batch()/DeviceRun")
    lib = _lib.require_cuda()
    dev = _dev()
    stream = _lib.stream_handle()
    lean = cfg.ps >= STEP_CHUNK_MIN_PS and bk.NAME == "cuda" and cfg.dim <= 256
    main = torch.cuda.current_stream()
    # fitness first (8 bytes per row): the stable sort and the coordinator draws run while the rows
    # stream in on a second stream
    fit = _to_device(pop.fitness, dev)
    if lean:
        copy = _copy_stream(dev)
        with torch.cuda.stream(copy):
            pos = _to_device(pop.positions, dev)
        pos.record_stream(main)
    else:
        pos = _to_device(pop.positions, dev)
    order = torch.empty(cfg.ps, dtype=torch.int32, device=dev)
    _lib.check(lib.apo_sort_order(_lib.ptr(fit), cfg.ps, _lib.ptr(order), stream), "apo_sort_order")
    in_dr = torch.empty(cfg.ps, dtype=torch.uint8, device=dev)
    _lib.check(lib.apo_select_dr(cfg.seed, iteration + 1, cfg.ps, cfg.pf_max, _lib.ptr(in_dr), None, stream),
               "apo_select_dr")
    if lean:
        # large populations: no snapshot gather (the update reads rows through order[]); finished rank
        # chunks are copied back while the next chunk updates
        from .kernels import cuda_backend

        main.wait_stream(copy)
        hp, hf, warned = cuda_backend.run_updates_to_host(pos, fit, in_dr, cfg, obj, iteration, iteration + 1,
                                                          order=order)
    elif cfg.ps >= STEP_CHUNK_MIN_PS and bk.NAME == "cuda":  # D > 256: the warp kernel reads rank-ordered rows
        from .kernels import cuda_backend

        idx = order.long()
        hp, hf, warned = cuda_backend.run_updates_to_host(pos.index_select(0, idx), fit.index_select(0, idx), in_dr,
                                                          cfg, obj, iteration, iteration + 1)
    else:
        idx = order.long()
        snap_pos = pos.index_select(0, idx).contiguous()
        snap_fit = fit.index_select(0, idx).contiguous()
        new_pos, new_fit, _acc, warned = bk.run_updates(snap_pos, snap_fit, in_dr, cfg, obj, iteration,
                                                        iteration + 1, parallel=(mode.kind == PARALLEL),
                                                        workers=workers)
        hp, hf = _to_host(new_pos, new_fit)
    return Population(hp, hf, iteration=iteration + 1, fe_count=pop.fe_count + cfg.ps,
                      warnings=pop.warnings + warned)


# ---------------------------------------------------------------------------
# device-resident runs


class DeviceRun:
    """A population resident in HBM driven by the C-ABI run handle."""

    def __init__(self, cfg: ApoConfig, obj: Objective, stream=None):
        import torch

        self.lib = _lib.require_cuda()
        self.cfg = cfg
        self.obj = obj
        self.dobj = device_objective(obj, cfg.dim)
        self.stream = stream
        sched = np.ascontiguousarray(schedule_table(cfg.max_iterations)) if cfg.max_iterations else np.zeros(3)
        pdr = np.ascontiguousarray(p_dr_table(cfg.ps))
        h = C.c_void_p()
        _lib.check(self.lib.apo_run_create(C.byref(h), cfg.ps, cfg.dim, cfg.max_iterations, cfg.seed,
                                           cfg.neighbor_pairs, cfg.pf_max, cfg.bounds.lower, cfg.bounds.upper,
                                           cfg.eps, self.dobj.ref, sched.ctypes.data, pdr.ctypes.data,
                                           rng_code(cfg), _lib.stream_handle(stream)), "apo_run_create")
        self.handle = h
        self._torch = torch

    def initialize(self):
        _lib.check(self.lib.apo_run_initialize(self.handle), "apo_run_initialize")

    def load(self, pop: Population):
        """Resume from a checkpointed population (reference row order) after pop.iteration iterations."""
        pos = np.ascontiguousarray(pop.positions, dtype=np.float64)
        fit = np.ascontiguousarray(pop.fitness, dtype=np.float64)
        if pos.shape != (self.cfg.ps, self.cfg.dim) or fit.shape != (self.cfg.ps,):
            raise ValueError("population shape does not match the run configuration")
        _lib.check(self.lib.apo_run_load(self.handle, pos.ctypes.data, fit.ctypes.data, 1, int(pop.iteration),
                                         int(pop.warnings)), "apo_run_load")
        self.start_iteration = int(pop.iteration)

    def iterate(self, n: int):
        _lib.check(self.lib.apo_run_iterate(self.handle, n), "apo_run_iterate")

    def counters(self):
        it, fe, w = C.c_int64(), C.c_int64(), C.c_int64()
        _lib.check(self.lib.apo_run_counters(self.handle, C.byref(it), C.byref(fe), C.byref(w)), "apo_run_counters")
        return it.value, fe.value, w.value

    def trace(self, n: int) -> np.ndarray:
        out = np.empty(n + 1)
        _lib.check(self.lib.apo_run_trace(self.handle, out.ctypes.data, n), "apo_run_trace")
        return out

    def best(self):
        f = C.c_double()
        row = C.c_int64()
        x = np.empty(self.cfg.dim)
        _lib.check(self.lib.apo_run_best(self.handle, C.byref(f), x.ctypes.data, C.byref(row)), "apo_run_best")
        return f.value, x, row.value

    def population(self):
        """(positions, fitness) in reference row order, host numpy arrays (views of page-locked
        buffers from torch's caching host allocator: the copy runs at full PCIe rate and a repeated
        call reuses the pages instead of faulting fresh ones in)."""
        pos = self._torch.empty((self.cfg.ps, self.cfg.dim), dtype=self._torch.float64, pin_memory=True)
        fit = self._torch.empty(self.cfg.ps, dtype=self._torch.float64, pin_memory=True)
        _lib.check(self.lib.apo_run_population(self.handle, pos.data_ptr(), fit.data_ptr(), 1),
                   "apo_run_population")
        return pos.numpy(), fit.numpy()

    def profile(self, enable: bool = True):
        _lib.check(self.lib.apo_run_profile(self.handle, 1 if enable else 0), "apo_run_profile")

    def profile_read(self):
        """(summed ms, launches) of the fused update kernel since profile()."""
        ms, n = C.c_double(), C.c_int64()
        _lib.check(self.lib.apo_run_profile_read(self.handle, C.byref(ms), C.byref(n)), "apo_run_profile_read")
        return ms.value, n.value

    def profile_split(self):
        """(candidate-kernel ms, CEC evaluation-kernel ms, iterations) since profile()."""
        a, b, n = C.c_double(), C.c_double(), C.c_int64()
        _lib.check(self.lib.apo_run_profile_split(self.handle, C.byref(a), C.byref(b), C.byref(n)),
                   "apo_run_profile_split")
        return a.value, b.value, n.value

    def update_path(self) -> str:
        """Kernels of one iteration's update: "fused" (one kernel), "cec_split", "cec_fused", "cec_gemm",
        "basic_split" (apo_run_update_path)."""
        p = C.c_int()
        _lib.check(self.lib.apo_run_update_path(self.handle, C.byref(p)), "apo_run_update_path")
        return ("fused", "cec_split", "cec_fused", "cec_gemm", "basic_split")[p.value]

    def close(self):
        if self.handle:
            self.lib.apo_run_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def rng_code(cfg: ApoConfig) -> int:
    """APO_RNG_KEYED (0, reference stream, oracle mode) or APO_RNG_PHILOX (1, production)."""
    return 1 if cfg.rng == "philox" else 0


def _batch_fits(cfg: ApoConfig, objectives=()) -> bool:
    """Whether (ps, dim) and these objectives fit the shared-memory batch kernel."""
    lib = _lib.require_cuda()
    objs = [resolve_objective(o) for o in objectives]
    if not objs:
        return int(lib.apo_run_batch_max_elems(cfg.ps, cfg.dim)) > 0
    descs = (_lib.apo_objective * len(objs))()
    for k, o in enumerate(objs):
        descs[k] = device_objective(o, cfg.dim).struct
    return bool(lib.apo_run_batch_fits(cfg.ps, cfg.dim, descs, len(objs)))


def run(cfg: ApoConfig, objective, mode: Optional[EngineMode] = None, backend: Optional[str] = None) -> RunResult:
    """Full run: initialise, then iterate within the iteration / evaluation budget (engine.py:175-212)."""
    mode = mode or EngineMode.sequential()
    obj = resolve_objective(objective)
    bk = _resolve_backend(obj, backend)
    workers = resolve_workers(mode, bk)
    _check(cfg, obj)
    n_iters = cfg.iterations_within_budget()
    started = time.perf_counter()
    if cfg.ps <= BATCH_PS_LIMIT and _batch_fits(cfg, [obj]):
        b = run_batch(cfg, [obj], [cfg.seed], want_population=True)
        seconds = time.perf_counter() - started
        return RunResult(best_position=b.best_position[0], best_fitness=float(b.best_fitness[0]), trace=b.trace[0],
                         iterations_run=n_iters, fe_count=cfg.ps * (1 + n_iters), warnings=int(b.warnings[0]),
                         wall_clock_seconds=seconds, mode=mode.kind, workers=workers, backend=bk.NAME,
                         config_echo=cfg,
                         population=Population(b.final_pos[0], b.final_fit[0], iteration=n_iters,
                                               fe_count=cfg.ps * (1 + n_iters), warnings=int(b.warnings[0])))
    dr = DeviceRun(cfg, obj)
    try:
        dr.initialize()
        dr.iterate(n_iters)
        it, fe, warned = dr.counters()
        trace = dr.trace(it)
        best_f, best_x, _ = dr.best()
        pos, fit = dr.population()
    finally:
        dr.close()
    seconds = time.perf_counter() - started
    return RunResult(best_position=best_x, best_fitness=best_f, trace=trace, iterations_run=it, fe_count=fe,
                     warnings=warned, wall_clock_seconds=seconds, mode=mode.kind, workers=workers, backend=bk.NAME,
                     config_echo=cfg,
                     population=Population(pos, fit, iteration=it, fe_count=fe, warnings=warned))


def resume(cfg: ApoConfig, objective, population: Population, backend: Optional[str] = None) -> RunResult:
    """Continue a run from a checkpointed Population (e.g. RunResult.population or a step() result) up to
    cfg's iteration / evaluation budget, on the device-resident loop.  Exact: the continuation equals the
    uninterrupted run (every draw is keyed by seed, iteration, individual and slot -- rng.py:1-19).
    The reference has no checkpointing; this is SURVEY.md 8(f) item 4."""
    obj = resolve_objective(objective)
    bk = _resolve_backend(obj, backend)
    _check(cfg, obj)
    if population.size != cfg.ps or population.dim != cfg.dim:
        raise ValueError("population shape does not match the configuration")
    n_total = cfg.iterations_within_budget()
    start = int(population.iteration)
    if not 0 <= start <= n_total:
        raise ValueError(f"population.iteration {start} outside [0, {n_total}]")
    started = time.perf_counter()
    dr = DeviceRun(cfg, obj)
    try:
        dr.load(population)
        dr.iterate(n_total - start)
        it, fe, warned = dr.counters()
        trace = dr.trace(it)[start:]
        trace[0] = float(np.min(population.fitness))
        best_f, best_x, _ = dr.best()
        pos, fit = dr.population()
    finally:
        dr.close()
    return RunResult(best_position=best_x, best_fitness=best_f, trace=trace, iterations_run=it, fe_count=fe,
                     warnings=warned, wall_clock_seconds=time.perf_counter() - started, mode=SEQUENTIAL, workers=1,
                     backend=bk.NAME, config_echo=cfg,
                     population=Population(pos, fit, iteration=it, fe_count=fe, warnings=warned))


@dataclass
class BatchResult:
    """Outcome of ``run_batch``/``run_many``: arrays indexed by run."""

    best_fitness: np.ndarray
    best_position: np.ndarray
    trace: Optional[np.ndarray]
    warnings: np.ndarray
    final_pos: Optional[np.ndarray] = None
    final_fit: Optional[np.ndarray] = None
    seconds: float = 0.0
    objectives: tuple = ()
    seeds: tuple = ()


def run_batch(cfg: ApoConfig, objectives: Sequence, seeds: Sequence[int], want_trace: bool = True,
              want_population: bool = False, device_out: bool = False, stream=None,
              threads_per_run: int = 0) -> BatchResult:
    """Independent runs (same ps/dim/bounds/T), each resident in one CTA's shared memory, on the current GPU.

    threads_per_run = 0 lets the library pick the launch shape (apo_run_batch_shaped); pass 256 when
    several batches run concurrently on different streams so their CTAs share the SMs."""
    import torch

    lib = _lib.require_cuda()
    objs = [resolve_objective(o) for o in objectives]
    if len(objs) != len(seeds):
        raise ValueError("one objective per seed")
    for o in objs:
        _check(cfg, o)
    if not _batch_fits(cfg, list({id(o): o for o in objs}.values())):
        raise ValueError(f"ps*dim = {cfg.ps * cfg.dim} does not fit the shared-memory batch kernel")
    n = len(objs)
    dev = _dev()
    n_iters = cfg.iterations_within_budget()
    descs = (_lib.apo_objective * n)()
    dobjs = {}
    for k, o in enumerate(objs):
        d = dobjs.setdefault(id(o), device_objective(o, cfg.dim))
        descs[k] = d.struct
    seeds_t = torch.as_tensor(np.array([int(s) for s in seeds], dtype=np.uint64).view(np.int64), device=dev)
    sched = torch.as_tensor(np.array(schedule_table(cfg.max_iterations))
                            if cfg.max_iterations else np.zeros(3), device=dev)
    pdr = torch.as_tensor(np.array(p_dr_table(cfg.ps)), device=dev)
    best_fit = torch.empty(n, dtype=torch.float64, device=dev)
    best_pos = torch.empty((n, cfg.dim), dtype=torch.float64, device=dev)
    trace = torch.empty((n, n_iters + 1), dtype=torch.float64, device=dev) if want_trace else None
    fpos = torch.empty((n, cfg.ps, cfg.dim), dtype=torch.float64, device=dev) if want_population else None
    ffit = torch.empty((n, cfg.ps), dtype=torch.float64, device=dev) if want_population else None
    warn = torch.zeros(n, dtype=torch.int64, device=dev)
    if stream is not None:
        # inputs were staged on the current stream; the caching allocator must not hand any of these
        # blocks to other work until the kernel on `stream` is done with them
        stream.wait_stream(torch.cuda.current_stream())
        for t in (seeds_t, sched, pdr, best_fit, best_pos, trace, fpos, ffit, warn):
            if t is not None:
                t.record_stream(stream)
        for d in dobjs.values():  # an Objective's tables may be freed while the kernel still reads them
            for t in d.keep:
                t.record_stream(stream)
    t0 = time.perf_counter()
    _lib.check(lib.apo_run_batch_shaped(n, _lib.ptr(seeds_t), descs, cfg.ps, cfg.dim, cfg.max_iterations, n_iters,
                                        cfg.neighbor_pairs, cfg.pf_max, cfg.bounds.lower, cfg.bounds.upper, cfg.eps,
                                        _lib.ptr(sched), _lib.ptr(pdr), _lib.ptr(best_fit), _lib.ptr(best_pos),
                                        _lib.ptr(trace), _lib.ptr(fpos), _lib.ptr(ffit), _lib.ptr(warn),
                                        rng_code(cfg), int(threads_per_run), _lib.stream_handle(stream)),
               "apo_run_batch_shaped")
    if device_out:
        return BatchResult(best_fit, best_pos, trace, warn, fpos, ffit, 0.0, tuple(o.name for o in objs),
                           tuple(seeds))

    if stream is not None:  # the host copies below run on the current stream: order them after the kernel
        torch.cuda.current_stream().wait_stream(stream)

    def host(t):
        return None if t is None else t.cpu().numpy()

    res = BatchResult(host(best_fit), host(best_pos), host(trace), host(warn), host(fpos), host(ffit), 0.0,
                      tuple(o.name for o in objs), tuple(seeds))
    res.seconds = time.perf_counter() - t0
    return res


def empty_cache() -> None:
    """Return the library's pooled device memory (run buffers, scratch) to the driver, like
    torch.cuda.empty_cache() does for torch's allocator."""
    _lib.check(_lib.require_cuda().apo_release_cached_memory(), "apo_release_cached_memory")


def run_many(cfg: ApoConfig, objectives: Sequence, seeds: Sequence[int], want_trace: bool = False,
             group=None, batch_fn=None) -> BatchResult:
    """Seeds x objectives sharded across the ranks of torch.distributed (if initialised).

    Run k goes to rank k % world_size; there is no collective while runs
    execute -- one all-gather of the per-run results at the end.  Results
    are identical for any world size (every draw is keyed by seed, not by
    placement).  ``batch_fn`` (default ``run_batch``) runs this rank's share; the CPU tests pass an
    oracle stand-in to exercise the sharding and the gather without a device.
    """
    import torch
    import torch.distributed as dist

    batch_fn = batch_fn or run_batch
    objs = [resolve_objective(o) for o in objectives]
    world = dist.get_world_size(group) if dist.is_available() and dist.is_initialized() else 1
    rank = dist.get_rank(group) if world > 1 else 0
    mine = list(range(rank, len(objs), world))
    local = batch_fn(cfg, [objs[k] for k in mine], [seeds[k] for k in mine], want_trace=want_trace) if mine else None
    if world == 1:
        return local
    n_iters = cfg.iterations_within_budget()
    width = 2 + cfg.dim + (n_iters + 1 if want_trace else 0)
    rows = np.full((len(mine), width), np.nan)
    for a, k in enumerate(mine):
        rows[a, 0] = k
        rows[a, 1] = local.best_fitness[a]
        rows[a, 2:2 + cfg.dim] = local.best_position[a]
        if want_trace:
            rows[a, 2 + cfg.dim:] = local.trace[a]
    per = -(-len(objs) // world)
    buf = np.full((per, width + 1), np.nan)
    buf[:len(mine), :width] = rows
    buf[:len(mine), width] = local.warnings if local is not None else 0
    backend = dist.get_backend(group)
    tdev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
    t = torch.as_tensor(buf, device=tdev)
    gathered = [torch.empty_like(t) for _ in range(world)]
    dist.all_gather(gathered, t, group=group)
    allrows = np.concatenate([g.cpu().numpy() for g in gathered])
    allrows = allrows[~np.isnan(allrows[:, 0])]
    allrows = allrows[np.argsort(allrows[:, 0], kind="stable")]
    return BatchResult(best_fitness=allrows[:, 1].copy(), best_position=allrows[:, 2:2 + cfg.dim].copy(),
                       trace=allrows[:, 2 + cfg.dim:width].copy() if want_trace else None,
                       warnings=allrows[:, width].astype(np.int64), objectives=tuple(o.name for o in objs),
                       seeds=tuple(seeds))


# ---------------------------------------------------------------------------
# seed-sweep benchmark (engine.py:215-284)


@dataclass
class ModeAggregate:
    mode: str
    workers: int
    best_fitness: list
    seconds: list
    results: list = field(repr=False, default_factory=list)

    @property
    def avg_best_fitness(self) -> float:
        return fmean(self.best_fitness)

    @property
    def avg_seconds(self) -> float:
        return fmean(self.seconds)


@dataclass
class BenchmarkResult:
    objective_name: str
    runs: int
    base_seed: int
    per_mode: dict
    speedup: Optional[float]

    def aggregate(self, kind: str) -> ModeAggregate:
        return self.per_mode[kind]


def benchmark(cfg: ApoConfig, objective, runs: int, modes: Sequence[EngineMode] = (),
              backend: Optional[str] = None) -> BenchmarkResult:
    if runs < 1:
        raise ValueError(f"runs must be >= 1, got {runs}")
    obj = resolve_objective(objective)
    mode_list = list(modes) or [EngineMode.sequential(), EngineMode.parallel()]
    per_mode: dict = {}
    for mode in mode_list:
        if mode.kind in per_mode:
            raise ValueError(f"duplicate mode {mode.kind!r} in benchmark request")
        agg = ModeAggregate(mode.kind, 0, [], [])
        for r in range(runs):
            res = run(replace(cfg, seed=cfg.seed + r), obj, mode, backend=backend)
            agg.workers = res.workers
            agg.best_fitness.append(res.best_fitness)
            agg.seconds.append(res.wall_clock_seconds)
            agg.results.append(res)
        per_mode[mode.kind] = agg
    speedup = None
    if SEQUENTIAL in per_mode and PARALLEL in per_mode:
        par = per_mode[PARALLEL].avg_seconds
        speedup = per_mode[SEQUENTIAL].avg_seconds / par if par > 0.0 else math.inf
    return BenchmarkResult(obj.name, runs, cfg.seed, per_mode, speedup)
