"""One population sharded by rank over the processes of a torch.distributed group.

BASELINE config 4 ("pop=1,000,000, population sharded over 8 GPUs with a
per-iteration NVLink allgather").  The reference has no distributed code: its
only parallelism is CPU threads over individuals with results independent of
the worker count (test_engine.py:209-217).  Here the same
contract holds across GPUs: a sharded run reproduces the single-GPU run bit
for bit, for any number of processes.

Per iteration, on every process (all on torch's current stream, so NCCL and
the kernels are ordered):

1. ``apo_shard_begin`` -- stable sort of the replicated fitness + the
   coordinator's Dr set (core.py:263-278, 504-513).  Identical everywhere, so
   no exchange is needed to agree on ranks.
2. ``apo_shard_update_range(lo, hi)`` -- the fused update of this process's
   ranks, reading any row of the replicated population (partners,
   neighbours, pairs span all ranks: core.py:344-397) and writing rows by rank.
3. all-gather of rows [lo, hi) of the next position/fitness buffers (NCCL
   over NVLink), so every process again holds the whole population -- now in
   rank order, which is exactly the reference's row order (engine.py:167-172).
   Each process's ranks come in `blocks` pieces (ShardPlan), and the gather of
   piece s is issued asynchronously as soon as it is updated, so NVLink
   traffic overlaps the update of piece s+1.

Traffic per iteration and GPU: (N-1)/N of the population (8 * ps * ld bytes)
received; SURVEY.md §8e explains why that bounds strong scaling at D = 100.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional

import numpy as np

from . import _lib
from .core import ApoConfig, p_dr_table, schedule_table
from .objectives import device_objective, resolve_objective

GROUP = 32  # the update kernel owns ranks in groups of 32 (apo_group.cuh)


@dataclass(frozen=True)
class ShardPlan:
    """Rank ranges of a population split over `world` processes, in whole groups of 32.

    With blocks = S > 1 the ranks are dealt out in S rounds: block s of process r is the range of
    `chunk` ranks starting at (s * world + r) * chunk.  Block s of every process is then one contiguous
    span of the buffer, so it can be all-gathered in place as soon as it is updated while block s+1
    computes (which process updates a rank is free: every process holds the whole population)."""

    ps: int
    world: int
    blocks: int = 1

    @property
    def chunk(self) -> int:
        per = -(-self.ps // (self.world * self.blocks))
        return -(-per // GROUP) * GROUP

    @property
    def ps_pad(self) -> int:
        return self.chunk * self.world * self.blocks

    def block(self, rank: int, s: int) -> tuple:
        lo = min((s * self.world + rank) * self.chunk, self.ps)
        return lo, min(lo + self.chunk, self.ps)

    def ranges(self, rank: int) -> list:
        return [self.block(rank, s) for s in range(self.blocks)]

    def range(self, rank: int) -> tuple:
        if self.blocks != 1:
            raise ValueError("range() is for single-block plans; use ranges()")
        return self.block(rank, 0)


def _dist(group):
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized():
        return dist, dist.get_world_size(group), dist.get_rank(group)
    return None, 1, 0


class _DeviceShard:
    """The CUDA side of a shard (C ABI apo_shard_*); buffers are torch tensors so NCCL can move them."""

    def __init__(self, cfg: ApoConfig, obj, plan: ShardPlan, stream=None):
        import torch

        self.lib = _lib.require_cuda()
        dev = torch.device("cuda", torch.cuda.current_device())
        self.ld = cfg.dim + (cfg.dim & 1)
        self.pos = [torch.zeros((plan.ps_pad, self.ld), dtype=torch.float64, device=dev) for _ in range(2)]
        self.fit = [torch.full((plan.ps_pad,), float("inf"), dtype=torch.float64, device=dev) for _ in range(2)]
        self.dobj = device_objective(obj, cfg.dim)
        sched = np.ascontiguousarray(schedule_table(cfg.max_iterations)) if cfg.max_iterations else np.zeros(3)
        pdr = np.ascontiguousarray(p_dr_table(cfg.ps))
        h = C.c_void_p()
        rng = 1 if cfg.rng == "philox" else 0
        _lib.check(self.lib.apo_shard_create(C.byref(h), cfg.ps, cfg.dim, self.ld, cfg.max_iterations, cfg.seed,
                                             cfg.neighbor_pairs, cfg.pf_max, cfg.bounds.lower, cfg.bounds.upper,
                                             cfg.eps, self.dobj.ref, sched.ctypes.data, pdr.ctypes.data, rng,
                                             _lib.ptr(self.pos[0]), _lib.ptr(self.pos[1]), _lib.ptr(self.fit[0]),
                                             _lib.ptr(self.fit[1]), _lib.stream_handle(stream)), "apo_shard_create")
        self.handle = h
        self.cur = 0

    def initialize(self):
        _lib.check(self.lib.apo_shard_initialize(self.handle), "apo_shard_initialize")
        self.cur = 0

    def begin(self):
        _lib.check(self.lib.apo_shard_begin(self.handle), "apo_shard_begin")

    def update_range(self, lo: int, hi: int):
        _lib.check(self.lib.apo_shard_update_range(self.handle, lo, hi), "apo_shard_update_range")

    def next_buffers(self):
        return self.pos[self.cur ^ 1], self.fit[self.cur ^ 1]

    def end(self):
        _lib.check(self.lib.apo_shard_end(self.handle), "apo_shard_end")
        self.cur ^= 1

    def current(self):
        return self.pos[self.cur], self.fit[self.cur]

    def counters(self, n: int):
        keys = np.zeros(n + 1, dtype=np.uint64)
        w = C.c_int64()
        _lib.check(self.lib.apo_shard_counters(self.handle, keys.ctypes.data, n, C.byref(w)), "apo_shard_counters")
        return keys, w.value

    def close(self):
        if getattr(self, "handle", None):
            self.lib.apo_shard_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def encode_keys(x) -> np.ndarray:
    """doubles -> order-preserving u64 keys (-0.0 == +0.0, NaN last), as apo_device.cuh sort_key."""
    x = np.asarray(x, dtype=np.float64)
    b = x.view(np.uint64)
    k = np.where((b >> np.uint64(63)) == 1, ~b, b | np.uint64(1 << 63))
    k = np.where(x == 0.0, np.uint64(1 << 63), k)
    return np.where(np.isnan(x), np.uint64(0xFFFFFFFFFFFFFFFF), k).astype(np.uint64)


def decode_keys(keys: np.ndarray) -> np.ndarray:
    """Order-preserving u64 keys (apo_device.cuh sort_key) -> doubles."""
    k = keys.astype(np.uint64)
    neg = (k >> np.uint64(63)) == 0
    bits = np.where(neg, ~k, k & np.uint64(0x7FFFFFFFFFFFFFFF))
    out = bits.view(np.float64).copy()
    out[k == np.uint64(0xFFFFFFFFFFFFFFFF)] = np.nan
    return out


class ShardedRun:
    """A single population sharded by rank over a process group (or over `virtual_world` ranges in one
    process: the same kernels and layout without the exchange -- used to check partition independence)."""

    def __init__(self, cfg: ApoConfig, objective, group=None, virtual_world: Optional[int] = None, stream=None,
                 engine=None, blocks: Optional[int] = None):
        self.cfg = cfg
        self.obj = resolve_objective(objective)
        self.dist, self.world, self.rank = _dist(group)
        self.group = group
        # blocks per process: the exchange of block s overlaps the update of block s+1 (4 by default when
        # there is an exchange; never more than one group of 32 ranks per block and process)
        world = virtual_world if virtual_world is not None else self.world
        if blocks is None:
            blocks = 4 if self.world > 1 else 1
        blocks = max(1, min(int(blocks), -(-cfg.ps // (GROUP * world))))
        if virtual_world is not None:
            if self.world != 1:
                raise ValueError("virtual_world is for single-process runs")
            self.plan = ShardPlan(cfg.ps, virtual_world, blocks)
        else:
            self.plan = ShardPlan(cfg.ps, self.world, blocks)
        self.virtual = virtual_world is not None
        # `engine` replaces the device shard only in tests of this orchestration (tests/test_shard.py)
        self.dev = engine(cfg, self.obj, self.plan) if engine is not None else _DeviceShard(cfg, self.obj, self.plan,
                                                                                              stream)
        self.iterations = 0

    def initialize(self):
        self.dev.initialize()
        self.iterations = 0

    def _exchange_block(self, s: int):
        """Start the in-place all-gather of block s (rows + fitness) of the next buffers; NCCL runs it on
        its own stream, so the update of block s+1 proceeds on the compute stream meanwhile."""
        pos, fit = self.dev.next_buffers()
        c, w = self.plan.chunk, self.world
        base = s * w * c
        mine = base + self.rank * c
        return [self.dist.all_gather_into_tensor(pos[base:base + w * c], pos[mine:mine + c], group=self.group,
                                                 async_op=True),
                self.dist.all_gather_into_tensor(fit[base:base + w * c], fit[mine:mine + c], group=self.group,
                                                 async_op=True)]

    def iterate(self, n: int):
        if self.iterations + n > self.cfg.max_iterations:
            raise ValueError("iteration budget exceeded")
        for _ in range(n):
            self.dev.begin()
            if self.virtual:
                for r in range(self.plan.world):
                    for lo, hi in self.plan.ranges(r):
                        self.dev.update_range(lo, hi)
            else:
                works = []
                for s, (lo, hi) in enumerate(self.plan.ranges(self.rank)):
                    self.dev.update_range(lo, hi)
                    if self.world > 1:
                        works += self._exchange_block(s)
                for wk in works:  # the compute stream waits for every block before the next sort
                    wk.wait()
            self.dev.end()
            self.iterations += 1

    def population(self):
        """(positions [ps, dim], fitness [ps]) in reference row order, host numpy."""
        pos, fit = self.dev.current()
        return (pos[:self.cfg.ps, :self.cfg.dim].cpu().numpy().copy(), fit[:self.cfg.ps].cpu().numpy().copy())

    def trace_and_warnings(self):
        """Best-so-far trace (entries 0..iterations) and warnings, reduced over the group."""
        import torch

        keys, warns = self.dev.counters(self.iterations)
        if self.world > 1:
            dev = "cuda" if self.dist.get_backend(self.group) == "nccl" else "cpu"
            # order-preserving keys compare as unsigned; flip the top bit to compare as signed for MIN
            t = torch.as_tensor((keys ^ np.uint64(1 << 63)).view(np.int64).copy(), device=dev)
            self.dist.all_reduce(t, op=self.dist.ReduceOp.MIN, group=self.group)
            keys = t.cpu().numpy().view(np.uint64) ^ np.uint64(1 << 63)
            w = torch.tensor([warns], dtype=torch.int64, device=dev)
            self.dist.all_reduce(w, group=self.group)
            warns = int(w.item())
        return decode_keys(keys), warns

    def close(self):
        self.dev.close()
