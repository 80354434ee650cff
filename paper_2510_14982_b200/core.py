"""Run configuration, population state and the host-side schedule constants.

API parity with protozoa.core (ApoConfig, ConfigError, Individual,
Population and the schedule functions).  The per-individual operators run
on the device (csrc/apo_update.cuh); what stays on the host is what the
reference also computes on the host with libm, so the device reads
bit-identical constants:

* ``schedule_table(T)``: (p_ah, f_mult, decay) per iteration
  (numba_backend.py:357-366, core.py:220-250);
* ``p_dr_table(ps)``: the dormancy threshold per rank
  (numba_backend.py:173-175, core.py:240-246).
"""

from __future__ import annotations

import math
from dataclasses import dataclass
from functools import lru_cache
from typing import NamedTuple, Optional

import numpy as np

from . import rng
from .objectives import Bounds

SLOT_DECISION, SLOT_SIGN, SLOT_MASK_SIZE, SLOT_MAGNITUDE, SLOT_FORAGE, SLOT_PARTNER = range(6)
VECTOR_BASE = 8
MASK_BASE = 1 << 32
PAIRS_BASE = 1 << 33
COORD_SLOT_PF = 0
COORD_SLOT_DR_PERM = 1

DORMANCY = "dormancy"
REPRODUCTION = "reproduction"
AUTOTROPH = "autotroph"
HETEROTROPH = "heterotroph"
OPERATIONS = (DORMANCY, REPRODUCTION, AUTOTROPH, HETEROTROPH)


class ConfigError(ValueError):
    """An ApoConfig violates one or more invariants."""


@dataclass(frozen=True)
class ApoConfig:
    """Run parameters (core.py:98-146 of the reference); every violated rule is reported."""

    ps: int
    dim: int
    bounds: Bounds
    max_iterations: int
    neighbor_pairs: int = 1
    pf_max: float = 0.1
    max_fes: Optional[int] = None
    seed: int = 0
    eps: float = 2.0 ** -52
    # "keyed": the reference's fmix64 stream (oracle mode, bit-exact with the reference);
    # "philox": Philox4x32-10 production stream (same algorithm, statistically equivalent)
    rng: str = "keyed"

    def violations(self) -> list:
        bad = []
        if self.ps < 1:
            bad.append(f"ps must be >= 1, got {self.ps}")
        if self.dim < 1:
            bad.append(f"dim must be >= 1, got {self.dim}")
        elif self.bounds.dim != self.dim:
            bad.append(f"bounds cover {self.bounds.dim} dims but dim is {self.dim}")
        if self.max_iterations < 0:
            bad.append(f"max_iterations must be >= 0, got {self.max_iterations}")
        if self.neighbor_pairs < 1:
            bad.append(f"neighbor_pairs must be >= 1, got {self.neighbor_pairs}")
        elif self.ps >= 2 and self.neighbor_pairs > self.ps - 1:
            bad.append(f"neighbor_pairs must be <= ps - 1 = {self.ps - 1}, got {self.neighbor_pairs}")
        if not 0.0 < self.pf_max <= 1.0:
            bad.append(f"pf_max must be in (0, 1], got {self.pf_max}")
        if self.max_fes is not None and self.max_fes < 1:
            bad.append(f"max_fes must be >= 1 when set, got {self.max_fes}")
        if not 0 <= self.seed < 2 ** 64:
            bad.append(f"seed must be in [0, 2**64), got {self.seed}")
        if not (math.isfinite(self.eps) and self.eps > 0.0):
            bad.append(f"eps must be a positive finite float, got {self.eps}")
        if self.rng not in ("keyed", "philox"):
            bad.append(f"rng must be 'keyed' or 'philox', got {self.rng!r}")
        return bad

    def __post_init__(self) -> None:
        bad = self.violations()
        if bad:
            raise ConfigError("invalid configuration:\n" + "\n".join(f"  - {b}" for b in bad))

    @property
    def iteration_span(self) -> int:
        return max(self.max_iterations - 1, 1)

    def iterations_within_budget(self) -> int:
        """Iterations engine.run executes (engine.py:191-193): t runs while fe < max_fes."""
        if self.max_fes is None:
            return self.max_iterations
        n = 0
        fe = self.ps
        while n < self.max_iterations and fe < self.max_fes:
            n += 1
            fe += self.ps
        return n


@dataclass
class Individual:
    position: np.ndarray
    fitness: float


@dataclass
class Population:
    """Positions [ps, dim] + fitness [ps] + run counters (core.py:157-196)."""

    positions: np.ndarray
    fitness: np.ndarray
    iteration: int = 0
    fe_count: int = 0
    warnings: int = 0

    def __post_init__(self) -> None:
        self.positions = np.ascontiguousarray(self.positions, dtype=np.float64)
        self.fitness = np.ascontiguousarray(self.fitness, dtype=np.float64)
        if self.positions.ndim != 2:
            raise ValueError(f"positions must be 2-D, got shape {self.positions.shape}")
        if self.fitness.shape != (self.positions.shape[0],):
            raise ValueError("fitness length must match the number of rows in positions")

    @property
    def size(self) -> int:
        return self.positions.shape[0]

    @property
    def dim(self) -> int:
        return self.positions.shape[1]

    def individual(self, i: int) -> Individual:
        if not 1 <= i <= self.size:
            raise IndexError(f"index must be in [1, {self.size}], got {i}")
        return Individual(self.positions[i - 1].copy(), float(self.fitness[i - 1]))

    def best(self) -> Individual:
        return self.individual(int(np.argmin(self.fitness)) + 1)


class UpdateDecision(NamedTuple):
    operation: str
    draw: float
    threshold: float


# ---------------------------------------------------------------------------
# schedules (host, libm)


def iteration_ratio(iteration: int, max_iterations: int) -> float:
    return iteration / max(max_iterations - 1, 1)


def p_autotroph_heterotroph(iteration: int, max_iterations: int) -> float:
    return 0.5 * (1.0 + math.cos(iteration_ratio(iteration, max_iterations) * math.pi))


def p_dormancy_reproduction(i: int, ps: int) -> float:
    return 0.5 * (1.0 - math.cos((1.0 - i / ps) * math.pi))


def rank_weight(fit_a: float, fit_b: float, eps: float) -> float:
    return math.exp(-abs(fit_a / (fit_b + eps)))


def iteration_scalars(iteration: int, max_iterations: int):
    """(p_ah, f_mult, decay) exactly as numba_backend.py:424-431 builds them."""
    ratio = iteration_ratio(iteration, max_iterations)
    return (p_autotroph_heterotroph(iteration, max_iterations), 1.0 + math.cos(ratio * math.pi), 1.0 - ratio)


@lru_cache(maxsize=16)
def schedule_table(max_iterations: int) -> np.ndarray:
    """[max_iterations, 3] of (p_ah, f_mult, decay)."""
    t = np.array([iteration_scalars(k, max_iterations) for k in range(max_iterations)], dtype=np.float64)
    t = t.reshape(max_iterations, 3)
    t.setflags(write=False)
    return t


@lru_cache(maxsize=16)
def p_dr_table(ps: int) -> np.ndarray:
    """Dormancy threshold per rank, libm cos as numba_backend.py:174-175."""
    cos, pi = math.cos, math.pi
    t = np.fromiter((0.5 * (1.0 - cos((1.0 - i / ps) * pi)) for i in range(1, ps + 1)), dtype=np.float64, count=ps)
    t.setflags(write=False)
    return t


# ---------------------------------------------------------------------------
# coordinator draws (host copies of core.py:263-278, for API parity; the
# device path computes them in csrc/apo_kernels.cu)


def proportion_fraction(key: rng.StreamKey, pf_max: float) -> float:
    return pf_max * rng.draw_uniform(key.advanced(COORD_SLOT_PF))


def select_dr_indices(ps: int, pf: float, key: rng.StreamKey) -> np.ndarray:
    return rng.randperm(ps, int(math.ceil(ps * pf)), key.advanced(COORD_SLOT_DR_PERM))


def decide_operation(i: int, in_dr: bool, iteration: int, cfg: ApoConfig, key: rng.StreamKey) -> UpdateDecision:
    u = rng.draw_uniform(key.advanced(SLOT_DECISION))
    if in_dr:
        thr = p_dormancy_reproduction(i, cfg.ps)
        return UpdateDecision(DORMANCY if u < thr else REPRODUCTION, u, thr)
    thr = p_autotroph_heterotroph(iteration, cfg.max_iterations)
    return UpdateDecision(AUTOTROPH if u < thr else HETEROTROPH, u, thr)


def sort_by_fitness(pop: Population) -> Population:
    """Stable ascending reorder (core.py:504-513) -- host convenience."""
    order = np.argsort(pop.fitness, kind="stable")
    return Population(pop.positions[order].copy(), pop.fitness[order].copy(), iteration=pop.iteration,
                      fe_count=pop.fe_count, warnings=pop.warnings)
