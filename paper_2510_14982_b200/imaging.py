"""Threshold search driven by the optimizer (API parity with protozoa.imaging).

The objective interface is the reference's: a 256-entry value table read at
round_half_up(x0) (objectives.py:183-192) built from the image histogram
(imaging.py:197-228).  The histogram is computed on the device
(``apo_histogram_u8``, shared-memory privatised); the 256-entry variance
table is host arithmetic over 256 integers, kept identical to the
reference's so the device objective reads bit-identical values.

PGM/PPM parsing is out of scope for the hot path; an
image is any 2-D uint8 array.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, replace
from typing import NamedTuple, Optional

import numpy as np

from .core import ApoConfig
from .engine import EngineMode, RunResult, run
from .objectives import KAPUR_ML, OTSU_ML, Bounds, Objective, table_objective


@dataclass
class GrayImage:
    pixels: np.ndarray

    def __post_init__(self) -> None:
        self.pixels = np.ascontiguousarray(self.pixels, dtype=np.uint8)
        if self.pixels.ndim != 2 or self.pixels.size == 0:
            raise ValueError(f"pixels must be a non-empty 2-D array, got shape {self.pixels.shape}")

    @property
    def height(self) -> int:
        return self.pixels.shape[0]

    @property
    def width(self) -> int:
        return self.pixels.shape[1]


@dataclass
class Histogram:
    counts: np.ndarray
    total: int

    def __post_init__(self) -> None:
        self.counts = np.ascontiguousarray(self.counts, dtype=np.int64)
        if self.counts.shape != (256,):
            raise ValueError("counts must have exactly 256 entries")
        if int(self.counts.sum()) != self.total or self.total <= 0:
            raise ValueError("total must be positive and equal the sum of counts")


def histogram_device(pixels):
    """256-bin counts of a uint8 tensor/array on the GPU -> int64 CUDA tensor."""
    import torch

    from . import _lib

    lib = _lib.require_cuda()
    px = torch.as_tensor(np.ascontiguousarray(pixels)) if isinstance(pixels, np.ndarray) else pixels
    px = px.to(device="cuda", dtype=torch.uint8).contiguous().view(-1)
    if px.data_ptr() % 16:
        px = px.clone()
    counts = torch.empty(256, dtype=torch.int64, device=px.device)
    _lib.check(lib.apo_histogram_u8(_lib.ptr(px), px.numel(), _lib.ptr(counts), _lib.stream_handle()),
               "apo_histogram_u8")
    return counts


def histogram(img: GrayImage) -> Histogram:
    """Intensity histogram (imaging.py:197-200), computed on the device."""
    counts = histogram_device(img.pixels).cpu().numpy()
    return Histogram(counts, int(img.pixels.size))


def between_class_variance(hist: Histogram, t: int) -> float:
    """omega0*omega1*(mu0-mu1)^2 for class 0 = intensities <= t (imaging.py:203-223)."""
    if not 0 <= t <= 255:
        raise ValueError(f"t must be in [0, 255], got {t}")
    c = hist.counts
    n0 = int(c[: t + 1].sum())
    n1 = hist.total - n0
    if n0 == 0 or n1 == 0:
        return 0.0
    idx = np.arange(256, dtype=np.int64)
    s0 = int((idx[: t + 1] * c[: t + 1]).sum())
    s1 = int((idx * c).sum()) - s0
    w0 = n0 / hist.total
    w1 = n1 / hist.total
    diff = s0 / n0 - s1 / n1
    return w0 * w1 * (diff * diff)


def variance_table(hist: Histogram) -> np.ndarray:
    return np.array([between_class_variance(hist, t) for t in range(256)])


def brute_force_otsu(hist: Histogram) -> tuple:
    """Exhaustive t = 0..255, ties -> smallest t (imaging.py:231-240)."""
    table = variance_table(hist)
    best_t, best_v = 0, table[0]
    for t in range(1, 256):
        if table[t] > best_v:
            best_t, best_v = t, table[t]
    return best_t, float(best_v)


def round_half_up(x: float) -> int:
    return int(math.floor(x + 0.5))


class ThresholdResult(NamedTuple):
    threshold: int
    variance: float
    run: RunResult


def apo_threshold(img: GrayImage, cfg: Optional[ApoConfig] = None, ps: int = 100, iterations: int = 50,
                  seed: int = 0, mode: Optional[EngineMode] = None, backend: Optional[str] = None) -> ThresholdResult:
    """Maximum-variance threshold by minimising the negated table (imaging.py:255-284)."""
    table = variance_table(histogram(img))
    objective = table_objective("negated_between_class_variance", -table)
    box = Bounds(0.0, 255.0, 1)
    cfg = (ApoConfig(ps=ps, dim=1, bounds=box, max_iterations=iterations, seed=seed) if cfg is None
           else replace(cfg, dim=1, bounds=box))
    result = run(cfg, objective, mode=mode, backend=backend)
    t = min(max(round_half_up(float(result.best_position[0])), 0), 255)
    return ThresholdResult(t, -result.best_fitness, result)


def apply_threshold(img: GrayImage, t: int) -> GrayImage:
    if not 0 <= t <= 255:
        raise ValueError(f"t must be in [0, 255], got {t}")
    return GrayImage(np.where(img.pixels > t, 255, 0).astype(np.uint8))


# ---------------------------------------------------------------------------
# Multilevel thresholding (BASELINE config 3; no reference counterpart: the
# reference stops at one threshold).  Definitions: DESIGN.md and
# oracle/threshold_oracle.c; k = 1 Otsu reduces to the reference's
# between_class_variance up to rounding.

METHODS = {"otsu": (0, OTSU_ML), "kapur": (1, KAPUR_ML)}
TABLE_LEN = 515
MAX_THRESHOLDS = 32


def threshold_tables_device(counts, method: str):
    """515-entry prefix table (apo_threshold_tables) of a 256-bin histogram -> CUDA tensor."""
    import torch

    from . import _lib

    if method not in METHODS:
        raise ValueError(f"method must be one of {tuple(METHODS)}, got {method!r}")
    lib = _lib.require_cuda()
    c = counts if isinstance(counts, torch.Tensor) else torch.as_tensor(np.ascontiguousarray(counts, dtype=np.int64))
    c = c.to(device="cuda", dtype=torch.int64).contiguous()
    if c.numel() != 256:
        raise ValueError("counts must have 256 bins")
    tab = torch.empty(TABLE_LEN, dtype=torch.float64, device=c.device)
    _lib.check(lib.apo_threshold_tables(_lib.ptr(c), METHODS[method][0], _lib.ptr(tab), _lib.stream_handle()),
               "apo_threshold_tables")
    return tab


def multilevel_objective(counts, k: int, method: str = "otsu") -> Objective:
    """Objective over k thresholds in [0, 255]: -(between-class variance) or -(total class entropy)."""
    if not 1 <= k <= MAX_THRESHOLDS:
        raise ValueError(f"k must be in [1, {MAX_THRESHOLDS}], got {k}")
    tab = threshold_tables_device(counts, method).cpu().numpy()
    return Objective(f"{method}_{k}", METHODS[method][1], min_dim=1, table=tab)


class MultiThresholdResult(NamedTuple):
    thresholds: tuple
    value: float  # between-class variance (otsu) or total entropy (kapur) at the thresholds
    run: RunResult


def thresholds_of(x) -> tuple:
    """Sorted integer thresholds the objective reads from a position."""
    return tuple(sorted(min(max(round_half_up(float(v)), 0), 255) for v in x))


def apo_multithreshold(img, k: int, method: str = "otsu", cfg: Optional[ApoConfig] = None, ps: int = 100,
                       iterations: int = 50, seed: int = 0) -> MultiThresholdResult:
    """k thresholds maximising Otsu's between-class variance or Kapur's entropy (histogram on the GPU)."""
    pixels = img.pixels if isinstance(img, GrayImage) else img
    counts = histogram_device(pixels)
    obj = multilevel_objective(counts, k, method)
    box = Bounds(0.0, 255.0, k)
    cfg = (ApoConfig(ps=ps, dim=k, bounds=box, max_iterations=iterations, seed=seed) if cfg is None
           else replace(cfg, dim=k, bounds=box))
    result = run(cfg, obj)
    return MultiThresholdResult(thresholds_of(result.best_position), -result.best_fitness, result)


def multilevel_value(counts, thresholds, method: str = "otsu") -> float:
    """Objective value (positive) of integer thresholds, evaluated on the device."""
    from .objectives import evaluate_batch

    obj = multilevel_objective(counts, len(thresholds), method)
    return -float(evaluate_batch(obj, np.asarray(thresholds, dtype=np.float64)[None, :])[0])
