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


# ---------------------------------------------------------------------------
# Netpbm ingestion (API parity with imaging.py:78-194 of the reference; SURVEY.md
# §8f item 3).  Host-side parsing -- the pixels then go to the GPU histogram.

class ImageFormatError(ValueError):
    """Malformed or unsupported PGM/PPM data; ``offset`` is the byte where parsing failed."""

    def __init__(self, message: str, offset: int):
        super().__init__(f"{message} (at byte {offset})")
        self.offset = offset


_WS = b" \t\n\r\x0b\x0c"


def _tokens(data: bytes):
    """Yield (token, offset) over a Netpbm header/ASCII raster: whitespace and '#' comments skipped."""
    pos, n = 0, len(data)
    while True:
        while pos < n:
            c = data[pos:pos + 1]
            if c == b"#":
                while pos < n and data[pos:pos + 1] not in (b"\n", b"\r"):
                    pos += 1
            elif c in _WS:
                pos += 1
            else:
                break
        if pos >= n:
            yield None, n
            return
        start = pos
        while pos < n and data[pos:pos + 1] not in _WS and data[pos:pos + 1] != b"#":
            pos += 1
        yield data[start:pos], start


def load_image(data: bytes) -> GrayImage:
    """PGM (P2/P5) or PPM (P3/P6) bytes, maxval 255, to a grey image (colour by BT.601 luminance,
    rounded half up).  Errors carry the byte offset of the first problem."""
    if not isinstance(data, (bytes, bytearray)):
        raise TypeError("load_image expects bytes")
    data = bytes(data)
    toks = _tokens(data)

    def need(what):
        tok, off = next(toks)
        if tok is None:
            raise ImageFormatError(f"unexpected end of data while reading {what}", off)
        return tok, off

    def unsigned(what):
        tok, off = need(what)
        if not tok.isdigit():
            raise ImageFormatError(f"expected an unsigned integer for {what}, got {tok[:20]!r}", off)
        return int(tok), off

    magic, off = need("the format magic")
    if magic not in (b"P2", b"P3", b"P5", b"P6"):
        raise ImageFormatError(f"unsupported format magic {magic[:8]!r}; expected P2, P3, P5 or P6", off)
    width, off = unsigned("the width")
    if width < 1:
        raise ImageFormatError(f"width must be >= 1, got {width}", off)
    height, off = unsigned("the height")
    if height < 1:
        raise ImageFormatError(f"height must be >= 1, got {height}", off)
    maxval, off = unsigned("the maximum value")
    if maxval != 255:
        raise ImageFormatError(f"only maxval 255 is supported, got {maxval}", off)
    chans = 3 if magic in (b"P3", b"P6") else 1
    count = width * height * chans
    if magic in (b"P5", b"P6"):
        pos = off + len(str(maxval))
        if pos >= len(data) or data[pos:pos + 1] not in _WS:
            raise ImageFormatError("expected a whitespace byte before the raster", pos)
        raster = data[pos + 1:pos + 1 + count]
        if len(raster) < count:
            raise ImageFormatError(f"raster truncated: expected {count} bytes, found {len(raster)}", len(data))
        values = np.frombuffer(raster, dtype=np.uint8).copy()
    else:
        values = np.empty(count, dtype=np.uint8)
        for k in range(count):
            v, off = unsigned("a raster value")
            if v > 255:
                raise ImageFormatError(f"raster value {v} exceeds maxval 255", off)
            values[k] = v
    if chans == 3:
        rgb = values.reshape(height, width, 3).astype(np.float64)
        y = np.floor(0.299 * rgb[..., 0] + 0.587 * rgb[..., 1] + 0.114 * rgb[..., 2] + 0.5)
        return GrayImage(np.clip(y, 0.0, 255.0).astype(np.uint8))
    return GrayImage(values.reshape(height, width))


def load_image_file(path) -> GrayImage:
    with open(path, "rb") as fh:
        return load_image(fh.read())


def write_pgm(img: GrayImage, binary: bool = True) -> bytes:
    """P5 (default) or P2 bytes; both round-trip through load_image pixel for pixel."""
    head = f"{'P5' if binary else 'P2'}\n{img.width} {img.height}\n255\n".encode("ascii")
    if binary:
        return head + img.pixels.tobytes()
    return head + ("\n".join(" ".join(map(str, row.tolist())) for row in img.pixels) + "\n").encode("ascii")
