"""Objectives, bounds and the objective registry (API parity with protozoa.objectives).

The six reference functions are the unshifted, unrotated basic forms
(objectives.py:3-12 of the reference) with the same integer codes, so an
``Objective`` built here or by the reference means the same thing to the
kernels.  Evaluation itself happens on the device (csrc/apo_objective.cuh);
``evaluate`` is a one-point convenience over the batched kernel.

Codes the reference does not have (CEC2022, multilevel thresholding) live in
separate registries (``cec2022.CEC2022_NAMES``, ``imaging``) so that
``FUNCTION_NAMES`` stays exactly the reference's six names
(test_objectives.py:157-162 of the reference freezes it).
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field
import weakref
from functools import lru_cache
from typing import Any, Callable, Optional

import numpy as np

SPHERE = 0
BENT_CIGAR = 1
HIGH_CONDITIONED_ELLIPTIC = 2
HGBAT = 3
ROSENBROCK = 4
GRIEWANK = 5
TABLE = 6
OTSU_ML = 7   # multilevel Otsu over prefix tables (no reference counterpart)
KAPUR_ML = 8  # multilevel Kapur
EXTERNAL = -1


@dataclass(frozen=True)
class Bounds:
    """Box constraint [lower, upper]^dim (objectives.py:45-63)."""

    lower: float
    upper: float
    dim: int

    def __post_init__(self) -> None:
        if not (math.isfinite(self.lower) and math.isfinite(self.upper)):
            raise ValueError("bounds must be finite")
        if not self.lower < self.upper:
            raise ValueError(f"lower must be < upper, got [{self.lower}, {self.upper}]")
        if self.dim < 1:
            raise ValueError(f"dim must be >= 1, got {self.dim}")

    @property
    def span(self) -> float:
        return self.upper - self.lower


def clamp(x: np.ndarray, bounds: Bounds) -> np.ndarray:
    """Component-wise projection onto the box; NaN passes through."""
    if x.shape != (bounds.dim,):
        raise ValueError(f"expected shape ({bounds.dim},), got {x.shape}")
    return np.clip(x, bounds.lower, bounds.upper)


@dataclass(frozen=True)
class Objective:
    """A named minimisation target.

    ``code`` selects the device implementation, ``table`` feeds the lookup
    objective, ``func`` holds an external callable, ``data`` carries extra
    per-objective device data (CEC2022 shift/rotation/shuffle).
    """

    name: str
    code: int
    min_dim: int = 1
    table: Optional[np.ndarray] = field(default=None, repr=False)
    func: Optional[Callable[[np.ndarray], float]] = field(default=None, repr=False)
    data: Any = field(default=None, repr=False, compare=False)


@lru_cache(maxsize=None)
def elliptic_weights(dim: int) -> np.ndarray:
    """(10^6)^(i/(D-1)) with Python's scalar pow, as objectives.py:88-102 does."""
    if dim == 1:
        return np.ones(1)
    w = np.array([10.0 ** (6.0 * i / (dim - 1)) for i in range(dim)])
    w.setflags(write=False)
    return w


FUNCTION_NAMES = ("sphere", "bent_cigar", "high_conditioned_elliptic", "hgbat", "rosenbrock", "griewank")

_REGISTRY = {
    "sphere": Objective("sphere", SPHERE),
    "bent_cigar": Objective("bent_cigar", BENT_CIGAR),
    "high_conditioned_elliptic": Objective("high_conditioned_elliptic", HIGH_CONDITIONED_ELLIPTIC, min_dim=2),
    "hgbat": Objective("hgbat", HGBAT, min_dim=2),
    "rosenbrock": Objective("rosenbrock", ROSENBROCK, min_dim=2),
    "griewank": Objective("griewank", GRIEWANK),
}

# Resolvers for names outside FUNCTION_NAMES (e.g. "cec2022_f6"); modules
# register a callable name -> Objective (see cec2022.py).
_EXTRA_RESOLVERS: list = []


def register_resolver(fn) -> None:
    _EXTRA_RESOLVERS.append(fn)


def get_objective(name: str) -> Objective:
    """Look up a built-in objective by name (objectives.py:174-180)."""
    if name in _REGISTRY:
        return _REGISTRY[name]
    for resolve in _EXTRA_RESOLVERS:
        obj = resolve(name)
        if obj is not None:
            return obj
    raise ValueError(f"unknown objective {name!r}; valid ids: {', '.join(FUNCTION_NAMES)}")


def table_objective(name: str, table: np.ndarray) -> Objective:
    """table[round_half_up(x[0])], index clamped (objectives.py:183-192)."""
    t = np.ascontiguousarray(table, dtype=np.float64)
    if t.ndim != 1 or t.size < 1:
        raise ValueError("table must be a non-empty 1-D array")
    return Objective(name, TABLE, min_dim=1, table=t)


def external_objective(func: Callable[[np.ndarray], float], name: str = "external", min_dim: int = 1) -> Objective:
    if not callable(func):
        raise TypeError("func must be callable")
    return Objective(name, EXTERNAL, min_dim=min_dim, func=func)


def resolve_objective(objective) -> Objective:
    if isinstance(objective, Objective):
        return objective
    if isinstance(objective, str):
        return get_objective(objective)
    if callable(objective):
        return external_objective(objective)
    raise TypeError(f"cannot interpret {objective!r} as an objective")


# ---------------------------------------------------------------------------
# Device descriptors


class DeviceObjective:
    """An Objective's C-ABI descriptor plus the device tensors it points to."""

    def __init__(self, obj: Objective, dim: int, device=None):
        import torch

        from . import _lib

        if obj.code == EXTERNAL:
            raise ValueError("external objective functions cannot run on the cuda backend")
        self.obj_ref = weakref.ref(obj)  # the cache must not keep its key's Objective alive
        self.dim = dim
        dev = device or torch.device("cuda", torch.cuda.current_device())
        self.keep = []
        table = None
        if obj.code == HIGH_CONDITIONED_ELLIPTIC:
            table = np.asarray(elliptic_weights(dim))
        elif obj.code in (TABLE, OTSU_ML, KAPUR_ML):
            table = obj.table
        self.struct = _lib.apo_objective()
        self.struct.code = int(obj.code)
        data = getattr(obj, "data", None)  # the reference's Objective has no CEC2022 data
        if data is not None and hasattr(data, "arrays"):  # CEC2022
            shift, rot, shuffle = obj.data.arrays(dim)
            rot_t = np.ascontiguousarray(np.transpose(rot, (0, 2, 1)))
            arrays = [("shift", shift), ("rot_t", rot_t), ("shuffle", shuffle)]
            rotation = getattr(data, "rotation", "dmma")
            if rotation == "auto":  # DMMA tables; the device loop may still pick FMAs at small D
                self.struct.flags = 1  # APO_OBJ_FMA_SMALL_D
                rotation = "dmma"
            if dim <= 104 and rotation == "dmma":
                # zero-padded M^T for the DMMA evaluation kernel (include/apo_b200.h)
                nt = 2 if dim <= 16 else 4 if dim <= 32 else 7 if dim <= 56 else 13
                n4 = (dim + 3) // 4 * 4
                pad = np.zeros((rot_t.shape[0], n4, 8 * nt))
                pad[:, :dim, :dim] = rot_t
                if obj.code - 100 in (6, 7, 8):  # hybrids: output column j holds z[shuffle[j]-1]
                    pad[0, :dim, :dim] = rot_t[0][:, np.asarray(shuffle) - 1]
                arrays.append(("rot_pad", pad))
                table = elliptic_weights(dim)  # ELLIPS weights 10^(6i/(D-1)), host libm like the oracle
            elif rotation == "dmma" and obj.code - 100 in (1, 2, 3, 4, 5, 6, 7, 8, 10):
                # D > 104: the rotated component's M^T padded for the DMMA GEMM (apo_cec_gemm.cu)
                comp = 1 if obj.code - 100 == 10 else 0
                kp, np_ = (dim + 15) // 16 * 16, (dim + 63) // 64 * 64
                gm = np.zeros((kp, np_))
                gm[:dim, :dim] = rot_t[comp]
                if obj.code - 100 in (6, 7, 8):
                    gm[:dim, :dim] = rot_t[0][:, np.asarray(shuffle) - 1]
                arrays.append(("rot_gemm", gm))
            for field, arr in arrays:
                t = torch.as_tensor(np.array(arr), device=dev)
                self.keep.append(t)
                setattr(self.struct, field, t.data_ptr())
        if table is not None:
            t = torch.as_tensor(np.array(table, dtype=np.float64), device=dev)
            self.keep.append(t)
            self.struct.table = t.data_ptr()
            self.struct.table_len = int(t.numel())
        else:
            self.struct.table = None
            self.struct.table_len = 0

    @property
    def ref(self):
        import ctypes

        return ctypes.byref(self.struct)


_DEV_CACHE: dict = {}


def device_objective(obj: Objective, dim: int) -> DeviceObjective:
    import torch

    key = (id(obj), obj.name, obj.code, dim, torch.cuda.current_device())
    hit = _DEV_CACHE.get(key)
    if hit is not None and hit.obj_ref() is obj:
        return hit
    d = DeviceObjective(obj, dim)
    _DEV_CACHE[key] = d
    # the entry (and its device tables) goes when the Objective does: per-call objectives such as the
    # threshold ones would otherwise accumulate
    weakref.finalize(obj, _DEV_CACHE.pop, key, None)
    return d


def evaluate_batch(objective, x) -> np.ndarray:
    """Fitness of every row of x ([n, dim]) on the device."""
    import torch

    from . import _lib

    obj = resolve_objective(objective)
    lib = _lib.require_cuda()
    xt = torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64)) if isinstance(x, np.ndarray) else x
    was_numpy = isinstance(x, np.ndarray)
    xt = xt.to(device="cuda", dtype=torch.float64).contiguous()
    if xt.ndim == 1:
        xt = xt.unsqueeze(0)
    n, dim = xt.shape
    out = torch.empty(n, dtype=torch.float64, device=xt.device)
    dobj = device_objective(obj, dim)
    _lib.check(lib.apo_evaluate(_lib.ptr(xt), n, dim, dim, dobj.ref, _lib.ptr(out), _lib.stream_handle()),
               "apo_evaluate")
    return out.cpu().numpy() if was_numpy else out


def evaluate_unchecked(objective: Objective, x: np.ndarray) -> float:
    if objective.code == EXTERNAL:
        return float(objective.func(x))
    return float(evaluate_batch(objective, np.asarray(x, dtype=np.float64)[None, :])[0])


def evaluate(objective, x: np.ndarray) -> float:
    """Evaluate at one point after validating it (objectives.py:231-243)."""
    obj = resolve_objective(objective)
    x = np.asarray(x, dtype=np.float64)
    if x.ndim != 1 or x.size < obj.min_dim:
        raise ValueError(f"{obj.name} needs a 1-D point with >= {obj.min_dim} components, got shape {x.shape}")
    if not np.all(np.isfinite(x)):
        raise ValueError(f"{obj.name}: input has non-finite components")
    return evaluate_unchecked(obj, x)
