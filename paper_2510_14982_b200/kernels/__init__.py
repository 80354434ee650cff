"""Backend plug-in boundary (API parity with protozoa.kernels).

The reference selects a backend module with ``get_backend(name)``
(kernels/__init__.py:47-56) and calls its ``run_updates`` from
``engine.step`` (engine.py:163-166).  This package registers exactly one
backend, ``"cuda"`` (cuda_backend.py): the sm_100a kernels behind the C ABI
of libapo_b200.so.  There is deliberately no CPU backend -- requesting
``numba`` or ``numpy`` names the reference package instead.
"""

from __future__ import annotations

import os

ENV_VAR = "PROTOZOA_KERNELS"
_CHOICES = ("auto", "cuda")


def _detect_default() -> str:
    choice = os.environ.get(ENV_VAR, "auto").strip().lower() or "auto"
    if choice not in _CHOICES:
        raise ValueError(f"{ENV_VAR} must be one of {_CHOICES} for this package, got {choice!r}")
    return "cuda"


DEFAULT_BACKEND = _detect_default()


def get_backend(name: str | None = None):
    resolved = (name or DEFAULT_BACKEND).strip().lower()
    if resolved in ("cuda", "auto"):
        from . import cuda_backend

        return cuda_backend
    raise ValueError(f"unknown backend {name!r}; this package provides only 'cuda' "
                     "(the CPU backends live in the reference package)")


def available_backends() -> tuple:
    return ("cuda",)
