"""The C-ABI library loads and exports every symbol include/apo_b200.h declares (CPU-only)."""

import os
import re

import pytest

from conftest import ROOT


def _declared():
    src = open(os.path.join(ROOT, "include", "apo_b200.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(apo_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_the_boundary():
    names = _declared()
    for must in ("apo_run_updates", "apo_run_batch", "apo_run_create", "apo_run_iterate", "apo_select_dr",
                 "apo_sort_order", "apo_initialize", "apo_evaluate", "apo_histogram_u8"):
        assert must in names


def test_library_exports_every_declared_symbol():
    from paper_2510_14982_b200 import _lib

    if not os.path.exists(_lib.LIB_PATH):
        _lib.build()
    lib = _lib.load()
    for name in _declared():
        assert hasattr(lib, name), name
    assert set(_lib.PROTOTYPES) >= set(_declared())
    assert lib.apo_abi_version() == 4


def test_library_is_sm100a():
    import subprocess

    from paper_2510_14982_b200 import _lib

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_no_cpu_fallback_without_a_device():
    import torch

    if torch.cuda.is_available():
        pytest.skip("device present")
    import numpy as np

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import _lib

    cfg = pz.ApoConfig(ps=4, dim=2, bounds=pz.Bounds(-1.0, 1.0, 2), max_iterations=3)
    with pytest.raises(_lib.ApoError):
        pz.run(cfg, "sphere")
    with pytest.raises(_lib.ApoError):
        pz.evaluate("sphere", np.zeros(2))
