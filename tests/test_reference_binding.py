"""The drop-in boundary exercised from the reference's side (INTEGRATION.md Options A and B).

Option B: the flat C entry ``apo_run_updates`` -- exactly the argument tuple the numba backend packs
(kernels/numba_backend.py:358-366) -- bound with ctypes as INTEGRATION.md shows, against the step
vectors the reference produced (tests/golden/steps.npz).

Option A: the UNMODIFIED reference package (installed offline into ``baseline/_ref`` by
``pip install --no-index --no-deps --target baseline/_ref``; git-ignored, it travels to the GPU box
with the snapshot) with the maintainer's three-line ``get_backend`` branch applied by monkeypatch:
``protozoa.step``/``protozoa.run`` with ``backend="cuda"`` must equal the reference's own numba backend
run in the same process.  Skipped when baseline/_ref is absent.
"""

import ctypes as C
import math
import os
import sys

import numpy as np
import pytest

from conftest import GOLDEN, ROOT

REF_SITE = os.path.join(ROOT, "baseline", "_ref")


def _groups(path):
    data = np.load(os.path.join(GOLDEN, path))
    groups = {}
    for key in data.files:
        name, field = key.split("/", 1)
        groups.setdefault(name, {})[field] = data[key]
    return groups


@pytest.fixture(scope="module")
def ref_protozoa():
    if not os.path.isdir(os.path.join(REF_SITE, "protozoa")):
        pytest.skip("reference not installed in baseline/_ref")
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join("/tmp", "numba_cache_refbinding"))
    sys.path.insert(0, REF_SITE)
    try:
        import protozoa
    finally:
        sys.path.remove(REF_SITE)
    return protozoa


def test_reference_package_importable_from_baseline(ref_protozoa):
    """CPU: the installed reference is the one Option A plugs into (its plug-in entry exists)."""
    from protozoa import kernels

    assert callable(kernels.get_backend) and ref_protozoa.step and ref_protozoa.run
    assert "numpy" in kernels.available_backends()


# ---------------------------------------------------------------------------- GPU


def _flat_binding():
    """INTEGRATION.md Option B, verbatim argument order (include/apo_b200.h:103-107)."""
    from paper_2510_14982_b200 import _lib

    lib = C.CDLL(_lib.LIB_PATH)
    lib.apo_run_updates.restype = C.c_int
    lib.apo_run_updates.argtypes = [C.c_void_p] * 7 + [C.c_int64, C.c_int64, C.c_uint64, C.c_uint64, C.c_int64] + \
        [C.c_double] * 7 + [C.c_int64, C.c_void_p, C.c_int64, C.c_void_p, C.c_void_p, C.c_void_p]
    lib.apo_last_error.restype = C.c_char_p
    return lib


def run_updates_ffi(lib, positions, fitness, in_dr, *, ps, dim, seed, npairs, lower, upper, eps, T, iteration,
                    key_iteration, code, table):
    import torch

    dev = torch.device("cuda")
    pos = torch.as_tensor(np.ascontiguousarray(positions), device=dev)
    fit = torch.as_tensor(np.ascontiguousarray(fitness), device=dev)
    dr = torch.as_tensor(np.ascontiguousarray(in_dr, dtype=np.uint8), device=dev)
    out_pos, out_fit = torch.empty_like(pos), torch.empty_like(fit)
    acc = torch.empty(ps, dtype=torch.uint8, device=dev)
    warn = torch.zeros(1, dtype=torch.int64, device=dev)
    ratio = iteration / max(T - 1, 1)  # numba_backend.py:357-366, host libm
    p_ah, f_mult, decay = 0.5 * (1.0 + math.cos(ratio * math.pi)), 1.0 + math.cos(ratio * math.pi), 1.0 - ratio
    p_dr = torch.as_tensor(np.array([0.5 * (1.0 - math.cos((1.0 - i / ps) * math.pi)) for i in range(1, ps + 1)]),
                           device=dev)  # core.py:240-246
    tab = torch.as_tensor(np.ascontiguousarray(table, dtype=np.float64), device=dev)
    rc = lib.apo_run_updates(pos.data_ptr(), fit.data_ptr(), dr.data_ptr(), out_pos.data_ptr(), out_fit.data_ptr(),
                             acc.data_ptr(), None, ps, dim, seed, key_iteration, npairs, lower, upper, upper - lower,
                             eps, p_ah, f_mult, decay, code, tab.data_ptr(), tab.numel(), p_dr.data_ptr(),
                             warn.data_ptr(), torch.cuda.current_stream().cuda_stream)
    if rc != 0:
        raise RuntimeError(lib.apo_last_error().decode())
    return out_pos.cpu().numpy(), out_fit.cpu().numpy(), acc.cpu().numpy().astype(bool), int(warn.item())


@pytest.mark.gpu
@pytest.mark.parametrize("case", sorted(_groups("steps.npz")))
def test_flat_c_entry_vs_reference_steps(case):
    import oracle
    import paper_2510_14982_b200 as pz

    g = _groups("steps.npz")[case]
    ps, dim, T, seed, npairs, steps = (int(v) for v in g["cfg"])
    pf_max, lo, hi, eps = (float(v) for v in g["cfgf"])
    name = str(g["objective"])
    code, table = oracle.objective_table(name, dim)  # numba_backend.py:341-346: weights / table / dummy
    assert code == pz.get_objective(name).code
    lib = _flat_binding()
    for t in range(steps):
        op, of, acc, nw = run_updates_ffi(lib, g["snap_pos"][t], g["snap_fit"][t], g["in_dr"][t], ps=ps, dim=dim,
                                          seed=seed, npairs=npairs, lower=lo, upper=hi, eps=eps, T=T, iteration=t,
                                          key_iteration=t + 1, code=code, table=table)
        assert np.array_equal(op, g["out_pos"][t]) and np.array_equal(of, g["out_fit"][t]), (name, t)
        assert np.array_equal(acc, g["acc"][t]) and nw == int(g["warn"][t])


@pytest.fixture
def ref_with_cuda(ref_protozoa, monkeypatch):
    """The maintainer's get_backend branch (INTEGRATION.md Option A), applied without editing the reference."""
    from protozoa import kernels

    from paper_2510_14982_b200.kernels import cuda_backend

    stock = kernels.get_backend

    def get_backend(name=None):
        if (name or "").strip().lower() == "cuda":
            return cuda_backend
        return stock(name)

    monkeypatch.setattr(kernels, "get_backend", get_backend)
    return ref_protozoa


@pytest.mark.gpu
@pytest.mark.parametrize("name,ps,dim", [("rosenbrock", 200, 20), ("high_conditioned_elliptic", 64, 10),
                                         ("hgbat", 333, 7), ("bent_cigar", 1000, 50), ("sphere", 31, 1)])
def test_option_a_reference_engine_step_with_cuda_backend(ref_with_cuda, name, ps, dim):
    protozoa = ref_with_cuda
    cfg = protozoa.ApoConfig(ps=ps, dim=dim, bounds=protozoa.Bounds(-30.0, 30.0, dim), max_iterations=20, seed=11)
    pop = protozoa.initialize(cfg, name)
    for t in range(4):
        mode = protozoa.EngineMode.sequential()
        want = protozoa.step(pop, cfg, name, t, mode, backend="numba")
        got = protozoa.step(pop, cfg, name, t, mode, backend="cuda")
        assert np.array_equal(got.positions, want.positions) and np.array_equal(got.fitness, want.fitness)
        assert got.warnings == want.warnings and got.fe_count == want.fe_count
        pop = want


@pytest.mark.gpu
def test_option_a_reference_run_with_cuda_backend(ref_with_cuda):
    protozoa = ref_with_cuda
    cfg = protozoa.ApoConfig(ps=100, dim=20, bounds=protozoa.Bounds(-100.0, 100.0, 20), max_iterations=60, seed=4)
    want = protozoa.run(cfg, "rosenbrock", backend="numba")
    got = protozoa.run(cfg, "rosenbrock", backend="cuda")
    assert np.array_equal(got.trace, want.trace) and got.best_fitness == want.best_fitness
    assert np.array_equal(got.best_position, want.best_position)
    assert np.array_equal(got.population.positions, want.population.positions)


@pytest.mark.gpu
def test_option_a_rejects_external_objective_like_numba(ref_with_cuda):
    """External objectives are forced to numpy by the reference engine (engine.py:92-97); asking the
    cuda backend directly for one raises ValueError, as numba_backend.py:339-340 does."""
    from paper_2510_14982_b200.kernels import cuda_backend

    from protozoa.objectives import external_objective

    protozoa = ref_with_cuda
    obj = external_objective(lambda x: float(np.sum(x * x)), name="ext")
    cfg = protozoa.ApoConfig(ps=8, dim=2, bounds=protozoa.Bounds(-1.0, 1.0, 2), max_iterations=3)
    with pytest.raises(ValueError):
        cuda_backend.run_updates(np.zeros((8, 2)), np.zeros(8), np.zeros(8, bool), cfg, obj, 0, 1)
