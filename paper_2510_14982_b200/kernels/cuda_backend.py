"""The "cuda" backend: the reference's run_updates protocol on the B200.

Module protocol (kernels/numba_backend.py:26,48,323 of the reference):
``NAME``, ``max_workers()`` and ``run_updates(positions, fitness, in_dr,
cfg, objective, iteration, key_iteration, parallel, workers)`` returning
``(new_positions, new_fitness, accepted, warning_count)``.  Inputs are read
only.  numpy inputs give numpy outputs (host<->device copies included);
CUDA tensors stay on the device.  ``parallel``/``workers`` are accepted for
signature compatibility: results never depend on them.
"""

from __future__ import annotations

import numpy as np

from .. import _lib
from ..core import ApoConfig, iteration_scalars, p_dr_table
from ..objectives import EXTERNAL, Objective, device_objective

NAME = "cuda"


def max_workers() -> int:
    """Visible CUDA devices (the reference reports CPU threads)."""
    try:
        return max(1, int(_lib.load().apo_device_count()))
    except Exception:
        return 1


_PDR_DEV: dict = {}


def p_dr_device(ps: int, device):
    import torch

    key = (ps, str(device))
    t = _PDR_DEV.get(key)
    if t is None:
        t = torch.as_tensor(np.array(p_dr_table(ps)), device=device)
        _PDR_DEV[key] = t
    return t


def run_updates(positions, fitness, in_dr, cfg: ApoConfig, objective: Objective, iteration: int,
                key_iteration: int, parallel: bool = False, workers: int = 1):
    import torch

    if objective.code == EXTERNAL:
        raise ValueError("the cuda backend cannot call external objective functions")
    lib = _lib.require_cuda()
    host = not isinstance(positions, torch.Tensor)
    dev = torch.device("cuda", torch.cuda.current_device()) if host else positions.device
    pos = torch.as_tensor(np.ascontiguousarray(positions, dtype=np.float64) if host else positions,
                          dtype=torch.float64, device=dev).contiguous()
    fit = torch.as_tensor(np.ascontiguousarray(fitness, dtype=np.float64) if host else fitness,
                          dtype=torch.float64, device=dev).contiguous()
    dr = torch.as_tensor(np.ascontiguousarray(in_dr, dtype=np.uint8) if host else in_dr, device=dev)
    dr = dr.to(torch.uint8).contiguous()
    ps, dim = pos.shape
    if fit.shape != (ps,) or dr.shape != (ps,):
        raise ValueError("fitness and in_dr must have one entry per row of positions")
    out_pos = torch.empty_like(pos)
    out_fit = torch.empty_like(fit)
    acc = torch.empty(ps, dtype=torch.uint8, device=dev)
    warn = torch.zeros(1, dtype=torch.int64, device=dev)
    p_ah, f_mult, decay = iteration_scalars(iteration, cfg.max_iterations)
    dobj = device_objective(objective, dim)
    rc = lib.apo_run_updates_obj(
        _lib.ptr(pos), _lib.ptr(fit), _lib.ptr(dr), _lib.ptr(out_pos), _lib.ptr(out_fit), _lib.ptr(acc), None,
        ps, dim, cfg.seed, key_iteration, cfg.neighbor_pairs, cfg.bounds.lower, cfg.bounds.upper, cfg.eps,
        p_ah, f_mult, decay, dobj.ref, _lib.ptr(p_dr_device(ps, dev)), _lib.ptr(warn), _lib.stream_handle())
    _lib.check(rc, "apo_run_updates")
    if host:
        return out_pos.cpu().numpy(), out_fit.cpu().numpy(), acc.cpu().numpy().astype(bool), int(warn.item())
    return out_pos, out_fit, acc.bool(), int(warn.item())


def run_updates_to_host(pos, fit, in_dr, cfg: ApoConfig, objective: Objective, iteration: int, key_iteration: int,
                        chunks: int = 4, order=None):
    """run_updates on device tensors with the result delivered to page-locked host memory: the update
    runs in rank chunks (apo_run_updates_range) and each finished chunk is copied back on a second
    stream while the next one computes.  Returns (positions, fitness) numpy views and the warning count;
    bit-identical to run_updates.  With `order` (int32 rank -> row, the stable sort's result) pos/fit
    are NOT the rank-ordered snapshot but the caller's rows, read through order[] (no gather)."""
    import torch

    lib = _lib.require_cuda()
    dev = pos.device
    ps, dim = pos.shape
    out_pos = torch.empty_like(pos)
    out_fit = torch.empty_like(fit)
    warn = torch.zeros(1, dtype=torch.int64, device=dev)
    hp = torch.empty((ps, dim), dtype=torch.float64, pin_memory=True)
    hf = torch.empty(ps, dtype=torch.float64, pin_memory=True)
    p_ah, f_mult, decay = iteration_scalars(iteration, cfg.max_iterations)
    dobj = device_objective(objective, dim)
    pdr = p_dr_device(ps, dev)
    from ..engine import _copy_stream

    compute = torch.cuda.current_stream()
    copy = _copy_stream(dev)
    step = -(-ps // chunks)
    step = (step + 31) // 32 * 32
    for lo in range(0, ps, step):
        hi = min(ps, lo + step)
        if order is not None:
            _lib.check(lib.apo_run_updates_ordered(
                _lib.ptr(pos), _lib.ptr(fit), _lib.ptr(order), _lib.ptr(in_dr), _lib.ptr(out_pos), _lib.ptr(out_fit),
                None, None, ps, dim, cfg.seed, key_iteration, cfg.neighbor_pairs, cfg.bounds.lower,
                cfg.bounds.upper, cfg.eps, p_ah, f_mult, decay, dobj.ref, _lib.ptr(pdr), _lib.ptr(warn), lo, hi,
                _lib.stream_handle()), "apo_run_updates_ordered")
        else:
            _lib.check(lib.apo_run_updates_range(
                _lib.ptr(pos), _lib.ptr(fit), _lib.ptr(in_dr), _lib.ptr(out_pos), _lib.ptr(out_fit), None, None,
                ps, dim, cfg.seed, key_iteration, cfg.neighbor_pairs, cfg.bounds.lower, cfg.bounds.upper, cfg.eps,
                p_ah, f_mult, decay, dobj.ref, _lib.ptr(pdr), _lib.ptr(warn), lo, hi, _lib.stream_handle()),
                "apo_run_updates_range")
        copy.wait_stream(compute)
        with torch.cuda.stream(copy):
            hp[lo:hi].copy_(out_pos[lo:hi], non_blocking=True)
            hf[lo:hi].copy_(out_fit[lo:hi], non_blocking=True)
    for t in (out_pos, out_fit):
        t.record_stream(copy)
    copy.synchronize()
    return hp.numpy(), hf.numpy(), int(warn.item())


def scripted_step_device(pos, fit, cfg: ApoConfig, objective: Objective, iteration: int, draws):
    """One iteration on device tensors with every draw read from `draws` (rng.DrawTable, APO_RNG_TABLE):
    stable sort, the coordinator's set from its scripted pf and permutation draws, the fused update.
    Returns (next positions, next fitness, accepted, warnings) by rank; raises LookupError on the first
    unscripted draw (the reference's ScriptedStream contract, tests/test_acceptance.py:50-80)."""
    import math

    import torch

    from ..rng import COORDINATOR_INDEX

    if objective.code == EXTERNAL:
        raise ValueError("the cuda backend cannot call external objective functions")
    if draws.seed != cfg.seed or draws.iteration != iteration + 1:
        raise ValueError(f"draw table is for (seed {draws.seed}, iteration {draws.iteration}); this step reads "
                         f"(seed {cfg.seed}, iteration {iteration + 1})")
    lib = _lib.require_cuda()
    dev = pos.device
    ps, dim = pos.shape
    ind, ctr, val = draws.arrays()
    u = draws.uniforms()
    pf_key = (COORDINATOR_INDEX, 0)  # COORD_SLOT_PF
    if pf_key not in u:
        raise LookupError(f"unscripted draw at (individual {COORDINATOR_INDEX}, counter 0)")
    count = int(math.ceil(ps * (cfg.pf_max * u[pf_key])))  # core.py:263-278
    t_ind = torch.as_tensor(ind.view(np.int64), device=dev)
    t_ctr = torch.as_tensor(ctr.view(np.int64), device=dev)
    t_val = torch.as_tensor(val, device=dev)
    miss = torch.zeros(3, dtype=torch.int64, device=dev)
    header = torch.as_tensor(np.array([len(val), t_ind.data_ptr(), t_ctr.data_ptr(), t_val.data_ptr(),
                                       miss.data_ptr()], dtype=np.uint64).view(np.int64), device=dev)
    stream = _lib.stream_handle()
    order = torch.empty(ps, dtype=torch.int32, device=dev)
    _lib.check(lib.apo_sort_order(_lib.ptr(fit), ps, _lib.ptr(order), stream), "apo_sort_order")
    in_dr = torch.empty(ps, dtype=torch.uint8, device=dev)
    _lib.check(lib.apo_select_dr_scripted(_lib.ptr(header), ps, count, _lib.ptr(in_dr), stream),
               "apo_select_dr_scripted")
    idx = order.long()
    snap_pos = pos.index_select(0, idx).contiguous()
    snap_fit = fit.index_select(0, idx).contiguous()
    out_pos, out_fit = torch.empty_like(snap_pos), torch.empty_like(snap_fit)
    acc = torch.empty(ps, dtype=torch.uint8, device=dev)
    warn = torch.zeros(1, dtype=torch.int64, device=dev)
    p_ah, f_mult, decay = iteration_scalars(iteration, cfg.max_iterations)
    dobj = device_objective(objective, dim)
    _lib.check(lib.apo_run_updates_scripted(
        _lib.ptr(snap_pos), _lib.ptr(snap_fit), _lib.ptr(in_dr), _lib.ptr(out_pos), _lib.ptr(out_fit), _lib.ptr(acc),
        None, ps, dim, _lib.ptr(header), cfg.neighbor_pairs, cfg.bounds.lower, cfg.bounds.upper, cfg.eps, p_ah,
        f_mult, decay, dobj.ref, _lib.ptr(p_dr_device(ps, dev)), _lib.ptr(warn), stream), "apo_run_updates_scripted")
    m = miss.cpu().numpy().view(np.uint64)
    if m[0]:
        raise LookupError(f"unscripted draw at (individual {int(m[1])}, counter {int(m[2])})")
    return out_pos, out_fit, acc.bool(), int(warn.item())
