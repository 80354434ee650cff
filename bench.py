#!/usr/bin/env python
"""bench.py -- APO population-update throughput on B200 (driver contract).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--workload c4|c2]

A "step" is one APO iteration (stable sort -> coordinator draws -> fused
update of every protozoon) over the resident population.  Headline
workload (BASELINE.json config 4 at one GPU): ps = 1,000,000, D = 100,
objective ``--objective`` (default rosenbrock; F6/F10 are CEC2022 names
when built), 800 MB population in HBM (> L2, so no flush is needed).
Multi-GPU (torchrun): every rank runs its own independent population
(seed = rank), no collective on the data path -> weak scaling; time is the
max over ranks of CUDA-event time.

``--impl reference`` times the CPU restatement of the reference iteration
(oracle/, bit-identical to the reference's numba path) on this host's
cores, rank 0 only.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "protozoa-evals/sec"
UNIT = "evals/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=["c4", "c2", "c3", "c5"])
    ap.add_argument("--objective", default="cec2022_f6")
    ap.add_argument("--ps", type=int, default=1_000_000)
    ap.add_argument("--dim", type=int, default=100)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-shard", action="store_true")
    return ap.parse_args()


# ---------------------------------------------------------------------------
# distributed plumbing


def dist_setup(backend):
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            import torch

            torch.cuda.set_device(local)  # bind this rank's GPU before NCCL creates its communicator
            dist.init_process_group(backend=backend, device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend=backend)
    return rank, world, local


def barrier(world):
    if world > 1:
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ---------------------------------------------------------------------------
# clocks sampled during the timed region


class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        if self.proc is None:
            return out
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        rows = []
        for line in open(self.path):
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                rows.append(parts)
        os.unlink(self.path)
        if not rows:
            return out
        sm = [float(r[1]) for r in rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in rows for k in range(4) if r[5 + k].lower().startswith("active")})
        out.update(sm_mhz=statistics.median(sm) if sm else None, sm_max_mhz=max(mx) if mx else None,
                   reasons=reasons, samples=len(rows))
        return out


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


def profile_traffic(workload: str, objective: str):
    """dram bytes per update launch from the committed ncu --set full capture, if any."""
    path = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(path) as fh:
            return json.load(fh).get(f"{workload}:{objective}")
    except Exception:
        return None


def traffic_fields(key: str):
    """ncu DRAM bytes of ONE captured launch (profiles/traffic.json) and the algorithmic bytes of that
    same launch, so the two compare like with like (a span-averaged algorithmic figure would not)."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh).get("launches", {}).get(key)
    except Exception:
        t = None
    if not t:
        return {"traffic": None}
    return {"traffic": t.get("dram_bytes"), "traffic_launch": t.get("launch"),
            "traffic_algorithmic_bytes": t.get("algorithmic_bytes"),
            "traffic_over_algorithmic": (round(t["dram_bytes"] / t["algorithmic_bytes"], 3)
                                         if t.get("algorithmic_bytes") else None)}


def dmma_pipe_pct(key: str, objective: str = None):
    """DMMA pipe utilisation of the captured launch (profiles/traffic.json), if any."""
    try:
        with open(os.path.join(ROOT, "profiles", "traffic.json")) as fh:
            t = json.load(fh).get("launches", {}).get(key)
        return t.get("dmma_pipe_active_pct") if t else None
    except Exception:
        return None


# ---------------------------------------------------------------------------
# algorithmic bytes


def op_mix(seed: int, key_iteration: int, ps: int, p_ah: float, in_dr: np.ndarray) -> float:
    """Exact autotroph fraction of one iteration (population independent)."""
    from paper_2510_14982_b200 import rng

    i = np.arange(1, ps + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = rng._mix_vec(np.uint64(rng.H0) ^ np.uint64(seed))
        h = rng._mix_vec(np.uint64(h) ^ np.uint64(key_iteration))
        base = rng._mix_vec(np.uint64(h) ^ i)
        u = (rng._mix_vec(base) >> np.uint64(11)).astype(np.float64) * rng.INV_2_53
    return float(np.count_nonzero((~in_dr) & (u < p_ah))) / ps


def bytes_per_eval(dim: int, p_auto: float, npairs: int = 1) -> float:
    return 8.0 * dim * (2.0 + p_auto * (1 + 2 * npairs)) + 32.0


# ---------------------------------------------------------------------------


def fp64_peak():
    """Measured FP64 DMMA peak (tools/fp64_peak.cu on this pool's B200, profiles/r01_fp64_peak.json)."""
    try:
        with open(os.path.join(ROOT, "profiles", "r01_fp64_peak.json")) as fh:
            d = json.load(fh)
        return float(d["dmma_tflops_4chain"]), "measured (tools/fp64_peak.cu)"
    except Exception:
        return 37.0, "fallback"


def rotated_components(name: str) -> int:
    """Rotations per evaluation (the D x D contractions k_cec_eval runs)."""
    if not name.startswith("cec2022_f"):
        return 0
    fn = int(name[len("cec2022_f"):])
    return {9: 3, 10: 1, 11: 5, 12: 6}.get(fn, 1)


def c4_measure(args, name, rank, world, local, K, W):
    """Device-resident C4 run: CUDA-event time of K iterations + per-kernel split."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import _lib
    from paper_2510_14982_b200.core import iteration_scalars
    from paper_2510_14982_b200.engine import DeviceRun

    ps, dim = args.ps, args.dim
    # the run is exactly W + K iterations long, so the K timed steps carry the schedule (p_ah, f, decay:
    # numba_backend.py:357-366) from early autotroph-heavy iterations to the heterotroph-heavy end
    T = W + K
    obj = pz.get_objective(name)
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=T, seed=rank)
    run = DeviceRun(cfg, obj)
    run.initialize()
    run.iterate(W)
    torch.cuda.synchronize()
    run.profile(True)
    clocks = ClockSampler(local)
    barrier(world)
    torch.cuda.synchronize()
    clocks.start()
    stream = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    run.iterate(K)
    e1.record(stream)
    torch.cuda.synchronize()
    barrier(world)
    clk = clocks.stop()
    ms = e0.elapsed_time(e1)
    cand_ms, eval_ms, launches = run.profile_split()
    path = run.update_path()
    max_ms = max_over_ranks(ms, world)
    # algorithmic bytes of the timed candidate launches (population independent op mix)
    dev = torch.device("cuda", local)
    in_dr = torch.empty(ps, dtype=torch.uint8, device=dev)
    total_bytes, p_autos = 0.0, []
    for t in range(W, W + K):
        _lib.check(_lib.load().apo_select_dr(cfg.seed, t + 1, ps, cfg.pf_max, _lib.ptr(in_dr), None,
                                             _lib.stream_handle()))
        p_auto = op_mix(cfg.seed, t + 1, ps, iteration_scalars(t, T)[0], in_dr.cpu().numpy().astype(bool))
        p_autos.append(p_auto)
        total_bytes += ps * bytes_per_eval(dim, p_auto, cfg.neighbor_pairs)
    run.close()
    del run
    torch.cuda.empty_cache()
    n = max(launches, 1)
    peaks, peak_kind = measured_peaks()
    per_launch = total_bytes / K
    nrot = rotated_components(name)
    flops = ps * nrot * 2.0 * dim * dim
    pk, pk_src = fp64_peak()

    def hbm_entry(kernel, ms_sum, traffic_key):
        gbs = per_launch / (ms_sum / 1e3 / n) / 1e9
        return {"kernel": kernel, "bound": "hbm", "achieved": round(gbs, 1), "peak": peaks["hbm_gbs"], "unit": "GB/s",
                "frac": round(gbs / peaks["hbm_gbs"], 4), "peak_source": peak_kind,
                "kernel_ms_avg": round(ms_sum / n, 4), "kernel_share_of_step": round(ms_sum / ms, 4),
                "bytes_per_launch": per_launch, "bytes_per_eval": round(per_launch / ps, 1),
                "p_auto_mean": round(float(np.mean(p_autos)), 4), **traffic_fields(traffic_key)}

    def dmma_entry(kernel, ms_sum, traffic_key, also=None):
        tf = flops / (ms_sum / 1e3 / n) / 1e12
        e = {"kernel": kernel, "bound": "tensor", "achieved": round(tf, 2), "peak": pk, "unit": "TFLOP/s",
             "frac": round(tf / pk, 4), "peak_source": pk_src, "kernel_ms_avg": round(ms_sum / n, 4),
             "kernel_share_of_step": round(ms_sum / ms, 4), "flops_per_launch": flops,
             "flops_per_eval": nrot * 2.0 * dim * dim, **traffic_fields(traffic_key),
             "ncu_dmma_pipe_active_pct": dmma_pipe_pct(traffic_key, name)}
        e.update(also or {})
        return e

    if path == "cec_fused":
        # one kernel does the HBM-bound update and the DMMA rotation: report both roofs, bound = the
        # one it is closer to
        both = cand_ms + eval_ms
        d = dmma_entry("k_update_cec<13,4> (fused: candidates + DMMA f64 rotation + basic + greedy select)", both,
                       f"c4fused:{name}")
        h = hbm_entry(d["kernel"], both, f"c4fused:{name}")
        d["hbm"] = {k: h[k] for k in ("achieved", "peak", "unit", "frac", "bytes_per_launch", "bytes_per_eval",
                                      "p_auto_mean")}
        kernels = [d]
    elif path == "cec_split":
        kernels = [hbm_entry("k_update_group<SEL> (candidates only)", cand_ms, f"c4:{name}"),
                   dmma_entry("k_cec_eval (DMMA f64 m8n8k4 rotation + basic + greedy select)", eval_ms,
                              f"c4eval:{name}", {"also_reads_bytes_per_eval": 8 * dim + 16})]
    elif path == "basic_split":
        # candidates (HBM-bound) + lane-per-protozoon sequential evaluation: the update as a whole against
        # the HBM roof (the evaluation re-reads the 8 D bytes per candidate: reported beside it)
        e = hbm_entry("k_update_group<SEL> (candidates) + k_basic_eval (sequential fold + select)", cand_ms + eval_ms,
                      f"c4:{name}")
        e["split_ms"] = {"candidates": round(cand_ms / n, 4), "evaluate": round(eval_ms / n, 4)}
        e["eval_reread_bytes_per_eval"] = 8 * dim + 16
        kernels = [e]
    else:
        kernels = [hbm_entry("k_update_group<SEL> (fused update, " + path + ")", cand_ms + eval_ms, f"c4:{name}")]
    dominant = max(kernels, key=lambda k: k["kernel_ms_avg"])
    return dict(cfg=cfg, obj=obj, ms=ms, max_ms=max_ms, clocks=clk, kernels=kernels, dominant=dominant,
                launches=launches, path=path)


def c4_workload(name, ps, dim):
    return f"C4: single population ps={ps} D={dim} objective={name} (synthetic CEC2022 data)"


def bench_ours(args, rank, world, local):
    import torch

    torch.cuda.set_device(local)
    K, W = args.steps, args.warmup
    m = c4_measure(args, args.objective, rank, world, local, K, W)
    ps, dim = args.ps, args.dim
    value = world * ps * K / (m["max_ms"] / 1e3)
    roofline = dict(m["dominant"])
    result = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K, "warmup": W,
        "ms_per_step": m["max_ms"] / K, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "update_path": m["path"],
        "dtype": "f64", "data": "synthetic (keyed-hash initial population, seed = rank; synthetic CEC2022 "
                                "shift/rotation/shuffle data, cec2022.py)",
        "config": {"workload": c4_workload(args.objective, ps, dim), "ps": ps, "dim": dim,
                   "iterations_per_step": 1, "max_iterations": K + W,
                   "schedule": "the K timed steps are the last K of a (W+K)-iteration run (autotroph -> heterotroph)",
                   "l2": "inputs larger than L2 (2 x 800 MB population buffers)",
                   "parallelism": f"independent populations x{world} (seed = rank)" if world > 1 else "single GPU",
                   "rng": "keyed fmix64 (bit-exact with the reference)"},
        "roofline": roofline,
        "roofline_kernels": m["kernels"],
        "clocks": m["clocks"],
        # per iteration (profiles/r02_launches_c4.summary.txt): the stable sort = k_make_keys + CUB histogram,
        # exclusive sum and 8 onesweep passes (11); the coordinator's Dr = k_dr_draw + CUB histogram, exclusive
        # sum, 3 onesweep passes + k_dr_resolve (7, on the side stream); the update = k_update_group (+ the
        # evaluation kernel on the split paths).  CUB's kernels are templates compiled into libapo_b200.so.
        "gpu_launches": (18 + (2 if m["path"] in ("cec_split", "basic_split", "cec_gemm") else 1)) * K,
    }
    if not args.no_suite:
        # the other headline objective, and the memory-bound update on a reference objective (rosenbrock:
        # bit-pinned to the reference's own vectors) with its own HBM roofline
        for other in (("cec2022_f10" if args.objective != "cec2022_f10" else "cec2022_f6"), "rosenbrock"):
            m2 = c4_measure(args, other, rank, world, local, K, W)
            result["c4_" + other.replace("cec2022_", "")] = {
                "value": world * ps * K / (m2["max_ms"] / 1e3), "unit": UNIT, "ms_per_step": m2["max_ms"] / K,
                "workload": c4_workload(other, ps, dim), "update_path": m2["path"], "roofline": m2["dominant"],
                "roofline_kernels": m2["kernels"], "clocks": m2["clocks"]}
    if world > 1 and not args.no_shard:
        # N > 1: BASELINE config 4 as stated -- ONE population sharded over the N GPUs (strong scaling) is
        # the headline; the N independent populations above stay as the weak-scaling side line
        try:
            sh = bench_sharded(args, rank, world, local, K, W)
            result["c4_independent"] = {"value": value, "unit": UNIT, "ms_per_step": m["max_ms"] / K,
                                        "scaling": "weak", "workload": f"{world} independent C4 populations"}
            result["c4_sharded"] = sh
            result["value"] = sh["value"]
            result["ms_per_step"] = sh["ms_per_step"]
            result["scaling"] = "strong"
            result["config"]["workload"] = sh["workload"]
            result["config"]["parallelism"] = f"one population sharded by rank over {world} GPUs"
        except Exception as exc:  # never lose the main line over the secondary measurement
            result["c4_sharded"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            result["c2_sharded"] = bench_c2_sharded(rank, world)
        except Exception as exc:
            result["c2_sharded"] = {"error": f"{type(exc).__name__}: {exc}"[:300]}
    if not args.no_e2e:
        result["e2e"] = bench_e2e(m["cfg"], m["obj"], K, rank, world)
        result["e2e_run"] = bench_e2e_run(m["cfg"], m["obj"], rank, world)
    if not args.no_suite and rank == 0:
        result["suite_c1"] = bench_c1()
        result["suite_c2"] = bench_suite(world)
        result["suite_c3"] = bench_c3()
        result["suite_c5"] = bench_c5()
    if rank == 0 and world == 1 and not args.no_cpu:
        result["cpu_baseline"] = cpu_baseline(m["cfg"], args.objective)
        try:
            ros = result.get("c4_rosenbrock", {})
            result["cpu_baseline_numba"] = cpu_baseline_numba(
                {"value": ros.get("value"), "line": "c4_rosenbrock"} if ros else None)
        except Exception as exc:  # a reported baseline: never lose the main line over it
            result["cpu_baseline_numba"] = {"unavailable": f"{type(exc).__name__}: {exc}"[:200]}
    return result


def bench_sharded(args, rank, world, local, K, W):
    """C4 as BASELINE config 4 states it: ONE population of ps rows sharded by rank over the N GPUs,
    per-iteration NCCL all-gather of the updated rows (strong scaling; shard.ShardedRun)."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.shard import ShardedRun

    ps, dim = args.ps, args.dim
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=K + W, seed=0)
    run = ShardedRun(cfg, args.objective)
    run.initialize()
    run.iterate(W)
    torch.cuda.synchronize()
    barrier(world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run.iterate(K)
    e1.record()
    torch.cuda.synchronize()
    barrier(world)
    ms = max_over_ranks(e0.elapsed_time(e1), world)
    trace, _ = run.trace_and_warnings()
    run.close()
    return {"value": ps * K / (ms / 1e3), "unit": UNIT, "ms_per_step": ms / K, "scaling": "strong",
            "workload": f"C4 sharded: ONE population ps={ps} D={dim} {args.objective} split by rank over {world} GPUs, "
                        "NCCL all-gather of rows + fitness per iteration",
            "exchange_bytes_per_gpu_per_step": 8 * (dim + (dim & 1) + 1) * ps * (world - 1) / world,
            "best": float(trace[-1])}


def bench_e2e(cfg, obj, K, rank, world):
    """Same metric through the public API with HOST buffers: pz.step(Population) per iteration."""
    import torch

    import paper_2510_14982_b200 as pz

    import dataclasses

    W = 4  # warm-up: lazy init, first-touch of host pages, the two page-locked buffers step() alternates
    n = 10
    cfg = dataclasses.replace(cfg, max_iterations=W + n)
    pop = pz.initialize(cfg, obj)
    for t in range(W):
        pop = pz.step(pop, cfg, obj, t)
    torch.cuda.synchronize()
    barrier(world)
    per = []
    t0 = time.perf_counter()
    for t in range(W, W + n):
        ts = time.perf_counter()
        pop = pz.step(pop, cfg, obj, t)
        per.append(time.perf_counter() - ts)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, world)
    nb = 8 * cfg.ps * cfg.dim + 8 * cfg.ps
    return {"value": world * cfg.ps * n / dt, "unit": UNIT, "h2d_bytes_per_step": nb, "d2h_bytes_per_step": nb,
            "steps": n, "warmup": W, "step_ms": [round(1e3 * x, 1) for x in per],
            "api": "paper_2510_14982_b200.step(Population numpy) -> Population numpy (the reference-facing "
                   "per-iteration call; the whole population crosses PCIe both ways every step)"}


def bench_e2e_run(cfg, obj, rank, world, T=30):
    """A whole engine.run (the loop resident on the device) end to end: initialisation, T iterations,
    and the RunResult on the host (trace, best, final population D2H) -- evals/s over ps * T."""
    import dataclasses

    import torch

    import paper_2510_14982_b200 as pz

    c = dataclasses.replace(cfg, max_iterations=T)
    for _ in range(2):  # warm-up (allocations, first touch of the host result pages)
        pz.run(dataclasses.replace(c, max_iterations=3), obj)
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    res = pz.run(c, obj)
    dt = max_over_ranks(time.perf_counter() - t0, world)
    return {"value": world * c.ps * T / dt, "unit": UNIT, "iterations": T, "seconds": dt,
            "d2h_bytes": int(res.population.positions.nbytes + res.population.fitness.nbytes + res.trace.nbytes),
            "api": "paper_2510_14982_b200.run(cfg, objective) -> RunResult (host arrays)"}


def bench_suite(world):
    """BASELINE config 2: CEC2022 F1-F12 x 30 seeds (360 independent runs), D=20, ps=100, T=1000,
    one CTA per run with the population resident in shared memory (rank 0's GPU)."""
    import torch

    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=1000)
    names = [f"cec2022_f{k}" for k in range(1, 13) for _ in range(30)]
    seeds = [s for _ in range(12) for s in range(30)]
    pz.run_batch(cfg, names[:24], seeds[:24], want_trace=False, device_out=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    times = []
    for _ in range(3):  # the launch's time is its slowest SM's three co-resident runs: report the median
        e0.record()
        res = pz.run_batch(cfg, names, seeds, want_trace=False, device_out=True)
        e1.record()
        torch.cuda.synchronize()
        times.append(e0.elapsed_time(e1))
    ms = float(np.median(times))
    evals = len(names) * cfg.ps * cfg.max_iterations
    best = res.best_fitness.cpu().numpy().reshape(12, 30)
    return {"value": evals / (ms / 1e3), "unit": UNIT, "ms": ms, "ms_all": [round(t, 1) for t in times],
            "runs": len(names),
            "workload": "C2: CEC2022 F1-F12 (synthetic data) x 30 seeds, D=20, ps=100, T=1000, one CTA per run",
            "median_best_minus_fstar": [float(np.median(best[k]) - pz.cec2022.FSTAR[k]) for k in range(12)],
            "gpus": 1}


def bench_c2_sharded(rank, world):
    """BASELINE config 2 over the N GPUs: the 360 (objective, seed) runs round-robin over ranks through
    engine.run_many -- no collective while runs execute, one all-gather of per-run results at the end.
    Time: CUDA events around each rank's batch, max over ranks, plus the final gather (wall clock)."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.engine import run_many

    cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=1000)
    names = [f"cec2022_f{k}" for k in range(1, 13) for _ in range(30)]
    seeds = [s for _ in range(12) for s in range(30)]
    run_many(cfg, names[:2 * world], seeds[:2 * world])  # warm-up
    torch.cuda.synchronize()
    barrier(world)
    t0 = time.perf_counter()
    res = run_many(cfg, names, seeds)
    torch.cuda.synchronize()
    dt = max_over_ranks(time.perf_counter() - t0, world)
    evals = len(names) * cfg.ps * cfg.max_iterations
    return {"value": evals / dt, "unit": UNIT, "seconds": dt, "runs": len(names), "scaling": "strong",
            "workload": f"C2: CEC2022 F1-F12 x 30 seeds (360 runs) round-robin over {world} GPUs via run_many",
            "median_best_minus_fstar": [float(np.median(res.best_fitness[30 * k:30 * k + 30]) -
                                              pz.cec2022.FSTAR[k]) for k in range(12)]}


def bench_c1():
    """BASELINE config 1: CEC2022 F1 D=10, pop=50, 1000 iterations, one seed -- a latency regime (one CTA
    holds the whole run in shared memory); the oracle's single-threaded run of the same config beside it."""
    import torch

    import paper_2510_14982_b200 as pz

    cfg = pz.ApoConfig(ps=50, dim=10, bounds=pz.Bounds(-100.0, 100.0, 10), max_iterations=1000, seed=0)
    pz.run(cfg, "cec2022_f1")
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = pz.run(cfg, "cec2022_f1")
    gpu_s = time.perf_counter() - t0
    out = {"workload": "C1: CEC2022 F1 (synthetic data) D=10, ps=50, T=1000, seed 0, pz.run end to end",
           "seconds": gpu_s, "value": cfg.ps * (cfg.max_iterations + 1) / gpu_s, "unit": UNIT,
           "best_minus_fstar": res.best_fitness - 300.0}
    try:
        import oracle

        t0 = time.perf_counter()
        want = oracle.run(ps=50, dim=10, max_iterations=1000, seed=0, name="cec2022_f1", lower=-100.0, upper=100.0)
        cpu_s = time.perf_counter() - t0
        out["cpu_oracle_seconds"] = cpu_s
        out["cpu_oracle_best_minus_fstar"] = want["best_fitness"] - 300.0
    except Exception as exc:  # the oracle is a checker; its absence must not cost the GPU line
        out["cpu_oracle"] = f"unavailable: {exc}"[:200]
    return out


def bench_c3(threads_per_run=320):
    """BASELINE config 3: multilevel Otsu and Kapur (k = 2..5 thresholds) on a synthetic 4096x4096 8-bit
    image; ps=100, T=1000, 30 seeds per (method, k), the 8 batches on 8 concurrent streams."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200 import imaging

    rnd = np.random.default_rng(0)
    n = 4096 * 4096
    comp = rnd.random(n) < 0.5
    px = np.where(comp, rnd.normal(70.0, 12.0, n), rnd.normal(190.0, 14.0, n))
    img = np.clip(np.rint(px), 0, 255).astype(np.uint8)
    dimg = torch.as_tensor(img).cuda()
    imaging.histogram_device(dimg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    reps = 20
    for _ in range(reps):
        counts = imaging.histogram_device(dimg)
    e1.record()
    torch.cuda.synchronize()
    hist_ms = e0.elapsed_time(e1) / reps
    jobs = []
    for method in ("otsu", "kapur"):
        for k in (2, 3, 4, 5):
            obj = imaging.multilevel_objective(counts, k, method)
            cfg = pz.ApoConfig(ps=100, dim=k, bounds=pz.Bounds(0.0, 255.0, k), max_iterations=1000)
            jobs.append((method, k, obj, cfg))
    streams = [torch.cuda.Stream() for _ in jobs]
    for (m, k, obj, cfg), st in zip(jobs, streams):  # warm-up (compiles nothing; first-launch costs)
        pz.run_batch(cfg, [obj] * 2, [0, 1], want_trace=False, device_out=True, stream=st,
                     threads_per_run=threads_per_run)
    torch.cuda.synchronize()
    e0.record()
    cur = torch.cuda.current_stream()
    outs = []
    for (m, k, obj, cfg), st in zip(jobs, streams):
        st.wait_stream(cur)
        outs.append(pz.run_batch(cfg, [obj] * 30, list(range(30)), want_trace=False, device_out=True, stream=st,
                                 threads_per_run=threads_per_run))
    for st in streams:
        cur.wait_stream(st)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    evals = len(jobs) * 30 * 100 * 1000
    best = {f"{m}_k{k}": {"thresholds": list(imaging.thresholds_of(o.best_position[0].cpu().numpy())),
                          "value": -float(o.best_fitness.min())}
            for (m, k, _, _), o in zip(jobs, outs)}
    return {"value": evals / (ms / 1e3), "unit": UNIT, "ms": ms, "runs": len(jobs) * 30,
            "workload": "C3: Otsu + Kapur, k=2..5, synthetic 4096x4096 bimodal u8 image, ps=100, T=1000, 30 seeds",
            "histogram": {"ms": hist_ms, "gbs": n / (hist_ms / 1e3) / 1e9, "kernel": "k_histogram_u8"},
            "best": best, "prefix_tables": "shared memory (k_run_batch stages the 515-entry table per CTA)"}


def bench_c5(sizes=(10, 20, 50, 100, 1000), fns=(1, 4, 10), ps=10_000, iters=20, small=False):
    """BASELINE config 5: dimension sweep on rotated functions, DMMA (tensor-core) rotation vs the FMA
    path.  ps=10^4 device-resident loop (the paper's PS), `iters` timed iterations after 3 warm-up; with
    small=True also ps=100 x 30 seeds x 200 iterations (one CTA per run where it fits in SMEM)."""
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.engine import DeviceRun

    rows = []
    for fn in fns:
        for dim in sizes:
            for rot in ("dmma", "fma", "auto"):  # auto: what the library picks (FMA on this path at D <= 32)
                obj = pz.cec2022_objective(fn, rotation=rot)
                cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=iters + 3)
                run = DeviceRun(cfg, obj)
                run.initialize()
                run.iterate(3)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                run.iterate(iters)
                e1.record()
                torch.cuda.synchronize()
                ms = e0.elapsed_time(e1) / iters
                run.close()
                row = {"fn": fn, "dim": dim, "ps": ps, "rotation": rot, "ms_per_iteration": round(ms, 4),
                       "evals_per_s": ps / (ms / 1e3), "rotation_tflops": ps * 2.0 * dim * dim *
                       {9: 3, 10: 1, 11: 5, 12: 6}.get(fn, 1) / (ms / 1e3) / 1e12}
                if small:
                    scfg = pz.ApoConfig(ps=100, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=200)
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    if pz.engine._batch_fits(scfg, [obj]):
                        pz.run_batch(scfg, [obj] * 30, list(range(30)), want_trace=False, device_out=True)
                    else:
                        for sd in range(30):
                            pz.run(pz.ApoConfig(ps=100, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim),
                                                max_iterations=200, seed=sd), obj)
                    torch.cuda.synchronize()
                    row["ps100_30seeds_evals_per_s"] = 30 * 100 * 200 / (time.perf_counter() - t0)
                rows.append(row)
    return {"workload": f"C5: F{'/F'.join(str(f) for f in fns)} x D in {list(sizes)}, ps={ps}, DMMA vs FMA rotation",
            "rows": rows}


def cpu_baseline(cfg, objective, max_seconds=25.0):
    """The oracle's reference iteration (oracle.step, bit-identical to the reference) on all host cores."""
    import oracle

    nthreads = os.cpu_count() or 1
    pos, fit = oracle.initialize(cfg.seed, cfg.ps, cfg.dim, cfg.bounds.lower, cfg.bounds.upper, objective)
    done = 0
    t0 = time.perf_counter()
    while True:
        pos, fit, _, _ = oracle.step(pos, fit, seed=cfg.seed, iteration=done, max_iterations=cfg.max_iterations,
                                     name=objective, lower=cfg.bounds.lower, upper=cfg.bounds.upper,
                                     pf_max=cfg.pf_max, nthreads=nthreads)
        done += 1
        if time.perf_counter() - t0 > max_seconds / 2 or done >= 5:
            break
    dt = time.perf_counter() - t0
    return {"value": cfg.ps * done / dt, "unit": UNIT, "cores": nthreads, "kind": "port",
            "sample": f"{done} full iterations of ps={cfg.ps} D={cfg.dim} {objective} "
                      "(oracle.step: stable sort + gather + coordinator + OpenMP update)",
            "cpu": _cpu_model()}


def cpu_baseline_numba(gpu_line=None, ps=1_000_000, dim=100, steps=3, max_seconds=60.0):
    """BASELINE.md §2's CPU baseline: the UNMODIFIED reference (baseline/_ref, numba backend, parallel
    mode on every host core) stepping the C4 shape on its own objective rosenbrock, JIT warm-up excluded
    (as compare_backends.py:56).  The initial population is the oracle's (bit-identical to the reference's
    initialize, which alone takes ~30 s of Python at this size)."""
    ref_site = os.path.join(ROOT, "baseline", "_ref")
    if not os.path.isdir(os.path.join(ref_site, "protozoa")):
        return {"unavailable": "reference not installed in baseline/_ref"}
    os.environ.setdefault("NUMBA_CACHE_DIR", os.path.join(tempfile.gettempdir(), "numba_cache_bench"))
    sys.path.insert(0, ref_site)
    try:
        import protozoa
    finally:
        sys.path.remove(ref_site)
    import oracle

    nthreads = os.cpu_count() or 1
    cfg = protozoa.ApoConfig(ps=ps, dim=dim, bounds=protozoa.Bounds(-100.0, 100.0, dim), max_iterations=25, seed=0)
    mode = protozoa.EngineMode.parallel(nthreads)
    small = protozoa.ApoConfig(ps=64, dim=dim, bounds=protozoa.Bounds(-100.0, 100.0, dim), max_iterations=3)
    protozoa.step(protozoa.initialize(small, "rosenbrock"), small, "rosenbrock", 0, mode)  # numba JIT
    pos, fit = oracle.initialize(0, ps, dim, -100.0, 100.0, "rosenbrock")
    pop = protozoa.Population(pos, fit, iteration=0, fe_count=ps)
    done, t0 = 0, time.perf_counter()
    while done < steps and time.perf_counter() - t0 < max_seconds:
        pop = protozoa.step(pop, cfg, "rosenbrock", done, mode)
        done += 1
    dt = time.perf_counter() - t0
    out = {"value": ps * done / dt, "unit": UNIT, "cores": nthreads, "kind": "reference",
           "sample": f"{done} protozoa.step iterations (numba backend, EngineMode.parallel({nthreads})) of "
                     f"ps={ps} D={dim} rosenbrock, JIT excluded",
           "cpu": _cpu_model()}
    if gpu_line:
        out["gpu_same_workload"] = gpu_line
    return out


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return None


def bench_reference(args, rank, world):
    """CPU reference arm: rank 0 times oracle.step on the same workload with every host core."""
    if rank != 0:
        return None
    import oracle
    import paper_2510_14982_b200 as pz

    ps, dim, K, W = args.ps, args.dim, args.steps, args.warmup
    T = W + K  # the same schedule span as the GPU arm
    nthreads = os.cpu_count() or 1
    pos, fit = oracle.initialize(0, ps, dim, -100.0, 100.0, args.objective)
    step_args = dict(seed=0, max_iterations=T, name=args.objective, lower=-100.0, upper=100.0, nthreads=nthreads)
    t0 = time.perf_counter()
    for t in range(W):
        pos, fit, _, _ = oracle.step(pos, fit, iteration=t, **step_args)
    t_warm = (time.perf_counter() - t0) / max(W, 1)
    budget = 150.0
    k_run = max(1, min(K, int(budget / max(t_warm, 1e-3))))
    t0 = time.perf_counter()
    for t in range(W, W + k_run):
        pos, fit, _, _ = oracle.step(pos, fit, iteration=t, **step_args)
    dt = time.perf_counter() - t0
    value = ps * k_run / dt
    sample = (f"{k_run} of {K} requested full iterations (budget {budget:.0f} s) of ps={ps} D={dim} "
              f"{args.objective} via oracle.step")
    return {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": k_run, "warmup": W,
        "ms_per_step": dt * 1e3 / k_run, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic", "impl": "reference",
        "config": {"workload": c4_workload(args.objective, ps, dim), "ps": ps, "dim": dim, "iterations_per_step": 1},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port", "sample": sample,
                         "cpu": _cpu_model()},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def main():
    args = parse()
    if args.impl == "reference":
        rank = int(os.environ.get("RANK", "0"))
        world = int(os.environ.get("WORLD_SIZE", "1"))
        res = bench_reference(args, rank, world)
        if res is not None:
            print(json.dumps(res), flush=True)
        return
    rank, world, local = dist_setup("nccl")
    if args.workload in ("c2", "c3", "c5"):
        import torch

        torch.cuda.set_device(local)
        res = (bench_suite(world) if args.workload == "c2" else bench_c3() if args.workload == "c3"
               else bench_c5(small=True))
        if rank == 0:
            print(json.dumps({"metric": METRIC, **res, "n_gpus": world, "steps": 1, "warmup": 1}), flush=True)
        return
    res = bench_ours(args, rank, world, local)
    if rank == 0:
        print(json.dumps(res), flush=True)
    if world > 1:
        import torch.distributed as dist

        dist.barrier()  # rank 0 may still be running the single-GPU suites
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
