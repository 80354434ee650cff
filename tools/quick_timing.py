"""Scratch timing of the headline shapes (CUDA events, warm; not the bench)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

torch.cuda.set_device(0)
tag = os.environ.get("APO_LIB", "default").split("/")[-1]
names = sys.argv[1:] or ["rosenbrock", "griewank"]
for name in [n for n in names if n != "c2"]:
    cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=100, seed=0)
    dr = DeviceRun(cfg, pz.get_objective(name))
    dr.initialize()
    dr.iterate(3)
    torch.cuda.synchronize()
    dr.profile(True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    dr.iterate(10)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    kms, n = dr.profile_read()
    print(f"[{tag}] C4 {name}: {ms:.3f} ms/iter (update kernel {kms / n:.3f} ms) -> {1e6 / ms * 1e3 / 1e9:.3f} Gevals/s",
          flush=True)
    dr.close()
if "c2" in names or not sys.argv[1:]:
    cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=1000)
    nm = list(pz.FUNCTION_NAMES) * 60
    seeds = list(range(len(nm)))
    pz.run_batch(cfg, nm[:8], seeds[:8])
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pz.run_batch(cfg, nm, seeds, want_trace=False, device_out=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"[{tag}] C2-like batch 360 runs: {dt * 1e3:.1f} ms -> {360 * 100 * 1000 / dt / 1e9:.3f} Gevals/s", flush=True)
