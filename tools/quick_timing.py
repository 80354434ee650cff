"""Scratch timing of the two headline shapes (not the bench; CUDA events, warm)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

torch.cuda.set_device(0)
for name in ("rosenbrock", "griewank"):
    cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=20, seed=0)
    dr = DeviceRun(cfg, pz.get_objective(name))
    dr.initialize(); dr.iterate(3); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); dr.iterate(10); e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print(f"C4 {name}: {ms:.3f} ms/iter -> {1e6/ms*1e3/1e9:.3f} Gevals/s", flush=True)
    dr.close()

cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=1000)
names = list(pz.FUNCTION_NAMES) * 60
seeds = list(range(len(names)))
pz.run_batch(cfg, names[:8], seeds[:8]); torch.cuda.synchronize()
t0 = time.perf_counter(); r = pz.run_batch(cfg, names, seeds, want_trace=False); torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"C2-like batch 360 runs: {dt*1e3:.1f} ms -> {360*100*1000/dt/1e9:.3f} Gevals/s", flush=True)
