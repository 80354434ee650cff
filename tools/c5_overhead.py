"""Host vs device time per iteration of the device loop at small populations (C5 shapes); not a bench value."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

for name, ps, dim in (("cec2022_f1", 1000, 10), ("cec2022_f1", 10000, 10), ("cec2022_f1", 100000, 10),
                      ("cec2022_f1", 10000, 100), ("rosenbrock", 10000, 10)):
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=420, seed=0)
    run = DeviceRun(cfg, pz.get_objective(name))
    run.initialize()
    run.iterate(20)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    t0 = time.perf_counter()
    run.iterate(400)
    host = time.perf_counter() - t0
    e1.record()
    torch.cuda.synchronize()
    dev = e0.elapsed_time(e1)
    print(f"{name} ps={ps} D={dim}: device {dev / 400 * 1e3:.1f} us/iter, host enqueue {host / 400 * 1e6:.1f} us/iter")
    run.close()

# the update kernel's share (apo_run_profile: events around the update launch only)
for name, ps, dim in (("cec2022_f1", 10000, 10), ("rosenbrock", 10000, 10), ("cec2022_f1", 1000, 10)):
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=420, seed=0)
    run = DeviceRun(cfg, pz.get_objective(name))
    run.initialize()
    run.iterate(20)
    run.profile(True)
    run.iterate(200)
    torch.cuda.synchronize()
    ms, n = run.profile_read()
    print(f"{name} ps={ps} D={dim}: update {ms / n * 1e3:.1f} us/iter over {n} iterations ({run.update_path()})")
    run.close()
