"""C4 shape on the Philox production stream: device-loop ms per iteration (CUDA events); not a bench value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

tag = os.environ.get("APO_LIB", "default").split("/")[-1]
for name in ("rosenbrock", "cec2022_f6"):
    cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=13, seed=0,
                       rng="philox")
    run = DeviceRun(cfg, pz.get_objective(name))
    run.initialize()
    run.iterate(3)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    run.iterate(10)
    e1.record()
    torch.cuda.synchronize()
    print(f"[{tag}] philox C4 {name}: {e0.elapsed_time(e1) / 10:.3f} ms/iter")
    run.close()
