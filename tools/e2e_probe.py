"""Per-phase host timing of engine.step at the C4 shape (diagnosing e2e outliers; not a bench value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200 import engine

cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=40, seed=0)
orig_dev, orig_host = engine._to_device, engine._to_host
acc = {"h2d": 0.0, "d2h": 0.0}


def to_dev(arr, dev):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = orig_dev(arr, dev)
    torch.cuda.synchronize()
    acc["h2d"] += time.perf_counter() - t
    return out


def to_host(*ts):
    torch.cuda.synchronize()
    t = time.perf_counter()
    out = orig_host(*ts)
    acc["d2h"] += time.perf_counter() - t
    return out


engine._to_device, engine._to_host = to_dev, to_host
pop = pz.initialize(cfg, "cec2022_f6")
for it in range(30):
    acc["h2d"] = acc["d2h"] = 0.0
    t0 = time.perf_counter()
    pop = pz.step(pop, cfg, "cec2022_f6", it)
    dt = time.perf_counter() - t0
    print(f"step {it:2d}: {1e3 * dt:7.1f} ms  h2d {1e3 * acc['h2d']:6.1f}  d2h {1e3 * acc['d2h']:6.1f}  "
          f"pinned={pop.positions.base is not None}", flush=True)
print(torch.cuda.memory_stats().get("num_alloc_retries", 0), "alloc retries")
