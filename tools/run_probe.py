"""Phase timing of engine.run at the C4 shape (diagnosing e2e_run; not a bench value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=30, seed=0)
obj = pz.get_objective("cec2022_f6")
for rep in range(3):
    t = [time.perf_counter()]
    dr = DeviceRun(cfg, obj)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    dr.initialize()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    dr.iterate(30)
    torch.cuda.synchronize(); t.append(time.perf_counter())
    it, fe, w = dr.counters(); tr = dr.trace(it); b = dr.best()
    t.append(time.perf_counter())
    pos, fit = dr.population()
    t.append(time.perf_counter())
    dr.close()
    torch.cuda.synchronize(); t.append(time.perf_counter())
    names = ["create", "init", "iterate", "counters", "population", "close"]
    print(" ".join(f"{n} {1e3 * (t[i + 1] - t[i]):.1f}" for i, n in enumerate(names)), flush=True)
    t0 = time.perf_counter()
    pz.run(cfg, obj)
    print(f"pz.run {1e3 * (time.perf_counter() - t0):.1f} ms", flush=True)
