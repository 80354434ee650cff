"""Phase timing of the public step() path (host numpy population in/out); not a bench value."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz

name = sys.argv[1] if len(sys.argv) > 1 else "cec2022_f6"
ps = int(sys.argv[2]) if len(sys.argv) > 2 else 1_000_000
cfg = pz.ApoConfig(ps=ps, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=100, seed=0)
t0 = time.perf_counter()
pop = pz.initialize(cfg, name)
print(f"initialize {time.perf_counter() - t0:.3f} s")
for t in range(4):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pop = pz.step(pop, cfg, name, t)
    torch.cuda.synchronize()
    print(f"step {t}: {time.perf_counter() - t0:.3f} s")
