"""Short C4 run for ncu captures: init + N iterations of ps=1M, D=100 (never a bench value)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

name = sys.argv[1] if len(sys.argv) > 1 else "rosenbrock"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 4
dim = int(sys.argv[3]) if len(sys.argv) > 3 else 100
cfg = pz.ApoConfig(ps=1_000_000, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=100, seed=0)
run = DeviceRun(cfg, pz.get_objective(name))
run.initialize()
run.iterate(n)
torch.cuda.synchronize()
print("done", run.counters())
