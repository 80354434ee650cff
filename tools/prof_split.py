"""Per-kernel split of the C4 device loop (candidate kernel vs CEC evaluation kernel); not a bench value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

name = sys.argv[1] if len(sys.argv) > 1 else "cec2022_f6"
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 100
ps = int(sys.argv[3]) if len(sys.argv) > 3 else 1_000_000
rng = sys.argv[4] if len(sys.argv) > 4 else "keyed"
cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=100, seed=0, rng=rng)
run = DeviceRun(cfg, pz.get_objective(name))
run.initialize()
skip = int(sys.argv[5]) if len(sys.argv) > 5 else 3
run.iterate(skip)
torch.cuda.synchronize()
run.profile(True)
run.iterate(5)
a, b, n = run.profile_split()
print(f"{name} D={dim} ps={ps} rng={rng} from iteration {skip}: candidates {a / n:.3f} ms  evaluate {b / n:.3f} ms  per iteration")
