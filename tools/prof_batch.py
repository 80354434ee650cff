"""C2-shape batch for ncu captures (never a bench value)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz

cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=1000)
names = list(pz.FUNCTION_NAMES) * 60
pz.run_batch(cfg, names, list(range(len(names))), want_trace=False, device_out=True)
torch.cuda.synchronize()
print("done")
