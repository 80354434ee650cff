"""Device-loop time per iteration at small populations (launch-overhead regime); not a bench value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

name = sys.argv[1] if len(sys.argv) > 1 else "cec2022_f6"
dim = int(sys.argv[2]) if len(sys.argv) > 2 else 100
ps = int(sys.argv[3]) if len(sys.argv) > 3 else 10_000
its = int(sys.argv[4]) if len(sys.argv) > 4 else 50
cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=1000, seed=0)
run = DeviceRun(cfg, pz.get_objective(name))
run.initialize()
run.iterate(5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
import time
e0.record()
h0 = time.perf_counter()
run.iterate(its)
host = (time.perf_counter() - h0) * 1e3 / its
e1.record()
torch.cuda.synchronize()
print(f"{name} D={dim} ps={ps}: {e0.elapsed_time(e1) / its:.4f} ms per iteration (host enqueue {host:.4f} ms)")
run.close()
