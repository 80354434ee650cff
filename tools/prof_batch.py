"""C2 suite batch (CEC2022 F1-F12 x 30 seeds, D=20, ps=100, T=1000) for ncu captures (never a bench value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz

T = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
only = sys.argv[2] if len(sys.argv) > 2 else None
cfg = pz.ApoConfig(ps=100, dim=20, bounds=pz.Bounds(-100.0, 100.0, 20), max_iterations=T)
fns = [only] if only else [f"cec2022_f{k}" for k in range(1, 13)]
names = [n for n in fns for _ in range(30)]
pz.run_batch(cfg, names[:8], list(range(8)), want_trace=False, device_out=True)
torch.cuda.synchronize()
t0 = time.perf_counter()
pz.run_batch(cfg, names, list(range(len(names))), want_trace=False, device_out=True)
torch.cuda.synchronize()
print(f"{len(names)} runs x {T} iterations: {1e3 * (time.perf_counter() - t0):.1f} ms")
