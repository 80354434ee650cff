"""C1 latency breakdown: the one-CTA batch kernel alone (CUDA events) vs pz.run end to end (never a bench value)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import paper_2510_14982_b200 as pz

ps, dim, T = (int(a) for a in (sys.argv[1:4] if len(sys.argv) > 3 else (50, 10, 1000)))
name = sys.argv[4] if len(sys.argv) > 4 else "cec2022_f1"
cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=T, seed=0)
for _ in range(3):
    pz.run(cfg, name)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ks = []
for _ in range(5):
    e0.record()
    pz.run_batch(cfg, [name], [0], want_trace=True, device_out=True)
    e1.record()
    torch.cuda.synchronize()
    ks.append(e0.elapsed_time(e1))
ws = []
for _ in range(5):
    t0 = time.perf_counter()
    pz.run(cfg, name)
    ws.append(1e3 * (time.perf_counter() - t0))
print(f"ps={ps} D={dim} T={T} {name}: kernel {min(ks):.3f} ms ({1e3 * min(ks) / T:.2f} us/iter), "
      f"pz.run {min(ws):.3f} ms (median {sorted(ws)[2]:.3f})")
