"""C2 suite (CEC2022 F1-F12 x 30 seeds, D=20, ps=100, T=1000) under launch-shape overrides
(APO_BATCH_THREADS / APO_BATCH_WORKERS, one process each); not a bench value.

    python tools/c2_shapes.py 'default:' 't128w592:APO_BATCH_THREADS=128,APO_BATCH_WORKERS=592' ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import numpy as np
    import torch

    import paper_2510_14982_b200 as pz

    suffix = os.environ.get("C2_SUFFIX", "")  # "_fma": the lane-per-output FMA rotation instead of DMMA
    dim = int(os.environ.get("C2_DIM", "20"))
    cfg = pz.ApoConfig(ps=100, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=1000)
    names = [f"cec2022_f{k}{suffix}" for k in range(1, 13) for _ in range(30)]
    seeds = [s for _ in range(12) for s in range(30)]
    pz.run_batch(cfg, names[:24], seeds[:24], want_trace=False, device_out=True)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(3):
        e0.record()
        pz.run_batch(cfg, names, seeds, want_trace=False, device_out=True)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    print(f"ms {np.median(ts):.1f} all {[round(t, 1) for t in ts]}")
    sys.exit(0)
for spec in sys.argv[1:]:
    label, rest = spec.split(":", 1)
    env = dict(kv.split("=", 1) for kv in rest.split(",") if kv)
    out = subprocess.run([sys.executable, __file__, "--one"], env={**os.environ, **env}, capture_output=True,
                         text=True, timeout=600)
    print(f"{label:12s} {out.stdout.strip()} {out.stderr.strip()[-200:]}")
