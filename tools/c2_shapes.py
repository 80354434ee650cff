"""C2 suite (CEC2022 F1-F12 x 30 seeds, D=20, ps=100, T=1000) under launch-shape overrides
(APO_BATCH_THREADS / APO_BATCH_WORKERS, one process each); not a bench value.

    python tools/c2_shapes.py 'default:' 't128w592:APO_BATCH_THREADS=128,APO_BATCH_WORKERS=592' ...
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import bench

    r = bench.bench_suite(1)
    print(f"ms {r['ms']:.1f} all {r['ms_all']} evals/s {r['value']:.3e}")
    sys.exit(0)
for spec in sys.argv[1:]:
    label, rest = spec.split(":", 1)
    env = dict(kv.split("=", 1) for kv in rest.split(",") if kv)
    out = subprocess.run([sys.executable, __file__, "--one"], env={**os.environ, **env}, capture_output=True,
                         text=True, timeout=600)
    print(f"{label:12s} {out.stdout.strip()} {out.stderr.strip()[-200:]}")
