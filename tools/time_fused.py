"""Per-iteration time of the C4 device loop for a few launch variants (env knobs), with a population
checksum so variants can be compared for agreement; not a bench value.

    python tools/time_fused.py cec2022_f6 [iters] [skip]     # one process per env setting (statics)
"""
import os
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

VARIANTS = [("split", {"APO_CEC_FUSED": "0"}),
            ("fused12", {"APO_CEC_FUSED": "1", "APO_FUSED_WARPS": "12"})]
if os.environ.get("TIME_VARIANTS"):  # e.g. TIME_VARIANTS='pf1:APO_CEC_PREFETCH=1;pf0:APO_CEC_PREFETCH=0'
    VARIANTS = [(lab, dict(kv.split("=", 1) for kv in rest.split(",") if kv))
                for lab, rest in (v.split(":", 1) for v in os.environ["TIME_VARIANTS"].split(";"))]


def one(name, iters, skip):
    import numpy as np
    import torch

    import paper_2510_14982_b200 as pz
    from paper_2510_14982_b200.engine import DeviceRun

    cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=25, seed=0)
    run = DeviceRun(cfg, pz.get_objective(name))
    run.initialize()
    run.iterate(skip)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    run.iterate(iters)
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / iters
    pos, fit = run.population()
    print(f"{name} ms/iter {ms:.3f}  best {fit.min():.15g}  fitsum {np.sum(fit):.15g}  possum {np.sum(pos[:1000]):.15g}")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--one":
        one(sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
        sys.exit(0)
    name = sys.argv[1] if len(sys.argv) > 1 else "cec2022_f6"
    iters = sys.argv[2] if len(sys.argv) > 2 else "10"
    skip = sys.argv[3] if len(sys.argv) > 3 else "3"
    for label, env in VARIANTS:
        out = subprocess.run([sys.executable, __file__, "--one", name, iters, skip], env={**os.environ, **env},
                             capture_output=True, text=True, timeout=600)
        print(f"{label:8s} {out.stdout.strip()} {out.stderr.strip()[-300:]}")
