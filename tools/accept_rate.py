"""Fraction of protozoa whose fitness changed (accepted candidates) per iteration of the bench's C4 run
(ps = 1e6, D = 100, T = W + K = 13); not a bench value."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200.engine import DeviceRun

name = sys.argv[1] if len(sys.argv) > 1 else "cec2022_f6"
T = int(sys.argv[2]) if len(sys.argv) > 2 else 13
cfg = pz.ApoConfig(ps=1_000_000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=T, seed=0)
run = DeviceRun(cfg, pz.get_objective(name))
run.initialize()
prev = np.sort(run.population()[1])
for t in range(T):
    run.iterate(1)
    fit = run.population()[1]
    cur = np.sort(fit)
    # population() is in rank order of the last sort; compare as multisets is not enough -- use counts
    changed = np.count_nonzero(~np.isin(fit, prev))
    print(f"{name} t={t} changed {changed / fit.size:.3f}")
    prev = cur
