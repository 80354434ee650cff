"""Small end-to-end exercise of every kernel family for compute-sanitizer (not a test of values)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2510_14982_b200 as pz
from paper_2510_14982_b200 import engine, imaging
from paper_2510_14982_b200.shard import ShardedRun

for name, ps, dim in [("rosenbrock", 300, 37), ("cec2022_f6", 700, 50), ("cec2022_f10", 300, 20),
                      ("cec2022_f1", 300, 150), ("griewank", 200, 300), ("cec2022_f12", 260, 120)]:
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=4, seed=1)
    engine.BATCH_PS_LIMIT = 256
    pz.run(cfg, name)                      # batch (if it fits) or device loop
    engine.BATCH_PS_LIMIT = 0
    pz.run(cfg, name)                      # device loop
    pop = pz.initialize(cfg, name)
    pz.step(pop, cfg, name, 0)             # reference-facing path
    if dim <= 256:
        sh = ShardedRun(cfg, name, virtual_world=3)
        sh.initialize()
        sh.iterate(2)
        sh.close()
for ps in (3000, 30000):                   # tile sort + merge prologue, CUB prologue (device loop)
    engine.BATCH_PS_LIMIT = 0
    pz.run(pz.ApoConfig(ps=ps, dim=5, bounds=pz.Bounds(-5.0, 5.0, 5), max_iterations=3, seed=2, pf_max=1.0), "sphere")
ccfg = pz.ApoConfig(ps=70_000, dim=5, bounds=pz.Bounds(-5.0, 5.0, 5), max_iterations=3, seed=1)
for name in ("rosenbrock", "cec2022_f4"):                   # step(): rank-chunked update + overlapped D2H
    pz.step(pz.initialize(ccfg, name), ccfg, name, 0)
# round 2: the lean step (fitness first, rows read through the sort's order, basic-objective split in
# dense mode), the one-kernel fused CEC2022 update (opt-in) and the verification entries
lcfg = pz.ApoConfig(ps=70_000, dim=40, bounds=pz.Bounds(-5.0, 5.0, 40), max_iterations=3, seed=3)
for name in ("rosenbrock", "griewank", "cec2022_f6"):
    pz.step(pz.initialize(lcfg, name), lcfg, name, 1)
os.environ["APO_CEC_FUSED"] = "1"
engine.BATCH_PS_LIMIT = 0
pz.run(pz.ApoConfig(ps=3000, dim=100, bounds=pz.Bounds(-100.0, 100.0, 100), max_iterations=3, seed=4), "cec2022_f10")
del os.environ["APO_CEC_FUSED"]
from paper_2510_14982_b200 import _lib  # noqa: E402

xs = torch.linspace(-700.0, 700.0, 4096, dtype=torch.float64, device="cuda")
ys = torch.empty_like(xs)
_lib.check(_lib.load().apo_debug_cos(_lib.ptr(xs), _lib.ptr(ys), xs.numel(), _lib.stream_handle()))
z = torch.rand(37, 100, dtype=torch.float64, device="cuda")
fz = torch.empty(37, dtype=torch.float64, device="cuda")
for variant in (0, 1):
    _lib.check(_lib.load().apo_debug_cec_basic(9, _lib.ptr(z), 37, 100, None, _lib.ptr(fz), variant, _lib.stream_handle()))
scfg = pz.ApoConfig(ps=16, dim=10, bounds=pz.Bounds(-5.0, 5.0, 10), max_iterations=3)
pz.run_batch(scfg, ["cec2022_f12", "sphere", "cec2022_f7"] * 60, list(range(180)))  # persistent claims
pz.run_batch(scfg, ["cec2022_f1"] * 4, list(range(4)), threads_per_run=64)        # explicit CTA size
img = (np.arange(64 * 64) % 251).astype(np.uint8).reshape(64, 64)
pz.apo_multithreshold(img, 3, "kapur", ps=40, iterations=5)
pz.run(pz.ApoConfig(ps=64, dim=8, bounds=pz.Bounds(-5.0, 5.0, 8), max_iterations=5, rng="philox"), "cec2022_f4")
# round 2, later: lane-per-protozoon batch groups (D <= 8) and scripted draws (APO_RNG_TABLE kernels)
pz.run_batch(pz.ApoConfig(ps=100, dim=5, bounds=pz.Bounds(-5.0, 5.0, 5), max_iterations=4),
             ["rosenbrock", "griewank", "sphere"] * 3, list(range(9)))
from paper_2510_14982_b200.rng import COORDINATOR_INDEX, DrawTable  # noqa: E402

tcfg = pz.ApoConfig(ps=64, dim=10, bounds=pz.Bounds(-5.0, 5.0, 10), max_iterations=5, seed=3)
counters = list(range(6)) + [8 + d for d in range(10)] + [(1 << 32) + j for j in range(10)] + [1 << 33, (1 << 33) + 1]
table = DrawTable.from_stream(3, 2, range(1, 65), counters)
table.scalars.update(DrawTable.from_stream(3, 2, [COORDINATOR_INDEX], range(0, 65)).scalars)
for name in ("rosenbrock", "cec2022_f6"):
    pz.step(pz.initialize(tcfg, name), tcfg, name, 1, draws=table)
torch.cuda.synchronize()
print("sanitize exercise done")
