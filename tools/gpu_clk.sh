#!/bin/bash
# per-phase cycle counts of the batch kernel (build_variants/clk.so, -DAPO_BATCH_CLOCK); not a bench value
APO_LIB=build_variants/clk.so python -c "
import sys; sys.path.insert(0,'.')
import paper_2510_14982_b200 as pz
import torch
for name, ps, dim, thr in (('cec2022_f6', 100, 20, 0), ('cec2022_f6', 100, 20, 640), ('cec2022_f1', 100, 20, 640),
                           ('cec2022_f12', 100, 20, 640), ('cec2022_f1', 50, 10, 0)):
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=1000, seed=0)
    print(name, ps, dim, thr, flush=True)
    pz.run_batch(cfg, [name], [0], threads_per_run=thr)
    torch.cuda.synchronize()
" 2>&1 | grep -v "^$\|lpp warp" | tail -20
