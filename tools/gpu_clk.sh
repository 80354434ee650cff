#!/bin/bash
# per-phase cycle counts of the batch kernel (build_variants/clk.so, -DAPO_BATCH_CLOCK); not a bench value
for v in "0 4" "1 4" "1 32"; do
  set -- $v
  echo "LPP=$1 G=$2"
  APO_LIB=build_variants/clk.so APO_BATCH_LPP=$1 APO_BATCH_LPP_G=$2 python -c "
import sys; sys.path.insert(0,'.')
import paper_2510_14982_b200 as pz
import torch
for name, ps, dim in (('cec2022_f1', 50, 10), ('rosenbrock', 50, 10)):
    cfg = pz.ApoConfig(ps=ps, dim=dim, bounds=pz.Bounds(-100.0, 100.0, dim), max_iterations=1000, seed=0)
    print(name, ps, dim, flush=True)
    pz.run_batch(cfg, [name], [0])
    torch.cuda.synchronize()
" 2>&1 | grep -v "^$" | tail -12
done
