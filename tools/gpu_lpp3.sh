#!/bin/bash
# C3 (thresholds, D=2..5) under APO_BATCH_LPP / APO_BATCH_LPP_G; not a bench value
for v in "0 32" "1 10" "1 16" "1 32"; do
  set -- $v
  APO_BATCH_LPP=$1 APO_BATCH_LPP_G=$2 python -c "
import sys; sys.path.insert(0, '.')
import bench
r = [bench.bench_c3() for _ in range(2)]
print('LPP=$1 G=$2 C3 ms', [round(x['ms'], 1) for x in r], r[-1]['best']['otsu_k3'])
" 2>&1 | tail -1
done
python -m pytest tests/test_threshold.py -q -m gpu 2>&1 | tail -2
