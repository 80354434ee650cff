#!/bin/bash
C2_SUFFIX=_dmma python tools/c2_shapes.py 'c2_dmma:' 2>&1 | tail -1
C2_SUFFIX=_fma python tools/c2_shapes.py 'c2_fma:' 2>&1 | tail -1
C2_SUFFIX= python tools/c2_shapes.py 'c2_auto:' 2>&1 | tail -1
C2_DIM=10 C2_SUFFIX=_dmma python tools/c2_shapes.py 'c2d10_dmma:' 2>&1 | tail -1
C2_DIM=10 C2_SUFFIX=_fma python tools/c2_shapes.py 'c2d10_fma:' 2>&1 | tail -1
C2_DIM=50 C2_SUFFIX=_dmma python tools/c2_shapes.py 'c2d50_dmma:' 2>&1 | tail -1
C2_DIM=50 C2_SUFFIX=_fma python tools/c2_shapes.py 'c2d50_fma:' 2>&1 | tail -1
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
r = bench.bench_c5(sizes=(10, 20, 32, 50, 100), fns=(1, 4, 10))
for row in r['rows']: print(row['fn'], row['dim'], row['rotation'], row['ms_per_iteration'])
PY
