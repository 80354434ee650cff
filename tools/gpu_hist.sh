#!/bin/bash
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
r = bench.bench_c3()
print('hist', json.dumps(r['histogram']), 'c3 ms', r['ms'])
PY
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_threshold.py tests/test_netpbm.py -m gpu 2>&1 | tail -2
