#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -8
python - <<'PY'
import sys, json
sys.path.insert(0, '.')
import bench
r = bench.bench_c3()
print('hist', json.dumps(r['histogram']), 'c3 ms', r['ms'])
r = bench.bench_c5(sizes=(10, 32, 50), fns=(1,))
for row in r['rows']: print(row['fn'], row['dim'], row['rotation'], row['ms_per_iteration'])
PY
