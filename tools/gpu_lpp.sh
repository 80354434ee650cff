#!/bin/bash
# lane-per-protozoon batch groups: parity of the batch paths + timing with APO_BATCH_LPP=0/1
python -m pytest tests/test_gpu_parity.py -q -x -m gpu -k "batch or full_runs or random_conf" 2>&1 | tail -3
python -m pytest tests/test_cec.py tests/test_threshold.py tests/test_philox.py -q -m gpu 2>&1 | tail -3
for v in 0 1; do
  export APO_BATCH_LPP=$v
  echo "LPP=$v"
  python tools/prof_c1.py 2>&1 | tail -1
  for d in 2 5 8; do python tools/prof_c1.py 100 $d 1000 rosenbrock 2>&1 | tail -1; done
  python -c "
import sys; sys.path.insert(0, '.')
import bench
r = [bench.bench_c3() for _ in range(2)]
print('C3 ms', [round(x['ms'], 1) for x in r])
" 2>&1 | tail -1
done
