#!/bin/bash
# batch-kernel rank sort (branch-free count): batch parity + C1/C2/C3 timing; not bench values
python -m pytest tests/test_gpu_parity.py tests/test_cec.py tests/test_threshold.py -q -x -m gpu -k "batch or full_runs or random_conf or suite or threshold" 2>&1 | tail -2
python tools/prof_c1.py 2>&1 | tail -1
python tools/prof_c1.py 100 20 1000 cec2022_f6 2>&1 | tail -1
python tools/c2_shapes.py 'c2:' 'c2b:'
python -c "
import sys; sys.path.insert(0, '.')
import bench
r = [bench.bench_c3() for _ in range(2)]
print('C3 ms', [round(x['ms'], 1) for x in r])
" 2>&1 | tail -1
