#!/bin/bash
export TIME_VARIANTS='default:'
for f in cec2022_f6 rosenbrock; do timeout 120 python tools/time_fused.py $f 10 3; done 2>&1 | grep -v "^$"
python tools/c2_shapes.py 'c2:' 2>&1 | tail -1
python tools/prof_c1.py 2>&1 | tail -1
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -5
