#!/bin/bash
for f in cec2022_f6 rosenbrock; do timeout 120 python tools/time_fused.py $f 10 3; done 2>&1 | grep -v "^$"
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -5
