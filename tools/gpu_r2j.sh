#!/bin/bash
mkdir -p gpurun_out
export TIME_VARIANTS='fused:APO_BASIC_SPLIT_MIN_DIM=0;split:APO_BASIC_SPLIT_MIN_DIM=33'
for f in rosenbrock sphere griewank hgbat; do timeout 300 python tools/time_fused.py $f 10 3; done > gpurun_out/time_bsplit.txt 2>&1
cat gpurun_out/time_bsplit.txt
unset TIME_VARIANTS
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_gpu.log | tail -5
