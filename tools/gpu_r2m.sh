#!/bin/bash
mkdir -p gpurun_out
for v in 0 1; do for f in rosenbrock sphere griewank; do APO_BASIC_EVAL=$v timeout 120 python tools/prof_split.py $f; done; done 2>&1 | tee gpurun_out/split_basic2.txt
timeout 1200 python -m pytest -q -p no:cacheprovider -x tests/test_headline_parity.py tests/test_gpu_parity.py tests/test_shard.py > gpurun_out/pytest_m.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_m.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_m.log | tail -3
