#!/bin/bash
mkdir -p gpurun_out
for f in rosenbrock sphere griewank; do timeout 120 python tools/prof_split.py $f; done > gpurun_out/split_basic.txt 2>&1
cat gpurun_out/split_basic.txt
timeout 900 python -m pytest -q -p no:cacheprovider -x tests/test_headline_parity.py -k basic tests/test_gpu_parity.py > gpurun_out/pytest_k.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_k.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_k.log | tail -3
