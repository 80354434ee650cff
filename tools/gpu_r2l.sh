#!/bin/bash
mkdir -p gpurun_out
for f in rosenbrock sphere griewank; do timeout 120 python tools/prof_split.py $f; done > gpurun_out/split_basic.txt 2>&1
cat gpurun_out/split_basic.txt
python tools/c2_shapes.py 'default:' 't128w592:APO_BATCH_THREADS=128,APO_BATCH_WORKERS=592' 't128:APO_BATCH_THREADS=128' 't192w444:APO_BATCH_THREADS=192,APO_BATCH_WORKERS=444' 't256w296:APO_BATCH_THREADS=256,APO_BATCH_WORKERS=296' 't320w296:APO_BATCH_THREADS=320,APO_BATCH_WORKERS=296' 2>&1 | tail -8
timeout 1200 python -m pytest -q -p no:cacheprovider -x tests/test_headline_parity.py tests/test_gpu_parity.py tests/test_shard.py tests/test_reference_binding.py > gpurun_out/pytest_l.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_l.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_l.log | tail -3
