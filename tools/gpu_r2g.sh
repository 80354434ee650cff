#!/bin/bash
mkdir -p gpurun_out
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
grep -E "^FAILED|passed|failed" gpurun_out/pytest_gpu.log | head -30
timeout 900 python bench.py --no-suite --no-cpu --steps 5 > gpurun_out/bench_lean.json 2> gpurun_out/bench_lean.err
python -c "import json;d=json.load(open('gpurun_out/bench_lean.json'));print('e2e',d['e2e']['value'],d['e2e']['step_ms'])"
