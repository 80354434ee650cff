#!/bin/bash
# Full check of the tree: all GPU tests, smoke, the default bench line, the reference arm.
mkdir -p gpurun_out/final
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo "bench rc=$? seconds=$(( $(date +%s) - s ))" >> gpurun_out/final/bench.err
s=$(date +%s); timeout 900 python bench.py --impl reference > gpurun_out/final/bench_ref.json 2> gpurun_out/final/bench_ref.err; echo "ref rc=$? seconds=$(( $(date +%s) - s ))" >> gpurun_out/final/bench_ref.err
tail -3 gpurun_out/final/pytest_gpu.log; tail -2 gpurun_out/final/smoke.log
