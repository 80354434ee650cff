#!/bin/bash
mkdir -p gpurun_out
export TIME_VARIANTS='pf0:APO_CEC_PREFETCH=0;pf1:APO_CEC_PREFETCH=1'
for f in cec2022_f6 cec2022_f10; do timeout 600 python tools/time_fused.py $f 10 3; done > gpurun_out/time_pf.txt 2>&1
cat gpurun_out/time_pf.txt
unset TIME_VARIANTS
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider -x > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -5 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 1200 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
tail -c 1500 gpurun_out/bench.err; head -c 400 gpurun_out/bench.json
