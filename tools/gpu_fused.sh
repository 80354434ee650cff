#!/bin/bash
mkdir -p gpurun_out
for f in cec2022_f6 cec2022_f10 cec2022_f1 cec2022_f12; do timeout 600 python tools/time_fused.py $f 10 3; done > gpurun_out/time_fused.txt 2>&1
cat gpurun_out/time_fused.txt
bash tools/gpu_tests.sh tests/test_headline_parity.py tests/test_reference_binding.py tests/test_shard.py tests/test_cec.py tests/test_resume.py
