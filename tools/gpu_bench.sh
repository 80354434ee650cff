#!/bin/bash
mkdir -p gpurun_out
export TIME_VARIANTS='epi0:APO_CEC_EPI=0;epi1:APO_CEC_EPI=1'
timeout 300 python tools/time_fused.py cec2022_f6 10 3 2>&1 | grep -v "^$"
unset TIME_VARIANTS
APO_CEC_EPI=1 timeout 900 python -m pytest -q -p no:cacheprovider tests/test_headline_parity.py -k "c4_device_loop or sweep" 2>&1 | tail -2
s=$(date +%s); timeout 1200 python bench.py > gpurun_out/bench_full.json 2> gpurun_out/bench_full.err; echo "bench rc=$? seconds=$(( $(date +%s) - s ))"
