#!/bin/bash
mkdir -p gpurun_out
export TIME_VARIANTS='split:APO_CEC_FUSED=0;ws8:APO_CEC_FUSED=2,APO_WS_PRODUCERS=8;ws6:APO_CEC_FUSED=2,APO_WS_PRODUCERS=6;ws10:APO_CEC_FUSED=2,APO_WS_PRODUCERS=10;ws4:APO_CEC_FUSED=2,APO_WS_PRODUCERS=4'
for f in cec2022_f6 cec2022_f10; do timeout 300 python tools/time_fused.py $f 10 3; done > gpurun_out/time_ws.txt 2>&1
cat gpurun_out/time_ws.txt
unset TIME_VARIANTS
timeout 900 python -m pytest -q -p no:cacheprovider tests/test_headline_parity.py -k fused > gpurun_out/pytest_ws.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_ws.log
grep -E "^FAILED|passed|failed|rc=" gpurun_out/pytest_ws.log
