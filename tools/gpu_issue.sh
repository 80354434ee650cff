#!/bin/bash
# ring rows issued by lanes 0-3: device-loop parity (staged SEL kernels) + C4 timing vs the previous build
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_resume.py tests/test_shard.py -q -x -m gpu 2>&1 | tail -2
for rep in 1 2; do
  python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
  APO_LIB=build_variants/notable.so python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
done
