#!/bin/bash
# cost of the scripted-draw branch in uniform(Key): default build vs -DAPO_NO_RNG_TABLE, interleaved
for rep in 1 2; do
  python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
  APO_LIB=build_variants/notable.so python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
done
python -m pytest tests/test_scripted.py -q -m gpu 2>&1 | tail -2
python -m pytest tests/test_philox.py tests/test_reference_binding.py -q -m gpu 2>&1 | tail -2
