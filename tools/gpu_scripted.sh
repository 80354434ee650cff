#!/bin/bash
# scripted draws (APO_RNG_TABLE) + the paths the extra uniform() branch touches; headline timing check
python -m pytest tests/test_scripted.py tests/test_reference_binding.py tests/test_abi.py -q -m gpu 2>&1 | tail -15
python -m pytest tests/test_gpu_parity.py tests/test_philox.py tests/test_resume.py -q -x -m gpu 2>&1 | tail -3
python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -4
