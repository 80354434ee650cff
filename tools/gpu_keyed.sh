#!/bin/bash
# keyed-only hot kernels + Philox builds: every GPU test, then the C1/C2/C4 timings
timeout 2400 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -3
python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
python tools/c2_shapes.py "c2:" | tail -1
python tools/prof_c1.py 2>&1 | tail -1
