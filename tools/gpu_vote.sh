#!/bin/bash
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -2
bash tools/gpu_ab_bench.sh
python tools/c2_shapes.py "c2:" | tail -1
python tools/prof_c1.py 2>&1 | tail -1
