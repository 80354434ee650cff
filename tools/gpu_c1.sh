#!/bin/bash
for t in 256 384 512 640; do echo "threads=$t"; APO_BATCH_THREADS=$t python tools/prof_c1.py 2>&1 | tail -1; done
for t in 512 640; do echo "C2-like single run ps=100 D=20 threads=$t"; APO_BATCH_THREADS=$t python tools/prof_c1.py 100 20 1000 cec2022_f1 2>&1 | tail -1; done
