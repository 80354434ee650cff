#!/bin/bash
# A/B: update kernels without the npairs > 1 instantiation (-DAPO_NPAIRS1_ONLY)
for rep in 1 2; do
  python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
  APO_LIB=build_variants/np1.so python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
done
for lib in "" build_variants/np1.so; do
  APO_LIB=$lib python tools/c2_shapes.py "c2${lib:+_np1}:" | tail -1
  APO_LIB=$lib python tools/prof_c1.py 2>&1 | tail -1
done
