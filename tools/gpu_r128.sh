#!/bin/bash
# k_run_batch at 96 vs 128 registers (build_variants/r128.so), single-run shapes (512-thread CTA)
for lib in "" build_variants/r128.so; do
  echo "lib=${lib:-default}"
  export APO_LIB=$lib
  [ -z "$lib" ] && unset APO_LIB
  python tools/prof_c1.py 2>&1 | tail -1
  python tools/prof_c1.py 50 10 1000 rosenbrock 2>&1 | tail -1
  python tools/prof_c1.py 100 20 1000 cec2022_f6 2>&1 | tail -1
  python tools/prof_c1.py 100 5 1000 sphere 2>&1 | tail -1
done
