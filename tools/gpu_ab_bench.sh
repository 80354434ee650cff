#!/bin/bash
# A/B of two builds on the bench's C4 lines (timed span of the schedule), interleaved
for rep in 1 2; do
  for lib in "" build_variants/head.so; do
    for obj in rosenbrock cec2022_f6; do
      APO_LIB=$lib python bench.py --objective $obj --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-new}', '$obj', round(d['ms_per_step'],4))"
    done
  done
done
