#!/bin/bash
# k_basic_eval_direct loads in flight per lane: unroll 4 (default) / 8 / 16 on the C4 rosenbrock line
for rep in 1 2; do
  for lib in "" build_variants/u8.so build_variants/u16.so; do
    APO_LIB=$lib python bench.py --objective rosenbrock --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-u4}', round(d['ms_per_step'],4))"
  done
done
