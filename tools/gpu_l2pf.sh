#!/bin/bash
timeout 900 python -m pytest tests/test_headline_parity.py tests/test_cec.py -q -x -m gpu 2>&1 | tail -1
for rep in 1 2; do
  for lib in "" build_variants/nopf.so; do
    for obj in cec2022_f6 cec2022_f10; do
      APO_LIB=$lib python bench.py --objective $obj --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-new}', '$obj', round(d['ms_per_step'],4), d['roofline']['kernel_ms_avg'])"
    done
  done
done
