#!/bin/bash
# packed tail chunk in the candidates-only kernels: parity + C4 timing vs -DAPO_PACK_TAILS=0
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_cec.py tests/test_resume.py tests/test_shard.py tests/test_scripted.py tests/test_reference_binding.py -q -x -m gpu 2>&1 | tail -2
for rep in 1 2; do
  python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
  APO_LIB=build_variants/nopack.so python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2
done
for lib in "" build_variants/nopack.so; do
  for obj in cec2022_f6 rosenbrock; do
    APO_LIB=$lib python bench.py --objective $obj --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('${lib:-default}', '$obj', round(d['ms_per_step'],4), d['roofline']['kernel_ms_avg'], d['roofline']['frac'])"
  done
done
