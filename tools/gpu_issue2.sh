#!/bin/bash
# ring row sources resolved once per group + u32 TMA addressing: device-loop parity + C4 timing
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_headline_parity.py tests/test_resume.py tests/test_shard.py tests/test_philox.py tests/test_cec.py -q -x -m gpu 2>&1 | tail -2
for rep in 1 2; do python tools/quick_timing.py rosenbrock cec2022_f6 2>&1 | tail -2; done
python bench.py --objective rosenbrock --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench rosenbrock', round(d['ms_per_step'],4))"
python bench.py --no-cpu --no-suite --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench f6', round(d['ms_per_step'],4))"
