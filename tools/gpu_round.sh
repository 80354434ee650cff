#!/bin/bash
# One GPU call: gpu tests, smoke, bench, ncu launch list + full capture of the top kernel.
set -x
mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --objective cec2022_f6 --no-cpu --no-suite --no-e2e > gpurun_out/bench_f6.json 2> gpurun_out/bench_f6.err
timeout 600 python bench.py --objective cec2022_f10 --no-cpu --no-suite --no-e2e > gpurun_out/bench_f10.json 2> gpurun_out/bench_f10.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-suite > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/c4_update_rosen python tools/prof_c4.py rosenbrock 4 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update -s 3 -c 1 -o gpurun_out/c4_update_f6 python tools/prof_c4.py cec2022_f6 4 > gpurun_out/ncu_full_f6.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_run_batch -c 1 -o gpurun_out/c2_batch python tools/prof_batch.py > gpurun_out/ncu_batch.log 2>&1

# summarise captures on the box (reports are too large to bring back all of them)
for r in gpurun_out/*.ncu-rep; do
  b=${r%.ncu-rep}
  python tools/ncu_summary.py $r > $b.summary.txt 2>&1
  ncu -i $r --page raw --csv > $b.raw.csv 2>/dev/null
  ncu -i $r --page details --csv > $b.details.csv 2>/dev/null
  sz=$(stat -c %s $r); if [ $sz -gt 15000000 ]; then rm -f $r; fi
done
du -sh gpurun_out/*
echo done
