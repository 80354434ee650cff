#!/bin/bash
mkdir -p gpurun_out
timeout 900 python bench.py --no-suite --no-cpu --steps 5 > gpurun_out/bench_lean.json 2> gpurun_out/bench_lean.err
python -c "import json;d=json.load(open('gpurun_out/bench_lean.json'));print('e2e',d['e2e']['value'],d['e2e']['step_ms'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_update_group -s 3 -c 1 -o gpurun_out/rosen python tools/prof_split.py rosenbrock > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/rosen.ncu-rep 30 > gpurun_out/c4_k_update_group_rosenbrock_r2.summary.txt 2>&1
ncu -i gpurun_out/rosen.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/rosen.src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/rosen.src.csv 40 > gpurun_out/c4_k_update_group_rosenbrock_r2.lines.txt 2>&1
rm -f gpurun_out/rosen.src.csv gpurun_out/*.ncu-rep
head -30 gpurun_out/c4_k_update_group_rosenbrock_r2.summary.txt
