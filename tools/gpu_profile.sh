#!/bin/bash
# bench + launch list + ncu --set full of the C4 kernels, summarised on the box (reports stay there).
mkdir -p gpurun_out
OBJ=${1:-cec2022_f6}
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-suite > /dev/null 2>&1
python tools/launch_share.py gpurun_out/launches_c4.csv > gpurun_out/launches_c4.summary.txt 2>&1
for K in k_update_group k_cec_eval; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 3 -c 1 -o gpurun_out/$K python tools/prof_split.py $OBJ > /dev/null 2>&1
  python tools/ncu_summary.py gpurun_out/$K.ncu-rep 30 > gpurun_out/c4_${K}_$OBJ.summary.txt 2>&1
  ncu -i gpurun_out/$K.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$K.src.csv 2>/dev/null
  python tools/ncu_lines.py gpurun_out/$K.src.csv 40 > gpurun_out/c4_${K}_$OBJ.lines.txt 2>&1
  rm -f gpurun_out/$K.ncu-rep gpurun_out/$K.src.csv
done
ls -la gpurun_out
