#!/bin/bash
mkdir -p gpurun_out
for f in cec2022_f6 cec2022_f10 cec2022_f1; do timeout 600 python tools/time_fused.py $f 10 3; done > gpurun_out/time_eval.txt 2>&1
cat gpurun_out/time_eval.txt
timeout 600 python tools/prof_split.py cec2022_f6 > gpurun_out/split_f6.txt 2>&1; cat gpurun_out/split_f6.txt
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_cec_eval -s 3 -c 1 -o gpurun_out/k_cec_eval python tools/prof_split.py cec2022_f6 > /dev/null 2>&1
python tools/ncu_summary.py gpurun_out/k_cec_eval.ncu-rep 30 > gpurun_out/c4_k_cec_eval_f6_r2.summary.txt 2>&1
ncu -i gpurun_out/k_cec_eval.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/k_cec_eval.src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/k_cec_eval.src.csv 40 > gpurun_out/c4_k_cec_eval_f6_r2.lines.txt 2>&1
rm -f gpurun_out/k_cec_eval.src.csv gpurun_out/*.ncu-rep
head -40 gpurun_out/c4_k_cec_eval_f6_r2.summary.txt
