#!/bin/bash
# instruction/stall profile of the C4 candidate kernel at a late iteration (90 of 100), cec2022_f6
O=gpurun_out/cand; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_update_group -s 90 -c 1 -o $O/late python tools/prof_c4.py cec2022_f6 92 > $O/ncu.log 2>&1
ncu -i $O/late.ncu-rep --page source --csv --print-source cuda,sass > $O/late.src.csv 2>/dev/null
python tools/ncu_lines.py $O/late.src.csv 70 inst > $O/late.inst.txt 2>&1
python tools/ncu_lines.py $O/late.src.csv 50 > $O/late.lines.txt 2>&1
python tools/ncu_summary.py $O/late.ncu-rep > $O/late.summary.txt 2>&1
rm -f $O/late.src.csv $O/late.ncu-rep
