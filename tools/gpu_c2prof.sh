#!/bin/bash
O=gpurun_out/r02c2; mkdir -p $O
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_run_batch -c 1 -o $O/c2 python tools/prof_batch.py > /dev/null 2>&1
ncu -i $O/c2.ncu-rep --page source --csv --print-source cuda,sass > $O/c2.src.csv 2>/dev/null
python tools/ncu_lines.py $O/c2.src.csv 70 inst > $O/c2.inst.txt 2>&1
python tools/ncu_lines.py $O/c2.src.csv 40 > $O/c2.lines.txt 2>&1
rm -f $O/*.ncu-rep $O/*.src.csv
head -72 $O/c2.inst.txt
