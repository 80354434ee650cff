#!/bin/bash
# source-line stall/instruction profile of the batch kernel at C1 shape, LPP on (G=32) and off
O=gpurun_out/lpp; mkdir -p $O
for v in "1 32 rosenbrock" "0 4 rosenbrock" "1 32 cec2022_f1"; do
  set -- $v
  tag=lpp$1_g$2_$3
  APO_BATCH_LPP=$1 APO_BATCH_LPP_G=$2 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_run_batch -c 1 -o $O/$tag python tools/prof_c1.py 50 10 1000 $3 > /dev/null 2>&1
  ncu -i $O/$tag.ncu-rep --page source --csv --print-source cuda,sass > $O/$tag.src.csv 2>/dev/null
  python tools/ncu_lines.py $O/$tag.src.csv 50 > $O/$tag.lines.txt 2>&1
  python tools/ncu_lines.py $O/$tag.src.csv 50 inst > $O/$tag.inst.txt 2>&1
  ncu -i $O/$tag.ncu-rep --page details --csv > $O/$tag.details.csv 2>/dev/null
  rm -f $O/$tag.ncu-rep $O/$tag.src.csv
done
