#!/bin/bash
# round-2 evidence: bench line, launch list, ncu --set full of the C4 kernels + C2 batch, traffic.json
mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
timeout 1200 python bench.py > $O/bench.json 2> $O/bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_c4.csv python bench.py --steps 2 --warmup 1 --no-e2e --no-cpu --no-suite > /dev/null 2>&1
python tools/launch_share.py $O/launches_c4.csv > $O/launches_c4.summary.txt 2>&1
cap() {  # name kernel-regex objective
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 3 -c 1 -o $O/$1 python tools/prof_split.py $3 > /dev/null 2>&1
  python tools/ncu_summary.py $O/$1.ncu-rep 30 > $O/$1.summary.txt 2>&1
  ncu -i $O/$1.ncu-rep --page source --csv --print-source cuda,sass > $O/$1.src.csv 2>/dev/null
  python tools/ncu_lines.py $O/$1.src.csv 40 > $O/$1.lines.txt 2>&1
  rm -f $O/$1.src.csv
}
cap c4_k_update_group_cec2022_f6 k_update_group cec2022_f6
cap c4_k_cec_eval_cec2022_f6 k_cec_eval cec2022_f6
cap c4_k_cec_eval_cec2022_f10 k_cec_eval cec2022_f10
cap c4_k_update_group_rosenbrock k_update_group rosenbrock
cap c4_k_basic_eval_rosenbrock k_basic_eval rosenbrock
python tools/traffic_update.py c4:cec2022_f6=$O/c4_k_update_group_cec2022_f6.ncu-rep:cec2022_f6:3 \
  c4eval:cec2022_f6=$O/c4_k_cec_eval_cec2022_f6.ncu-rep:cec2022_f6:3 c4eval:cec2022_f10=$O/c4_k_cec_eval_cec2022_f10.ncu-rep:cec2022_f10:3 \
  c4:rosenbrock=$O/c4_k_update_group_rosenbrock.ncu-rep:rosenbrock:3 c4eval:rosenbrock=$O/c4_k_basic_eval_rosenbrock.ncu-rep:rosenbrock:3 > $O/traffic.log 2>&1
cp profiles/traffic.json $O/traffic.json
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_run_batch -c 1 -o $O/c2_batch python tools/prof_batch.py > /dev/null 2>&1
python tools/ncu_summary.py $O/c2_batch.ncu-rep 30 > $O/c2_batch.summary.txt 2>&1
rm -f $O/*.ncu-rep
ls -la $O; head -c 600 $O/bench.json; tail -3 $O/traffic.log
