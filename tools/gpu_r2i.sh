#!/bin/bash
mkdir -p gpurun_out
M=sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__issue_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,smsp__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__warp_issue_stalled_mio_throttle_per_warp_active.pct,smsp__warp_issue_stalled_short_scoreboard_per_warp_active.pct,smsp__warp_issue_stalled_math_pipe_throttle_per_warp_active.pct,smsp__warp_issue_stalled_wait_per_warp_active.pct,smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct
timeout 600 ncu --metrics $M --clock-control none -k regex:k_cec_eval -s 3 -c 1 --csv python tools/prof_split.py cec2022_f6 > gpurun_out/eval_smem_metrics.csv 2>&1
grep -E "k_cec_eval" gpurun_out/eval_smem_metrics.csv | awk -F'","' '{print $(NF-2), $(NF-1), $NF}'
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_run_batch -c 1 -o gpurun_out/c1 python tools/prof_c1.py > gpurun_out/prof_c1.log 2>&1
python tools/ncu_summary.py gpurun_out/c1.ncu-rep 30 > gpurun_out/c1_k_run_batch_r2.summary.txt 2>&1
ncu -i gpurun_out/c1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/c1.src.csv 2>/dev/null
python tools/ncu_lines.py gpurun_out/c1.src.csv 50 > gpurun_out/c1_k_run_batch_r2.lines.txt 2>&1
rm -f gpurun_out/c1.src.csv gpurun_out/*.ncu-rep
cat gpurun_out/prof_c1.log | tail -2; head -25 gpurun_out/c1_k_run_batch_r2.summary.txt
