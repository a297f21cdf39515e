#!/bin/bash
mkdir -p gpurun_out
cd "$(dirname "$0")" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o hashbench hashbench.cu && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o piperate piperate.cu && cd ..
./scripts/hashbench > gpurun_out/hashbench.txt 2>&1
./scripts/piperate > gpurun_out/piperate.txt 2>&1
timeout 300 ncu --metrics smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active,sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum,sm__cycles_elapsed.avg,smsp__cycles_active.avg,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio,smsp__average_warps_issue_stalled_wait_per_issue_active.ratio,smsp__average_warps_issue_stalled_not_selected_per_issue_active.ratio,smsp__average_warps_issue_stalled_dispatch_stall_per_issue_active.ratio,gpc__cycles_elapsed.avg.per_second,sm__inst_executed_pipe_fmaheavy.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_fmalite.avg.pct_of_peak_sustained_active -c 5 --csv ./scripts/hashbench > gpurun_out/hb_ncu.csv 2>&1
cat gpurun_out/hashbench.txt gpurun_out/piperate.txt
