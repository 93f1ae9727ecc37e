#!/bin/bash
# dfs_lab2: guarded / padded stack accesses vs the product step (timing + l1tex counters)
mkdir -p gpurun_out
./tools/microbench/dfs_lab2 18 6 3 > gpurun_out/r02_lab2_n18.jsonl 2>&1
./tools/microbench/dfs_lab2 20 7 2 > gpurun_out/r02_lab2_n20.jsonl 2>&1
M=l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,smsp__sass_inst_executed_op_shared_ld.sum,smsp__sass_inst_executed_op_shared_st.sum,smsp__inst_executed.sum,gpu__time_duration.sum,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --metrics $M --clock-control none --csv ./tools/microbench/dfs_lab2 18 6 1 > gpurun_out/r02_lab2_ncu_n18.csv 2>&1
