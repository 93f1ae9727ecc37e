set -x
mkdir -p gpurun_out
./tools/microbench/dfs_lab 18 6 3 > gpurun_out/lab_18_6.jsonl 2>&1
./tools/microbench/dfs_lab 20 7 1 > gpurun_out/lab_20_7.jsonl 2>&1
timeout 600 ncu --metrics l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,gpu__time_duration.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed --csv --log-file gpurun_out/lab_banks.csv ./tools/microbench/dfs_lab 18 6 1 > /dev/null 2>&1
cat gpurun_out/lab_*.jsonl
