# One GPU call: int-pipe microbench, block sweep, ncu full capture of the DFS kernel.
set -x
mkdir -p gpurun_out
./tools/microbench/intpeak > gpurun_out/intpeak.jsonl 2>&1
timeout 300 python tools/nqcount.py --n 18 --pre-rows 6 --sweep > gpurun_out/sweep18.jsonl 2>&1
timeout 300 python tools/nqcount.py --n 20 --pre-rows 6 --sweep --reps 1 > gpurun_out/sweep20.jsonl 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -s 1 -c 1 \
  -o gpurun_out/prof_dfs_n18 python tools/nqcount.py --n 18 --pre-rows 6 --reps 2 > gpurun_out/ncu_full.log 2>&1
cat gpurun_out/intpeak.jsonl gpurun_out/sweep18.jsonl gpurun_out/sweep20.jsonl; tail -3 gpurun_out/ncu_full.log
