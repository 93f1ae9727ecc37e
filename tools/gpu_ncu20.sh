mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/prof_dfs_n20_r7 python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 > gpurun_out/ncu20.log 2>&1
tail -2 gpurun_out/ncu20.log
