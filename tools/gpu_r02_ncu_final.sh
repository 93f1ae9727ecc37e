#!/bin/bash
# ncu --set full of the final DFS kernel (contiguous form, the bench's N=1 launch) at the
# bench workload, V4 (default) and the zero-conflict plane layout.
mkdir -p gpurun_out
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/r02_final_dfs_v4_n20_r7 python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 > gpurun_out/r02_final_ncu_v4.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/r02_final_dfs_planes_n20_r7 python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 --layout 1 > gpurun_out/r02_final_ncu_planes.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_final_launches.csv \
  python bench.py --single-launch --steps 2 --warmup 3 --no-cpu-baseline --no-e2e --no-execute > gpurun_out/r02_final_launches_bench.log 2>&1
