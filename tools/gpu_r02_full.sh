#!/bin/bash
# Round-2 full pass: GPU suite, both bench arms, ncu launch list + full captures at N=20 R=7.
mkdir -p gpurun_out
lscpu | grep "Model name" > gpurun_out/r02_host.txt; nproc >> gpurun_out/r02_host.txt
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02_pytest_gpu.log
timeout 600 python bench.py --impl reference > gpurun_out/r02_bench_ref.json 2> gpurun_out/r02_bench_ref.err
timeout 600 python bench.py > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err
# launch list of the bench's kernel in its single-launch form (the streaming launch waits for
# host publishes, which ncu's serialised launches would block)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_launches.csv \
  python bench.py --single-launch --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-execute > gpurun_out/r02_launches_bench.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/r02_dfs_v4_n20_r7 python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 > gpurun_out/r02_ncu_v4.log 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/r02_dfs_planes_n20_r7 python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 --layout 1 > gpurun_out/r02_ncu_planes.log 2>&1
timeout 300 python tools/nqcount.py --n 20 --pre-rows 7 --reps 3 --layout 1 > gpurun_out/r02_planes_time.log 2>&1
