# Profiles of the product DFS kernel: full ncu capture at N=18 (R=6), DRAM bytes of the
# bench workload (N=20, R=7), the launch list of one bench step, then a bench line.
set -x
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -s 1 -c 1 \
  -o gpurun_out/prof_dfs_n18 python tools/nqcount.py --n 18 --pre-rows 6 --reps 2 > gpurun_out/ncu_full.log 2>&1
timeout 900 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum --clock-control none \
  -k regex:nq_dfs_kernel -c 1 --csv --log-file gpurun_out/dram_n20_r7.csv python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 > gpurun_out/ncu_dram.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/ncu_bench.log 2>&1
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/bench.json; tail -3 gpurun_out/bench.err
