set -x
mkdir -p gpurun_out
./tools/microbench/dfs_lab 18 6 3 > gpurun_out/lab_18_6.jsonl 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:lab_kernel -c 1 -o gpurun_out/prof_ad_n18 ./tools/microbench/dfs_lab 18 6 1 2 > gpurun_out/ncu_ad.log 2>&1
cat gpurun_out/lab_*.jsonl; tail -2 gpurun_out/ncu_ad.log
