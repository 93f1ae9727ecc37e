set -x
mkdir -p gpurun_out

./tools/microbench/dfs_lab 18 6 3 > gpurun_out/lab_18_6.jsonl 2>&1
./tools/microbench/dfs_lab 20 7 1 > gpurun_out/lab_20_7.jsonl 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/lab_*.jsonl
