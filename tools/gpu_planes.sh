set -x
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -s 1 -c 1 \
  -o gpurun_out/prof_dfs_planes_n18 python tools/nqcount.py --n 18 --pre-rows 6 --reps 2 --layout 1 > gpurun_out/ncu_planes.log 2>&1
python tools/nqcount.py --n 20 --pre-rows 7 --reps 2 --layout 1 > gpurun_out/planes_n20.json
python tools/nqcount.py --n 20 --pre-rows 7 --reps 2 --layout 0 > gpurun_out/v4_n20.json
cat gpurun_out/pytest_gpu.log gpurun_out/planes_n20.json gpurun_out/v4_n20.json
