# Round-end style check: GPU tests, smoke, bench (default), launch list of a bench run.
set -x
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -5 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 900 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 900 python bench.py --impl reference > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_bench.log 2>&1
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log; cut -c1-400 gpurun_out/bench.json; cut -c1-300 gpurun_out/bench_ref.json
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:nq_dfs_kernel -c 1 \
  -o gpurun_out/prof_dfs_n20_r7_final python tools/nqcount.py --n 20 --pre-rows 7 --reps 1 > gpurun_out/ncu20_final.log 2>&1
tail -1 gpurun_out/ncu20_final.log
