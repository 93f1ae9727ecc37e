# GPU parity tests, smoke, one bench line (N=20, default R), and the launch list.
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 600 python bench.py ${BENCH_ARGS} > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_gpu.log gpurun_out/smoke.log gpurun_out/bench.json; tail -5 gpurun_out/bench.err
