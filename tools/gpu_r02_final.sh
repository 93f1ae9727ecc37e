#!/bin/bash
# Round-2 final pass: GPU suite, smoke, both bench arms, ncu launch list of the bench kernel.
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -n 30 > gpurun_out/r02_final_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_final_smoke.log 2>&1
timeout 600 python bench.py --impl reference > gpurun_out/r02_final_bench_ref.json 2> gpurun_out/r02_final_bench_ref.err
timeout 600 python bench.py > gpurun_out/r02_final_bench.json 2> gpurun_out/r02_final_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r02_final_launches.csv \
  python bench.py --single-launch --steps 2 --warmup 1 --no-cpu-baseline --no-e2e --no-execute --no-zero-conflict > gpurun_out/r02_final_launches.log 2>&1
