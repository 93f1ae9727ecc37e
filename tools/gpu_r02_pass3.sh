#!/bin/bash
# Round-2 re-check after the last code changes: GPU suite, smoke, both bench arms, launch list.
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02d_smoke.log 2>&1; echo "smoke exit $?" >> gpurun_out/r02d_smoke.log
timeout 1500 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/r02d_pytest_gpu.log
timeout 600 python bench.py --impl reference > gpurun_out/r02d_bench_ref.json 2> gpurun_out/r02d_bench_ref.err
timeout 600 python bench.py > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err
