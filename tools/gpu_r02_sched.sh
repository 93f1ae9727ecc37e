#!/bin/bash
# Round-2 scheduler pass: GPU suite, dispatcher emulation, N=27 projection via the product call.
set -x
mkdir -p gpurun_out
python -m pytest tests -m gpu -x -q 2>&1 | tail -20 > gpurun_out/r02_gputest.log
python tools/scaling_emulation.py --mode records --ks 1,2,4,8 > gpurun_out/r02_scaling_records.jsonl 2>&1
python tools/scaling_emulation.py --mode roots --ks 1,2,4,8 > gpurun_out/r02_scaling_roots.jsonl 2>&1
python tools/project_n27.py --n 21 --pre-rows 7 --stride 1000 --deepen 10 > gpurun_out/r02_projection_n21.jsonl 2>&1
python tools/project_n27.py --n 27 --pre-rows 7 --stride 1000000 --deepen 11 > gpurun_out/r02_projection_n27.jsonl 2>&1
