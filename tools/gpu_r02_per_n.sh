#!/bin/bash
# Per-N table through execute() on one B200 (N=16..23) and the k-GPU emulation at the
# N whose one-GPU occupancy k divides (N=18/19: 8 blocks/SM; N=21: 7).
mkdir -p gpurun_out
timeout 900 python tools/per_n.py --ns 16,17,18,19,20,21,22 --reps 2 > gpurun_out/r02_per_n.jsonl 2> gpurun_out/r02_per_n.err
timeout 1500 python tools/per_n.py --ns 23 --reps 1 >> gpurun_out/r02_per_n.jsonl 2>> gpurun_out/r02_per_n.err
timeout 300 python tools/scaling_emulation.py --n 18 --pre-rows 6 --ks 1,2,4,8 --reps 3 > gpurun_out/r02_scaling_n18.jsonl 2>> gpurun_out/r02_per_n.err
timeout 300 python tools/scaling_emulation.py --n 19 --pre-rows 7 --ks 1,2,4,8 --reps 3 > gpurun_out/r02_scaling_n19.jsonl 2>> gpurun_out/r02_per_n.err
timeout 600 python tools/scaling_emulation.py --n 21 --pre-rows 7 --ks 1,7 --blocks 7 --reps 2 > gpurun_out/r02_scaling_n21.jsonl 2>> gpurun_out/r02_per_n.err
