#!/bin/bash
# Re-run of the k-GPU emulation after the streaming-kernel changes (bus-reader lock,
# queue view in shared memory) and the one-worker contiguous launch (k = 1 baseline).
mkdir -p gpurun_out
timeout 600 python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,2,4,8 --reps 3 > gpurun_out/r02_scaling_stream_v2.jsonl 2> gpurun_out/r02_scaling_stream_v2.err
timeout 1500 python tools/scaling_emulation.py --n 22 --pre-rows 7 --ks 1,7 --blocks 7 --reps 1 > gpurun_out/r02_scaling_stream_n22_v2.jsonl 2> gpurun_out/r02_scaling_stream_n22_v2.err
