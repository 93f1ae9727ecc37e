#!/bin/bash
# Streaming-launch overhead probe: kernel time of the guided (streaming) launch vs the
# contiguous launch of the same device-resident frontier, then the same with the
# probe build's per-warp counters (-DNQB_STREAM_STATS).
set -x
mkdir -p gpurun_out
for cfg in "18 6" "18 7" "20 7" "20 8"; do
  set -- $cfg
  echo "n=$1 R=$2" | tee -a gpurun_out/r02_stream_probe.log
  timeout 300 python tools/span_probe.py --n $1 --pre-rows $2 --iters 2 2>&1 | tee -a gpurun_out/r02_stream_probe.log
done
timeout 600 python -c "
from paper_2511_12009_b200 import _build as b
b.NVCC_FLAGS.append('-DNQB_STREAM_STATS'); b.build(force=True)"
for cfg in "18 6" "18 7" "20 8"; do
  set -- $cfg
  echo "stats n=$1 R=$2" | tee -a gpurun_out/r02_stream_probe.log
  timeout 300 python tools/span_probe.py --n $1 --pre-rows $2 --iters 1 --mode both 2>&1 | tee -a gpurun_out/r02_stream_probe.log
done
