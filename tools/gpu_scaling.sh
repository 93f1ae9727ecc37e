mkdir -p gpurun_out
timeout 900 python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,2,4,8 > gpurun_out/scaling_n20_r7.jsonl 2>&1
timeout 900 python tools/scaling_emulation.py --n 20 --pre-rows 8 --ks 1,8 > gpurun_out/scaling_n20_r8.jsonl 2>&1
timeout 900 python tools/scaling_emulation.py --n 18 --pre-rows 7 --ks 1,2,4,8 > gpurun_out/scaling_n18_r7.jsonl 2>&1
cat gpurun_out/scaling_*.jsonl
