mkdir -p gpurun_out
nproc; lscpu | grep "Model name"
timeout 1500 python tools/cpu_projection.py --spec 18:6:1 --spec 20:7:128 --spec 22:7:5000 --spec 23:7:50000 --reps 3 > gpurun_out/cpu_projection.jsonl 2>&1
cat gpurun_out/cpu_projection.jsonl
