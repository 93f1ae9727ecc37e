mkdir -p gpurun_out
for spec in "7 batch" "7 expand" "8 batch" "8 expand"; do
  set -- $spec
  timeout 900 python bench.py --pre-rows $1 --e2e-mode $2 --no-cpu-baseline > gpurun_out/bm_$1_$2.json 2> gpurun_out/bm_$1_$2.err
  python -c "
import json; d=json.load(open('gpurun_out/bm_$1_$2.json')); print('$1 $2', round(d['ms_per_step'],1), '%.4e'%d['value'], '%.4e'%d['e2e']['value'], round(d['e2e']['ms_per_step'],1), d['e2e']['h2d_bytes_per_step'])" || tail -3 gpurun_out/bm_$1_$2.err
done
NQB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 2 --steps 2 --warmup 1 --pre-rows 8 --e2e-mode expand > gpurun_out/tr_exp.json 2> gpurun_out/tr_exp.err; echo "torchrun rc=$?"; cut -c1-300 gpurun_out/tr_exp.json; tail -2 gpurun_out/tr_exp.err
