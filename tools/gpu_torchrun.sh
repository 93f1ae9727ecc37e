# The multi-rank bench flow on a one-GPU box: 2 and 4 ranks sharing cuda:0 (gloo).
mkdir -p gpurun_out
for N in 2 4; do
  NQB_BENCH_SHARE_GPU=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N \
    --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus $N --steps 2 --warmup 1 \
    > gpurun_out/torchrun_$N.json 2> gpurun_out/torchrun_$N.err
  echo "N=$N rc=$?"; cat gpurun_out/torchrun_$N.json | cut -c1-600; tail -3 gpurun_out/torchrun_$N.err
done
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29512 \
  bench.py --impl reference --gpus 2 --steps 1 --warmup 1 > gpurun_out/torchrun_ref.json 2> gpurun_out/torchrun_ref.err
echo "ref rc=$?"; cut -c1-300 gpurun_out/torchrun_ref.json
