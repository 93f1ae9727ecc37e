# Q(24) on one B200 across several gpurun calls: a checkpointed run (16 chunks) that
# stops itself before the call limit and resumes from runs/n24.ckpt on the next call.
mkdir -p gpurun_out
RES=""
if [ -f runs/n24.ckpt ]; then cp runs/n24.ckpt gpurun_out/n24.ckpt; RES="--resume"; fi
timeout 3510 python -m paper_2511_12009_b200.cli solve --n 24 --pre-rows 7 --workers 1 --config config1 \
  --checkpoint gpurun_out/n24.ckpt --checkpoint-chunk 9058722 --checkpoint-interval-s 0 \
  --stop-after-s 2750 --time-limit-s 3440 $RES --format json > gpurun_out/n24_call.json 2> gpurun_out/n24_call.log
echo "rc=$?" >> gpurun_out/n24_call.log
tail -3 gpurun_out/n24_call.log; grep -E '"total"|"completed"|"calc_ms"' gpurun_out/n24_call.json | head -3
grep -c "^done" gpurun_out/n24.ckpt
