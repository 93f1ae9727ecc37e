# Q(24) on one B200 through the CLI / execute() path (device-side deepening R=5 -> 8).
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/solve24_clocks_start.txt
timeout 14000 python -m paper_2511_12009_b200.cli solve --n 24 --pre-rows 8 --partition strided --workers 1 \
  --format json > gpurun_out/solve24.json 2> gpurun_out/solve24.log
echo "rc=$?" >> gpurun_out/solve24.log
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active --format=csv >> gpurun_out/solve24_clocks_end.txt
tail -3 gpurun_out/solve24.log; grep '"total"\|calc_ms\|"nodes"' gpurun_out/solve24.json | head -4
