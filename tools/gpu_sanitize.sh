# compute-sanitizer memcheck / racecheck / synccheck of the DFS kernel on small boards.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/nqcount.py --n 12 --pre-rows 4 --reps 1 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/nqcount.py --n 12 --pre-rows 4 --reps 1 --layout 1 > gpurun_out/sanitize_memcheck_planes.log 2>&1
echo "memcheck planes rc=$?" >> gpurun_out/sanitize_summary.txt; tail -2 gpurun_out/sanitize_memcheck_planes.log >> gpurun_out/sanitize_summary.txt
# execute() through the device-deepening path (coarse roots -> level passes -> count)
for tool in memcheck racecheck; do
  NQB_DEVICE_EXPAND_MIN_RECORDS=0 timeout 600 compute-sanitizer --tool $tool --print-limit 20 \
    python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 6 --partition strided --workers 2 \
    > gpurun_out/sanitize_expand_$tool.log 2>&1
  echo "expand $tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -2 gpurun_out/sanitize_expand_$tool.log >> gpurun_out/sanitize_summary.txt
done
make -s -C tests/cpp && ./tests/cpp/test_dropin gpu >> gpurun_out/sanitize_summary.txt 2>&1
cat gpurun_out/sanitize_summary.txt
