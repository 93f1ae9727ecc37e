# compute-sanitizer memcheck / racecheck / synccheck of the DFS kernel on small boards.
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $tool --print-limit 20 python tools/nqcount.py --n 12 --pre-rows 4 --reps 1 > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> gpurun_out/sanitize_summary.txt
  tail -3 gpurun_out/sanitize_$tool.log >> gpurun_out/sanitize_summary.txt
done
timeout 600 compute-sanitizer --tool memcheck --print-limit 20 python tools/nqcount.py --n 12 --pre-rows 4 --reps 1 --layout 1 > gpurun_out/sanitize_memcheck_planes.log 2>&1
echo "memcheck planes rc=$?" >> gpurun_out/sanitize_summary.txt; tail -2 gpurun_out/sanitize_memcheck_planes.log >> gpurun_out/sanitize_summary.txt
make -s -C tests/cpp && ./tests/cpp/test_dropin gpu >> gpurun_out/sanitize_summary.txt 2>&1
cat gpurun_out/sanitize_summary.txt
