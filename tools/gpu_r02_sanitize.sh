# compute-sanitizer on the round-2 streaming path: guided dispatch (one streaming launch
# per worker fed through mapped host memory), with and without device deepening, and the
# stealing feeder; plus the contiguous kernel as before, and a pinned host batch read in
# place by the kernel (zero-copy) through nq_count and two streaming workers.
mkdir -p gpurun_out
S=gpurun_out/r02_sanitize_summary.txt
: > $S
run() {  # name, tool, command...
  local name=$1 tool=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 "$@" > gpurun_out/r02_sanitize_${name}_${tool}.log 2>&1
  echo "$name $tool rc=$?" >> $S
  tail -n 2 gpurun_out/r02_sanitize_${name}_${tool}.log >> $S
}
for tool in memcheck racecheck synccheck; do
  run contiguous $tool python tools/nqcount.py --n 12 --pre-rows 4 --reps 1
  run guided $tool python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 4 --partition guided --workers 2
  run stealing $tool python -m paper_2511_12009_b200.cli solve --n 12 --pre-rows 4 --partition stealing --workers 2 --chunk-size 64
done
for tool in memcheck racecheck; do
  run pinned $tool python tools/pinned_smoke.py
  NQB_DEVICE_EXPAND_MIN_RECORDS=0 run guided_deepen $tool python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 6 --partition guided --workers 2
done
cat $S
