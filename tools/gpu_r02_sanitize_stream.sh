mkdir -p gpurun_out
S=gpurun_out/r02_sanitize_race2.txt
: > $S
run() { local name=$1 tool=$2; shift 2
  timeout 900 compute-sanitizer --tool $tool --print-limit 20 "$@" > gpurun_out/r02_sanitize_${name}_${tool}.log 2>&1
  echo "$name $tool rc=$?" >> $S; tail -n 2 gpurun_out/r02_sanitize_${name}_${tool}.log >> $S; }
run guided racecheck python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 4 --partition guided --workers 2
run stealing racecheck python -m paper_2511_12009_b200.cli solve --n 12 --pre-rows 4 --partition stealing --workers 2 --chunk-size 64
run pinned racecheck python tools/pinned_smoke.py
run pinned memcheck python tools/pinned_smoke.py
NQB_DEVICE_EXPAND_MIN_RECORDS=0 run guided_deepen racecheck python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 6 --partition guided --workers 2
run guided synccheck python -m paper_2511_12009_b200.cli solve --n 13 --pre-rows 4 --partition guided --workers 2
cat $S
