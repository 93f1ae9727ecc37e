# Bit-exact large-N counts on one B200 (device-resident frontier, kernel time).
mkdir -p gpurun_out
for spec in "21 7" "22 7"; do
  set -- $spec
  timeout 1500 python tools/nqcount.py --n $1 --pre-rows $2 --reps 1 >> gpurun_out/bigN.jsonl 2>&1
done
cat gpurun_out/bigN.jsonl
