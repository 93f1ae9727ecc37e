# Validate and measure intra-warp tail donation (nq_ctx_set_balance).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q 2>&1 | tail -4 > gpurun_out/pytest_gpu.log
for b in 0 1; do
  timeout 600 python tools/nqcount.py --n 18 --pre-rows 6 --reps 3 --balance $b >> gpurun_out/donate_n18.jsonl 2>&1
  timeout 600 python tools/nqcount.py --n 18 --pre-rows 7 --reps 3 --balance $b >> gpurun_out/donate_n18.jsonl 2>&1
  timeout 600 python tools/nqcount.py --n 20 --pre-rows 7 --reps 2 --balance $b >> gpurun_out/donate_n20.jsonl 2>&1
  timeout 900 python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,8 --balance $b >> gpurun_out/donate_scaling.jsonl 2>&1
  timeout 900 python tools/scaling_emulation.py --n 18 --pre-rows 7 --ks 1,8 --balance $b >> gpurun_out/donate_scaling.jsonl 2>&1
done
cat gpurun_out/pytest_gpu.log
python - <<'PY'
import json
for f in ("gpurun_out/donate_n18.jsonl", "gpurun_out/donate_n20.jsonl"):
    for l in open(f):
        try: d = json.loads(l)
        except Exception: print(l.strip()); continue
        print(f.split("/")[-1], d["n"], d["pre_rows"], "balance", d["balance"], d["kernel_ms"], d["ok"])
for l in open("gpurun_out/donate_scaling.jsonl"):
    try: d = json.loads(l)
    except Exception: print(l.strip()); continue
    print("scaling", d["k"], "balance", d["balance"], d["T_k_ms"], d["efficiency"], d["solutions"])
PY
