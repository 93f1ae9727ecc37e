mkdir -p gpurun_out
timeout 800 python -m pytest tests/test_gpu_parity.py -q -k "expan or deepen" 2>&1 | tail -3
for spec in "7 batch" "7 expand" "8 expand"; do
  set -- $spec
  timeout 900 python bench.py --pre-rows $1 --e2e-mode $2 --no-cpu-baseline > gpurun_out/bm_$1_$2.json 2> gpurun_out/bm_$1_$2.err
  python -c "
import json; d=json.load(open('gpurun_out/bm_$1_$2.json')); print('$1 $2', round(d['ms_per_step'],1), '%.4e'%d['value'], '%.4e'%d['e2e']['value'], round(d['e2e']['ms_per_step'],1), d['e2e']['h2d_bytes_per_step'])" || tail -3 gpurun_out/bm_$1_$2.err
done
