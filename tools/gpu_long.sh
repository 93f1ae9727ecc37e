# N=21 projection validation, N=27 projection, then N=23 through the CLI (scheduler path).
mkdir -p gpurun_out
timeout 600 python tools/project_n27.py --n 21 --pre-rows 7 --stride 1000 --deepen 10 > gpurun_out/proj21.jsonl 2>&1
timeout 900 python tools/project_n27.py --n 27 --pre-rows 7 --stride 1000000 --deepen 11 > gpurun_out/proj27.jsonl 2>&1
tail -1 gpurun_out/proj21.jsonl; tail -1 gpurun_out/proj27.jsonl
timeout 2000 python -m paper_2511_12009_b200.cli solve --n 23 --pre-rows 7 --partition guided --format json > gpurun_out/solve23.json 2> gpurun_out/solve23.log
tail -3 gpurun_out/solve23.log; grep '"total"\|calc_ms\|nodes' gpurun_out/solve23.json | head -5
