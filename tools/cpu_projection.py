#!/usr/bin/env python3
"""Reference CPU path timed on systematic frontier slices, projected to full counts
("For N=20, 22 and 23, time the same fixed systematic frontier slices
... report the projected full time and label it projected").

Runs the UNMODIFIED reference execute_batch (oracle/_ref/libnqref.so: stealing, chunk
64, config1, lastrow, all host threads) on records i ≡ 0 (mod K) of the R-frontier;
projected full time = calc_ms × K. Median of `--reps` runs. Test/benchmark
infrastructure only (it loads the oracle build).

    python tools/cpu_projection.py --spec 20:7:128 --spec 22:7:5000 --spec 23:7:50000
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
sys.path.insert(0, os.path.join(REPO, "tests"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--spec", action="append", default=[], help="N:R:stride")
    ap.add_argument("--reps", type=int, default=3)
    args = ap.parse_args()
    from oracle_ctypes import Reference
    from paper_2511_12009_b200 import nqueens as nq

    ref = Reference()
    threads = os.cpu_count() or 1
    try:
        model = next(l.split(":", 1)[1].strip() for l in subprocess.run(
            ["lscpu"], capture_output=True, text=True).stdout.splitlines() if l.startswith("Model name"))
    except (StopIteration, OSError):
        model = "unknown"
    for spec in args.spec or ["20:7:128"]:
        n, r, k = map(int, spec.split(":"))
        sl = nq.generate_slice(n, r, k, 0)
        times, total = [], None
        for _ in range(args.reps):
            total, calc_ms, processed = ref.execute_batch(n, r, sl, workers=threads, chunk=64,
                                                          strategy=2, variant=1, config_index=0)
            assert processed == len(sl)
            times.append(calc_ms)
        med = statistics.median(times)
        print(json.dumps({"n": n, "pre_rows": r, "stride": k, "slice_records": len(sl),
                          "slice_weighted_total": total, "calc_ms_median": med,
                          "calc_ms_runs": times, "projected_full_s": med * k / 1e3,
                          "projected_full_days": med * k / 1e3 / 86400, "threads": threads,
                          "cpu": model, "label": "projected"}), flush=True)


if __name__ == "__main__":
    main()
