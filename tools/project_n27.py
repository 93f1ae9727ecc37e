#!/usr/bin/env python3
"""Projected wall time of a full N-Queens count from timed frontier slices (BASELINE
config 5: "N=27 timed frontier slices ... to project full 27/28-Queens wall time").

Method:
  1. systematic slice of the R-frontier: records with index ≡ o (mod K), for several
     offsets o (the frontier's cost rises with index, so a stride sample is stratified);
  2-3. the slice is counted through the product's scheduler call a user makes,
     execute_batch_expand (nq_solve_batch_expand): guided chunks of the slice's records
     are shipped to the GPU, deepened there to depth D (so the slice becomes enough
     GPU-sized records, ~10^5-10^7 nodes each, to keep every lane busy) and counted;
     time = the scheduler's device span (CUDA events, first launch -> last kernel end),
     the host wall time of the call is reported beside it;
  4. projection: T_full(1 GPU) = T_slice * K (each sampled record's subtree is counted
     completely), T_full(G GPUs) = T_full(1 GPU) / G (the scheduler's work split;
     no inter-GPU exchange). The spread over offsets is the error bar.
Also projects the total node count (nodes_slice * K) and, when the full answer is known
(OEIS), checks the scaled solution estimate.

    python tools/project_n27.py --n 27 --pre-rows 7 --stride 1000000 --deepen 11
    python tools/project_n27.py --n 21 --pre-rows 7 --stride 1000 --deepen 10   # validation
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

OEIS = {20: 39029188884, 21: 314666222712, 22: 2691008701644, 23: 24233937684440,
        24: 227514171973736, 25: 2207893435808352, 26: 22317699616364044,
        27: 234907967154122528}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=27)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--stride", type=int, default=1_000_000)
    ap.add_argument("--offsets", default="")
    ap.add_argument("--deepen", type=int, default=11)
    ap.add_argument("--gpus", type=int, default=8, help="GPU count the projection is quoted for")
    args = ap.parse_args()

    import numpy as np
    from paper_2511_12009_b200 import nqueens as nq

    offsets = ([int(x) for x in args.offsets.split(",")] if args.offsets else
               [0, args.stride // 3, 2 * args.stride // 3])
    full = nq.count_subproblems(args.n, args.pre_rows)
    opts = nq.ExecuteOptions(config=nq.builtin_configs[0],
                             plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 1), devices=[0])
    rows = []
    for o in offsets:
        t0 = time.perf_counter()
        sl = nq.generate_slice(args.n, args.pre_rows, args.stride, o)
        gen_s = time.perf_counter() - t0
        rep = nq.execute_batch_expand(args.n, args.deepen, sl, opts)
        dev_ms = max(w.span_ms for w in rep.workers)
        rows.append({"offset": o, "slice_records": len(sl),
                     "deepened_records": sum(w.processed for w in rep.workers),
                     "launches": sum(w.chunks for w in rep.workers),
                     "host_gen_s": round(gen_s, 3), "kernel_ms": dev_ms, "call_wall_ms": rep.calc_ms,
                     "nodes": rep.nodes, "solutions": rep.total,
                     "nodes_per_s": rep.nodes / (dev_ms * 1e-3),
                     "call": "execute_batch_expand (nq_solve_batch_expand), guided, 1 GPU"})
        print(json.dumps(rows[-1]), flush=True)

    k = args.stride
    t1 = [x["kernel_ms"] * 1e-3 * k for x in rows]           # full count on 1 GPU, s
    nodes = [x["nodes"] * k for x in rows]
    sols = [x["solutions"] * k for x in rows]
    out = {
        "n": args.n, "pre_rows": args.pre_rows, "frontier_records": full, "stride": k,
        "deepen_to": args.deepen, "offsets": offsets,
        "projected_nodes": statistics.mean(nodes),
        "projected_solutions": statistics.mean(sols),
        "projected_s_1gpu": statistics.mean(t1),
        "projected_s_1gpu_spread": [min(t1), max(t1)],
        f"projected_s_{args.gpus}gpu": statistics.mean(t1) / args.gpus,
        f"projected_days_{args.gpus}gpu": statistics.mean(t1) / args.gpus / 86400,
        "mean_nodes_per_s_1gpu": statistics.mean(x["nodes_per_s"] for x in rows),
        "slices": rows,
    }
    if args.n in OEIS:
        out["oeis"] = OEIS[args.n]
        out["solution_estimate_rel_err"] = out["projected_solutions"] / OEIS[args.n] - 1
    print(json.dumps(out))


if __name__ == "__main__":
    main()
