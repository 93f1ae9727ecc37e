#!/usr/bin/env python3
"""Projected wall time of a full N-Queens count from timed frontier slices (BASELINE
config 5: "N=27 timed frontier slices ... to project full 27/28-Queens wall time").

Method:
  1. systematic slice of the R-frontier: records with index ≡ o (mod K), for several
     offsets o (the frontier's cost rises with index, so a stride sample is stratified);
  2. each slice record is deepened on the host to depth D (nq_expand), so the slice
     becomes enough GPU-sized records (~10^5-10^7 nodes each) to keep every lane busy;
  3. the deepened slice is counted on one B200 with the product kernel (device-resident,
     CUDA-event kernel time);
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
import ctypes
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
    ap.add_argument("--layout", type=int, default=0)
    args = ap.parse_args()

    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq

    offsets = ([int(x) for x in args.offsets.split(",")] if args.offsets else
               [0, args.stride // 3, 2 * args.stride // 3])
    full = nq.count_subproblems(args.n, args.pre_rows)
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    _lib.check(_lib.lib.nq_ctx_set_layout(ctx, args.layout))
    rows = []
    for o in offsets:
        t0 = time.perf_counter()
        sl = nq.generate_slice(args.n, args.pre_rows, args.stride, o)
        deep = nq.expand(args.n, sl, args.deepen)
        gen_s = time.perf_counter() - t0
        dev = torch.from_numpy(deep.view(np.int32).reshape(-1, 4)).cuda()
        r = _lib.NqResult()
        _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.deepen, _lib.VARIANT_LASTROW,
                                            ctypes.c_void_p(dev.data_ptr()), len(deep),
                                            ctypes.byref(r)))
        rows.append({"offset": o, "slice_records": len(sl), "deepened_records": len(deep),
                     "host_gen_s": round(gen_s, 3), "kernel_ms": r.kernel_ms,
                     "nodes": r.nodes, "solutions": r.solutions,
                     "nodes_per_s": r.nodes / (r.kernel_ms * 1e-3)})
        print(json.dumps(rows[-1]), flush=True)
        del dev
    _lib.lib.nq_ctx_destroy(ctx)

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
