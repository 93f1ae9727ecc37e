#!/usr/bin/env python3
"""k-GPU runs of the product's dynamic dispatcher, emulated on ONE B200.

The multi-GPU path (nq_sched.cpp) has no inter-GPU traffic: each GPU runs one persistent
streaming launch that its host thread feeds with chunks from ONE guided dispenser
(nq_dispatch_*), and the per-GPU partials are summed on the host. This tool runs exactly
that code with k workers on device 0 (devices = [0] * k), each worker's launch capped at
8/k resident blocks per SM (NQB_BLOCKS_PER_SM) so that every worker owns 1/k of every SM:
k "virtual GPUs" of 1/k of a B200 each, fed by the real dispenser and feeders.

On one device the total hardware is fixed, so perfect balance gives T_k = T_1 and the
efficiency is T_1 / T_k, with T_k = the slowest worker's device span (CUDA events: first
operation -> end of its kernel). Caveat: when a virtual GPU runs dry its blocks leave
the SMs and the remaining workers' blocks get a larger share of each SM, which a real
idle GPU would not give them; the emulated end-phase imbalance is therefore a lower bound.

    python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,2,4,8            # 8 blocks/SM
    python tools/scaling_emulation.py --n 22 --pre-rows 7 --ks 1,7 --blocks 7     # 7 blocks/SM

--blocks must be the one-GPU occupancy of the workload (the stack depth sets it: 8 blocks
per SM at N=20 R=7, 7 at N=22 R=7), and k must divide it: otherwise one virtual GPU's
launch cannot be resident next to the others and only starts when one of them ends.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)


def one(n, r, k, reps, strategy):
    import numpy as np
    import torch
    from paper_2511_12009_b200 import nqueens as nq
    recs = nq.generate_packed(n, r)
    strat = nq.PartitionStrategy[strategy]
    weights = []
    if strat is nq.PartitionStrategy.weighted:  # the paper's 8-GPU weights
        w = list(nq.paper_gpu_weights)[:k]
        weights = [x / sum(w) for x in w] if k <= 8 else []
    chunk = 64 if strat is nq.PartitionStrategy.stealing else 0
    opts = nq.ExecuteOptions(config=nq.builtin_configs[0],
                             plan=nq.PartitionPlan(strat, k, weights, chunk),
                             devices=[0] * k)
    dev = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).cuda()
    best = None
    for _ in range(reps):
        rep = nq.execute_batch_device(n, r, [dev.data_ptr()] * k, len(recs), opts)
        span = max(w.span_ms for w in rep.workers)
        if best is None or span < best[0]:
            best = (span, rep)
    span, rep = best
    return {"k": k, "strategy": strategy, "T_k_ms": span,
            "spans_ms": [round(w.span_ms, 2) for w in rep.workers],
            "chunks": [w.chunks for w in rep.workers], "solutions": rep.total, "nodes": rep.nodes,
            "blocks_per_sm": int(os.environ.get("NQB_BLOCKS_PER_SM", "0"))}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--blocks", type=int, default=8, help="resident blocks per SM of one GPU")
    ap.add_argument("--strategy", default="guided",
                    choices=["guided", "stealing", "weighted", "uniform"],
                    help="weighted = the reference's default plan with the paper's 8-GPU weights")
    ap.add_argument("--child", type=int, default=0)
    args = ap.parse_args()
    if args.child:
        print(json.dumps(one(args.n, args.pre_rows, args.child, args.reps, args.strategy)))
        return
    t1 = None
    for k in [int(x) for x in args.ks.split(",")]:
        if args.blocks % k:
            raise SystemExit(f"k={k} does not divide --blocks {args.blocks}: the k launches "
                             f"would not all be resident at once")
        # enough hardware queues for k concurrent persistent launches on one device
        env = {**os.environ, "NQB_BLOCKS_PER_SM": str(max(1, args.blocks // k)),
               "CUDA_DEVICE_MAX_CONNECTIONS": "32"}
        out = subprocess.run([sys.executable, __file__, "--n", str(args.n), "--pre-rows",
                              str(args.pre_rows), "--reps", str(args.reps), "--child", str(k),
                              "--strategy", args.strategy],
                             capture_output=True, text=True, env=env, check=True).stdout
        row = json.loads(out.strip().splitlines()[-1])
        if k == 1:
            t1 = row["T_k_ms"]
        row["efficiency"] = t1 / row["T_k_ms"] if t1 else None
        row["virtual_gpu"] = f"1/{k} of every SM ({max(1, args.blocks // k)} blocks/SM)"
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
