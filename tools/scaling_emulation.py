#!/usr/bin/env python3
"""Per-GPU work of a k-GPU run, measured on one B200.

The multi-GPU path has no inter-GPU traffic: under torchrun each rank counts the
stratified shard i ≡ rank (mod k) of the frontier on its own GPU and only two integers
are reduced at the end (bench.py). The k-GPU wall time is therefore the slowest rank's
kernel time. This tool times every rank's shard, one after another, on the single GPU
available and reports T_k = max over ranks and the implied strong-scaling efficiency
T_1 / (k · T_k) — what the driver's 1/2/4/8-GPU runs measure, minus launch/host noise.

    python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,2,4,8
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--balance", type=int, default=1)
    args = ap.parse_args()

    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq

    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    _lib.check(_lib.lib.nq_ctx_set_balance(ctx, args.balance))
    t1 = None
    rows = []
    for k in [int(x) for x in args.ks.split(",")]:
        times, sols, nodes = [], 0, 0
        for rank in range(k):
            shard = nq.generate_slice(args.n, args.pre_rows, k, rank)
            dev = torch.from_numpy(shard.view(np.int32).reshape(-1, 4)).cuda()
            best = None
            for _ in range(args.reps):
                r = _lib.NqResult()
                _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                    ctypes.c_void_p(dev.data_ptr()), len(shard),
                                                    ctypes.byref(r)))
                best = r if best is None or r.kernel_ms < best.kernel_ms else best
            times.append(best.kernel_ms)
            sols += best.solutions
            nodes += best.nodes
            del dev
        tk = max(times)
        if k == 1:
            t1 = tk
        row = {"k": k, "balance": args.balance, "per_rank_ms": [round(t, 3) for t in times], "T_k_ms": round(tk, 3),
               "rank_spread": round(max(times) / min(times), 4), "solutions": sols, "nodes": nodes,
               "nodes_per_s_k_gpus": nodes / (tk * 1e-3),
               "efficiency": (t1 / (k * tk)) if t1 else None}
        rows.append(row)
        print(json.dumps(row), flush=True)
    _lib.lib.nq_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
