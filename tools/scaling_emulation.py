#!/usr/bin/env python3
"""k-GPU makespan of the product's GUIDED dispatcher, emulated on one B200.

The multi-GPU path (nq_sched.cpp) has no inter-GPU traffic: host threads (or one process
per GPU, torchrun) take guided chunks from ONE dispenser (nq_dispatch_*), each GPU counts
the chunks it takes, partials are summed on the host. A k-GPU run's time is therefore
set by the chunk sequence the dispenser hands out for W = k and by each chunk's time on
one GPU. This tool

  1. drains a dispenser created exactly as the scheduler creates it (count, guided,
     floor count/(128 k), W = k) to get the chunk sequence;
  2. times every chunk ALONE on the one GPU available (CUDA events; device-resident
     R-records for --mode records = bench.py's `value` path, or the chunk's coarse roots
     deepened on the device for --mode roots = execute()'s path);
  3. list-schedules the chunks onto k GPUs in dispenser order (each GPU takes the next
     chunk when its current one ends) and reports the makespan T_k and the strong-scaling
     efficiency T_1 / (k T_k).

Each chunk is timed with its own end-of-launch tail, which the scheduler's two launches
in flight per GPU hide, so T_k is conservative.

    python tools/scaling_emulation.py --n 20 --pre-rows 7 --ks 1,2,4,8 --mode records
"""
from __future__ import annotations

import argparse
import ctypes
import heapq
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def chunks_for(nq, count, k):
    with nq.Dispatcher.create(count, nq.PartitionStrategy.guided, 0, k) as d:
        out = []
        while (c := d.take()) is not None:
            out.append(c)
        return out


def makespan(times, k):
    """Greedy list scheduling in dispenser order onto k GPUs."""
    free = [0.0] * k
    heapq.heapify(free)
    for t in times:
        heapq.heappush(free, heapq.heappop(free) + t)
    return max(free)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--ks", default="1,2,4,8")
    ap.add_argument("--mode", default="records", choices=["records", "roots"])
    args = ap.parse_args()

    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq

    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    if args.mode == "records":
        recs = nq.generate_packed(args.n, args.pre_rows)
        dev = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).cuda()
        base = dev.data_ptr()
    else:
        coarse = max(2, args.pre_rows - 3)
        recs = nq.generate_packed(args.n, coarse)

    def time_chunk(f, n):
        r = _lib.NqResult()
        if args.mode == "records":
            _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                ctypes.c_void_p(base + 16 * f), n, ctypes.byref(r)))
            return r.kernel_ms, r.solutions, r.nodes
        part = np.ascontiguousarray(recs[f:f + n])
        torch.cuda.synchronize()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record()
        _lib.check(_lib.lib.nq_count_expand(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                            part.ctypes.data, n, ctypes.byref(r)))
        ev1.record()
        torch.cuda.synchronize()
        # the expand call runs on the context's own stream; bracket it on the host side
        return max(ev0.elapsed_time(ev1), r.kernel_ms), r.solutions, r.nodes

    time_chunk(0, min(len(recs), 4096))  # warm
    t1 = None
    for k in [int(x) for x in args.ks.split(",")]:
        seq = chunks_for(nq, len(recs), k)
        times, sols, nodes = [], 0, 0
        for f, n in seq:
            ms, s, nd = time_chunk(f, n)
            times.append(ms)
            sols += s
            nodes += nd
        tk = makespan(times, k)
        if k == 1:
            t1 = tk
        row = {"mode": args.mode, "n": args.n, "pre_rows": args.pre_rows, "k": k,
               "chunks": len(seq), "sum_chunk_ms": round(sum(times), 3), "T_k_ms": round(tk, 3),
               "ideal_ms": round(sum(times) / k, 3), "solutions": sols, "nodes": nodes,
               "nodes_per_s_k_gpus": nodes / (tk * 1e-3),
               "efficiency": (t1 / (k * tk)) if t1 else None,
               "largest_chunk_ms": round(max(times), 3), "last_chunks_ms": [round(t, 3) for t in times[-4:]]}
        print(json.dumps(row), flush=True)
    _lib.lib.nq_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
