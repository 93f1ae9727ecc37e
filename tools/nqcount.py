#!/usr/bin/env python3
"""Run the device counting path on one configuration (tuning sweeps, ncu captures).

    python tools/nqcount.py --n 18 --pre-rows 6 [--block 128] [--bps 0] [--order 1]
                            [--reps 3] [--sweep]

Prints one JSON line per configuration: kernel ms (CUDA events on the launching
stream), nodes/s and nodes per SM-clock, with the total checked against OEIS.
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

OEIS = [1, 0, 0, 2, 10, 4, 40, 92, 352, 724, 2680, 14200, 73712, 365596, 2279184, 14772512,
        95815104, 666090624, 4968057848, 39029188884, 314666222712, 2691008701644,
        24233937684440, 227514171973736, 2207893435808352, 22317699616364044,
        234907967154122528]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=18)
    ap.add_argument("--pre-rows", type=int, default=6)
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--bps", type=int, default=0)
    ap.add_argument("--order", type=int, default=1)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--sweep", action="store_true", help="blocks x blocks-per-SM sweep")
    ap.add_argument("--variant", type=int, default=1)
    ap.add_argument("--layout", type=int, default=0, help="0 = uint4 frames, 1 = 32-bit planes")
    ap.add_argument("--balance", type=int, default=1, help="1 = intra-warp tail donation")
    args = ap.parse_args()

    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq

    subs = nq.generate_packed(args.n, args.pre_rows)
    dev = torch.from_numpy(subs.view(np.int32).reshape(-1, 4)).cuda()
    props = torch.cuda.get_device_properties(0)
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    _lib.check(_lib.lib.nq_ctx_set_layout(ctx, args.layout))
    _lib.check(_lib.lib.nq_ctx_set_balance(ctx, args.balance))
    configs = [(args.block, args.bps)]
    if args.sweep:
        configs = [(b, k) for b in (64, 96, 128, 192, 256) for k in (0,)]
    for block, bps in configs:
        _lib.check(_lib.lib.nq_ctx_set_tuning(ctx, block, bps, args.order))
        best = None
        for _ in range(args.reps):
            r = _lib.NqResult()
            _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, args.variant,
                                                ctypes.c_void_p(dev.data_ptr()), len(subs),
                                                ctypes.byref(r)))
            if best is None or r.kernel_ms < best.kernel_ms:
                best = r
        ok = args.n > len(OEIS) or best.solutions == OEIS[args.n - 1]
        rate = best.nodes / (best.kernel_ms * 1e-3)
        print(json.dumps({"n": args.n, "pre_rows": args.pre_rows, "block": block or 128,
                          "bps": bps, "order": args.order, "layout": args.layout, "balance": args.balance, "records": len(subs),
                          "solutions": best.solutions, "ok": ok, "nodes": best.nodes,
                          "iterations": best.iterations, "kernel_ms": round(best.kernel_ms, 3),
                          "nodes_per_s": rate,
                          "nodes_per_sm_clk_at_max": rate / (props.multi_processor_count * 1.965e9)}),
              flush=True)
        if not ok:
            sys.exit(f"count mismatch: {best.solutions} != {OEIS[args.n - 1]}")
    _lib.lib.nq_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
