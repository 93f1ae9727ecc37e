#!/usr/bin/env python3
"""Kernel time vs device span of one guided (streaming) count and one contiguous count
of the same device-resident frontier (the streaming path's intrinsic overhead), e.g.
under ncu: python tools/span_probe.py --n 20 --pre-rows 7 --iters 1"""
import argparse
import ctypes
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--iters", type=int, default=4)
    ap.add_argument("--mode", default="both", choices=["both", "stream", "single"])
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq
    recs = nq.generate_packed(args.n, args.pre_rows)
    dev = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).cuda()
    o = nq.ExecuteOptions(config=nq.builtin_configs[0],
                          plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 1, [], 0), devices=[0])
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    for _ in range(args.iters):
        if args.mode in ("both", "stream"):
            t0 = time.perf_counter()
            # an explicit dispenser: one worker without one gets the contiguous launch
            o.dispatch = nq.Dispatcher.create(len(recs), nq.PartitionStrategy.guided, 0, 1)
            rep = nq.execute_batch_device(args.n, args.pre_rows, [dev.data_ptr()], len(recs), o)
            o.dispatch.close()
            o.dispatch = None
            w = rep.workers[0]
            print(f"stream: kernel_ms {w.kernel_ms:.2f} span_ms {w.span_ms:.2f} "
                  f"wall {(time.perf_counter() - t0) * 1e3:.2f} chunks {w.chunks}", flush=True)
        if args.mode in ("both", "single"):
            r = _lib.NqResult()
            _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                ctypes.c_void_p(dev.data_ptr()), len(recs),
                                                ctypes.byref(r)))
            print(f"single: kernel_ms {r.kernel_ms:.2f}", flush=True)
    _lib.lib.nq_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
