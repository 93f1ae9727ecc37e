#!/usr/bin/env python3
"""Kernel time of one contiguous count whose records are read (a) from HBM and (b) straight
from pinned host memory over the bus (the kernel reads each 16-B record once, when a
lane starts it), e.g. python tools/zero_copy_probe.py --n 20 --pre-rows 7"""
import argparse
import ctypes
import sys
import time

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=7)
    ap.add_argument("--iters", type=int, default=3)
    args = ap.parse_args()
    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq
    recs = nq.generate_packed(args.n, args.pre_rows)
    host = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).pin_memory()
    dev = host.cuda()
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    for _ in range(args.iters):
        for name, ptr in (("hbm", dev.data_ptr()), ("pinned-host", host.data_ptr())):
            r = _lib.NqResult()
            t0 = time.perf_counter()
            _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                ctypes.c_void_p(ptr), len(recs), ctypes.byref(r)))
            wall = (time.perf_counter() - t0) * 1e3
            print(f"{name}: kernel_ms {r.kernel_ms:.2f} wall_ms {wall:.2f} solutions {r.solutions} "
                  f"nodes {r.nodes}", flush=True)
    _lib.lib.nq_ctx_destroy(ctx)


if __name__ == "__main__":
    main()
