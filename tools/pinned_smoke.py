#!/usr/bin/env python3
"""Small zero-copy run for compute-sanitizer: a pinned host batch counted in place through
nq_count (contiguous) and nq_solve_batch over two streaming workers on device 0."""
import ctypes
import sys

sys.path.insert(0, __file__.rsplit("/tools/", 1)[0])


def main():
    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq
    n, r = 12, 4
    recs = nq.generate_packed(n, r)
    pinned = torch.from_numpy(recs.view(np.int32).reshape(-1, 4).copy()).pin_memory()
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    res = _lib.NqResult()
    _lib.check(_lib.lib.nq_count(ctx, n, r, _lib.VARIANT_LASTROW, ctypes.c_void_p(pinned.data_ptr()),
                                 len(recs), ctypes.byref(res)))
    o = _lib.NqSolveOpts()
    o.variant = _lib.VARIANT_LASTROW
    o.strategy = _lib.PARTITION_GUIDED
    o.worker_count = 2
    devs = (ctypes.c_int * 2)(0, 0)
    o.devices = devs
    o.n_devices = 2
    rep = _lib.NqReport()
    _lib.check(_lib.lib.nq_solve_batch(n, r, ctypes.c_void_p(pinned.data_ptr()), len(recs),
                                       ctypes.byref(o), ctypes.byref(rep)))
    _lib.lib.nq_ctx_destroy(ctx)
    assert res.solutions == rep.total == 14200, (res.solutions, rep.total)
    print(f"pinned ok: nq_count {res.solutions}, nq_solve_batch x2 workers {rep.total}")


if __name__ == "__main__":
    main()
