"""Generate tests/golden/*.json from the REFERENCE ITSELF (test infrastructure only).

Runs the unmodified reference headers compiled from /root/reference into
oracle/_ref/libnqref.so (oracle/Makefile) and records their outputs as fixtures, so the
GPU box — which has no /root/reference — can check parity against them.

    make -C oracle && python tests/golden/make_golden.py
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
from oracle_ctypes import Reference  # noqa: E402

# OEIS A000170; N=27 also subproblems.hpp:28.
OEIS_A000170 = [1, 0, 0, 2, 10, 4, 40, 92, 352, 724, 2680, 14200, 73712, 365596, 2279184,
                14772512, 95815104, 666090624, 4968057848, 39029188884, 314666222712,
                2691008701644, 24233937684440, 227514171973736, 2207893435808352,
                22317699616364044, 234907967154122528]

# Alg. 3 node counts (last-row loop iterations over the folded frontier), SURVEY.md
# Appendix B, computed there with the reference generator; N <= 16 re-derived by
# tests/test_oracle.py with the C restatement, N <= 20 by the GPU tests.
APPENDIX_B_NODES = {
    14: {5: 13463861, 6: 13343119, 7: 12925591},
    15: {5: 84372259, 6: 84140740, 7: 83191889},
    16: {5: 563126914, 6: 562707506, 7: 560708278},
    17: {5: 3960479916, 6: 3959755915, 7: 3955802368},
    18: {5: 29349696096, 6: 29348496950, 7: 29341087800},
    19: {5: 228485522213, 6: 228483606026, 7: 228470349555},
    20: {5: 1865473917695, 6: 1865470950135, 7: 1865448168709},
}


def recs(a: np.ndarray):
    return [[int(r["cols"]), int(r["diag"]), int(r["antidiag"]), int(r["row"])] for r in a]


def main():
    ref = Reference()
    out = {"source": "reference headers /root/reference/proj/include compiled by oracle/Makefile",
           "oeis_a000170": OEIS_A000170, "appendix_b_nodes": APPENDIX_B_NODES}

    # Frontier sizes (count_subproblems, subproblems.hpp:118) incl. the 27/7 anchor.
    sizes = {}
    for n in range(2, 28):
        for r in range(1, min(n, 9)):
            if n >= 24 and r > 7:
                continue
            sizes[f"{n},{r}"] = ref.count_subproblems(n, r)
    out["count_subproblems"] = sizes

    # Exact frontier records (generate, subproblems.hpp:110) for small plans.
    out["generate"] = {f"{n},{r}": recs(ref.generate(n, r))
                       for n, r in [(3, 1), (3, 2), (5, 1), (5, 2), (6, 3), (8, 3), (9, 2), (11, 3),
                                    (12, 4), (13, 2)]}

    # Export format bytes (write_batch, subproblems.hpp:169).
    out["write_batch"] = {f"{n},{r}": ref.write_batch(n, r) for n, r in [(5, 1), (5, 2), (14, 1), (9, 3)]}

    # Per-subproblem counts and high-water marks, all three reference kernels.
    per = {}
    for n in range(4, 13):
        for r in (1, 2, 3):
            if r >= n:
                continue
            a = ref.generate(n, r)
            it = [ref.count(0, n, rec) for rec in a]
            lr = [ref.count(1, n, rec) for rec in a]
            rc = [ref.count(2, n, rec)[0] for rec in a]
            per[f"{n},{r}"] = {"records": recs(a), "iterative": it, "lastrow": lr, "recursive": rc}
    out["per_subproblem"] = per

    # execute() totals through the reference scheduler (stealing, 4 workers, config1).
    tot = {}
    for n in range(2, 15):
        r = min(6, n - 1)
        a = ref.generate(n, r)
        t, _, processed = ref.execute_batch(n, r, a, workers=4, chunk=64)
        assert processed == len(a)
        tot[str(n)] = {"pre_rows": r, "total": t}
    out["execute_totals"] = tot

    path = os.path.join(HERE, "reference_golden.json")
    with open(path, "w") as f:
        json.dump(out, f, separators=(",", ":"))
    print(path, os.path.getsize(path), "bytes")


if __name__ == "__main__":
    main()
