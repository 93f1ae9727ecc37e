"""Pin systematic slices (records i ≡ 0 mod stride) of the N=16..23 frontiers: node count
and weighted total, computed with the C oracle (multi-threaded) on the slice the
REFERENCE's own generator picks (oracle/_ref, for_each_subproblem), its total
cross-checked against the reference build's execute_batch. These are the bench's
CPU-baseline samples and the independent node-count pins of the large-N GPU tests
(tests/test_gpu_parity.py::test_bench_samples_rederived_on_device, ::test_large_n_slices).

    python tests/golden/make_bench_samples.py
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle_ctypes import Oracle, Reference, reference_available  # noqa: E402
from paper_2511_12009_b200 import nqueens as nq  # noqa: E402

PLANS = [(20, 6, 256), (20, 6, 128), (20, 7, 256), (20, 7, 128), (20, 8, 256), (20, 8, 128), (18, 6, 16), (16, 5, 1),
         (21, 7, 1000), (22, 7, 10000), (23, 7, 100000)]


def main():
    o = Oracle()
    path = os.path.join(HERE, "bench_samples.json")
    out = json.load(open(path)) if os.path.exists(path) else {}
    for n, r, stride in PLANS:
        key = f"{n},{r},{stride}"
        if key in out:
            continue
        s = nq.generate_slice(n, r, stride, 0)
        if reference_available():
            assert (Reference().generate_slice(n, r, stride, 0) == s).all()
        total, nodes = o.solve_batch(n, s)
        if reference_available() and len(s) < 100000:
            assert Reference().execute_batch(n, r, s, workers=os.cpu_count())[0] == total
        out[key] = {"records": len(s), "nodes": nodes, "total": total}
        print(key, out[key], flush=True)
        json.dump(out, open(path, "w"), indent=1)


if __name__ == "__main__":
    main()
