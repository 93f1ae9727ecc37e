#!/usr/bin/env python3
"""bench.py — N-Queens DFS nodes/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 20] [--pre-rows R]
    python bench.py --impl reference ...          # the reference's own CPU path
    torchrun --nproc-per-node N bench.py --gpus N # one process per GPU

A step = one pass of the counting path over the whole N=20 folded frontier (R=6:
2,967,560 packed records, 1.865e12 DFS nodes): the persistent sm_100a DFS kernel,
its count reduction and the 64-byte result read-back. Under torchrun each rank counts
the stratified shard i ≡ rank (mod world) of the frontier (no data-path collective;
one all_reduce of the per-rank counts and a max of the per-rank times at the end).

value  — device-resident frontier, CUDA-event time of the step on the launching stream.
e2e    — nq_solve_batch() (execute_batch's counterpart) with the frontier in pinned HOST
         memory: H2D copy + kernel + result D2H inside the timed region, wall clock.
roofline — integer-issue bound: achieved = nodes/s × 18 algorithmic int ops per node
            vs the int-op peak measured live on this GPU (LOP3+IMAD 1:1
           stream, nq_measure_int_peak).
cpu_baseline — the reference's execute_batch (oracle/_ref/libnqref.so, built from the
           unmodified reference headers) on a systematic slice of the same frontier
           with all host threads (rank 0, N=1 only).
"""
from __future__ import annotations

import argparse
import ctypes
import json
import os
import statistics
import subprocess
import sys
import threading
import time

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "N-Queens wall time & DFS nodes/sec at 1/2/4/8 B200 (N=20–23), bit-exact counts"
OEIS = {16: 14772512, 17: 95815104, 18: 666090624, 19: 4968057848, 20: 39029188884,
        21: 314666222712, 22: 2691008701644, 23: 24233937684440}
INT_OPS_PER_NODE = 18  # algorithmic int ops of the minimal last-row body


def ncu_traffic(n, pre_rows, world):
    """DRAM bytes (read + write) per launch of the DFS kernel for this workload, from the
    committed ncu capture (profiles/ncu_dram.json), or None when not captured."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_dram.json")) as f:
            d = json.load(f)
    except OSError:
        return None
    e = d.get(f"{n},{pre_rows},{world}")
    return None if e is None else e["dram_bytes_per_launch"]


def ncu_limits():
    """The binding resource of the DFS kernel per the committed ncu capture."""
    try:
        with open(os.path.join(REPO, "profiles", "ncu_limits.json")) as f:
            d = json.load(f)
    except OSError:
        return None
    return {"resource": d["binding_resource"], "frac": d["smem_wavefronts_pct_of_peak"] / 100,
            "alu_pipe_frac": d["alu_pipe_pct"] / 100, "source": d["capture"]}


def load_samples():
    with open(os.path.join(REPO, "tests", "golden", "bench_samples.json")) as f:
        return json.load(f)


# ---------------------------------------------------------------------------------------
def shard(records, rank, world):
    """This rank's stratified shard of the frontier: records i ≡ rank (mod world). The
    DFS order's cost rises with index, so striding balances ranks."""
    import numpy as np
    return np.ascontiguousarray(records[rank::world])


def reduce_over_ranks(pg, counts, times, device):
    """Σ of the integer counts and max of the times over ranks (pg = torch.distributed
    or None). The only cross-rank traffic of the bench: no data-path collective."""
    import torch
    cnt = torch.tensor([int(c) for c in counts], dtype=torch.int64, device=device)
    tmax = torch.tensor([float(t) for t in times], dtype=torch.float64, device=device)
    if pg is not None:
        pg.all_reduce(cnt)
        pg.all_reduce(tmax, op=pg.ReduceOp.MAX)
    return [int(x) for x in cnt.tolist()], [float(x) for x in tmax.tolist()]


def dist_env():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return world, rank, local


class Clocks:
    """nvidia-smi sampler during the timed region (B200_PROFILING.md clocks line)."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    if out:
                        self.samples.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)
        self._t = threading.Thread(target=run, daemon=True)
        self._t.start()

    def stop(self):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4)
                          if len(s) > 3 + i and s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.samples)}


# ---------------------------------------------------------------------------------------
def cpu_reference_sample(n, pre_rows, stride, threads):
    """The reference's execute_batch on records i ≡ 0 (mod stride): (calc_ms, total, len)."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from oracle_ctypes import Reference, reference_available, Oracle
    from paper_2511_12009_b200 import nqueens as nq  # frontier only (host C++ generator)
    sample = nq.generate_slice(n, pre_rows, stride, 0)
    if reference_available():
        ref = Reference()
        # Warm the host threads first (the first parallel region of a process pays
        # thread start-up and clock ramp: ~0.1-0.5 s on the box), then time the sample.
        warm = sample[:: max(1, len(sample) // 2048)]
        ref.execute_batch(n, pre_rows, warm, workers=threads, chunk=64, strategy=2, variant=1,
                          config_index=0)
        total, calc_ms, processed = ref.execute_batch(n, pre_rows, sample, workers=threads,
                                                      chunk=64, strategy=2, variant=1,
                                                      config_index=0)
        assert processed == len(sample)
        return calc_ms, total, len(sample), "reference"
    o = Oracle()  # the C restatement when the reference build is absent
    t0 = time.perf_counter()
    total, _ = o.solve_batch(n, sample, threads=threads, chunk=64)
    return (time.perf_counter() - t0) * 1e3, total, len(sample), "port"


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    samples = load_samples()
    key = f"{args.n},{args.pre_rows},{args.ref_stride}"
    if key not in samples:
        print(json.dumps({"impl": "reference",
                          "unavailable": f"no pinned node count for sample {key}"}))
        return 0
    nodes = samples[key]["nodes"]
    threads = os.cpu_count() or 1
    times = []
    total = None
    kind = "reference"
    for i in range(args.warmup + args.steps):
        ms, total, length, kind = cpu_reference_sample(args.n, args.pre_rows, args.ref_stride, threads)
        assert total == samples[key]["total"], (total, samples[key]["total"])
        if i >= args.warmup:
            times.append(ms)
    ms = sum(times) / len(times)
    v = nodes / (ms / 1e3)
    sample = (f"N={args.n} R={args.pre_rows} frontier records i%{args.ref_stride}==0 "
              f"({length} records, {nodes} nodes, total {total})")
    line = {"metric": METRIC, "value": v, "unit": "nodes/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (deterministic frontier)",
            "config": {"workload": f"N={args.n} R={args.pre_rows} full-frontier count",
                       "n": args.n, "pre_rows": args.pre_rows, "sample_stride": args.ref_stride},
            "cpu_baseline": {"value": v, "unit": "nodes/s", "cores": threads, "kind": kind,
                             "sample": sample},
            "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---------------------------------------------------------------------------------------
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--block", type=int, default=0)
    ap.add_argument("--blocks-per-sm", type=int, default=0)
    ap.add_argument("--order", type=int, default=1, help="1 = expensive end first")
    ap.add_argument("--ref-stride", type=int, default=256)
    ap.add_argument("--cpu-stride", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-mode", default="batch", choices=["batch", "expand"],
                    help="batch: nq_solve_batch on the host R-frontier shard; expand: the "
                         "coarse (R-3) frontier shard over PCIe, deepened on the device "
                         "(nq_count_expand)")
    args = ap.parse_args()
    world, rank, local = dist_env()
    if args.pre_rows is None:
        # R=7: 22.8 M finer subtrees keep every lane busy to the end (lane efficiency
        # 99.7% vs 97.9% at R=6, tools/microbench/dfs_lab.cu) and the shallower stack
        # fits one more block per SM.
        # R=7 at every world size: with the kernel's tail donation the slowest of 8
        # stratified shards runs at 99.4% of ideal (tools/scaling_emulation.py; 95.4%
        # without donation), and the shard is 8x smaller to ship than at R=8.
        args.pre_rows = 7 if args.n >= 19 else 6
    if args.impl == "reference":
        return run_reference_arm(args)

    import numpy as np
    import torch
    from paper_2511_12009_b200 import _lib
    from paper_2511_12009_b200 import nqueens as nq

    # NQB_BENCH_SHARE_GPU=1 (testing only): every rank on cuda:0 with gloo, so the
    # multi-rank flow (shards, barrier, reductions, rank-0 line) runs on a one-GPU box.
    share = os.environ.get("NQB_BENCH_SHARE_GPU") == "1"
    if share:
        local = 0
    torch.cuda.set_device(local)
    pg = None
    red_device = "cuda"
    if world > 1:
        import torch.distributed as dist
        if share:
            dist.init_process_group("gloo")
            red_device = "cpu"
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    # ---- inputs: this rank's stratified shard of the folded frontier, resident in HBM
    n_records = nq.count_subproblems(args.n, args.pre_rows)
    if world == 1:
        mine = nq.generate_packed(args.n, args.pre_rows)
    else:  # generate only this rank's stride (= shard(full, rank, world)), not the whole stream
        mine = nq.generate_slice(args.n, args.pre_rows, world, rank)
    host = torch.from_numpy(mine.view(np.int32).reshape(-1, 4)).pin_memory()
    dev = host.cuda()
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device="cuda")  # > 126 MB L2

    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(local, ctypes.byref(ctx)))
    _lib.check(_lib.lib.nq_ctx_set_tuning(ctx, args.block, args.blocks_per_sm, args.order))

    def step_device():
        r = _lib.NqResult()
        _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                            ctypes.c_void_p(dev.data_ptr()), len(mine),
                                            ctypes.byref(r)))
        return r

    dev_list = (ctypes.c_int * 1)(local)
    e2e_opts = _lib.NqSolveOpts()
    e2e_opts.variant = _lib.VARIANT_LASTROW
    e2e_opts.strategy = _lib.PARTITION_STRIDED
    e2e_opts.worker_count = 1
    e2e_opts.n_devices = 1
    e2e_opts.devices = dev_list

    coarse = max(2, args.pre_rows - 3)
    if args.e2e_mode == "expand":
        roots = nq.generate_slice(args.n, coarse, world, rank)
        host_roots = torch.from_numpy(roots.view(np.int32).reshape(-1, 4)).pin_memory()
        e2e_h2d_bytes = nq.count_subproblems(args.n, coarse) * 16
    else:
        e2e_h2d_bytes = n_records * 16

    def step_e2e():
        """Host inputs -> device -> count -> result read-back, every step. batch:
        execute_batch's GPU counterpart (nq_solve_batch) on this rank's host R-records;
        expand: this rank's coarse records, deepened and counted on the device."""
        if args.e2e_mode == "expand":
            r = _lib.NqResult()
            _lib.check(_lib.lib.nq_count_expand(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                ctypes.c_void_p(host_roots.data_ptr()), len(roots),
                                                ctypes.byref(r)))
            return r.solutions, r.nodes
        rep = _lib.NqReport()
        _lib.check(_lib.lib.nq_solve_batch(args.n, args.pre_rows, ctypes.c_void_p(host.data_ptr()),
                                           len(mine), ctypes.byref(e2e_opts), ctypes.byref(rep)))
        return rep.total, rep.nodes

    def barrier():
        torch.cuda.synchronize()
        if pg:
            pg.barrier()

    for _ in range(args.warmup):
        step_device()

    clocks = Clocks(local)
    clocks.start()
    barrier()
    dev_ms, nodes, sols = [], 0, 0
    res = None
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        res = step_device()
        dev_ms.append(res.kernel_ms)
        nodes += res.nodes
        sols += res.solutions
    barrier()
    clk = clocks.stop()
    t_dev = sum(dev_ms)

    e2e_ms = None
    if not args.no_e2e:
        step_e2e()
        barrier()
        t0 = time.perf_counter()
        e2e_nodes = 0
        e2e_sols = set()
        for _ in range(args.steps):
            sols_e2e, nodes_e2e = step_e2e()
            e2e_nodes += nodes_e2e
            e2e_sols.add(sols_e2e)
        barrier()
        e2e_ms = (time.perf_counter() - t0) * 1e3
        if len(e2e_sols) != 1:
            raise SystemExit(f"e2e counts differ between steps: {sorted(e2e_sols)}")

    # ---- cross-rank reduction: Σ counts, max time (host-side; 5 numbers per rank)
    e2e_sol = next(iter(e2e_sols)) if e2e_ms is not None else 0
    (nodes_all, sols_all, e2e_sol_all), (t_dev_max, e2e_max) = reduce_over_ranks(
        pg, [nodes, sols, e2e_sol], [t_dev, e2e_ms or 0.0], red_device)
    per_step_sols = sols_all // args.steps
    if args.n in OEIS and per_step_sols != OEIS[args.n]:
        raise SystemExit(f"count mismatch: {per_step_sols} != OEIS {OEIS[args.n]}")
    if e2e_ms is not None and e2e_sol_all != per_step_sols:
        raise SystemExit(f"e2e count mismatch: {e2e_sol_all} != {per_step_sols}")

    if rank != 0:
        if pg:
            pg.destroy_process_group()
        return 0

    value = nodes_all / (t_dev_max / 1e3)
    ops, mhz = nq.measure_int_peak(local)
    achieved = value * INT_OPS_PER_NODE
    line = {
        "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev_max / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (deterministic folded frontier; no dataset)",
        "config": {"workload": f"N={args.n} R={args.pre_rows} full-frontier count",
                   "n": args.n, "pre_rows": args.pre_rows, "records": n_records,
                   "solutions": per_step_sols, "nodes_per_step": nodes_all // args.steps,
                   "parallelism": f"stratified shard x{world}" if world > 1 else "1 GPU",
                   "l2": "flushed between steps (256 MiB write, untimed)",
                   "block": args.block or 128, "order": "expensive-first" if args.order else "stream"},
        "wall_ms": t_dev_max / args.steps,
        "gpu_launches": args.steps,
        "roofline": {"bound": "int", "achieved": achieved / 1e12, "peak": ops / 1e12,
                     "unit": "Tint-op/s", "frac": achieved / ops,
                     "traffic": ncu_traffic(args.n, args.pre_rows, world),
                     "peak_source": f"measured live on this GPU: LOP3+IMAD 1:1 int32 stream, "
                                    f"all SMs, {mhz:.0f} MHz (nq_measure_int_peak)",
                     "ops_per_node": INT_OPS_PER_NODE,
                     "algorithmic": f"{INT_OPS_PER_NODE} int ops per DFS node x "
                                    f"{nodes_all // args.steps} nodes per launch",
                     "binding_limit": ncu_limits()},
        "clocks": clk,
    }
    if e2e_ms is not None:
        line["e2e"] = {"value": nodes_all / (e2e_max / 1e3), "unit": "nodes/s",
                       "h2d_bytes_per_step": e2e_h2d_bytes, "d2h_bytes_per_step": 64 * world,
                       "mode": ("nq_count_expand: coarse R-3 frontier over PCIe, deepened on the device"
                                if args.e2e_mode == "expand" else
                                "nq_solve_batch (execute_batch) on the host R-frontier"),
                       "ms_per_step": e2e_max / args.steps}
    if world == 1 and not args.no_e2e:
        # BASELINE.md §3 wall time: one warm execute() — host generation of the frontier,
        # dispatch, the counting launch and the reduction — through nq_solve.
        rep = _lib.NqReport()
        for _ in range(2):  # the first call also maps the stream-ordered pool; report the second
            _lib.check(_lib.lib.nq_solve(args.n, args.pre_rows, ctypes.byref(e2e_opts), ctypes.byref(rep)))
        if args.n in OEIS and rep.total != OEIS[args.n]:
            raise SystemExit(f"execute() count mismatch: {rep.total}")
        line["execute_wall_ms"] = {"generation_ms": rep.generation_ms, "calc_ms": rep.calc_ms,
                                   "total_ms": rep.generation_ms + rep.calc_ms,
                                   "call": "nq_solve (execute): generate + H2D + count + D2H"}
    if world == 1 and not args.no_cpu_baseline:
        samples = load_samples()
        key = f"{args.n},{args.pre_rows},{args.cpu_stride}"
        if key in samples:
            threads = os.cpu_count() or 1
            ms, total, length, kind = cpu_reference_sample(args.n, args.pre_rows, args.cpu_stride, threads)
            assert total == samples[key]["total"]
            line["cpu_baseline"] = {
                "value": samples[key]["nodes"] / (ms / 1e3), "unit": "nodes/s", "cores": threads,
                "kind": kind,
                "sample": f"N={args.n} R={args.pre_rows} records i%{args.cpu_stride}==0 "
                          f"({length} records, {samples[key]['nodes']} nodes, {ms:.0f} ms)"}
    print(json.dumps(line))
    _lib.lib.nq_ctx_destroy(ctx)
    if pg:
        pg.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
