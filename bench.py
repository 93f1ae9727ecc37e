#!/usr/bin/env python3
"""bench.py — N-Queens DFS nodes/s on B200 (BASELINE.json metric), one JSON line.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--n 20] [--pre-rows R]
    python bench.py --impl reference ...            # the reference's own CPU path
    torchrun --nproc-per-node N bench.py --gpus N   # one process per GPU

A step = one full count of the N=20 folded frontier (R=7: 22,781,426 packed records,
1.865e12 DFS nodes) through the product's multi-GPU scheduler (execute_batch's
counterpart, csrc/nq_sched.cpp): host-side GUIDED dynamic chunk dispatch (big chunks
from the expensive end first, shrinking to the end), one host thread per GPU feeding
ONE persistent streaming launch of the sm_100a DFS kernel (one GPU alone: the whole
frontier as one contiguous launch), per-GPU u64 partials summed on the host with
checked adds. No NCCL anywhere:
  * one process (--gpus N, no torchrun): nq_solve_batch_device over devices 0..N-1;
  * torchrun (one process per GPU): every rank runs the same scheduler on its own GPU,
    all drawing chunks from ONE dispenser in POSIX shared memory (nq_dispatch_*), each
    posting its partial into its slot; gloo (CPU) only for the barriers and the max of
    the per-rank device times.

value  — frontier resident in HBM on every GPU (replicated, copied before timing), CUDA
         events: per GPU, first enqueued launch -> end of its last kernel; max over GPUs.
e2e    — nq_solve_batch with the frontier in pinned HOST memory, read in place by the
         kernels over PCIe (each record once, by the GPU that takes it), the count,
         results D2H; host wall clock, max over ranks.
roofline — integer-issue bound: achieved = per-GPU nodes/s x 18 algorithmic int ops per
           node vs the int-op peak measured live (nq_measure_int_peak).
cpu_baseline — the reference's execute_batch (oracle/_ref/libnqref.so, built from the
           unmodified reference headers) on a systematic slice of the same frontier with
           all host threads (N=1 only).
Every step's count is checked against OEIS A000170.
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
OEIS = {8: 92, 9: 352, 10: 724, 11: 2680, 12: 14200, 13: 73712, 14: 365596, 15: 2279184,
        16: 14772512, 17: 95815104, 18: 666090624, 19: 4968057848, 20: 39029188884,
        21: 314666222712, 22: 2691008701644, 23: 24233937684440}
INT_OPS_PER_NODE = 18  # algorithmic int ops of the minimal last-row body


def load_profile_json(name):
    try:
        with open(os.path.join(REPO, "profiles", name)) as f:
            return json.load(f)
    except OSError:
        return None


def ncu_traffic(n, pre_rows):
    """DRAM bytes (read + write) per launch of the DFS kernel for this workload, from the
    committed ncu capture (profiles/ncu_dram.json), or None when not captured."""
    d = load_profile_json("ncu_dram.json") or {}
    e = d.get(f"{n},{pre_rows},1")
    return None if e is None else e["dram_bytes_per_launch"]


def ncu_limits():
    """The binding resource of the DFS kernel per the committed ncu capture."""
    d = load_profile_json("ncu_limits.json")
    if not d:
        return None
    keys = ("binding_resource", "smem_wavefronts_pct_of_peak", "alu_pipe_pct", "issue_active_pct",
            "smem_wavefronts_per_node", "sass_inst_per_node", "capture")
    return {k: d[k] for k in keys if k in d}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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

    def __init__(self, devices):
        self.devices = ",".join(str(d) for d in devices)
        self.samples = []
        self._stop = threading.Event()
        self._t = None

    def start(self):
        def run():
            while not self._stop.is_set():
                try:
                    out = subprocess.run(
                        ["nvidia-smi", "-i", self.devices, f"--query-gpu={self.FIELDS}",
                         "--format=csv,noheader,nounits"], capture_output=True, text=True,
                        timeout=5).stdout.strip()
                    for line in out.splitlines():
                        self.samples.append([x.strip() for x in line.split(",")])
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
                "samples": len(self.samples), "devices": self.devices}


# ---- the reference arm: ONLY oracle/_ref (the unmodified reference headers) -------------
def reference_sample(n, pre_rows, stride, threads, warm=True):
    """The reference's own generator (for_each_subproblem) picks records i ≡ 0 (mod
    stride); the reference's execute_batch (stealing, chunk 64, lastrow, config1) counts
    them on `threads` host threads. Returns (calc_ms, total, records)."""
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from oracle_ctypes import Reference
    ref = Reference()
    sample = ref.generate_slice(n, pre_rows, stride, 0)
    if warm:  # thread start-up and clock ramp of the first parallel region: untimed
        ref.execute_batch(n, pre_rows, sample[:: max(1, len(sample) // 2048)], workers=threads,
                          chunk=64, strategy=2, variant=1, config_index=0)
    total, calc_ms, processed = ref.execute_batch(n, pre_rows, sample, workers=threads, chunk=64,
                                                  strategy=2, variant=1, config_index=0)
    assert processed == len(sample)
    return calc_ms, total, len(sample)


def load_samples():
    with open(os.path.join(REPO, "tests", "golden", "bench_samples.json")) as f:
        return json.load(f)


def run_reference_arm(args):
    world, rank, _ = dist_env()
    if rank != 0:
        return 0
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from oracle_ctypes import reference_available
    if not reference_available():
        print(json.dumps({"impl": "reference",
                          "unavailable": "oracle/_ref/libnqref.so (the reference build) is missing"}))
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
    length = total = 0
    for i in range(args.warmup + args.steps):
        ms, total, length = reference_sample(args.n, args.pre_rows, args.ref_stride, threads,
                                             warm=(i == 0))
        if total != samples[key]["total"]:
            raise SystemExit(f"reference sample count {total} != pinned {samples[key]['total']}")
        if i >= args.warmup:
            times.append(ms)
    ms = sum(times) / len(times)
    v = nodes / (ms / 1e3)
    sample = (f"N={args.n} R={args.pre_rows} frontier records i%{args.ref_stride}==0 of the "
              f"reference's own stream ({length} records, {nodes} nodes, total {total}); "
              f"timed: the reference's execute_batch calc_ms (stealing, chunk 64, lastrow)")
    line = {"metric": METRIC, "value": v, "unit": "nodes/s", "impl": "reference",
            "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "u32", "data": "synthetic (deterministic frontier)",
            "config": {"workload": f"N={args.n} R={args.pre_rows} full-frontier count",
                       "n": args.n, "pre_rows": args.pre_rows, "sample_stride": args.ref_stride,
                       "same_config": False,
                       "why_sample": "the full count would take ~%.0f min on these host cores; the "
                                     "slice is a systematic 1/%d sample of the same frontier"
                                     % (ms * args.ref_stride / 60000.0, args.ref_stride)},
            "cpu_baseline": {"value": v, "unit": "nodes/s", "cores": threads,
                             "cpu_model": cpu_model(), "kind": "reference", "sample": sample},
            "e2e": {"value": v, "unit": "nodes/s", "h2d_bytes_per_step": 0,
                    "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


# ---- the B200 arm -------------------------------------------------------------------------
class Scheduler:
    """Drives the product's scheduler (nq_solve_batch_device / nq_solve_batch) on a set of
    devices, optionally drawing chunks from a shared dispenser."""

    def __init__(self, args, devices, dispatch=None):
        from paper_2511_12009_b200 import _lib
        self._lib = _lib
        self.args = args
        self.devices = devices
        self.dev_arr = (ctypes.c_int * len(devices))(*devices)
        o = _lib.NqSolveOpts()
        o.variant = _lib.VARIANT_LASTROW
        o.strategy = {"guided": _lib.PARTITION_GUIDED, "stealing": _lib.PARTITION_STEALING,
                      "strided": _lib.PARTITION_STRIDED}[args.dispatch]
        o.chunk = args.chunk
        o.worker_count = len(devices)
        o.n_devices = len(devices)
        o.devices = self.dev_arr
        if dispatch is not None:
            o.dispatch = dispatch.handle
        self.opts = o

    def device_resident(self, dev_ptrs, count):
        _lib = self._lib
        ptrs = (ctypes.c_void_p * len(dev_ptrs))(*dev_ptrs)
        rep = _lib.NqReport()
        _lib.check(_lib.lib.nq_solve_batch_device(self.args.n, self.args.pre_rows, ptrs, count,
                                                  ctypes.byref(self.opts), ctypes.byref(rep)))
        return rep

    def host(self, host_ptr, count):
        _lib = self._lib
        rep = _lib.NqReport()
        _lib.check(_lib.lib.nq_solve_batch(self.args.n, self.args.pre_rows, ctypes.c_void_p(host_ptr),
                                           count, ctypes.byref(self.opts), ctypes.byref(rep)))
        return rep

    def execute(self):
        _lib = self._lib
        rep = _lib.NqReport()
        _lib.check(_lib.lib.nq_solve(self.args.n, self.args.pre_rows, ctypes.byref(self.opts),
                                     ctypes.byref(rep)))
        return rep


def workers_of(rep):
    return [rep.workers[i] for i in range(rep.worker_count)]


def span_ms(rep):
    return max(w.span_ms for w in workers_of(rep))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--n", "--board", dest="n", type=int, default=20)
    ap.add_argument("--pre-rows", type=int, default=None)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--dispatch", default="guided", choices=["guided", "stealing", "strided"],
                    help="scheduler strategy (strided: host-input e2e only)")
    ap.add_argument("--chunk", type=int, default=0, help="guided floor / stealing chunk (0 = auto)")
    ap.add_argument("--single-launch", action="store_true",
                    help="1 GPU only: count the whole frontier in one persistent launch "
                         "(nq_count_device) instead of through the scheduler")
    ap.add_argument("--ref-stride", type=int, default=256)
    ap.add_argument("--cpu-stride", type=int, default=128)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-execute", action="store_true")
    ap.add_argument("--no-zero-conflict", action="store_true",
                    help="skip timing the zero-bank-conflict plane layout beside the default")
    args = ap.parse_args()
    if args.pre_rows is None:
        # R=7: 22.8 M finer subtrees keep every lane busy to the end (lane efficiency
        # 99.7% vs 97.9% at R=6) and the shallower stack fits one more block per SM.
        args.pre_rows = 7 if args.n >= 19 else 6
    if args.impl == "reference":
        return run_reference_arm(args)
    world, _, _ = dist_env()
    if world > 1:
        return run_torchrun(args)
    return run_single_process(args)


def check_total(n, total, what):
    if n in OEIS and total != OEIS[n]:
        raise SystemExit(f"{what}: count {total} != OEIS A000170({n}) = {OEIS[n]}")


def frontier(args):
    import numpy as np
    import torch
    from paper_2511_12009_b200 import nqueens as nq
    recs = nq.generate_packed(args.n, args.pre_rows)
    host = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).pin_memory()
    return recs, host


def roofline(value_per_gpu, nodes_per_step, device):
    from paper_2511_12009_b200 import nqueens as nq
    ops, mhz = nq.measure_int_peak(device)
    achieved = value_per_gpu * INT_OPS_PER_NODE
    return {"bound": "int", "achieved": achieved / 1e12, "peak": ops / 1e12,
            "unit": "Tint-op/s", "frac": achieved / ops,
            "peak_source": f"measured live on this GPU: LOP3+IMAD 1:1 int32 stream, all SMs, "
                           f"{mhz:.0f} MHz (nq_measure_int_peak)",
            "ops_per_node": INT_OPS_PER_NODE,
            "algorithmic": f"{INT_OPS_PER_NODE} int ops per DFS node x {nodes_per_step} nodes "
                           f"per step, per GPU",
            "binding_limit": ncu_limits()}


def run_single_process(args):
    import torch
    from paper_2511_12009_b200 import _lib
    G = args.gpus
    if torch.cuda.device_count() < G:
        raise SystemExit(f"--gpus {G} but only {torch.cuda.device_count()} CUDA devices visible")
    devices = list(range(G))
    recs, host = frontier(args)
    count = len(recs)
    devs = [host.to(f"cuda:{d}") for d in devices]
    flush = [torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{d}") for d in devices]
    sched = Scheduler(args, devices)
    if args.single_launch and G != 1:
        raise SystemExit("--single-launch is a 1-GPU mode")
    if args.dispatch == "strided" and not args.single_launch:
        args.single_launch = G == 1
    ctx = None
    if args.single_launch:
        ctx = ctypes.c_void_p()
        _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))

    def step_value():
        """(device ms, nodes, total, launches) of one full count, inputs in HBM."""
        if ctx is not None:
            r = _lib.NqResult()
            _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                                ctypes.c_void_p(devs[0].data_ptr()), count,
                                                ctypes.byref(r)))
            return r.kernel_ms, r.nodes, r.solutions, 1
        rep = sched.device_resident([d.data_ptr() for d in devs], count)
        return span_ms(rep), rep.nodes, rep.total, sum(w.launches for w in workers_of(rep))

    def flush_l2():
        for f in flush:
            f.zero_()
        for d in devices:
            torch.cuda.synchronize(d)

    for _ in range(args.warmup):
        step_value()
    clocks = Clocks(devices)
    clocks.start()
    dev_ms, nodes_steps, launches = [], [], 0
    for _ in range(args.steps):
        flush_l2()
        ms, nodes, total, nl = step_value()
        check_total(args.n, total, "device-resident step")
        dev_ms.append(ms)
        nodes_steps.append(nodes)
        launches += nl
    for d in devices:
        torch.cuda.synchronize(d)
    clk = clocks.stop()
    if len(set(nodes_steps)) != 1:
        raise SystemExit(f"node counts differ between steps: {sorted(set(nodes_steps))}")
    nodes_per_step = nodes_steps[0]
    t_dev = sum(dev_ms)
    value = nodes_per_step * args.steps / (t_dev / 1e3)
    line = base_line(args, G, value, t_dev, nodes_per_step, count, clk, launches,
                     "1 process, one host thread per GPU" if G > 1 else "1 GPU")
    line["roofline"] = roofline(value / G, nodes_per_step // G, 0)
    line["roofline"]["traffic"] = ncu_traffic(args.n, args.pre_rows) if G == 1 else None
    line["device_ms_per_step"] = dev_ms

    if not args.no_e2e:
        e2e_sched = sched
        if args.dispatch == "strided":
            e2e_sched = Scheduler(args, devices)
        e2e_sched.host(host.data_ptr(), count)  # warm: pinned staging, pooled contexts
        wall = []
        for _ in range(args.steps):
            for d in devices:
                torch.cuda.synchronize(d)
            t0 = time.perf_counter()
            rep = e2e_sched.host(host.data_ptr(), count)
            wall.append((time.perf_counter() - t0) * 1e3)
            check_total(args.n, rep.total, "e2e step")
        line["e2e"] = {"value": nodes_per_step * args.steps / (sum(wall) / 1e3), "unit": "nodes/s",
                       # the pinned frontier is read in place by the kernels over PCIe: every
                       # record crosses the bus once, to the GPU that takes it
                       "h2d_bytes_per_step": count * 16, "d2h_bytes_per_step": 80 * sum(
                           w.launches for w in workers_of(rep)),
                       "ms_per_step": sum(wall) / args.steps,
                       "call": f"nq_solve_batch (execute_batch) on the pinned host frontier, "
                               f"{args.dispatch} dispatch over {G} GPU(s): the kernels read the "
                               f"records in place over PCIe (zero-copy, each record once), "
                               f"{'streaming' if G > 1 else 'contiguous'} count, result "
                               f"read-back; host wall clock"}
    if not args.no_execute:
        rep = None
        for _ in range(2):  # the first call also maps the stream-ordered pool; report the second
            rep = sched.execute()
        check_total(args.n, rep.total, "execute()")
        line["execute_wall_ms"] = {"generation_ms": rep.generation_ms, "calc_ms": rep.calc_ms,
                                   "total_ms": rep.generation_ms + rep.calc_ms,
                                   "call": f"nq_solve (execute): coarse frontier on the host, "
                                           f"deepened + counted on {G} GPU(s), {args.dispatch}"}
    if G == 1 and not args.no_zero_conflict:
        line["zero_conflict_layout"] = zero_conflict_layout(args, devs[0], count, flush_l2)
    if G == 1 and not args.no_cpu_baseline:
        line["cpu_baseline"] = cpu_baseline(args)
    print(json.dumps(line))
    if ctx is not None:
        _lib.lib.nq_ctx_destroy(ctx)
    return 0


def zero_conflict_layout(args, dev, count, flush_l2):
    """The north star's zero-bank-conflict configuration, timed beside the default: the
    same count with the 32-bit plane stack (NQ_LAYOUT_PLANES: lane t owns bank t in four
    word planes), one contiguous launch, checked. Its per-instruction ncu evidence (0
    excess wavefronts on every LDS/STS at this workload) is profiles/r02_ncu_dfs_planes_n20_r7.md."""
    from paper_2511_12009_b200 import _lib
    ctx = ctypes.c_void_p()
    _lib.check(_lib.lib.nq_ctx_create(0, ctypes.byref(ctx)))
    _lib.check(_lib.lib.nq_ctx_set_layout(ctx, _lib.LAYOUT_PLANES))
    try:
        r = _lib.NqResult()
        flush_l2()
        _lib.check(_lib.lib.nq_count_device(ctx, args.n, args.pre_rows, _lib.VARIANT_LASTROW,
                                            ctypes.c_void_p(dev.data_ptr()), count, ctypes.byref(r)))
        check_total(args.n, r.solutions, "plane-layout count")
        return {"layout": "32-bit planes", "ms": r.kernel_ms,
                "nodes_per_s": r.nodes / (r.kernel_ms * 1e-3),
                "ncu_excess_smem_wavefronts_per_instruction": 0,
                "evidence": "profiles/r02_ncu_dfs_planes_n20_r7.md"}
    finally:
        _lib.lib.nq_ctx_destroy(ctx)


def cpu_baseline(args):
    samples = load_samples()
    key = f"{args.n},{args.pre_rows},{args.cpu_stride}"
    sys.path.insert(0, os.path.join(REPO, "tests"))
    from oracle_ctypes import reference_available
    if key not in samples or not reference_available():
        return None
    threads = os.cpu_count() or 1
    ms, total, length = reference_sample(args.n, args.pre_rows, args.cpu_stride, threads)
    if total != samples[key]["total"]:
        raise SystemExit(f"reference sample count {total} != pinned {samples[key]['total']}")
    return {"value": samples[key]["nodes"] / (ms / 1e3), "unit": "nodes/s", "cores": threads,
            "cpu_model": cpu_model(), "kind": "reference",
            "sample": f"N={args.n} R={args.pre_rows} records i%{args.cpu_stride}==0 "
                      f"({length} records, {samples[key]['nodes']} nodes, {ms:.0f} ms)"}


def base_line(args, n_gpus, value, t_dev, nodes_per_step, count, clk, launches, parallelism):
    return {
        "metric": METRIC, "value": value, "unit": "nodes/s", "n_gpus": n_gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": t_dev / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32",
        "data": "synthetic (deterministic folded frontier; no dataset)",
        "config": {"workload": f"N={args.n} R={args.pre_rows} full-frontier count",
                   "n": args.n, "pre_rows": args.pre_rows, "records": count,
                   "solutions": OEIS.get(args.n), "nodes_per_step": nodes_per_step,
                   "parallelism": parallelism,
                   "dispatch": "single persistent launch" if args.single_launch else
                               f"{args.dispatch} dispatch with one worker: the whole frontier as "
                               f"one contiguous launch (expensive end first)" if n_gpus == 1 and
                               os.environ.get("WORLD_SIZE", "1") == "1" else
                               f"{args.dispatch} host-side dynamic chunks fed into one streaming launch per GPU",
                   "l2": "flushed between steps (256 MiB write per GPU, untimed)"},
        "wall_ms": t_dev / args.steps,
        "gpu_launches": launches,
        "clocks": clk,
    }


def run_torchrun(args):
    """One process per GPU: the same scheduler in every rank, chunks from ONE dispenser in
    POSIX shared memory, partials posted per rank and summed on the host. gloo (CPU) carries
    the barriers and the max of the per-rank device times; there is no NCCL."""
    import torch
    import torch.distributed as dist
    from paper_2511_12009_b200 import nqueens as nq
    world, rank, local = dist_env()
    if os.environ.get("NQB_BENCH_SHARE_GPU") == "1":  # testing: every rank on cuda:0
        local = 0
    torch.cuda.set_device(local)
    dist.init_process_group("gloo")
    recs, host = frontier(args)
    count = len(recs)
    dev = host.to(f"cuda:{local}")
    flush = torch.empty(256 * 1024 * 1024, dtype=torch.uint8, device=f"cuda:{local}")
    run_id = os.environ.get("TORCHELASTIC_RUN_ID", "x") + "-" + os.environ.get("MASTER_PORT", "0")
    name = f"/nqb200-{run_id}"
    strategy = nq.PartitionStrategy[args.dispatch if args.dispatch != "strided" else "guided"]
    if rank == 0:
        disp = nq.Dispatcher.create(count, strategy, args.chunk, world, name=name)
    dist.barrier()
    if rank != 0:
        disp = nq.Dispatcher.attach(name)
    dist.barrier()
    if rank == 0:  # every rank has it mapped: unlink the name so nothing outlives the job
        ctypes.CDLL(None).shm_unlink(name.encode())
    if args.dispatch == "strided":
        args.dispatch = "guided"
    sched = Scheduler(args, [local], dispatch=disp)

    def one_pass(fn):
        """One cooperative pass; returns (this rank's report, summed (sols, nodes, recs))."""
        dist.barrier()
        rep = fn()
        disp.post(rank, rep.total, rep.nodes, sum(w.processed for w in workers_of(rep)))
        dist.barrier()
        summed = disp.sum(world) if rank == 0 else None
        dist.barrier()
        if rank == 0:
            disp.reset()
        return rep, summed

    dev_pass = lambda: sched.device_resident([dev.data_ptr()], count)  # noqa: E731
    for _ in range(args.warmup):
        one_pass(dev_pass)
    clocks = Clocks([local])
    if rank == 0:
        clocks.start()
    spans, launches, nodes_steps = [], 0, []
    for _ in range(args.steps):
        flush.zero_()
        torch.cuda.synchronize()
        rep, summed = one_pass(dev_pass)
        spans.append(span_ms(rep) if rep.worker_count else 0.0)
        launches += sum(w.launches for w in workers_of(rep))
        if rank == 0:
            check_total(args.n, summed[0], "device-resident step")
            if summed[2] != count:
                raise SystemExit(f"{summed[2]} records counted, expected {count}")
            nodes_steps.append(summed[1])
    clk = clocks.stop() if rank == 0 else None
    t = torch.tensor(spans + [float(launches)], dtype=torch.float64)
    tmax = t.clone()
    dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    tsum = t.clone()
    dist.all_reduce(tsum, op=dist.ReduceOp.SUM)
    step_ms = tmax[:-1].tolist()
    total_launches = int(tsum[-1].item())

    e2e = None
    if not args.no_e2e:
        host_pass = lambda: sched.host(host.data_ptr(), count)  # noqa: E731
        one_pass(host_pass)  # warm
        wall = []
        for _ in range(args.steps):
            torch.cuda.synchronize()
            dist.barrier()
            t0 = time.perf_counter()
            rep, summed = one_pass(host_pass)
            wall.append((time.perf_counter() - t0) * 1e3)
            if rank == 0:
                check_total(args.n, summed[0], "e2e step")
        w = torch.tensor(wall, dtype=torch.float64)
        dist.all_reduce(w, op=dist.ReduceOp.MAX)
        nl = torch.tensor([float(sum(x.launches for x in workers_of(rep)))], dtype=torch.float64)
        dist.all_reduce(nl, op=dist.ReduceOp.SUM)
        e2e = (w.tolist(), int(nl.item()))
    if rank == 0:
        if len(set(nodes_steps)) != 1:
            raise SystemExit(f"node counts differ between steps: {sorted(set(nodes_steps))}")
        nodes_per_step = nodes_steps[0]
        t_dev = sum(step_ms)
        value = nodes_per_step * args.steps / (t_dev / 1e3)
        line = base_line(args, world, value, t_dev, nodes_per_step, count, clk, total_launches,
                         f"{world} processes (torchrun), one GPU each, one shared host dispenser")
        line["roofline"] = roofline(value / world, nodes_per_step // world, local)
        line["roofline"]["traffic"] = None
        line["device_ms_per_step"] = step_ms
        if e2e is not None:
            line["e2e"] = {"value": nodes_per_step * args.steps / (sum(e2e[0]) / 1e3),
                           "unit": "nodes/s", "h2d_bytes_per_step": count * 16,
                           "d2h_bytes_per_step": 80 * e2e[1],
                           "ms_per_step": sum(e2e[0]) / args.steps,
                           "call": "nq_solve_batch per rank on its pinned host frontier (read in "
                                   "place over PCIe, each record by the GPU that takes it), chunks "
                                   "from the shared dispenser; host wall clock "
                                   "incl. the barriers, max over ranks"}
        print(json.dumps(line))
    disp.close(unlink=False)
    dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
