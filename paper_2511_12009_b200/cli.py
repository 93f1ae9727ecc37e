"""Command-line front end over the GPU path, mirroring the reference CLI
(tools/nqueens_cli.cpp): `solve`, `subcount` and `bench` with the same option names,
defaults, log lines and exit codes (0 ok, 2 config error, 3 overflow, 1 other), plus
`--gpus` / `--devices`. `solve --checkpoint FILE [--resume]` and `resume FILE` run the
chunk-granular checkpointed count (nq_solve_checkpointed); `layout` (the analytical bank
model) is replaced by ncu evidence and tests/test_layout_banks.py.

    python -m paper_2511_12009_b200.cli solve --n 20 --pre-rows 7 --workers 8 --partition guided
    python -m paper_2511_12009_b200.cli subcount --n 27 --pre-rows 7
    python -m paper_2511_12009_b200.cli bench --n-min 12 --n-max 16 --r-min 4 --r-max 6
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

EXIT_OK, EXIT_OTHER, EXIT_CONFIG, EXIT_OVERFLOW, EXIT_CHECKPOINT = 0, 1, 2, 3, 4


def _workers(flag):
    if flag is not None:
        return flag
    env = os.environ.get("NQUEENS_WORKERS")  # nqueens_cli.cpp:51-58
    if env and env.isdigit() and int(env) >= 1:
        return int(env)
    return 1


def _default_weights(nq, k):  # nqueens_cli.cpp:43-49
    w = list(nq.paper_gpu_weights)
    return [w[i] if i < 8 else w[-1] for i in range(k)]


def do_solve(nq, a):
    pre = a.pre_rows if a.pre_rows is not None else min(max(6, 1), max(1, a.n - 1))
    cfg = nq.find_config(a.config)
    if cfg is None:
        raise nq.ConfigError(f"unknown stack config '{a.config}' (known: config1..config5)")
    kernel = {"iterative": nq.KernelVariant.iterative, "lastrow": nq.KernelVariant.lastrow}.get(a.kernel)
    if kernel is None:
        raise nq.ConfigError(f"unknown kernel '{a.kernel}'")
    strategy = nq.partition_strategy_from(a.partition)
    devices = [int(x) for x in a.devices.split(",")] if a.devices else (
        list(range(a.gpus)) if a.gpus else None)
    # one worker per listed device unless --workers / NQUEENS_WORKERS say otherwise
    workers = _workers(a.workers) if (a.workers is not None or not devices) else len(devices)
    weights = []
    if strategy is nq.PartitionStrategy.weighted:
        weights = ([float(x) for x in a.weights.split(",")] if a.weights
                   else _default_weights(nq, workers))
    if a.export_subproblems and a.n > 1:
        with open(a.export_subproblems, "w") as f:
            nq.write_batch(f, nq.GenerationPlan(a.n, pre))
    to_stdout = a.format == "log"
    log = (lambda line: print(line, flush=True)) if to_stdout else (lambda line: print(line, file=sys.stderr))
    opts = nq.ExecuteOptions(kernel=kernel, config=cfg,
                             plan=nq.PartitionPlan(strategy, workers, weights, a.chunk_size),
                             log=log, devices=devices)
    if a.checkpoint:
        cancel = _sigint_event()
        opts.cancel = cancel
        timer = None
        if getattr(a, "time_limit_s", 0):
            import threading
            # Daemon + cancelled on return: a finished run must not wait for the limit.
            timer = threading.Timer(a.time_limit_s, cancel.set)
            timer.daemon = True
            timer.start()
        try:
            rep = _run_interruptible(lambda: nq.execute_checkpointed(
                a.n, pre, opts, a.checkpoint, chunk=a.checkpoint_chunk,
                flush_interval_s=a.checkpoint_interval_s, resume=a.resume,
                stop_after_s=getattr(a, "stop_after_s", 0.0)), cancel)
        finally:
            if timer is not None:
                timer.cancel()
        if rep.completed:
            log(nq.log_result_line(a.n, rep.total, rep.calc_ms))
        else:
            log(f"interrupted: progress saved to {a.checkpoint}")
    else:
        rep = nq.execute(a.n, pre, opts)
    if a.format == "json":
        print(json.dumps(rep.to_json(), indent=2))
    elif a.format == "csv":
        print("worker,assigned,processed,partial_sum,elapsed_ms")
        for w in rep.workers:
            print(f"{w.worker},{w.assigned},{w.processed},{w.partial_sum},{w.elapsed_ms}")
        print(f"total,,,{rep.total},{rep.calc_ms}")
    return EXIT_OK


def _run_interruptible(fn, cancel):
    """Runs fn in a worker thread so the main thread keeps handling SIGINT/SIGTERM (a
    Python signal handler cannot run while the main thread is inside a C call)."""
    import threading
    box = {}

    def work():
        try:
            box["r"] = fn()
        except BaseException as e:  # noqa: BLE001 — re-raised in the main thread
            box["e"] = e

    t = threading.Thread(target=work, daemon=True)
    t.start()
    while t.is_alive():
        t.join(0.2)
    if "e" in box:
        raise box["e"]
    return box["r"]


def _sigint_event():
    """SIGINT / SIGTERM set a cancel event (nqueens_cli.cpp:24-26, :310-311)."""
    import signal
    import threading
    ev = threading.Event()
    for sig in (signal.SIGINT, signal.SIGTERM):
        signal.signal(sig, lambda *_: ev.set())
    return ev


def do_resume(nq, a):
    d = nq.checkpoint_details(a.checkpoint)
    print(f"resuming n={d['n']} R={d['pre_rows']} kernel={d['kernel'].name} chunk={d['chunk']}: "
          f"{d['done_chunks']}/{d['chunks']} chunks already counted", file=sys.stderr)
    # the kernel variant and chunk size are part of the file's identity: take them from it
    a.n, a.pre_rows, a.resume, a.checkpoint_chunk = d["n"], d["pre_rows"], True, d["chunk"]
    a.kernel = d["kernel"].name
    return do_solve(nq, a)


def do_subcount(nq, a):
    if a.export_subproblems:
        with open(a.export_subproblems, "w") as f:
            nq.write_batch(f, nq.GenerationPlan(a.n, a.pre_rows))
    t0 = time.perf_counter()
    count = nq.count_subproblems(a.n, a.pre_rows)
    print(nq.log_generation_line((time.perf_counter() - t0) * 1e3, count))
    return EXIT_OK


def do_bench(nq, a):  # nqueens_cli.cpp:224-271, median calc_ms per cell, uniform partition
    workers = _workers(a.workers)
    print("n,r,config,kernel,reps,median_ms,total,ratio")
    for cname in a.configs.split(","):
        cfg = nq.find_config(cname)
        if cfg is None:
            raise nq.ConfigError(f"unknown stack config '{cname}' (known: config1..config5)")
        for kname in a.kernels.split(","):
            kernel = {"iterative": nq.KernelVariant.iterative, "lastrow": nq.KernelVariant.lastrow}[kname]
            for r in range(a.r_min, a.r_max + 1):
                prev = None
                for n in range(a.n_min, a.n_max + 1):
                    ok = n == 1 or (r < n and nq.required_depth(n, r, kernel is nq.KernelVariant.lastrow)
                                    <= cfg.max_depth())
                    if not ok:
                        print(f"{n},{r},{cname},{kname},{a.reps},skipped,,")
                        prev = None
                        continue
                    times, total = [], 0
                    for _ in range(a.reps):
                        opts = nq.ExecuteOptions(kernel=kernel, config=cfg,
                                                 plan=nq.PartitionPlan(nq.PartitionStrategy.uniform, workers))
                        rep = nq.execute(n, 0 if n == 1 else r, opts)
                        times.append(rep.calc_ms)
                        total = rep.total
                    times.sort()
                    ratio = f"{total / prev}" if prev else ""
                    print(f"{n},{r},{cname},{kname},{a.reps},{times[len(times) // 2]},{total},{ratio}")
                    prev = total
    return EXIT_OK


def main(argv=None):
    ap = argparse.ArgumentParser(prog="nqueens")
    sub = ap.add_subparsers(dest="cmd", required=True)
    s = sub.add_parser("solve", help="count solutions for one board size")
    s.add_argument("--n", type=int, required=True)
    s.add_argument("--pre-rows", type=int, default=None)
    s.add_argument("--config", default="config2")
    s.add_argument("--workers", type=int, default=None)
    s.add_argument("--partition", default="weighted")
    s.add_argument("--weights", default="")
    s.add_argument("--kernel", default="lastrow")
    s.add_argument("--format", default="log", choices=["json", "csv", "log"])
    s.add_argument("--chunk-size", type=int, default=4096)
    s.add_argument("--export-subproblems", default="")
    s.add_argument("--gpus", type=int, default=0, help="use devices 0..G-1 (default: all visible)")
    s.add_argument("--devices", default="", help="explicit comma-separated device list")
    s.add_argument("--checkpoint", default="", help="checkpoint file (chunk-granular progress)")
    s.add_argument("--resume", action="store_true", help="continue the run in --checkpoint")
    s.add_argument("--checkpoint-chunk", type=int, default=0, help="records per chunk (0 = auto)")
    s.add_argument("--checkpoint-interval-s", type=float, default=30.0,
                   help="rewrite the checkpoint at most this often")
    s.add_argument("--time-limit-s", type=float, default=0.0,
                   help="checkpointed runs: cancel (and save progress) after this many seconds")
    s.add_argument("--stop-after-s", type=float, default=0.0,
                   help="checkpointed runs: start no new chunk after this many seconds")
    rs = sub.add_parser("resume", help="continue an interrupted checkpointed run")
    rs.add_argument("checkpoint")
    rs.add_argument("--format", default="log", choices=["json", "csv", "log"])
    rs.add_argument("--checkpoint-interval-s", type=float, default=30.0)
    rs.add_argument("--time-limit-s", type=float, default=0.0)
    rs.add_argument("--stop-after-s", type=float, default=0.0)
    rs.add_argument("--config", default="config2")
    rs.add_argument("--workers", type=int, default=None)
    rs.add_argument("--gpus", type=int, default=0, help="use devices 0..G-1 (default: all visible)")
    rs.add_argument("--devices", default="", help="explicit comma-separated device list")
    for k, v in (("partition", "stealing"), ("weights", ""), ("kernel", "lastrow"),
                 ("chunk_size", 4096), ("export_subproblems", "")):
        rs.set_defaults(**{k: v})
    c = sub.add_parser("subcount", help="count generated subproblems")
    c.add_argument("--n", type=int, required=True)
    c.add_argument("--pre-rows", type=int, required=True)
    c.add_argument("--export-subproblems", default="")
    b = sub.add_parser("bench", help="benchmark sweep, CSV on stdout")
    b.add_argument("--n-min", type=int, default=12)
    b.add_argument("--n-max", type=int, default=15)
    b.add_argument("--r-min", type=int, default=4)
    b.add_argument("--r-max", type=int, default=7)
    b.add_argument("--configs", default="config2")
    b.add_argument("--kernels", default="lastrow")
    b.add_argument("--reps", type=int, default=3)
    b.add_argument("--workers", type=int, default=None)
    try:
        a = ap.parse_args(argv)
    except SystemExit as e:
        return EXIT_OK if e.code == 0 else EXIT_CONFIG
    from . import nqueens as nq
    try:
        return {"solve": do_solve, "subcount": do_subcount, "bench": do_bench,
                "resume": do_resume}[a.cmd](nq, a)
    except nq.ConfigError as e:
        print(f"config error: {e}", file=sys.stderr)
        return EXIT_CONFIG
    except OverflowError as e:
        print(f"overflow: {e}", file=sys.stderr)
        return EXIT_OVERFLOW
    except nq.CheckpointError as e:
        print(f"checkpoint error: {e}", file=sys.stderr)
        return EXIT_CHECKPOINT
    except Exception as e:  # noqa: BLE001 — the reference maps everything else to 1
        print(f"error: {e}", file=sys.stderr)
        return EXIT_OTHER


if __name__ == "__main__":
    sys.exit(main())
