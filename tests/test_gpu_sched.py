"""GPU: the multi-GPU scheduler (csrc/nq_sched.cpp) with more workers than devices.

On a one-GPU box a device list that repeats device 0 (devices = [0, 0, 0, 0]) runs the
whole multi-device code path — one host thread per worker, per-worker contexts, the
dynamic dispenser, one streaming launch per worker, host checked sums — against one
device. Every total is compared with OEIS A000170 and every node count with Appendix B
(independent pins: the reference generator's profile).
"""
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

from paper_2511_12009_b200 import nqueens as nq

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

Q = {16: 14772512, 18: 666090624, 20: 39029188884}


def opts(strategy, devices, chunk=0, workers=None):
    return nq.ExecuteOptions(config=nq.builtin_configs[0],
                             plan=nq.PartitionPlan(strategy, workers or len(devices), [], chunk),
                             devices=devices)


@pytest.mark.parametrize("n,r", [(18, 6), (20, 7)])
@pytest.mark.parametrize("strategy,chunk", [(nq.PartitionStrategy.strided, 0),
                                            (nq.PartitionStrategy.guided, 0),
                                            (nq.PartitionStrategy.stealing, 65536)])
def test_four_workers_on_one_device(golden, n, r, strategy, chunk):
    """Four workers share device 0: distinct contexts (the repeated-device race of round
    1 is gone), every record counted once, totals and nodes exact."""
    recs = nq.generate_packed(n, r)
    rep = nq.execute_batch(n, r, recs, opts(strategy, [0, 0, 0, 0], chunk))
    assert rep.total == Q[n] and rep.completed
    assert rep.nodes == golden["appendix_b_nodes"][str(n)][str(r)]
    assert sum(w.processed for w in rep.workers) == len(recs)
    assert sum(w.partial_sum for w in rep.workers) == rep.total
    kms = [w.kernel_ms for w in rep.workers]
    print(f"\nN={n} R={r} {strategy.name}: per-worker kernel_ms {['%.1f' % k for k in kms]}, "
          f"chunks {[w.chunks for w in rep.workers]}, launches {[w.launches for w in rep.workers]}, "
          f"span {['%.1f' % w.span_ms for w in rep.workers]}")
    if strategy is not nq.PartitionStrategy.strided:
        # one streaming launch per worker; workers sharing ONE device may find the
        # dispenser drained by the first worker's kernel (it holds every SM)
        assert all(w.launches == 1 for w in rep.workers)
        assert sum(w.chunks for w in rep.workers) >= 1


def test_device_resident_batch_guided(golden):
    """nq_solve_batch_device: the frontier resident on the device, workers launch on
    sub-ranges of it (bench.py's `value` path)."""
    n, r = 18, 6
    recs = nq.generate_packed(n, r)
    dev = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).cuda()
    for devices in ([0], [0, 0], [0, 0, 0]):
        rep = nq.execute_batch_device(n, r, [dev.data_ptr()] * len(devices), len(recs),
                                      opts(nq.PartitionStrategy.guided, devices))
        assert rep.total == Q[n] and rep.nodes == golden["appendix_b_nodes"]["18"]["6"]
        assert sum(w.processed for w in rep.workers) == len(recs)
        assert all(w.span_ms > 0 for w in rep.workers)
    with pytest.raises(nq.ConfigError, match="not strided"):
        nq.execute_batch_device(n, r, [dev.data_ptr()], len(recs),
                                opts(nq.PartitionStrategy.strided, [0]))


def test_execute_guided_deepens_on_the_device(golden):
    """execute() with guided dispatch over 3 workers: chunks of the coarse R-3 frontier,
    deepened on the device and counted (the N=27-capable path)."""
    rep = nq.execute(20, 7, opts(nq.PartitionStrategy.guided, [0, 0, 0]))
    assert rep.total == Q[20] and rep.completed
    assert rep.nodes == golden["appendix_b_nodes"]["20"]["7"]
    assert rep.task_count == 22781426


def test_shared_dispenser_in_one_process(golden):
    """Two execute_batch calls drawing from one named dispenser split the work between
    them (the torchrun layout, here two threads of one process)."""
    import threading
    n, r = 18, 6
    recs = nq.generate_packed(n, r)
    name = f"/nqb200-gputest-{os.getpid()}"
    with nq.Dispatcher.create(len(recs), nq.PartitionStrategy.guided, 0, 2, name=name) as d:
        reps = [None, None]

        def run(i):
            reps[i] = nq.execute_batch(n, r, recs, nq.ExecuteOptions(
                config=nq.builtin_configs[0], plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 1),
                devices=[0], dispatch=d))
        ts = [threading.Thread(target=run, args=(i,)) for i in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
    assert reps[0].total + reps[1].total == Q[n]
    assert reps[0].nodes + reps[1].nodes == golden["appendix_b_nodes"]["18"]["6"]
    assert sum(w.processed for rep in reps for w in rep.workers) == len(recs)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _bench(cmd, env=None, timeout=600):
    out = subprocess.run(cmd, cwd=REPO, capture_output=True, text=True, timeout=timeout,
                         env={**os.environ, **(env or {})})
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, out.stdout
    return json.loads(lines[0])


def test_bench_torchrun_two_ranks_one_gpu():
    """bench.py under torchrun: 2 ranks (both on cuda:0 for this test), one shared
    dispenser, host-summed partials, no NCCL; the line reports both GPUs' work."""
    line = _bench([sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=2",
                   "--master-addr=127.0.0.1", f"--master-port={_free_port()}", "bench.py",
                   "--gpus", "2", "--board", "16", "--pre-rows", "6", "--steps", "3", "--warmup", "3"],
                  env={"NQB_BENCH_SHARE_GPU": "1"})
    assert line["n_gpus"] == 2 and line["config"]["solutions"] == Q[16]
    assert line["gpu_launches"] >= 2 * 3 and line["e2e"]["value"] > 0
    assert "shared host dispenser" in line["config"]["parallelism"]


def test_bench_single_process_multi_worker():
    """bench.py --gpus 1 through the scheduler (guided) and as one persistent launch."""
    for extra in ([], ["--single-launch"]):
        line = _bench([sys.executable, "bench.py", "--n", "16", "--pre-rows", "6", "--steps", "3",
                       "--warmup", "3", "--no-cpu-baseline"] + extra)
        assert line["n_gpus"] == 1 and line["config"]["solutions"] == Q[16]
        assert line["value"] > 1e10 and line["e2e"]["value"] > 0
        assert line["roofline"]["frac"] > 0


@pytest.mark.parametrize("strategy", list(nq.PartitionStrategy))
def test_empty_and_single_record_batches_every_strategy(strategy):
    """Edge cases of the scheduler (test_scheduler.cpp:121-130): an empty batch counts 0
    and completes; a single record (with a non-default multiplier) is counted once,
    weighted, whatever the strategy and worker count."""
    from paper_2511_12009_b200 import _lib
    empty = np.zeros(0, dtype=_lib.SUB_DTYPE)
    for workers in (1, 3):
        o = nq.ExecuteOptions(config=nq.builtin_configs[0],
                              plan=nq.PartitionPlan(strategy, workers, [], 16), devices=[0])
        rep = nq.execute_batch(12, 4, empty, o)
        assert rep.total == 0 and rep.completed and rep.nodes == 0
        one = nq.generate_packed(12, 4)[100:101].copy()
        want = nq.count_each(12, one, nq.KernelVariant.lastrow, pre_rows=4)[0][0]
        one["row"] = (one["row"] & 0xFF) | (5 << 8)          # multiplier 5
        rep = nq.execute_batch(12, 4, one, o)
        assert rep.total == 5 * int(want) and rep.completed
        assert sum(w.processed for w in rep.workers) == 1


def test_streaming_launch_costs_about_a_contiguous_launch(golden):
    """One worker fed through an explicit dispenser runs the streaming launch; at N=18 R=7
    it consumes ~3e8 records/s, the case whose every chunk boundary used to send all
    warps over the bus at once (4x slower). Within 10% of the contiguous launch of the
    same records, with identical totals and Alg. 3 nodes."""
    n, r = 18, 7
    recs = nq.generate_packed(n, r)
    dev = torch.from_numpy(recs.view(np.int32).reshape(-1, 4)).cuda()
    o = opts(nq.PartitionStrategy.guided, [0])
    best = {}
    for _ in range(3):
        for mode in ("contiguous", "streaming"):
            o.dispatch = (nq.Dispatcher.create(len(recs), nq.PartitionStrategy.guided, 0, 1)
                          if mode == "streaming" else None)
            rep = nq.execute_batch_device(n, r, [dev.data_ptr()], len(recs), o)
            if o.dispatch is not None:
                o.dispatch.close()
            assert rep.total == Q[n] and rep.nodes == golden["appendix_b_nodes"][str(n)][str(r)]
            best[mode] = min(best.get(mode, 1e9), rep.workers[0].span_ms)
    print(best)
    assert best["streaming"] < 1.10 * best["contiguous"], best
