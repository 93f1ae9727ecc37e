"""The multi-GPU scheduler's host-side dynamic dispenser (csrc/nq_dispatch.cpp), on CPU:
the product library itself, no device and no stand-in for the counting kernel.

* guided / stealing chunk streams cover every record exactly once (scheduler.hpp:351-362);
* a NAMED dispenser in POSIX shared memory is shared by two processes (gloo world_size 2,
  the torchrun layout of bench.py): concurrent takes still partition the records, the
  per-rank partials posted into slots are summed (checked) on the host, and a reset
  starts the next pass.
"""
import json
import os
import socket
import sys

import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)
sys.path.insert(0, REPO)

from paper_2511_12009_b200 import nqueens as nq  # noqa: E402


def drain(d):
    out = []
    while (c := d.take()) is not None:
        out.append(c)
    return out


def assert_partition(chunks, count):
    pos = 0
    for f, n in sorted(chunks):
        assert f == pos and n >= 1
        pos += n
    assert pos == count


@pytest.mark.parametrize("count,workers", [(1, 1), (1000, 4), (22781426, 8), (30880, 8), (7, 16)])
def test_guided_covers_every_record_once_expensive_end_first(count, workers):
    with nq.Dispatcher.create(count, nq.PartitionStrategy.guided, 0, workers) as d:
        info = d.info()
        assert info["chunk"] == max(count // (128 * workers), 1)
        chunks = drain(d)
        assert_partition(chunks, count)
        assert chunks[0][0] + chunks[0][1] == count     # first chunk ends at the expensive end
        firsts = [f for f, _ in chunks]
        assert firsts == sorted(firsts, reverse=True)   # then walks toward the cheap front
        sizes = [n for _, n in chunks]
        assert all(a >= b for a, b in zip(sizes, sizes[1:]) if b >= info["chunk"])
        cap = max(count // (16 * workers), info["chunk"])
        assert sizes[0] == min(count, max(min(count // (2 * workers), cap), info["chunk"]))
        assert max(sizes) <= max(cap, 1)        # no chunk larger than 1/16 of a worker's share


def test_stealing_is_the_reference_cursor():
    with nq.Dispatcher.create(1000, nq.PartitionStrategy.stealing, 64, 3) as d:
        chunks = drain(d)
    assert chunks == [(i, min(64, 1000 - i)) for i in range(0, 1000, 64)]


def test_reset_starts_a_new_pass():
    with nq.Dispatcher.create(500, nq.PartitionStrategy.guided, 10, 2) as d:
        a = drain(d)
        assert d.take() is None
        d.reset()
        assert drain(d) == a


def test_bad_dispensers_are_rejected():
    with pytest.raises(nq.ConfigError, match="stealing or guided"):
        nq.Dispatcher.create(10, nq.PartitionStrategy.strided, 0, 1)
    with pytest.raises(nq.ConfigError, match="chunk_size"):
        nq.Dispatcher.create(10, nq.PartitionStrategy.stealing, 0, 1)
    with pytest.raises(nq.ConfigError):
        nq.Dispatcher.create(10, nq.PartitionStrategy.guided, 0, 65)    # > NQ_MAX_WORKERS
    with pytest.raises(nq.ConfigError):
        nq.Dispatcher.attach("/nqb200-test-no-such-segment")


def test_sum_needs_every_slot_and_checks_overflow():
    with nq.Dispatcher.create(10, nq.PartitionStrategy.guided, 0, 2) as d:
        d.post(0, 5, 50, 4)
        with pytest.raises(nq.ConfigError):
            d.sum(2)                                       # slot 1 has not posted
        d.post(1, 7, 70, 6)
        assert d.sum(2) == (12, 120, 10)
        d.post(1, 2**64 - 1, 0, 0)
        with pytest.raises(OverflowError):
            d.sum(2)


def test_solve_batch_rejects_a_dispenser_of_another_size():
    """Checked before any device is touched, so it runs on CPU."""
    import numpy as np
    recs = nq.generate_packed(10, 3)
    with nq.Dispatcher.create(len(recs) + 1, nq.PartitionStrategy.guided, 0, 1) as d:
        opts = nq.ExecuteOptions(plan=nq.PartitionPlan(nq.PartitionStrategy.guided, 1), dispatch=d)
        with pytest.raises(nq.ConfigError, match="dispenser covers"):
            nq.execute_batch(10, 3, np.ascontiguousarray(recs), opts)


def _rank(rank, world, port, name, count, out_dir):
    sys.path.insert(0, REPO)
    import torch.distributed as dist

    from paper_2511_12009_b200 import nqueens as nq

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    if rank == 0:
        d = nq.Dispatcher.create(count, nq.PartitionStrategy.guided, 0, world, name=name)
    dist.barrier()
    if rank != 0:
        d = nq.Dispatcher.attach(name)
    passes = []
    for _ in range(3):
        dist.barrier()
        mine = []
        while (c := d.take()) is not None:
            mine.append(c)
        # stand-in partial: a checkable function of the records this rank took
        sol = sum(sum(range(f, f + n)) for f, n in mine)
        d.post(rank, sol, 2 * sol, sum(n for _, n in mine))
        dist.barrier()
        summed = d.sum(world) if rank == 0 else None
        gathered = [None] * world
        dist.all_gather_object(gathered, mine)
        dist.barrier()
        if rank == 0:
            d.reset()
        passes.append({"summed": summed, "chunks": gathered})
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump(passes, f)
    dist.barrier()
    d.close(unlink=(rank == 0))
    dist.destroy_process_group()


def test_two_processes_share_one_dispenser(tmp_path):
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    world, count = 2, 200_000
    name = f"/nqb200-test-{os.getpid()}-{port}"
    mp.spawn(_rank, args=(world, port, name, count, str(tmp_path)), nprocs=world, join=True)
    passes = json.load(open(tmp_path / "r0.json"))
    for p in passes:
        every = [tuple(c) for per_rank in p["chunks"] for c in per_rank]
        assert_partition(every, count)                      # exactly once across processes
        want = count * (count - 1) // 2
        assert p["summed"] == [want, 2 * want, count]
    assert not os.path.exists("/dev/shm" + name)           # the owner unlinked it
