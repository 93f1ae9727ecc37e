"""The multi-rank bench path (torchrun, one process per GPU) exercised on CPU with the
gloo backend at world_size 2: each rank counts its stratified shard of the frontier
(here with the C oracle standing in for the GPU), then bench.reduce_over_ranks sums the
counts and takes the max time — the same functions bench.py runs over NCCL."""
import json
import os
import sys

import pytest
import torch.multiprocessing as mp

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)


def _rank(rank, world, port, out_dir):
    sys.path.insert(0, REPO)
    sys.path.insert(0, HERE)
    import torch.distributed as dist

    import bench
    from oracle_ctypes import Oracle

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    o = Oracle()
    full = o.generate(12, 4)
    mine = bench.shard(full, rank, world)
    total, nodes = o.solve_batch(12, mine, threads=1)
    (nodes_all, total_all), (tmax,) = bench.reduce_over_ranks(dist, [nodes, total],
                                                              [float(rank + 1)], "cpu")
    with open(os.path.join(out_dir, f"r{rank}.json"), "w") as f:
        json.dump({"records": len(mine), "nodes_all": nodes_all, "total_all": total_all,
                   "tmax": tmax, "first": int(mine["cols"][0]) if len(mine) else -1}, f)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_two_rank_shard_and_reduce(tmp_path, world, oracle):
    import socket
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.spawn(_rank, args=(world, port, str(tmp_path)), nprocs=world, join=True)
    res = [json.load(open(tmp_path / f"r{r}.json")) for r in range(world)]
    full = oracle.generate(12, 4)
    want_total, want_nodes = oracle.solve_batch(12, full)
    assert want_total == 14200
    assert sum(r["records"] for r in res) == len(full)           # shards partition the frontier
    assert res[0]["first"] == int(full["cols"][0]) and res[1]["first"] == int(full["cols"][1])
    for r in res:                                                # every rank sees the same sums
        assert r["total_all"] == want_total and r["nodes_all"] == want_nodes
        assert r["tmax"] == float(world)                         # max over ranks


def test_rank_slice_equals_shard(oracle):
    """bench.py generates a rank's records with nq_generate_slice(stride=world,
    offset=rank); that must be exactly shard(full, rank, world)."""
    import numpy as np
    sys.path.insert(0, REPO)
    import bench
    from paper_2511_12009_b200 import nqueens as nq
    full = nq.generate_packed(14, 5)
    for world in (2, 3, 8):
        for rank in range(world):
            assert np.array_equal(nq.generate_slice(14, 5, world, rank), bench.shard(full, rank, world))
