"""Multi-rank host logic on CPU (gloo, world_size 2): sharding and the occupancy exchange.

The GPU run uses the same code over NCCL (bench.py under torchrun); every
rank must reach the same decisions from the all-gathered occupancy alone.
"""

import os
import socket

import pytest
import torch.multiprocessing as mp

from paper_2503_08461_b200 import shard


def test_lpt_shard_balanced_and_deterministic():
    toks = [1088] * 32
    parts = shard.lpt_shard(toks, 4)
    assert sorted(i for p in parts for i in p) == list(range(32))
    assert [len(p) for p in parts] == [8, 8, 8, 8]
    var = [640, 1536, 900, 1000, 1200, 700, 800, 1500]
    parts = shard.lpt_shard(var, 2)
    loads = [sum(var[i] for i in p) for p in parts]
    assert abs(loads[0] - loads[1]) <= max(var)
    assert parts == shard.lpt_shard(var, 2)


def test_assign_arrivals_rule():
    occ = [[100, 0, 0, 0], [100, 0, 0, 0], [50, 0, 0, 0]]
    assert shard.assign_arrivals(occ, [10, 10, 10]) == [0, 1, 0]
    occ = [[10, 5, 0, 0], [30, 0, 0, 0]]
    assert shard.assign_arrivals(occ, [40, 1]) == [1, 0]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        ex = shard.OccupancyExchange()
        decisions = []
        free = [1000, 1400]
        queued = [0, 0]
        for tick in range(5):
            occ = ex.gather(free[rank], queued[rank], tick, 7 * rank)
            arrivals = [100 + 10 * tick, 50, 300]
            ranks = shard.assign_arrivals(occ, arrivals)
            decisions.append((occ, ranks))
            for r, b in zip(ranks, arrivals):
                if r == rank:
                    queued[rank] += b
        q.put((rank, decisions))
    finally:
        dist.destroy_process_group()


def test_occupancy_exchange_gloo_world2():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert out[0] == out[1], "ranks diverged on the replicated decision"
    occ0, ranks0 = out[0][0]
    assert occ0 == [[1000, 0, 0, 0], [1400, 0, 0, 7]]
    assert ranks0 == [1, 1, 1]  # 1400-100-50 still beats 1000
