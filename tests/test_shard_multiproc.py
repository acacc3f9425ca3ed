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


def _serve_worker(rank, world, port, q):
    import torch.distributed as dist

    from paper_2503_08461_b200 import engine, serving
    from paper_2503_08461_b200.kv import CompressorSpec, ModelConfig
    from paper_2503_08461_b200.scheduling import parse_policy

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        trace = serving.c5_trace(n=400)
        model = ModelConfig("llava-7b", 32, 32, 128, 2)
        sim = engine.Simulator([], model=model, compressor=CompressorSpec(), cost=engine.CostModel(),
                               policy=parse_policy(serving.C5_POLICY),
                               capacity_bytes=serving.C5_CAPACITY, safety_requests=trace)
        out, owner = serving.route_and_run(sim, trace, __import__(
            "paper_2503_08461_b200.shard", fromlist=["x"]).OccupancyExchange(), rank, world)
        q.put((rank, owner, sorted(r.request_id for r in out.records),
               [r.first_token_s - r.arrival_s for r in out.records]))
    finally:
        dist.destroy_process_group()


def test_routed_serving_two_ranks_agree_and_cover_the_trace():
    """Config 5's routed engine on 2 gloo ranks: identical routing on both ranks, every
    request served exactly once by the rank the routing chose, all of them complete."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_serve_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=300) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    (_, own0, ids0, tt0), (_, own1, ids1, tt1) = res
    assert own0 == own1 and set(own0) == {0, 1}
    assert ids0 == [i for i, r in enumerate(own0) if r == 0]
    assert ids1 == [i for i, r in enumerate(own0) if r == 1]
    assert min(tt0 + tt1) > 0


def test_routed_serving_one_rank_is_the_plain_run():
    from paper_2503_08461_b200 import engine, serving
    from paper_2503_08461_b200.kv import CompressorSpec, ModelConfig
    from paper_2503_08461_b200.scheduling import parse_policy

    trace = serving.c5_trace(n=300)
    model = ModelConfig("llava-7b", 32, 32, 128, 2)
    kw = dict(model=model, compressor=CompressorSpec(), cost=engine.CostModel(),
              capacity_bytes=serving.C5_CAPACITY)
    plain = engine.simulate(trace, policy=parse_policy(serving.C5_POLICY), **kw)
    sim = engine.Simulator([], policy=parse_policy(serving.C5_POLICY), safety_requests=trace, **kw)
    routed, owner = serving.route_and_run(sim, trace, None, 0, 1)
    assert owner == [0] * len(trace)
    assert [vars(r) for r in routed.records] == [vars(r) for r in plain.records]
    assert routed.pool.ledger == plain.pool.ledger
