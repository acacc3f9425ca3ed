"""Config 5: a serving trace through prefill -> compress -> decode with the compression
stage executed for real on the B200 pool.

The pipeline is ``engine.Simulator`` -- the restated reference engine (stage queues, the
dynamic policy ``bmin=6,bmax=64,wmax_ms=3000,aging=on``, memory admission with reserved
bytes and safety margins, decode run to completion, release at completion;
reference engine.py / scheduling.py) -- with two device seams:

* the compress stage is ``engine.DeviceCompress``: each batch the policy forms goes
  through ``KVCachePool.compress_batch`` (one batched press per compressor: Knorm
  factor 2 for even request ids, SnapKV window 32 factor 4 for odd ones, or the
  reference's mean-pool factor 5 chunk fold) and the measured CUDA-event time of those
  calls is the stage's duration (reference: the cost formula of engine.py:128-136);
* every prefill batch writes its KV into the admitted handles' blocks layer by layer
  through the real P.Store kernel (``write_prefill_kv``); decode steps grow the blocks
  on the device (``append_decode_batch``).

Prefill and decode durations stay the reference cost model's (simulated seconds):
they are not on the compression path. TTFT = first token - arrival (metrics.py:75-78).

Multi-GPU (``serve_routed``): every rank holds the whole trace and its own engine and
pool. Before each ``tick_s`` window all ranks all-gather their engine's occupancy
(int64[4]: free bytes, queued raw bytes, in-flight, compress backlog --
``shard.OccupancyExchange``, NCCL) and apply the same ``shard.assign_arrivals`` rule to
the window's arrivals, so every rank makes the same routing decision without a
broadcast. No collective touches the compression itself.
"""

from __future__ import annotations

from dataclasses import dataclass, replace

import numpy as np

from . import engine as eng
from . import shard
from . import workload as wl
from .kv import CompressorSpec, MapKind, ModelConfig, PressKind
from .pool import KVCachePool
from .scheduling import parse_policy

C5_POLICY = "dynamic:bmin=6,bmax=64,wmax_ms=3000,aging=on"   # experiment.py:57
C5_CAPACITY = 60 * 10 ** 9                                   # experiment.py:55 (GB = 1e9)
KNORM = CompressorSpec(factor=2, press=PressKind.KNORM)
SNAPKV = CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32, pool_kernel=7)
REFERENCE = CompressorSpec(factor=5, map_kind=MapKind.MEAN_POOL)   # experiment.py:58-60


def c5_trace(rate: float = 40.0, n: int = 2000, seed: int = 0) -> list[wl.RequestSpec]:
    """BASELINE config 5: the reference ``highload`` preset at ``rate`` req/s."""
    return wl.generate(replace(wl.WORKLOAD_PRESETS["highload"], rate_req_per_s=rate,
                               num_requests=n, seed=seed))


def mixed_compressor(rid: int) -> CompressorSpec:
    return KNORM if rid % 2 == 0 else SNAPKV


class DeviceInputs:
    """SnapKV window queries for up to ``max_batch`` members (device, pool dtype) and the
    synthetic prefill output the P.Store writes draw from; generated once per run."""

    def __init__(self, pool: KVCachePool, max_batch: int, max_rows: int, seed: int = 0):
        import torch

        cfg = pool.config
        dev, dt = pool.device, pool._native.torch_dtype
        gen = torch.Generator(device=dev).manual_seed(seed)
        self.q = torch.randn((max_batch, cfg.num_layers, pool.num_q_heads, 32, cfg.head_dim),
                             generator=gen, device=dev).to(dt)
        self.k = torch.randn((max_rows, cfg.num_kv_heads, cfg.head_dim), generator=gen,
                             device=dev).to(dt)
        self.v = torch.randn((max_rows, cfg.num_kv_heads, cfg.head_dim), generator=gen,
                             device=dev).to(dt)

    def press(self, comp: CompressorSpec, n: int) -> dict:
        if comp.press is PressKind.SNAPKV:
            return {"q_window": self.q[:n]}
        return {}

    def write_prefill(self, pool: KVCachePool, handles, now: float) -> None:
        rows = sum(h.spec.total_tokens for h in handles)
        if rows > self.k.shape[0]:
            raise ValueError("prefill batch exceeds the synthetic prefill buffer")
        for layer in range(pool.config.num_layers):
            pool.write_prefill_kv(handles, layer, self.k[:rows], self.v[:rows])


def _device_sim(pool, requests, compressor_for, policy, cost, inputs, safety=None):
    return eng.Simulator(
        requests, model=pool.config, compressor=compressor_for(0), cost=cost,
        policy=parse_policy(policy) if isinstance(policy, str) else policy,
        capacity_bytes=pool.capacity_bytes, pool_mode=pool.mode, pool=pool,
        compress_stage=eng.DeviceCompress(inputs.press), compressor_for=compressor_for,
        prefill_writer=inputs.write_prefill, safety_requests=safety)


def make_inputs(pool: KVCachePool, trace, max_batch: int = 64, seed: int = 0) -> DeviceInputs:
    longest = max(r.input_tokens for r in trace)
    return DeviceInputs(pool, max_batch, max_batch * longest, seed)


def serve(pool: KVCachePool, requests, *, compressor_for=mixed_compressor,
          policy=C5_POLICY, cost: eng.CostModel | None = None,
          inputs: DeviceInputs | None = None) -> eng.SimOutput:
    """One rank, one pool: the whole trace through the engine with device compression."""
    inputs = inputs or make_inputs(pool, requests)
    pool.set_profiling(True)
    return _device_sim(pool, requests, compressor_for, policy, cost or eng.CostModel(),
                       inputs).run()


def serve_routed(pool: KVCachePool, trace, exchange: shard.OccupancyExchange | None,
                 rank: int, world: int, *, compressor_for=mixed_compressor, policy=C5_POLICY,
                 cost: eng.CostModel | None = None, tick_s: float = 0.05,
                 inputs: DeviceInputs | None = None):
    """Tick-routed multi-GPU serving on the device pool. Returns (SimOutput of this rank,
    rank of every request). Every rank must call it with the same trace."""
    inputs = inputs or make_inputs(pool, trace)
    pool.set_profiling(True)
    sim = _device_sim(pool, [], compressor_for, policy, cost or eng.CostModel(), inputs,
                      safety=trace)
    return route_and_run(sim, trace, exchange, rank, world, tick_s)


def route_and_run(sim: eng.Simulator, trace, exchange: shard.OccupancyExchange | None,
                  rank: int, world: int, tick_s: float = 0.05):
    """Drive an (empty) engine through ``trace`` with per-tick replicated routing: before
    each ``tick_s`` window every rank all-gathers ``sim.occupancy()`` and assigns the
    window's arrivals with ``shard.assign_arrivals``; this rank injects its own and
    advances to the window's end. With ``world == 1`` this is exactly ``sim.run()``."""
    owner = [-1] * len(trace)
    i, t = 0, 0.0
    while i < len(trace):
        window = []
        while i < len(trace) and trace[i].arrival_time <= t + tick_s:
            window.append(i)
            i += 1
        if world == 1:
            ranks = [0] * len(window)
        else:
            occ = exchange.gather(*sim.occupancy()) if exchange is not None else None
            if occ is None or len(occ) != world:
                raise RuntimeError("routed serving needs an initialised process group")
            ranks = shard.assign_arrivals(occ, [sim._footprint(trace[j])[1] for j in window])
        mine = []
        for j, r in zip(window, ranks):
            owner[j] = r
            if r == rank:
                mine.append(trace[j])
        sim.inject(mine)
        t += tick_s
        sim.advance(t)
    sim.advance()
    return sim.finish(), owner


@dataclass
class ServingReport:
    """Summary of one rank's serving run (the bench's c5 line)."""

    ttft: list
    compress_s: float
    compress_batches: int
    raw_tokens: int
    kept_tokens: int
    launches: int
    paths: dict
    batch_sizes: list

    @classmethod
    def of(cls, out: eng.SimOutput) -> "ServingReport":
        logs = out.compress_batches
        paths = {"tc": 0, "simt": 0, "chunk": 0}
        for b in logs:
            for k, v in (b.paths or {}).items():
                paths[k] += v
        return cls([r.first_token_s - r.arrival_s for r in out.records],
                   sum(b.duration_s for b in logs), len(logs), sum(b.raw_tokens for b in logs),
                   sum(b.kept_tokens for b in logs), sum(b.launches for b in logs), paths,
                   [b.members for b in logs])

    def summary(self) -> dict:
        tt = np.asarray(self.ttft) if self.ttft else np.zeros(1)
        return {"requests": len(self.ttft), "ttft_p50_s": float(np.percentile(tt, 50)),
                "ttft_mean_s": float(tt.mean()), "ttft_p90_s": float(np.percentile(tt, 90)),
                "compress_batches": self.compress_batches,
                "compress_batch_p50": float(np.median(self.batch_sizes)) if self.batch_sizes else 0,
                "compressed_tokens": self.raw_tokens, "kept_tokens": self.kept_tokens,
                "compress_ms_total": self.compress_s * 1e3,
                "compress_tokens_per_s": self.raw_tokens / self.compress_s if self.compress_s else None,
                "paths": self.paths}


def reference_sim_ttft(trace, world: int = 1, compressor: CompressorSpec = REFERENCE,
                       policy: str = C5_POLICY, capacity: int = C5_CAPACITY,
                       model: ModelConfig | None = None) -> dict:
    """the reference pipeline with its *simulated* compress cost (this
    module's engine in cost-model mode replays the reference bit for bit), sharded
    ``request_id % world`` into independent runs. Host-only, ~1 s for 2000 requests."""
    model = model or ModelConfig("llava-7b", 32, 32, 128, 2)
    ttft = []
    for g in range(world):
        shard_reqs = [r for r in trace if r.request_id % world == g]
        out = eng.simulate(shard_reqs, model=model, compressor=compressor, cost=eng.CostModel(),
                           policy=parse_policy(policy), capacity_bytes=capacity)
        ttft += [r.first_token_s - r.arrival_s for r in out.records]
    return {"ttft_p50_s": float(np.percentile(ttft, 50)), "ttft_mean_s": float(np.mean(ttft))}
