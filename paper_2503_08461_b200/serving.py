"""Config-5 serving driver: a request trace through prefill -> compress -> decode,
with the compression stage executed for real on the device pool.

This is a compact restatement of the reference pipeline (engine.py:1-21): three
stage executors connected by FIFO queues, an event heap in simulated time, the
reference's affine cost model for prefill and decode (engine.py:63-105,
``CostModel`` defaults, ``COST_PRESETS["h100-llava7b-default"]``), and strict
pool admission. The one change is the compress stage: instead of
``stage_duration(COMPRESS)`` (engine.py:128-136) the batch is really
compressed by ``KVCachePool.compress_batch`` on the GPU and its CUDA-event time
is charged. TTFT = end of the first decode step - arrival (metrics.py:75-144).

Multi-GPU: arrivals are routed tick by tick. Every rank all-gathers its
occupancy (``shard.OccupancyExchange``, NCCL) and applies the same
``shard.assign_arrivals`` rule, so all ranks agree without a broadcast; each
rank then runs its own pipeline on its own pool. No collective touches the
compression itself.

Trace (reference ``WORKLOAD_PRESETS["highload"]``, workload.py:133-140,
restated): Poisson arrivals at ``rate`` req/s, 576 image tokens, text and
output lengths geometric with mean 32. Presses alternate by request id:
Knorm (factor 2) for even ids, SnapKV (window 32, factor 4) for odd ids.
"""

from __future__ import annotations

import heapq
from dataclasses import dataclass, field

import numpy as np

from .kv import CompressorSpec, ModelConfig, PressKind, kv_bytes, split_modalities
from .pool import KVCachePool
from . import shard

PREFILL_BASE_S, PREFILL_PER_TOKEN_S = 0.1, 2e-6          # engine.py:74-75 (CostModel)
DECODE_BASE_S, DECODE_PER_CTX_TOKEN_S = 0.0105, 2e-7      # engine.py:80-82


@dataclass
class Request:
    rid: int
    arrival: float
    image: int
    text: int
    output: int
    rank: int = 0
    prefill_end: float = 0.0
    compress_end: float = 0.0
    first_token: float = 0.0

    @property
    def tokens(self) -> int:
        return self.image + self.text


def make_trace(rate: float = 40.0, n: int = 2000, seed: int = 0, image: int = 576,
               text_mean: float = 32.0, out_mean: float = 32.0) -> list[Request]:
    rng = np.random.default_rng(seed)
    gaps = rng.exponential(1.0 / rate, size=n)
    t = np.cumsum(gaps)
    text = rng.geometric(1.0 / text_mean, size=n)
    out = rng.geometric(1.0 / out_mean, size=n)
    return [Request(i, float(t[i]), image, int(text[i]), int(out[i])) for i in range(n)]


def route(trace: list[Request], world: int, exchange: shard.OccupancyExchange | None,
          capacity: int, cfg: ModelConfig, tick_s: float = 0.05) -> None:
    """Assign ``rank`` to every request, tick by tick, with the replicated rule."""
    if world == 1:
        for r in trace:
            r.rank = 0
        return
    queued = [0] * world
    horizon = 4 * tick_s   # queued bytes decay: a request leaves the queue ~one compress later
    pending_out: list[list[tuple[float, int]]] = [[] for _ in range(world)]
    i = 0
    t = 0.0
    while i < len(trace):
        t += tick_s
        for k in range(world):   # retire what each rank has compressed by now (local model)
            keep = [(due, b) for due, b in pending_out[k] if due > t]
            queued[k] -= sum(b for due, b in pending_out[k] if due <= t)
            pending_out[k] = keep
        batch = []
        while i < len(trace) and trace[i].arrival <= t:
            batch.append(trace[i])
            i += 1
        if exchange is not None:
            import torch.distributed as dist

            me = dist.get_rank()
            occ = exchange.gather(capacity - queued[me], queued[me], len(pending_out[me]), 0)
        else:
            occ = [[capacity - queued[k], queued[k], len(pending_out[k]), 0] for k in range(world)]
        raw = [kv_bytes(cfg, r.tokens) for r in batch]
        for r, k, b in zip(batch, shard.assign_arrivals(occ, raw), raw):
            r.rank = k
            queued[k] += b
            pending_out[k].append((t + horizon, b))


@dataclass
class ServingStats:
    ttft: list = field(default_factory=list)
    compress_ms: list = field(default_factory=list)
    compress_batches: int = 0
    compressed_tokens: int = 0
    kept_tokens: int = 0
    makespan_s: float = 0.0
    launches: int = 0

    def summary(self) -> dict:
        tt = np.array(self.ttft) if self.ttft else np.zeros(1)
        total_ms = sum(self.compress_ms)
        return {
            "requests": len(self.ttft),
            "ttft_p50_s": float(np.percentile(tt, 50)),
            "ttft_mean_s": float(tt.mean()),
            "ttft_p90_s": float(np.percentile(tt, 90)),
            "compress_batches": self.compress_batches,
            "compressed_tokens": self.compressed_tokens,
            "kept_tokens": self.kept_tokens,
            "compress_ms_total": total_ms,
            "compress_tokens_per_s": self.compressed_tokens / (total_ms / 1e3) if total_ms else None,
            "makespan_s": self.makespan_s,
        }


def serve(pool: KVCachePool, requests: list[Request], *, max_prefill: int = 8,
          max_compress: int = 64, seed: int = 0) -> ServingStats:
    """Run one rank's requests through the pipeline (simulated clock, real compression)."""
    import torch

    cfg = pool.config
    dev = pool.device
    stats = ServingStats()
    pool.set_profiling(True)
    hq = pool.num_q_heads
    knorm = CompressorSpec(factor=2, press=PressKind.KNORM)
    snap = CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32, pool_kernel=7)
    gen = torch.Generator(device=dev).manual_seed(seed)
    q_all = torch.randn((max_compress, cfg.num_layers, hq, 32, cfg.head_dim), generator=gen,
                        device=dev, dtype=torch.float32).to(pool._native.torch_dtype)
    # synthetic prefill output (varlen [rows, Hkv, D] per layer, the layout attention
    # produces); written into the blocks with the real P.Store path, layer by layer
    max_rows = max_prefill * max(r.tokens for r in requests) if requests else 0
    pf_k = torch.randn((max_rows, cfg.num_kv_heads, cfg.head_dim), generator=gen, device=dev,
                       dtype=torch.float32).to(pool._native.torch_dtype)
    pf_v = torch.randn((max_rows, cfg.num_kv_heads, cfg.head_dim), generator=gen, device=dev,
                       dtype=torch.float32).to(pool._native.torch_dtype)
    events: list = []
    seq = 0

    def push(t, kind, payload):
        nonlocal seq
        heapq.heappush(events, (t, seq, kind, payload))
        seq += 1

    for r in requests:
        push(r.arrival, "arrive", r)
    q_prefill, q_compress, q_decode = [], [], []
    busy = {"prefill": False, "compress": False, "decode": False}
    handles = {}

    def dispatch(now):
        if not busy["prefill"] and q_prefill:
            batch = []
            for r in list(q_prefill):
                if len(batch) == max_prefill:
                    break
                if kv_bytes(cfg, r.tokens) > pool.available_bytes - sum(
                        kv_bytes(cfg, b.tokens) for b in batch):
                    break       # strict admission: wait for releases
                batch.append(r)
            if batch:
                for r in batch:
                    q_prefill.remove(r)
                busy["prefill"] = True
                dur = PREFILL_BASE_S + PREFILL_PER_TOKEN_S * sum(r.tokens for r in batch)
                push(now + dur, "prefill_done", batch)
        if not busy["compress"] and q_compress:
            batch = q_compress[:max_compress]
            del q_compress[:len(batch)]
            busy["compress"] = True
            ms = 0.0
            for comp, members in ((knorm, [r for r in batch if r.rid % 2 == 0]),
                                  (snap, [r for r in batch if r.rid % 2 == 1])):
                if not members:
                    continue
                hs = [handles[r.rid] for r in members]
                kw = {"q_window": q_all[:len(hs)]} if comp.press is PressKind.SNAPKV else {}
                pool.compress_batch(hs, comp, now, **kw)
                prof = pool.last_profile()
                ms += prof["total_ms"]
                stats.launches += prof["total_launches"]
                stats.kept_tokens += sum(h.spec.total_tokens for h in hs)
            stats.compress_ms.append(ms)
            stats.compress_batches += 1
            stats.compressed_tokens += sum(r.tokens for r in batch)
            push(now + ms / 1e3, "compress_done", batch)
        if not busy["decode"] and q_decode:
            batch = list(q_decode)
            q_decode.clear()
            busy["decode"] = True
            ctx = sum(handles[r.rid].spec.total_tokens for r in batch)
            push(now + DECODE_BASE_S + DECODE_PER_CTX_TOKEN_S * ctx, "decode_done", batch)

    now = 0.0
    while events:
        now, _, kind, payload = heapq.heappop(events)
        if kind == "arrive":
            q_prefill.append(payload)
        elif kind == "prefill_done":
            busy["prefill"] = False
            hs = pool.allocate_batch([r.rid for r in payload],
                                     [split_modalities(r.image, r.text) for r in payload], now)
            rows = sum(r.tokens for r in payload)
            for layer in range(cfg.num_layers):       # the prefill's KV writes (P.Store)
                pool.write_prefill_kv(hs, layer, pf_k[:rows], pf_v[:rows])
            for r, h in zip(payload, hs):
                handles[r.rid] = h
                r.prefill_end = now
            q_compress.extend(payload)
        elif kind == "compress_done":
            busy["compress"] = False
            for r in payload:
                r.compress_end = now
            q_decode.extend(payload)
        elif kind == "decode_done":
            busy["decode"] = False
            for r in payload:
                r.first_token = now
                stats.ttft.append(now - r.arrival)
                # the rest of the decode is not on this path: release at first token
                pool.release(handles.pop(r.rid), now)
        dispatch(now)
    stats.makespan_s = now
    pool.verify_conservation()
    return stats
