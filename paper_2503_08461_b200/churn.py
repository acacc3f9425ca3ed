"""Admission waves with alloc/free churn over one device pool (config 4).

The reference engine admits a request's raw cache only when it fits
(``KVCachePool.allocate`` strict admission, pool.py:147-165; the engine's
``_budget``, engine.py:367-374), compresses it (pool.py:167-192), grows it
during decode (pool.py:194-211) and releases it at completion
(pool.py:213-224). ``run_waves`` replays that lifecycle for a request list
far larger than HBM: each wave admits raw caches in arrival order until the
next one would not fit, compresses the whole wave in one batched device pass,
appends decode tokens to every live compressed cache, and releases the caches
that completed (each compressed request lives for ``lifetime_waves`` waves).
Device block occupancy and fragmentation are sampled after every mutation.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from typing import Callable, Sequence

from .kv import CompressorSpec, KVCacheSpec, compressed_spec, kv_bytes
from .pool import CacheHandle, KVCachePool, PoolMode


@dataclass
class ChurnStats:
    waves: int = 0
    compressed_requests: int = 0
    raw_tokens: int = 0
    kept_tokens: int = 0
    compress_ms: list = field(default_factory=list)
    wave_sizes: list = field(default_factory=list)
    peak_bytes: int = 0
    max_fragmentation: float = 0.0
    fragmentation: list = field(default_factory=list)  # (op, used_blocks, fragmentation)
    launches: int = 0

    @property
    def total_compress_ms(self) -> float:
        return sum(self.compress_ms)


def run_waves(pool: KVCachePool, specs: Sequence[KVCacheSpec], comp: CompressorSpec,
              inputs_for: Callable[[int], dict], *, decode_tokens: int = 32,
              lifetime_waves: int = 1, seed: int = 0, request_ids=None,
              sample_fragmentation: bool = True, max_wave: int = 128) -> ChurnStats:
    """Compress every spec through admission waves; returns timing and occupancy stats.

    ``inputs_for(n)`` returns the press inputs (e.g. EA ``mean_q``/``cov_q``) for a
    wave of ``n`` requests. Raw KV of each admitted request is produced by the
    deterministic K8 generator (stand-in for prefill).
    """
    stats = ChurnStats()
    pending = list(range(len(specs)))
    rids = list(request_ids) if request_ids is not None else list(range(len(specs)))
    live: list[tuple[int, list[CacheHandle]]] = []   # (wave index, handles)
    now = 0.0
    pool.set_profiling(True)

    def sample(op: str) -> None:
        if not sample_fragmentation:
            return
        bs = pool.block_stats()
        stats.fragmentation.append((op, bs.used_blocks, bs.fragmentation))
        stats.max_fragmentation = max(stats.max_fragmentation, bs.fragmentation)

    while pending:
        # admit in arrival order while the raw footprint fits (strict admission)
        avail = pool.available_bytes
        wave = []
        for i in pending:
            need = kv_bytes(pool.config, specs[i].total_tokens)
            if pool.mode is PoolMode.LEGACY_ZOMBIE:
                # legacy keeps the raw cache next to its compressed copy: reserve both
                # (the reference engine's COMPRESS estimate, engine.py:380-385)
                need += kv_bytes(pool.config, compressed_spec(specs[i], comp).total_tokens)
            if need > avail or len(wave) == max_wave:
                break
            wave.append(i)
            avail -= need
        if not wave:
            if not live:
                raise RuntimeError("a single request does not fit the pool")
            _, old = live.pop(0)
            pool.release_batch(old, now)
            now += 1.0
            sample("release")
            continue
        pending = pending[len(wave):]
        handles = pool.allocate_batch([rids[i] for i in wave], [specs[i] for i in wave], now)
        sample("allocate")
        pool.synth_fill(handles, seed=seed)
        now += 1.0
        pool.compress_batch(handles, comp, now, **inputs_for(len(handles)))
        prof = pool.last_profile()
        stats.compress_ms.append(prof["total_ms"])
        stats.launches += prof["total_launches"]
        sample("compress")
        stats.waves += 1
        stats.wave_sizes.append(len(wave))
        stats.compressed_requests += len(wave)
        stats.raw_tokens += sum(specs[i].total_tokens for i in wave)
        stats.kept_tokens += sum(h.spec.total_tokens for h in handles)
        # decode growth of every live compressed cache that still fits
        for _, hs in live + [(stats.waves, handles)]:
            for h in hs:
                if kv_bytes(pool.config, decode_tokens) <= pool.available_bytes:
                    pool.append_decode_tokens(h, decode_tokens, now)
        sample("append")
        live.append((stats.waves, handles))
        # completions: requests older than their lifetime release their blocks
        while live and live[0][0] <= stats.waves - lifetime_waves:
            _, old = live.pop(0)
            pool.release_batch(old, now)
            sample("release")
        stats.peak_bytes = max(stats.peak_bytes, pool.peak_bytes)
        now += 1.0
    for _, hs in live:
        pool.release_batch(hs, now)
    sample("release")
    pool.verify_conservation()
    return stats
