#!/usr/bin/env python
"""Benchmark of the batched KV-cache compression stage (FastCache hot path) on B200.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config c2] [--impl ours|reference]

One *step* = one ``KVCachePool.compress_batch`` over one synthetic batch whose
raw KV is already resident in the paged pool (Knorm / SnapKV / EA scoring +
top-k + in-place compaction + tail-block free). Between steps the batch is
released, re-allocated and re-filled by the K8 generator (untimed; the 18 GB
refill also flushes L2 -- inputs are larger than L2 anyway). Step time is
measured with CUDA events on the launch stream and summed over K steps,
bracketed by barrier + synchronize, max over ranks.

``e2e`` is the same metric through the public API with HOST buffers: every
step copies the batch's raw KV from pinned host memory into the pool
(H2D + ingest kernel), compresses, and reads the kept indices back (D2H).

``--impl reference`` times the CPU reference arm (the oracle port of the same
pass, oracle/cpu_pipeline.py) on the host cores, rank 0 only.

Multi-GPU (torchrun): requests are sharded across ranks -- every rank
compresses its own independent batch (weak scaling); no collective on the
data path, NCCL only for the barrier / max-over-ranks timing.
"""

from __future__ import annotations

import argparse
import gc
import json
import os
import statistics
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    # name: (description, L, H, D, dtype, press, factor, n_req, lengths fn)
    "c1": "tiny synthetic KV (4 layers, 8 heads, head_dim 64, batch 4, seq 512) Knorm 50%, fp32",
    "c2": "LLaVA-1.5-7B-shaped KV (32 layers, 32 heads, d=128, 576 image + 512 text tokens) "
          "batch 32, Knorm 50%, fp16",
    "c3": "LLaVA-1.5-7B-shaped KV batch 64, SnapKV (window 32, pool 7) at 25% keep, "
          "variable-length requests (576 img + text U[64,960])",
    "c3l": "SnapKV (window 32, pool 7) at 25% keep on c4w's 64 mixed-length requests (1k-8k "
           "tokens): segments beyond the 2048-token TMEM ring take the two-pass tensor-core path",
    "c3g": "SnapKV (window 32, pool 7) at 25% keep with GQA: Llama-3-8B-shaped KV (32 layers, 8 kv "
           "heads, 32 query heads, d=128), c3's 64 variable-length requests",
    "c4g": "ExpectedAttention at 25% keep with GQA: Llama-3-8B-shaped KV (8 kv / 32 query heads), "
           "c4w's 64 mixed-length requests (1k-8k tokens)",
    "c4w": "ExpectedAttention at 25% keep, 64 mixed-length requests (1k-8k tokens; one admission "
           "wave of config 4)",
    "c4": "ExpectedAttention at 25% keep on 256 mixed-length requests (1k-8k tokens) with pool "
          "alloc/free churn (admission waves, 140 GB pool) and fragmentation accounting",
    "c2m": "LLaVA-1.5-7B-shaped KV (32 layers, 32 heads, d=128, 576 image + 512 text tokens) "
           "batch 32 through the reference's own compressor (compress_tensor MEAN_POOL, factor 5, "
           "kv.py:211-239) folded into the pool blocks (K7, SURVEY.md §8(f) row 1), fp16",
    "c2d": "decode after compression: config 2's batch (32 x 1088 tokens, Knorm 50% -> 544) "
           "then 64 decode steps, each = append one token per request + per layer write K/V and "
           "paged attention over the compacted blocks (SURVEY.md §8(f) row 2)",
    "c2p": "prefill KV ingest (P.Store): config 2's batch (32 x 1088 tokens) written layer by "
           "layer from the varlen [rows, H, D] prefill layout into the paged blocks",
    "c5": "synthetic serving trace at 40 req/s (2000 requests, highload shape), request-sharded "
          "by NCCL occupancy exchange, mixed Knorm/SnapKV, TTFT and compression throughput",
}


STRONG = {"c3", "c3g", "c3l", "c4g", "c4w", "c4"}
Q_HEADS = {"c3g": 32, "c4g": 32}   # query heads when they differ from the kv heads (GQA)


def workload(name: str):
    import numpy as np

    from paper_2503_08461_b200 import (
        CompressorSpec,
        MapKind,
        ModelConfig,
        PressKind,
        split_modalities,
    )

    if name == "c1":
        cfg = ModelConfig("tiny", 4, 8, 64, 4)
        specs = [split_modalities(0, 512)] * 4
        return cfg, "float32", specs, CompressorSpec(factor=2, press=PressKind.KNORM)
    if name == "c2":
        cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
        specs = [split_modalities(576, 512)] * 32
        return cfg, "float16", specs, CompressorSpec(factor=2, press=PressKind.KNORM)
    if name == "c2m":
        cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
        specs = [split_modalities(576, 512)] * 32
        return cfg, "float16", specs, CompressorSpec(factor=5, map_kind=MapKind.MEAN_POOL)
    if name == "c3":
        cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
        txt = np.random.default_rng(0).integers(64, 961, 64)
        specs = [split_modalities(576, int(t)) for t in txt]
        return cfg, "float16", specs, CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32,
                                                      pool_kernel=7)
    if name == "c3g":
        cfg = ModelConfig("llama-3-8b", 32, 8, 128, 2)
        txt = np.random.default_rng(0).integers(64, 961, 64)
        specs = [split_modalities(576, int(t)) for t in txt]
        return cfg, "float16", specs, CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32,
                                                      pool_kernel=7)
    if name == "c4g":
        cfg = ModelConfig("llama-3-8b", 32, 8, 128, 2)
        lens = np.random.default_rng(0).integers(1024, 8193, 256)[:64]
        specs = [split_modalities(576, int(t) - 576) for t in lens]
        return cfg, "float16", specs, CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION,
                                                      n_sink=4)
    if name == "c3l":
        cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
        lens = np.random.default_rng(0).integers(1024, 8193, 256)[:64]
        specs = [split_modalities(576, int(t) - 576) for t in lens]
        return cfg, "float16", specs, CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32,
                                                      pool_kernel=7)
    if name in ("c4w", "c4"):
        cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
        lens = np.random.default_rng(0).integers(1024, 8193, 256)
        lens = lens[:64] if name == "c4w" else lens
        specs = [split_modalities(576, int(t) - 576) for t in lens]
        return cfg, "float16", specs, CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION,
                                                      n_sink=4)
    raise SystemExit(f"unknown config {name}")


def alg_bytes(cfg, specs, comp, hq=None) -> int:
    """SURVEY.md §8(d) algorithmic HBM bytes of one batch (R raw, C kept)."""
    from paper_2503_08461_b200 import PressKind, compressed_spec, kv_bytes

    raw = sum(kv_bytes(cfg, s.total_tokens) for s in specs)
    kept = sum(kv_bytes(cfg, compressed_spec(s, comp).total_tokens) for s in specs)
    lhq = cfg.num_layers * (hq or cfg.num_kv_heads)
    if comp.press is PressKind.KNORM:
        return raw // 2 + 2 * kept
    if comp.press is PressKind.SNAPKV:
        return raw // 2 + 2 * kept + len(specs) * lhq * comp.window * cfg.head_dim * cfg.bytes_per_element
    if comp.press is PressKind.EXPECTED_ATTENTION:
        return raw + 2 * kept + len(specs) * lhq * (cfg.head_dim + cfg.head_dim ** 2) * 4
    return raw + kept


def measured_peak():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        with open(path) as f:
            return float(json.load(f)["hbm_gbs"]), "measured"
    except (OSError, KeyError, ValueError):
        return 6650.0, "fallback"


class ClockSampler:
    """nvidia-smi-equivalent clock / throttle sampling (NVML) during the timed region."""

    def __init__(self, index: int, period: float = 0.01):
        self.index, self.period = index, period
        self.samples, self.reasons = [], set()
        self.max_mhz = None
        self._stop = threading.Event()
        self._thr = None

    def __enter__(self):
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nv = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._nv = None
            return self
        self._thr = threading.Thread(target=self._run, daemon=True)
        self._thr.start()
        return self

    def _run(self):
        nv = self._nv
        names = {
            "hw_slowdown": getattr(nv, "nvmlClocksEventReasonHwSlowdown", 0x8),
            "sw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonSwThermalSlowdown", 0x20),
            "hw_thermal_slowdown": getattr(nv, "nvmlClocksEventReasonHwThermalSlowdown", 0x40),
            "sw_power_cap": getattr(nv, "nvmlClocksEventReasonSwPowerCap", 0x4),
            "hw_power_brake_slowdown": getattr(nv, "nvmlClocksEventReasonHwPowerBrakeSlowdown", 0x80),
        }
        # every 10 ms while the timed region runs, plus once more as it ends, so even a
        # ~20-ms region (c3g's 5 steps) carries a few samples
        while True:
            stopping = self._stop.is_set()
            try:
                mhz = nv.nvmlDeviceGetClockInfo(self._h, nv.NVML_CLOCK_SM)
                mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self._h)
                self.samples.append(mhz)
                for k, bit in names.items():
                    if mask & bit:
                        self.reasons.add(k)
            except Exception:  # noqa: BLE001
                pass
            if stopping:
                break
            self._stop.wait(self.period)

    def __exit__(self, *exc):
        self._stop.set()
        if self._thr is not None:
            self._thr.join()
        return False

    def summary(self):
        med = statistics.median(self.samples) if self.samples else None
        return {"sm_mhz": med, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                "samples": len(self.samples)}


def press_inputs(comp, cfg, n, device, torch, seed, hq=None):
    from paper_2503_08461_b200 import PressKind

    hq = hq or cfg.num_kv_heads
    gen = torch.Generator(device=device).manual_seed(seed)
    if comp.press is PressKind.SNAPKV:
        q = torch.randn((n, cfg.num_layers, hq, comp.window, cfg.head_dim),
                        generator=gen, device=device, dtype=torch.float32).half()
        return {"q_window": q}
    if comp.press is PressKind.EXPECTED_ATTENTION:
        d = cfg.head_dim
        mu = torch.randn((n, cfg.num_layers, hq, d), generator=gen, device=device) / d ** 0.5
        a = torch.randn((hq, d, d), generator=gen, device=device)
        cov1 = a @ a.transpose(-1, -2) / d
        cov = cov1.expand(n, cfg.num_layers, -1, -1, -1).contiguous()
        return {"mean_q": mu.contiguous(), "cov_q": cov}
    return {}


def traffic_from_profile(config: str):
    path = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    try:
        with open(path) as f:
            return json.load(f).get("dram_bytes_per_launch")
    except (OSError, ValueError):
        return None


def _scaled_traffic(config: str, alg_bytes: int):
    path = os.path.join(ROOT, "profiles", f"ncu_{config}.json")
    try:
        with open(path) as f:
            ratio = json.load(f).get("traffic_over_alg")
        return None if ratio is None else ratio * alg_bytes
    except (OSError, ValueError):
        return None


def _allreduce(value: float, op: str, device) -> float:
    """Max/sum over ranks (NCCL on the GPU tensor, gloo on a CPU copy)."""
    import torch
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size() == 1:
        return value
    dev = device if dist.get_backend() == "nccl" else torch.device("cpu")
    t = torch.tensor([value], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX if op == "max" else dist.ReduceOp.SUM)
    return float(t.item())


def run_serving_bench(args, rank, world, local_rank):
    """Config 5: the reference highload trace at 40 req/s through the restated reference
    engine (dynamic policy, admission, decode to completion) with the compress stage run
    on the device pool and charged its measured time; request-routed over the ranks by the
    NCCL occupancy all-gather. Reported beside the reference's simulated-compress TTFT for
    the same trace and policy."""
    import numpy as np
    import torch

    from paper_2503_08461_b200 import KVCachePool, ModelConfig, serving, shard

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
    trace = serving.c5_trace()
    ex = shard.OccupancyExchange(device=device) if world > 1 else None

    def one_run(compressor_for, reqs):
        pool = KVCachePool(cfg, serving.C5_CAPACITY, device=device, kv_dtype="float16",
                           max_handles=1024, max_tokens_per_handle=4096,
                           num_q_heads=cfg.num_kv_heads)
        inputs = serving.make_inputs(pool, reqs)
        out, owner = serving.serve_routed(pool, reqs, ex, rank, world,
                                          compressor_for=compressor_for, inputs=inputs)
        rep = serving.ServingReport.of(out)
        del pool, inputs, out
        gc.collect()
        torch.cuda.empty_cache()
        return rep, owner

    # warm-up: the first 200 requests of the trace (kernels, allocator, P.Store)
    for _ in range(max(1, args.warmup // 3)):
        one_run(serving.mixed_compressor, trace[:200])
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(device.index) as clocks:
        mixed, owner = one_run(serving.mixed_compressor, trace)
        refc, _ = one_run(lambda rid: serving.REFERENCE, trace)
    max_s = _allreduce(mixed.compress_s, "max", device)
    tokens = _allreduce(float(mixed.raw_tokens), "sum", device)

    def gather_ttft(rep):
        if world == 1:
            return rep.ttft
        parts = [None] * world
        torch.distributed.all_gather_object(parts, rep.ttft)
        return [x for p in parts for x in p]

    tt_mixed, tt_ref = gather_ttft(mixed), gather_ttft(refc)
    sim = serving.reference_sim_ttft(trace, world) if rank == 0 else {}
    sim_same = serving.reference_sim_ttft(trace, 1) if rank == 0 and world > 1 else sim
    shares = [owner.count(k) for k in range(world)]
    return {
        "metric": "compressed KV tokens/s", "value": tokens / max_s,
        "unit": "tokens/s", "n_gpus": world, "steps": mixed.compress_batches,
        "warmup": max(1, args.warmup // 3), "ms_per_step": max_s * 1e3 / max(1, mixed.compress_batches),
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f16",
        "data": "synthetic trace (reference highload preset @ 40 req/s, 2000 requests, seed 0; "
                "workload.generate restated draw for draw)",
        "config": {"workload": f"c5: {CONFIGS['c5']}", "requests": len(trace), "rate_rps": 40.0,
                   "policy": serving.C5_POLICY, "pool_capacity_bytes_per_gpu": serving.C5_CAPACITY,
                   "compressors": "mixed: Knorm factor 2 (even ids) / SnapKV w32 factor 4 (odd ids)",
                   "parallelism": f"x{world}: arrivals routed per 50 ms tick from an all-gather "
                                  "of int64[4] engine occupancy; no data-path collective",
                   "requests_per_rank": shares,
                   "timing": "step = one compress batch the dynamic policy formed; its duration "
                             "is the CUDA-event time of compress_batch (press + tail-block free); "
                             "prefill/decode: reference cost model (simulated seconds)"},
        "ttft_p50_s": float(np.percentile(tt_mixed, 50)), "ttft_mean_s": float(np.mean(tt_mixed)),
        "ttft_p90_s": float(np.percentile(tt_mixed, 90)),
        "reference_compressor_run": {
            "compressor": "meanpool factor 5 (the reference default), chunk fold on the device",
            "ttft_p50_s": float(np.percentile(tt_ref, 50)), "ttft_mean_s": float(np.mean(tt_ref)),
            "compress_tokens_per_s": refc.raw_tokens / refc.compress_s if refc.compress_s else None},
        "reference_simulated": {
            "what": "same trace, policy and compressor with the reference's simulated compress "
                    "cost (0.01 s + 1e-5 s/token), request_id % G shards (BASELINE.md §5); "
                    "engine restatement pinned bit-for-bit to the reference "
                    "(tests/test_refengine_dropin.py)",
            "ttft_p50_s": sim.get("ttft_p50_s"), "ttft_mean_s": sim.get("ttft_mean_s"),
            "g1_ttft_p50_s": sim_same.get("ttft_p50_s"), "baseline_md_g1_p50_s": 2.306},
        "serving_rank0": mixed.summary(), "gpu_launches": mixed.launches + refc.launches,
        "paths": mixed.paths, "clocks": clocks.summary(),
    }


def run_churn_bench(args, rank, world, local_rank):
    """Config 4: every step compresses all requests through admission waves with churn."""
    import torch

    from paper_2503_08461_b200 import KVCachePool, churn, shard

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cfg, dtype, specs, comp = workload(args.config)
    total_tokens = sum(s.total_tokens for s in specs)
    mine = shard.lpt_shard([s.total_tokens for s in specs], world)[rank]
    specs = [specs[i] for i in mine]
    capacity = int(os.environ.get("FASTCACHE_C4_CAPACITY", 140 * 10 ** 9)) // world
    max_wave = 128
    pool = KVCachePool(cfg, capacity, device=device, kv_dtype=dtype, max_handles=512,
                       max_tokens_per_handle=8192 + 2048, num_q_heads=cfg.num_kv_heads)
    full = press_inputs(comp, cfg, max_wave, device, torch, seed=1234 + rank)

    def inputs_for(n):
        return {k: v[:n] for k, v in full.items()}

    rids = [rank * 1_000_000 + i for i in range(len(specs))]
    for _ in range(args.warmup):
        churn.run_waves(pool, specs, comp, inputs_for, request_ids=rids, max_wave=max_wave,
                        sample_fragmentation=False)
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    runs = []
    with ClockSampler(device.index) as clocks:
        for _ in range(args.steps):
            runs.append(churn.run_waves(pool, specs, comp, inputs_for, request_ids=rids,
                                        max_wave=max_wave))
    torch.cuda.synchronize(device)
    my_ms = sum(r.total_compress_ms for r in runs)
    if world > 1:
        torch.distributed.barrier()
    max_ms = _allreduce(my_ms, "max", device)
    peak, peak_kind = measured_peak()
    abytes = alg_bytes(cfg, specs, comp)
    achieved = abytes * args.steps / (my_ms / 1e3) / 1e9
    r0 = runs[-1]
    return {
        "metric": "compressed KV tokens/s", "value": total_tokens * args.steps / (max_ms / 1e3),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic (oracle/synth.py generator)",
        "config": {"workload": f"c4: {CONFIGS['c4']}", "press": comp.press.value,
                   "factor": comp.factor, "requests_total": 256, "requests_this_gpu": len(specs),
                   "pool_capacity_bytes_per_gpu": capacity,
                   "parallelism": f"LPT request shards x{world}; no data-path collective",
                   "timing": "CUDA events around each wave's compress_batch, summed"},
        "roofline": {"bound": "hbm", "kernel": "ea_tc_kernel (one launch per admission wave)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "frac_of_nominal_8tbs": achieved / 8000.0,
                     "traffic": _scaled_traffic("c4w", abytes),
                     "traffic_note": "DRAM bytes per step = ncu traffic/algorithmic ratio of one "
                                     "c4w wave (profiles/ncu_c4w.json) x this step's algorithmic bytes",
                     "alg_bytes_per_step": abytes},
        "churn": {"waves": r0.waves, "wave_sizes": r0.wave_sizes, "peak_bytes": r0.peak_bytes,
                  "max_fragmentation": r0.max_fragmentation,
                  "final_fragmentation": r0.fragmentation[-2][2] if len(r0.fragmentation) > 1 else None,
                  "kept_tokens": r0.kept_tokens, "raw_tokens": r0.raw_tokens},
        "gpu_launches": sum(r.launches for r in runs),
        "clocks": clocks.summary(),
    }


def run_decode_bench(args, rank, world, local_rank):
    """Decode over compacted blocks: tokens/s of decode steps and the attention kernel's HBM
    roofline (K/V bytes of every live token, every layer)."""
    import torch

    from paper_2503_08461_b200 import KVCachePool, compressed_spec, kv_bytes

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cfg, dtype, specs, comp = workload("c2")
    n, L, H, D = len(specs), cfg.num_layers, cfg.num_kv_heads, cfg.head_dim
    steps_per_run = 64
    cap = sum(kv_bytes(cfg, s.total_tokens) for s in specs)
    pool = KVCachePool(cfg, cap, device=device, kv_dtype=dtype, max_handles=2 * n,
                       max_tokens_per_handle=max(s.total_tokens for s in specs) + 64,
                       num_q_heads=H)
    tdt = getattr(torch, dtype)
    gen = torch.Generator(device=device).manual_seed(rank)
    k = torch.randn((L, n, H, D), generator=gen, device=device).to(tdt)
    v = torch.randn((L, n, H, D), generator=gen, device=device).to(tdt)
    q = torch.randn((L, n, H, D), generator=gen, device=device).to(tdt)
    out = torch.empty((n, H, D), dtype=tdt, device=device)
    stream = torch.cuda.current_stream(device)
    rids = [rank * 1_000_000 + i for i in range(n)]
    step_ms, attn_ms, attn_bytes, launches = [], [], 0, 0
    attn_dev_ms = []
    from paper_2503_08461_b200 import _native

    def run(timed):
        nonlocal attn_bytes, launches
        hs = pool.allocate_batch(rids, specs, 0.0)
        pool.synth_fill(hs, seed=17)
        pool.compress_batch(hs, comp, 1.0)
        torch.cuda.synchronize(device)
        for st in range(steps_per_run):
            l0 = _native.launch_count()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(2 * L + 2)]
            ev[0].record(stream)
            pool.append_decode_batch(hs, 1, 2.0 + st)
            for layer in range(L):
                pool.write_decode_kv(hs, layer, k[layer], v[layer])
                ev[1 + 2 * layer].record(stream)
                pool.decode_attention(hs, layer, q[layer], out=out)
                ev[2 + 2 * layer].record(stream)
            ev[-1].record(stream)
            ev[-1].synchronize()
            if timed:
                step_ms.append(ev[0].elapsed_time(ev[-1]))
                attn_ms.append(sum(ev[1 + 2 * i].elapsed_time(ev[2 + 2 * i]) for i in range(L)) / L)
                live = sum(h.spec.total_tokens for h in hs)
                attn_bytes += live * 2 * H * D * cfg.bytes_per_element + 2 * n * H * D * cfg.bytes_per_element
                launches += _native.launch_count() - l0
        if timed:
            # device time of the attention kernel alone: 32 back-to-back launches (the host
            # runs ahead of the GPU here, unlike in the step loop where Python paces it)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize(device)
            e0.record(stream)
            for layer in range(L):
                pool.decode_attention(hs, layer, q[layer], out=out)
            e1.record(stream)
            e1.synchronize()
            attn_dev_ms.append(e0.elapsed_time(e1) / L)
        pool.release_batch(hs, 99.0)

    for _ in range(args.warmup):
        run(False)
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(device.index) as clocks:
        for _ in range(args.steps):
            run(True)
        torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    total_ms = sum(step_ms)
    max_ms = _allreduce(total_ms, "max", device)
    n_steps = len(step_ms)
    peak, peak_kind = measured_peak()
    live = sum(compressed_spec(s, comp).total_tokens for s in specs) + n * steps_per_run
    final_bytes = live * 2 * H * D * cfg.bytes_per_element + 2 * n * H * D * cfg.bytes_per_element
    achieved = final_bytes / (statistics.mean(attn_dev_ms) / 1e3) / 1e9
    return {
        "metric": "decode tokens/s over compressed caches", "value": n * n_steps * world / (max_ms / 1e3),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max_ms / n_steps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic (K8 generator; random q/k/v)",
        "config": {"workload": f"c2d: {CONFIGS['c2d']}", "requests_per_gpu": n,
                   "decode_steps_per_run": steps_per_run, "layers": L,
                   "timing": "CUDA events per decode step (append + 32 x (write K/V + attention)); "
                             "attention kernel events per layer"},
        "roofline": {"bound": "hbm", "kernel": "decode_attn_kernel (paged, split-KV)",
                     "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
                     "frac": achieved / peak, "traffic": None,
                     "alg_bytes_per_launch": final_bytes,
                     "attn_us_per_layer": 1e3 * statistics.mean(attn_dev_ms),
                     "attn_us_per_layer_in_step": 1e3 * statistics.mean(attn_ms),
                     "note": "achieved = K/V bytes of every live token (kept + 64 decoded per "
                             "request) + q/out, over the device time of back-to-back launches"},
        "tpot_ms": max_ms / n_steps,
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }


def run_prefill_bench(args, rank, world, local_rank):
    """P.Store: write_prefill_kv of every layer of config 2's batch (HBM read + write)."""
    import torch

    from paper_2503_08461_b200 import KVCachePool, kv_bytes

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cfg, dtype, specs, _ = workload("c2")
    n, L, H, D = len(specs), cfg.num_layers, cfg.num_kv_heads, cfg.head_dim
    rows = sum(s.total_tokens for s in specs)
    cap = sum(kv_bytes(cfg, s.total_tokens) for s in specs)
    pool = KVCachePool(cfg, cap, device=device, kv_dtype=dtype, max_handles=2 * n,
                       max_tokens_per_handle=max(s.total_tokens for s in specs) + 64)
    tdt = getattr(torch, dtype)
    gen = torch.Generator(device=device).manual_seed(rank)
    k = torch.randn((L, rows, H, D), generator=gen, device=device).to(tdt)
    v = torch.randn((L, rows, H, D), generator=gen, device=device).to(tdt)
    stream = torch.cuda.current_stream(device)
    rids = [rank * 1_000_000 + i for i in range(n)]
    from paper_2503_08461_b200 import _native

    times, launches = [], 0

    def step_once(timed):
        nonlocal launches
        hs = pool.allocate_batch(rids, specs, 0.0)
        torch.cuda.synchronize(device)
        l0 = _native.launch_count()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for layer in range(L):
            pool.write_prefill_kv(hs, layer, k[layer], v[layer])
        e1.record(stream)
        e1.synchronize()
        if timed:
            times.append(e0.elapsed_time(e1))
            launches += _native.launch_count() - l0
        pool.release_batch(hs, 1.0)

    for _ in range(args.warmup):
        step_once(False)
    with ClockSampler(device.index) as clocks:
        for _ in range(args.steps):
            step_once(True)
    ms = statistics.mean(times)
    max_ms = _allreduce(sum(times), "max", device)
    peak, peak_kind = measured_peak()
    moved = 2 * cap                                   # read the varlen K/V, write the blocks
    achieved = moved / (ms / 1e3) / 1e9
    return {
        "metric": "prefill KV ingested tokens/s", "value": rows * world * len(times) / (max_ms / 1e3),
        "unit": "tokens/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": max_ms / len(times), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f16", "data": "synthetic (random K/V)",
        "config": {"workload": f"c2p: {CONFIGS['c2p']}", "requests_per_gpu": n,
                   "timing": "CUDA events around the 32 per-layer write_prefill_kv calls"},
        "roofline": {"bound": "hbm", "kernel": "write_prefill_tma_kernel (TMA head-group tiles -> "
                                                 "whole-chunk bulk stores)", "achieved": achieved,
                     "peak": peak, "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak,
                     "traffic": _scaled_traffic("r02_c2p", moved),
                     "traffic_note": "DRAM bytes per step = the ncu traffic/algorithmic ratio of one "
                                     "layer's launch (profiles/ncu_r02_c2p.json) x the step's bytes",
                     "alg_bytes_per_step": moved},
        "gpu_launches": launches,
        "clocks": clocks.summary(),
    }


def run_ours(args, rank, world, local_rank):
    """The headline press config, then (default c2 run) the c3 / c4w legs in the same
    process, each with its own roofline, clocks and sampled parity."""
    import torch

    result = press_leg(args, args.config, rank, world, local_rank, with_e2e=args.e2e_steps > 0)
    legs = [x for x in args.legs.split(",") if x and x != args.config] if args.legs else []
    if legs:
        result["legs"] = {}
        for name in legs:
            gc.collect()                # pools and their handles reference each other
            torch.cuda.empty_cache()
            leg = press_leg(args, name, rank, world, local_rank, with_e2e=False)
            result["legs"][name] = {k: leg[k] for k in (
                "value", "unit", "ms_per_step", "scaling", "dtype", "config", "hbm_gbs_per_gpu",
                "kept_tokens_per_s", "roofline", "gpu_launches", "clocks", "parity", "paths")
                if k in leg}
    return result


def press_leg(args, name, rank, world, local_rank, with_e2e):
    """One press config: W warm-up + K timed compress_batch steps over a batch resident in the
    pool (CUDA events on the launch stream, max over ranks), then one untimed extra batch
    checked against the oracle on a sample of segments (``parity``)."""
    import torch

    from paper_2503_08461_b200 import KVCachePool, compressed_spec, kv_bytes

    from paper_2503_08461_b200 import shard

    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    cfg, dtype, specs, comp = workload(name)
    strong = name in STRONG
    job_kept = sum(compressed_spec(s, comp).total_tokens for s in specs) * (1 if strong else world)
    if strong:  # fixed total work, LPT-balanced request shards
        total_tokens = sum(s.total_tokens for s in specs)
        specs = [specs[i] for i in shard.lpt_shard([s.total_tokens for s in specs], world)[rank]]
    n = len(specs)
    raw_tokens = sum(s.total_tokens for s in specs)
    job_tokens = total_tokens if strong else raw_tokens * world
    cap = sum(kv_bytes(cfg, s.total_tokens) for s in specs)
    hq = Q_HEADS.get(name, cfg.num_kv_heads)
    pool = KVCachePool(cfg, cap, device=device, kv_dtype=dtype, max_handles=max(64, 2 * n),
                       max_tokens_per_handle=max(s.total_tokens for s in specs) + 64,
                       num_q_heads=hq, block_size=args.block_size)
    pool.set_profiling(True)
    ins = press_inputs(comp, cfg, n, device, torch, seed=1234 + rank, hq=hq)
    rids = [rank * 1_000_000 + i for i in range(n)]
    stream = torch.cuda.current_stream(device)

    def fill():
        hs = pool.allocate_batch(rids, specs, 0.0)
        pool.synth_fill(hs, seed=SYNTH_SEED)
        return hs

    press_ms, step_ms, launches, press_launches = [], [], 0, 0
    for i in range(args.warmup):
        hs = fill()
        pool.compress_batch(hs, comp, 1.0, **ins)
        pool.release_batch(hs, 2.0)
    torch.cuda.synchronize(device)
    if world > 1:
        torch.distributed.barrier()
    with ClockSampler(device.index) as clocks:
        for i in range(args.steps):
            hs = fill()
            ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            ev0.record(stream)
            pool.compress_batch(hs, comp, 1.0, **ins)
            ev1.record(stream)
            prof = pool.last_profile()
            ev1.synchronize()
            step_ms.append(ev0.elapsed_time(ev1))
            press_ms.append(prof["press_ms"])
            launches += prof["total_launches"]
            press_launches += prof["press_launches"]
            pool.release_batch(hs, 2.0)
        torch.cuda.synchronize(device)
    paths = pool.last_paths()
    if world > 1:
        torch.distributed.barrier()
    total_ms = sum(step_ms)
    max_ms = _allreduce(total_ms, "max", device)
    value = job_tokens * args.steps / (max_ms / 1e3)
    abytes = alg_bytes(cfg, specs, comp, Q_HEADS.get(name))
    peak, peak_kind = measured_peak()
    press_avg = statistics.mean(press_ms)
    achieved = abytes / (press_avg / 1e3) / 1e9
    kernel = {"chunk": "chunk_pool_kernel (reference compress_tensor fold into the blocks)",
              "knorm": "press_kernel<KNORM> (score + top-k + in-place compaction)",
              "snapkv": "snapkv_tc_kernel (tcgen05 window QK^T + softmax/pool + top-k + compaction)",
              "expected_attention": "ea_tc_kernel (tcgen05 K.[Sigma;mu] + softmax*|V| + top-k + "
                                    "compaction)"}.get(comp.press.value, "press kernel")
    result = {
        "metric": "compressed KV tokens/s",
        "value": value,
        "unit": "tokens/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": max_ms / args.steps,
        "higher_is_better": True,
        "scaling": "strong" if strong else "weak",
        "vs_baseline": None,
        "dtype": {"float16": "f16", "bfloat16": "bf16", "float32": "f32"}[dtype],
        "data": "synthetic (deterministic counter-based KV generator, oracle/synth.py)",
        "config": {
            "workload": f"{name}: {CONFIGS[name]}",
            "press": comp.press.value, "factor": comp.factor, "block_size": args.block_size,
            "requests_per_gpu": n,
            "raw_tokens_per_gpu": raw_tokens,
            "parallelism": f"request-sharded x{world} ({'LPT shards of one batch' if strong else 'one batch per GPU'}; no data-path collective)",
            "l2": "inputs larger than L2 (raw KV %.1f GB/GPU) and re-filled between steps"
                  % (cap / 1e9),
            "timing": "CUDA events on the launch stream around compress_batch, summed over steps",
        },
        "hbm_gbs_per_gpu": abytes * args.steps / (max_ms / 1e3) / 1e9,
        "kept_tokens_per_s": job_kept * args.steps / (max_ms / 1e3),
        "roofline": {
            "bound": "hbm", "kernel": kernel,
            "achieved": achieved, "peak": peak, "peak_kind": peak_kind, "unit": "GB/s",
            "frac": achieved / peak, "traffic": traffic_from_profile(name),
            "frac_of_nominal_8tbs": achieved / 8000.0,
            "peak_note": "peak = MEASURED_PEAKS.json hbm_gbs, a 1:1 read/write copy; the press "
                         "mix is read-heavy (Knorm 2:1), which HBM serves faster than a copy, so "
                         "frac can exceed 1 (ncu DRAM throughput is the cross-check)",
            "alg_bytes_per_step": abytes,
            "press_launches_per_step": press_launches / args.steps,
            "press_ms": press_avg,
        },
        "gpu_launches": launches,
        "paths": paths,
        "clocks": clocks.summary(),
    }
    if args.parity_segments > 0:
        result["parity"] = sampled_parity(pool, fill, specs, comp, ins, dtype, rids,
                                          args.parity_segments, device, world)
    if with_e2e:
        result["e2e"] = run_e2e(args, pool, cfg, dtype, specs, comp, ins, rids, device, world,
                                job_tokens)
    del pool
    return result


SYNTH_SEED = 17


def sampled_parity(pool, fill, specs, comp, ins, dtype, rids, n_segments, device, world):
    """Untimed: one more batch, compressed with indices + scores, checked on ``n_segments``
    sampled (request, layer, head) segments against the CPU oracle (oracle/parity.py, the
    checker only), summed over ranks."""
    import torch

    from oracle import parity
    from paper_2503_08461_b200 import PressKind

    hs = fill()
    want = comp.press is not PressKind.CHUNK      # the chunk fold has no scores / indices
    res = pool.compress_batch(hs, comp, 1.0, return_indices=want, return_scores=want, **ins)
    t0 = time.perf_counter()
    rep = parity.check_batch(pool, hs, specs, comp, res, dtype=dtype, seed=SYNTH_SEED, keys=rids,
                             inputs=ins, n_segments=n_segments)
    rep["check_s"] = time.perf_counter() - t0
    pool.verify_conservation()
    pool.release_batch(hs, 2.0)
    del res
    torch.cuda.synchronize(device)
    if world > 1:
        rep["segments"] = int(_allreduce(float(rep["segments"]), "sum", device))
        rep["mismatches"] = int(_allreduce(float(rep["mismatches"]), "sum", device))
        rep["max_score_rel_err"] = _allreduce(rep["max_score_rel_err"], "max", device)
    return rep


E2E_MAX_PINNED_BYTES = 64 * 10 ** 9


def run_e2e(args, pool, cfg, dtype, specs, comp, ins, rids, device, world, job_tokens):
    """Same metric through the public API with host buffers: every step hands the pool the
    batch's raw KV in pinned host memory (``compress_batch(host_kv=...)``) plus the press
    inputs (H2D), and reads the kept indices back (D2H)."""
    import torch

    from paper_2503_08461_b200 import PoolMode, PressKind, kv_bytes

    stream = torch.cuda.current_stream(device)
    # Pinned-host budget per rank: <= 64 GB and <= 40% of host RAM shared by the ranks of
    # this node. A batch above it is measured on its largest prefix that fits (the path is
    # PCIe-bound, so tokens/s per request does not depend on how many are in the batch).
    try:
        ram = os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES")
    except (ValueError, OSError):
        ram = 2 * E2E_MAX_PINNED_BYTES
    local_world = int(os.environ.get("LOCAL_WORLD_SIZE", "1"))
    budget = min(E2E_MAX_PINNED_BYTES, int(0.4 * ram) // max(1, local_world))
    m, acc = 0, 0
    for s_ in specs:
        b_ = kv_bytes(cfg, s_.total_tokens)
        if acc + b_ > budget:
            break
        acc += b_
        m += 1
    if m == 0:
        return {"value": None, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0,
                "skipped": f"one request's raw KV exceeds the {budget / 1e9:.0f} GB pinned budget"}
    sample = None if m == len(specs) else f"first {m} of {len(specs)} requests per rank " \
        f"({acc / 1e9:.1f} GB pinned; budget {budget / 1e9:.0f} GB)"
    specs, rids = specs[:m], rids[:m]
    ins = {k: v[:m].contiguous() for k, v in ins.items()}
    n = len(specs)
    shapes = [(cfg.num_layers, 2, cfg.num_kv_heads, s.total_tokens, cfg.head_dim) for s in specs]
    tdt = getattr(torch, dtype)
    hs = pool.allocate_batch(rids, specs, 0.0)
    pool.synth_fill(hs, seed=SYNTH_SEED)
    host = []
    for h, shp in zip(hs, shapes):
        buf = torch.empty(shp, dtype=tdt, pin_memory=True)
        buf.copy_(pool.load_tokens(h))
        host.append(buf)
    pool.release_batch(hs, 0.0)
    host_ins = {k: v.cpu().pin_memory() for k, v in ins.items()}
    dev_ins = {k: torch.empty_like(v) for k, v in ins.items()}
    split = pool.mode is PoolMode.POOLED and comp.press in (PressKind.KNORM, PressKind.SNAPKV)
    raw_bytes = sum(b.numel() * b.element_size() for b in host)
    kept_tokens = None
    kept_host = None
    times, d2h = [], 0
    for step in range(args.warmup + args.e2e_steps):
        hs = pool.allocate_batch(rids, specs, 0.0)
        torch.cuda.synchronize(device)
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        for k, v in host_ins.items():
            dev_ins[k].copy_(v, non_blocking=True)
        res = pool.compress_batch(hs, comp, 1.0, return_indices=True, host_kv=host, **dev_ins)
        flat = torch.cat([k.reshape(-1) for k in res.kept_idx])
        if kept_host is None:
            kept_host = torch.empty(flat.shape, dtype=flat.dtype, pin_memory=True)
        kept_host.copy_(flat, non_blocking=True)
        ev1.record(stream)
        ev1.synchronize()
        if step >= args.warmup:
            times.append(ev0.elapsed_time(ev1))
            d2h = kept_host.numel() * kept_host.element_size()
        kept_tokens = sum(h.spec.total_tokens for h in hs)
        pool.release_batch(hs, 2.0)
    max_ms = _allreduce(sum(times), "max", device)
    tokens = _allreduce(float(sum(s_.total_tokens for s_ in specs)), "sum", device) * len(times)
    bpt = cfg.bytes_per_token
    kv_h2d = (raw_bytes // 2 + kept_tokens * bpt // 2) if split else raw_bytes
    h2d = kv_h2d + sum(v.numel() * v.element_size() for v in host_ins.values())
    return {"value": tokens / (max_ms / 1e3), "unit": "tokens/s",
            "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
            "ms_per_step": max_ms / len(times),
            "pcie_gbs": (h2d + d2h) / (max_ms / len(times) / 1e3) / 1e9,
            "sample": sample,
            "path": ("pinned host KV -> compress_batch(host_kv=...): " +
                     ("K planes DMA (double-buffered staging) -> score/select/compact -> kept V "
                      "rows zero-copy from host" if split else "K+V DMA -> compress") +
                     "; press inputs H2D; kept indices D2H")}


def cpu_reference(args, cfg, dtype, specs, comp, reps: int | None = None):
    """The oracle port of the same pass, timed on the host cores (bounded sample)."""
    import numpy as np

    from oracle import cpu_pipeline
    from paper_2503_08461_b200 import PressKind

    workers = len(os.sched_getaffinity(0))
    s0 = specs[0]
    segs = [seg.token_count for seg in s0.segments]
    rng = np.random.default_rng(0)
    np_dt = {"float16": np.float16, "float32": np.float32, "bfloat16": np.float32}[dtype]
    kv = rng.standard_normal((cfg.num_layers, 2, cfg.num_kv_heads, s0.total_tokens, cfg.head_dim),
                             dtype=np.float32).astype(np_dt)
    if comp.press in (PressKind.SNAPKV, PressKind.EXPECTED_ATTENTION):
        return cpu_press_sample(cfg, dtype, specs, comp, workers)
    note = ""
    n_req = reps or workers
    r = cpu_pipeline.time_knorm_requests(kv, segs, comp.factor, n_req, workers,
                                         cfg.bytes_per_element)
    sample = (f"{n_req} requests x {cfg.num_layers} layers x {cfg.num_kv_heads} heads x "
              f"{s0.total_tokens} tokens (oracle/cpu_pipeline.knorm_compress_request: Knorm scores, "
              f"stable top-k, ascending K/V gather), one request per process, KV drawn once and "
              f"shared{note}")
    return {"value": r["tokens_per_s"], "unit": "tokens/s", "cores": r["workers"], "kind": "port",
            "sample": sample, "seconds": r["seconds"],
            "cpu_model": _cpu_model(),
            "literal_reference_path": literal_reference_path(cfg, kv, segs, comp)}


def cpu_press_sample(cfg, dtype, specs, comp, workers):
    """SnapKV / EA on the host: the oracle press (float64 scores, stable top-k, K/V gather)
    on a bounded sample of (layer, head) pairs of the batch's longest request, extrapolated
    to every (request, layer, head) of the batch."""
    import numpy as np

    from oracle import cpu_pipeline
    from paper_2503_08461_b200 import PressKind

    s0 = max(specs, key=lambda s: s.total_tokens)
    segs = [seg.token_count for seg in s0.segments]
    t_len, d = s0.total_tokens, cfg.head_dim
    rng = np.random.default_rng(0)
    np_dt = np.float16 if dtype == "float16" else np.float32
    k = rng.standard_normal((t_len, d), dtype=np.float32).astype(np_dt)
    v = rng.standard_normal((t_len, d), dtype=np.float32).astype(np_dt)
    if comp.press is PressKind.SNAPKV:
        kw = {"q_win": rng.standard_normal((1, comp.window, d)).astype(np.float32),
              "window": comp.window, "pool_kernel": comp.pool_kernel}
        kind = "snapkv"
    else:
        a = rng.standard_normal((1, d, d))
        kw = {"mean_q": rng.standard_normal((1, d)) / d ** 0.5, "cov_q": a @ a.transpose(0, 2, 1) / d,
              "n_sink": comp.n_sink}
        kind = "expected_attention"
    n_pairs = 4 * workers
    r = cpu_pipeline.time_press_pairs(k, v, segs, comp.factor, kind, n_pairs, workers, **kw)
    # every pair of the batch, scaled by length (the work is linear in T at fixed D)
    pairs_total = sum(s.total_tokens for s in specs) / t_len * cfg.num_layers * cfg.num_kv_heads
    secs = r["seconds_per_pair"] * pairs_total / r["workers"]
    tokens = sum(s.total_tokens for s in specs)
    return {"value": tokens / secs, "unit": "tokens/s", "cores": r["workers"], "kind": "port",
            "sample": f"{n_pairs} (layer, head) pairs of a {t_len}-token request "
                      f"(oracle/cpu_pipeline.press_compress_pair: {kind} float64 scores, stable "
                      f"top-K_r, K/V gather) on {r['workers']} processes, extrapolated linearly "
                      f"in tokens to the whole batch", "seconds": secs,
            "cpu_model": _cpu_model()}


def literal_reference_path(cfg, kv, segs, comp, layers: int = 2):
    """SURVEY.md §8(d) CPU path 1: the reference's own tensor compressor -- compress_tensor
    (MEAN_POOL, kv.py:211-239, restated in oracle/chunk.py) on every (layer, K|V, head,
    modality segment), one thread, timed on ``layers`` layers and extrapolated to L."""
    import numpy as np

    from oracle import chunk

    t0 = time.perf_counter()
    for layer in range(layers):
        for kvi in range(2):
            for head in range(cfg.num_kv_heads):
                start = 0
                for n in segs:
                    chunk.compress_tensor(kv[layer, kvi, head, start:start + n], comp.factor, "meanpool")
                    start += n
    secs = (time.perf_counter() - t0) * cfg.num_layers / layers
    tokens = kv.shape[3]
    return {"value": tokens / secs, "unit": "tokens/s", "cores": 1, "kind": "port",
            "sample": f"1 request x {layers} of {cfg.num_layers} layers x {cfg.num_kv_heads} heads x "
                      f"K|V x segments {list(segs)}, compress_tensor MEAN_POOL factor {comp.factor}, "
                      "extrapolated linearly to all layers"}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for ln in f:
                if ln.startswith("model name"):
                    return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


def run_reference(args):
    cfg, dtype, specs, comp = workload(args.config if args.config not in ("c5", "c2d", "c2p") else "c2")
    times = []
    last = None
    for i in range(args.warmup + args.steps):
        last = cpu_reference(args, cfg, dtype, specs, comp)
        if i >= args.warmup:
            times.append(last["seconds"])
    tokens = last["value"] * last["seconds"]
    value = tokens * len(times) / sum(times)
    cb = dict(last)
    cb["value"] = value
    return {
        "metric": "compressed KV tokens/s", "value": value, "unit": "tokens/s", "n_gpus": 0,
        "ranks": int(os.environ.get("WORLD_SIZE", "1")), "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * sum(times) / len(times), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f16" if dtype == "float16" else dtype,
        "data": "synthetic", "impl": "reference",
        "config": {"workload": f"{args.config}: {CONFIGS[args.config]}",
                   "note": "CPU reference arm: the reference has no tensor-level press "
                           "(SURVEY.md §0); this is the oracle port of the same pass"},
        "cpu_baseline": cb,
        "e2e": {"value": value, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }


def _free_port() -> int:
    import socket

    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        return sk.getsockname()[1]


def self_launch(args) -> int:
    """``--gpus N`` without a torchrun environment: re-exec this script as N ranks under
    ``torch.distributed.run`` (one process per GPU, NCCL). On a box with fewer GPUs than N
    the ranks share the visible GPUs over gloo (a multi-rank path check, flagged in the
    output). NCCL's INIT log (communicator size per rank) goes to stderr."""
    import subprocess

    import torch

    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    env.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if torch.cuda.device_count() < args.gpus:
        env["FASTCACHE_DIST_BACKEND"] = "gloo"
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={_free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c2", choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--block-size", type=int, default=16,
                    help="pool block size in tokens for the press configs (default 16)")
    ap.add_argument("--legs", default=None,
                    help="extra press configs measured in the same run (default for c2: c3,c4w)")
    ap.add_argument("--parity-segments", type=int, default=64,
                    help="sampled (request, layer, head) segments checked against the oracle "
                         "after the timed region (0 = off)")
    args = ap.parse_args()
    if args.legs is None:
        args.legs = "c3,c4w" if args.config == "c2" else ""
    if args.warmup < 3:
        raise SystemExit("--warmup must be >= 3")
    if args.gpus < 1:
        raise SystemExit("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(self_launch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}: launch one rank per GPU "
                         f"(torchrun --nproc-per-node {args.gpus}) or drop WORLD_SIZE")
    if args.impl == "reference":
        if rank == 0:
            print(json.dumps(run_reference(args)), flush=True)
        return
    import torch

    # FASTCACHE_DIST_BACKEND=gloo lets several ranks share one GPU (multi-rank path checks on
    # a box with fewer GPUs than ranks); the default is one rank per GPU over NCCL.
    backend = os.environ.get("FASTCACHE_DIST_BACKEND", "nccl")
    shared = torch.cuda.device_count() < world
    local_rank = local_rank % max(1, torch.cuda.device_count())
    if world > 1:
        torch.cuda.set_device(local_rank)
        if backend == "nccl":
            torch.distributed.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            torch.distributed.init_process_group(backend)
    if args.config == "c4":
        result = run_churn_bench(args, rank, world, local_rank)
    elif args.config == "c5":
        result = run_serving_bench(args, rank, world, local_rank)
    elif args.config == "c2d":
        result = run_decode_bench(args, rank, world, local_rank)
    elif args.config == "c2p":
        result = run_prefill_bench(args, rank, world, local_rank)
    else:
        result = run_ours(args, rank, world, local_rank)
    if world > 1:
        result.setdefault("config", {})["backend"] = backend
        if shared:
            result["config"]["shared_device"] = (
                f"{world} ranks on {torch.cuda.device_count()} visible GPU(s) over {backend}: a "
                "multi-rank path check, not a scaling number")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cfg, dtype, specs, comp = workload(args.config if args.config not in ("c5", "c2d", "c2p") else "c2")
        result["cpu_baseline"] = cpu_reference(args, cfg, dtype, specs, comp)
    if rank == 0:
        print(json.dumps(result), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
