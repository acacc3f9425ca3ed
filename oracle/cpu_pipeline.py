"""Vectorised CPU restatement of one compression pass (the timed CPU reference arm).

TEST / BASELINE INFRASTRUCTURE ONLY (see oracle/__init__.py): bench.py times
this as ``cpu_baseline`` (kind "port") and as ``--impl reference``; tests
check it equals the per-segment oracle (tests/test_oracle_pipeline.py).

The reference has no tensor-level press: its compression
stage is a cost formula plus ``compressed_spec`` + ``transition_compressed``
(engine.py:501-510). This is the same algorithm the GPU runs -- Knorm scores
with the restated summation order, stable (score desc, index asc) top-K_r,
ascending gather of K and V -- written for a CPU: one vectorised pass over a
whole request [L, 2, H, T, D].
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import press


def knorm_compress_request(kv: np.ndarray, seg_tokens, factor: int, bytes_per_element: int = 2):
    """kv: [L, 2, H, T, D] stored dtype -> (kept [L, H, K_r] int32, compacted [L, 2, H, K_r, D])."""
    n_layers, _, n_heads, t_len, d = kv.shape
    k_r = press.kept_budget(seg_tokens, factor)
    keys = kv[:, 0].astype(np.float32).reshape(-1, d)
    scores = press.knorm_scores(keys, bytes_per_element).reshape(n_layers * n_heads, t_len)
    ikeys = press.float_keys(scores).astype(np.int64)
    order = np.argsort(-ikeys, axis=1, kind="stable")[:, :k_r]
    kept = np.sort(order, axis=1).astype(np.int32).reshape(n_layers, n_heads, k_r)
    idx = kept[:, None, :, :, None]
    compacted = np.take_along_axis(kv, np.broadcast_to(idx, (n_layers, 2, n_heads, k_r, 1)), axis=3)
    return kept, compacted


def _worker(args):
    kv, seg_tokens, factor, bpe, reps = args
    t0 = time.perf_counter()
    for _ in range(reps):
        knorm_compress_request(kv, seg_tokens, factor, bpe)
    return time.perf_counter() - t0


_SHARED = {}


def _forked_worker(reps):
    kv, seg_tokens, factor, bpe = _SHARED["job"]
    t0 = time.perf_counter()
    for _ in range(reps):
        knorm_compress_request(kv, seg_tokens, factor, bpe)
    return time.perf_counter() - t0


def time_knorm_requests(kv: np.ndarray, seg_tokens, factor: int, n_requests: int,
                        workers: int | None = None, bytes_per_element: int = 2) -> dict:
    """Time ``n_requests`` independent request compressions on ``workers`` processes.

    Every request reuses the same KV array (forked, copy-on-write): the cost of
    the pass does not depend on the values. Returns the wall time of the
    slowest worker and the derived input-token throughput.
    """
    import multiprocessing as mp

    workers = workers or len(os.sched_getaffinity(0))
    workers = max(1, min(workers, n_requests))
    reps = [n_requests // workers + (1 if i < n_requests % workers else 0) for i in range(workers)]
    _SHARED["job"] = (kv, list(seg_tokens), factor, bytes_per_element)
    t0 = time.perf_counter()
    if workers == 1:
        times = [_forked_worker(reps[0])]
    else:
        ctx = mp.get_context("fork")
        with ctx.Pool(workers) as pool:
            times = pool.map(_forked_worker, reps)
    wall = time.perf_counter() - t0
    tokens = n_requests * kv.shape[3]
    return {"seconds": max(times), "wall_s": wall, "workers": workers, "tokens": tokens,
            "tokens_per_s": tokens / max(times)}


# ---------------------------------------------------------------------------
# SnapKV / ExpectedAttention: the press itself on a sample of (layer, head) pairs
# ---------------------------------------------------------------------------


def press_compress_pair(k_rows, v_rows, seg_tokens, factor: int, press_kind: str, *,
                        q_win=None, mean_q=None, cov_q=None, window: int = 32,
                        pool_kernel: int = 7, n_sink: int = 4):
    """One (request, layer, kv-head): oracle scores (float64), stable top-K_r, K/V gather."""
    kf = k_rows.astype(np.float32)
    if press_kind == "snapkv":
        s = press.snapkv_scores(kf, q_win, window, pool_kernel)
    else:
        s = press.expected_attention_scores(kf, v_rows.astype(np.float32), mean_q, cov_q, n_sink)
    kept = press.select(s, seg_tokens, factor)
    return kept, k_rows[kept], v_rows[kept]


def _pair_worker(reps):
    args, kw = _SHARED["pair"]
    t0 = time.perf_counter()
    for _ in range(reps):
        press_compress_pair(*args, **kw)
    return time.perf_counter() - t0


def time_press_pairs(k_rows, v_rows, seg_tokens, factor: int, press_kind: str, n_pairs: int,
                     workers: int | None = None, **kw) -> dict:
    """Time ``n_pairs`` (layer, head) compressions of one request shape on ``workers``
    processes; returns seconds per pair (slowest worker x workers / pairs)."""
    import multiprocessing as mp

    workers = workers or len(os.sched_getaffinity(0))
    workers = max(1, min(workers, n_pairs))
    reps = [n_pairs // workers + (1 if i < n_pairs % workers else 0) for i in range(workers)]
    _SHARED["pair"] = ((k_rows, v_rows, list(seg_tokens), factor, press_kind), kw)
    if workers == 1:
        times = [_pair_worker(reps[0])]
    else:
        with mp.get_context("fork").Pool(workers) as pool:
            times = pool.map(_pair_worker, reps)
    return {"seconds": max(times), "workers": workers, "pairs": n_pairs,
            "seconds_per_pair": max(times) / max(reps)}
