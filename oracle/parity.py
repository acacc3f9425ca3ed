"""Sampled oracle check of a full-size compress batch (the parity leg of bench.py and of
the BASELINE-scale GPU tests).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py): this module is the checker that
runs AFTER a timed region, never inside it, and nothing in the product package
imports it.

A BASELINE-scale batch (c2: 32 requests x 32 layers x 32 heads; c4w: 64 requests of
up to 8k tokens) is far too large to regenerate and re-score whole on the CPU. The
raw KV came from the counter-based generator (``synth``), so any single
(request, layer, kv-head) segment can be regenerated bit for bit from
``(seed, request key, layer, kv, head)``. This module draws a deterministic sample of
such segments -- always including the first and last layer and head of the longest
and the shortest request, plus seeded random picks -- and checks, per segment, with
the bars of SURVEY.md §8(c) / the BASELINE.json north star:

* scores: Knorm bit-exact against ``press.knorm_scores`` (the kernel's fp32 order);
  SnapKV / ExpectedAttention within ``rtol`` (1e-5) of the float64 oracle, forced
  keeps (+inf) in the same places;
* kept indices: Knorm exactly ``press.select``; SnapKV / EA the oracle set up to
  tolerated boundary swaps (``press.kept_set_mismatch``);
* compacted payload: the K and V rows now stored at ranks 0..K_r-1 are bit copies of
  the regenerated raw rows the GPU selected;
* the reference chunk compressor (MEAN_POOL / SEEDED_LINEAR folded into the pool): the
  stored rows equal ``chunk.compress_tensor`` of each modality segment (pinned to the
  reference's own golden vectors) -- bit-exact for MEAN_POOL on fp16/fp32, within 1e-2
  (bf16) / 1e-6 (fp32) for SEEDED_LINEAR, whose reference output is float64.
"""

from __future__ import annotations

import numpy as np

from . import chunk as ochunk
from . import press as opress
from . import synth as osynth


def sample_segments(lengths, num_layers: int, num_heads: int, n: int, seed: int = 0):
    """Deterministic (request, layer, head) triples: corners first, then seeded picks."""
    order = sorted(range(len(lengths)), key=lambda i: (-lengths[i], i))
    picks = []
    for r in dict.fromkeys((order[0], order[-1])):
        for layer in dict.fromkeys((0, num_layers - 1)):
            for head in dict.fromkeys((0, num_heads - 1)):
                picks.append((r, layer, head))
    rng = np.random.default_rng(seed)
    seen = set(picks)
    while len(picks) < n and len(seen) < len(lengths) * num_layers * num_heads:
        t = (int(rng.integers(len(lengths))), int(rng.integers(num_layers)),
             int(rng.integers(num_heads)))
        if t not in seen:
            seen.add(t)
            picks.append(t)
    return picks


def _stored_rows(pool, handle, layer, head, n):
    """Ranks 0..n-1 of (layer, head) straight from the paged layer view: [2, n, D]."""
    import torch

    cache = pool.kv_cache(layer)                   # [NB, 2, H, bs, D]
    bs = cache.shape[3]
    j = torch.arange(n, device=cache.device)
    seg = cache[handle.block_table.long()[j // bs], :, head, j % bs].transpose(0, 1).contiguous()
    if seg.dtype == torch.bfloat16:
        seg = seg.view(torch.int16)
    return seg.cpu().numpy()


def _check_chunk_rows(pool, handle, layer, head, k_st, v_st, seg_tokens, comp, dtype):
    kind = comp.map_kind.value
    got = _stored_rows(pool, handle, layer, head, opress.kept_budget(seg_tokens, comp.factor))
    for kv, raw in ((0, k_st), (1, v_st)):
        src = osynth.to_f32(raw, dtype) if dtype == "bfloat16" else raw
        parts, start = [], 0
        for n in (x for x in seg_tokens if x > 0):
            parts.append(ochunk.compress_tensor(src[start:start + n], comp.factor, kind, comp.seed))
            start += n
        want = np.concatenate(parts)
        if kind == "meanpool" and dtype != "bfloat16":
            if not np.array_equal(got[kv].view(np.uint8), want.astype(raw.dtype).view(np.uint8)):
                return f"{'KV'[kv]} rows differ from compress_tensor"
        else:
            g32 = osynth.to_f32(got[kv], dtype)
            w32 = osynth.to_f32(osynth.cast_dtype(want.astype(np.float32), dtype), dtype)
            tol = 1e-6 if dtype == "float32" else 1e-2
            if not np.allclose(g32, w32, rtol=tol, atol=1e-6):
                return f"{'KV'[kv]} rows beyond {tol} of compress_tensor"
    return None


def check_batch(pool, handles, raw_specs, comp, result, *, dtype: str, seed: int, keys,
                inputs: dict | None = None, n_segments: int = 64, rtol: float = 1e-5,
                dist: int = osynth.DIST_SCALED, sample_seed: int = 0) -> dict:
    """Check ``n_segments`` sampled segments of one compressed batch against the oracle.

    ``handles`` were filled by ``pool.synth_fill(handles, seed=seed, keys=keys)`` and then
    compressed with ``result = pool.compress_batch(..., return_indices=True,
    return_scores=True)``. ``raw_specs`` are the specs before compression. Returns
    ``{"segments": checked, "mismatches": m, "max_score_rel_err": e, "failures": [...]}``.
    """
    import torch

    from paper_2503_08461_b200 import PressKind

    cfg = pool.config
    L, H, D = cfg.num_layers, cfg.num_kv_heads, cfg.head_dim
    hq = pool.num_q_heads
    g = hq // H
    bpe = cfg.bytes_per_element
    inputs = inputs or {}
    lengths = [s.total_tokens for s in raw_specs]
    picks = sample_segments(lengths, L, H, n_segments, sample_seed)
    chunk_kind = comp.press is PressKind.CHUNK
    by_req: dict[int, list] = {}
    for r, layer, head in picks:
        by_req.setdefault(r, []).append((layer, head))
    failures, max_rel = [], 0.0
    torch.cuda.synchronize()
    for r, segs in sorted(by_req.items()):
        spec = raw_specs[r]
        t_len = spec.total_tokens
        seg_tokens = [s.token_count for s in spec.segments]
        k_r = opress.kept_budget(seg_tokens, comp.factor)
        scores_r = None if chunk_kind else result.scores[r]
        kept_r = None if chunk_kind else result.kept_idx[r]
        for layer, head in segs:
            tag = f"req {r} layer {layer} head {head}"
            k_st = osynth.head_values(seed, keys[r], layer, 0, head, t_len, D, dtype, dist)
            v_st = osynth.head_values(seed, keys[r], layer, 1, head, t_len, D, dtype, dist)
            k32, v32 = osynth.to_f32(k_st, dtype), osynth.to_f32(v_st, dtype)
            if chunk_kind:
                why = _check_chunk_rows(pool, handles[r], layer, head, k_st, v_st, seg_tokens,
                                        comp, dtype)
                if why:
                    failures.append(f"{tag}: {why}")
                continue
            got_s = scores_r[layer, head].cpu().numpy()
            got_k = kept_r[layer, head].cpu().numpy().astype(np.int64)
            if comp.press is PressKind.KNORM:
                want = opress.knorm_scores(k32, bpe)
                if not np.array_equal(got_s, want):
                    failures.append(f"{tag}: Knorm scores differ")
                want_k = opress.select(want, seg_tokens, comp.factor, comp.per_segment)
                if not np.array_equal(got_k, want_k):
                    failures.append(f"{tag}: Knorm kept set differs")
            else:
                sl = slice(head * g, (head + 1) * g)
                if comp.press is PressKind.SNAPKV:
                    q = inputs["q_window"][r, layer, sl].float().cpu().numpy()
                    want = opress.snapkv_scores(k32, q, comp.window, comp.pool_kernel)
                else:
                    mu = inputs["mean_q"][r, layer, sl].cpu().numpy()
                    cov = inputs["cov_q"][r, layer, sl].cpu().numpy()
                    want = opress.expected_attention_scores(k32, v32, mu, cov, comp.n_sink)
                got64 = got_s.astype(np.float64)
                fin = np.isfinite(want)
                if not np.array_equal(np.isfinite(got64), fin):
                    failures.append(f"{tag}: forced-keep positions differ")
                elif fin.any():
                    rel = float((np.abs(got64[fin] - want[fin]) / np.abs(want[fin])).max())
                    max_rel = max(max_rel, rel)
                    if rel > rtol:
                        failures.append(f"{tag}: score rel err {rel:.3g} > {rtol}")
                if comp.per_segment:
                    start = 0
                    for n_seg in (n for n in seg_tokens if n > 0):
                        part = got_k[(got_k >= start) & (got_k < start + n_seg)] - start
                        why = opress.kept_set_mismatch(part, want[start:start + n_seg],
                                                       opress.ceil_div(n_seg, comp.factor), rtol)
                        if why:
                            failures.append(f"{tag}: {why}")
                        start += n_seg
                else:
                    why = opress.kept_set_mismatch(got_k, want, k_r, rtol)
                    if why:
                        failures.append(f"{tag}: {why}")
            if got_k.shape[0] != k_r or got_k.min(initial=0) < 0 or got_k.max(initial=0) >= t_len:
                failures.append(f"{tag}: kept indices out of range")
                continue
            # ranks 0..K_r-1 of this (layer, head), read straight from the paged layer view
            cache = pool.kv_cache(layer)                   # [NB, 2, H, bs, D]
            bs = cache.shape[3]
            j = torch.arange(k_r, device=cache.device)
            blocks = handles[r].block_table.long()
            seg = cache[blocks[j // bs], :, head, j % bs].transpose(0, 1).contiguous()
            if seg.dtype == torch.bfloat16:
                seg = seg.view(torch.int16)
            got_rows = seg.cpu().numpy()
            want_rows = np.stack([k_st[got_k], v_st[got_k]])
            if not np.array_equal(got_rows.view(np.uint8), want_rows.view(np.uint8)):
                failures.append(f"{tag}: compacted K/V rows are not bit copies")
    checked = len(picks)
    bad = len({f.split(":")[0] for f in failures})
    return {"segments": checked, "mismatches": bad, "max_score_rel_err": max_rel,
            "failures": failures[:8], "rtol": rtol,
            "sample": f"{checked} (request, layer, kv-head) segments of {len(raw_specs)} requests "
                      f"(corners of the longest/shortest request + seeded picks), regenerated "
                      f"from the counter-based generator (seed {seed})"}
