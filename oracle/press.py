"""CPU restatement of the batched presses, the top-k and the compaction.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Parity status: the press formulas follow NVIDIA kvpress as restated in
SURVEY.md Appendix A. kvpress is not in /root/reference (no vendored copy, no
pinned version, no call site; the paper cites it at PAPER.md:55,101,113,297),
so these scores are **parity unpinned by the reference**; tests/ pins them
with known-answer tests. What the reference *does* pin is the budget:
K_r = compressed_spec(spec, CompressorSpec(factor=k)).total_tokens, i.e.
sum over modality segments of ceil(n_seg / k) (reference
pkg/src/kvservesim/kv.py:169-194).

Deliberate deviations from kvpress (documented in DESIGN.md):
* kept indices are emitted ascending (kvpress gathers in score order), so the
  cache keeps sequence order;
* forced-keep tokens (SnapKV window, EA sinks) score +inf instead of max(s);
* the SnapKV window attention stays fp32 through the mean (kvpress casts the
  softmax back to the model dtype before the mean).
"""

from __future__ import annotations

import math

import numpy as np

from . import synth

# ---------------------------------------------------------------------------
# budget (reference ceil rule)
# ---------------------------------------------------------------------------


def ceil_div(n: int, k: int) -> int:
    """kv.py:169-170."""
    return -(-n // k)


def kept_budget(seg_tokens, factor: int) -> int:
    """K_r = sum_seg ceil(n_seg / factor) (kv.py:185-193)."""
    return sum(ceil_div(int(n), factor) for n in seg_tokens if int(n) > 0)


# ---------------------------------------------------------------------------
# ordering and top-k
# ---------------------------------------------------------------------------


def float_keys(scores: np.ndarray) -> np.ndarray:
    """Order-preserving uint32 keys of float32 scores (larger score -> larger key).

    Same transform as the device radix select: negative floats are bit-inverted,
    non-negative floats get the sign bit set. (-0.0 sorts just below +0.0.)
    """
    u = np.ascontiguousarray(scores, dtype=np.float32).view(np.uint32)
    neg = (u & np.uint32(0x80000000)) != 0
    return np.where(neg, ~u, u | np.uint32(0x80000000)).astype(np.uint32)


def topk_ascending(scores: np.ndarray, k: int) -> np.ndarray:
    """Indices of the k best tokens by (score desc, index asc), returned ascending."""
    scores = np.asarray(scores, dtype=np.float32)
    if k >= scores.shape[0]:
        return np.arange(scores.shape[0], dtype=np.int32)
    keys = float_keys(scores).astype(np.int64)
    order = np.argsort(-keys, kind="stable")  # stable: ties keep index order
    return np.sort(order[:k]).astype(np.int32)


def select(scores: np.ndarray, seg_tokens, factor: int, per_segment: bool = False) -> np.ndarray:
    """Kept positions of one (request, layer, kv-head): ascending int32, length K_r."""
    segs = [int(n) for n in seg_tokens if int(n) > 0]
    if not per_segment:
        return topk_ascending(scores, kept_budget(segs, factor))
    out, start = [], 0
    for n in segs:
        out.append(topk_ascending(scores[start:start + n], ceil_div(n, factor)) + start)
        start += n
    return np.concatenate(out).astype(np.int32)


# ---------------------------------------------------------------------------
# Knorm
# ---------------------------------------------------------------------------


def knorm_lane_layout(head_dim: int, bytes_per_element: int) -> tuple[int, int, int]:
    """(lanes per row, 16-byte vectors per lane, elements per vector) of the device kernel.

    A row of D elements is read as D*bpe/16 16-byte vectors; min(that, 32) lanes
    share a row, each accumulating its vectors in order.
    """
    vecs = head_dim * bytes_per_element // 16
    lpr = min(vecs, 32)
    return lpr, vecs // lpr, 16 // bytes_per_element


def knorm_scores(k_rows_f32: np.ndarray, bytes_per_element: int) -> np.ndarray:
    """s_t = -||K_t||_2 in float32 with the device kernel's exact summation order.

    Lane j of a row accumulates x*x (each product rounded to fp32, then an fp32
    add; no FMA) over elements d = (j + v*LPR)*EPV + e for v, then e ascending;
    the LPR lane partials are combined by an xor butterfly (offsets LPR/2..1);
    then sqrt (correctly rounded) and negation. For fp16/bf16 inputs every x*x
    is exact in fp32, so only the add order matters.
    """
    x = np.asarray(k_rows_f32, dtype=np.float32)
    t, d = x.shape
    lpr, vpl, epv = knorm_lane_layout(d, bytes_per_element)
    sq = x * x                                            # fp32, rounded
    sq = sq.reshape(t, vpl, lpr, epv).transpose(0, 2, 1, 3).reshape(t, lpr, vpl * epv)
    acc = sq[:, :, 0].copy()
    for i in range(1, vpl * epv):
        acc = acc + sq[:, :, i]
    lanes = np.arange(lpr)
    off = lpr // 2
    while off >= 1:
        acc = acc + acc[:, lanes ^ off]
        off //= 2
    return (-np.sqrt(acc[:, 0])).astype(np.float32)


def knorm_scores_naive(k_rows_f32: np.ndarray) -> np.ndarray:
    """float64 -||K_t|| (order-independent truth for tolerance checks)."""
    x = np.asarray(k_rows_f32, dtype=np.float64)
    return -np.sqrt((x * x).sum(axis=1))


# ---------------------------------------------------------------------------
# SnapKV
# ---------------------------------------------------------------------------


def snapkv_scores(k_rows_f32: np.ndarray, q_win_f32: np.ndarray, window: int,
                  pool_kernel: int) -> np.ndarray:
    """SnapKV score of one (request, layer, kv-head); float64 truth.

    k_rows: [T, D]; q_win: [g, w, D] post-RoPE queries of the last w positions
    of the g query heads sharing this kv-head.
      a[j, t] = Q_j . K_t / sqrt(D), masked to -inf for t > T - w + j
      A = softmax_t(a)                          (over all T)
      s'[t] = mean_j A[j, t]                   for t < T - w
      s'' = avg_pool1d(s', p, stride 1, zero pad p//2, divide by p)
      s = mean over the g heads; s[t >= T - w] = +inf (forced keep)
    """
    k = np.asarray(k_rows_f32, dtype=np.float64)
    q = np.asarray(q_win_f32, dtype=np.float64)
    t_len, d = k.shape
    g, w, _ = q.shape
    if w != window:
        raise ValueError("q_win window mismatch")
    if t_len <= window:
        raise ValueError("SnapKV needs more tokens than the observation window")
    logits = np.einsum("gjd,td->gjt", q, k) / math.sqrt(d)
    j = np.arange(w)[:, None]
    tt = np.arange(t_len)[None, :]
    logits = np.where(tt > (t_len - w + j), -np.inf, logits)
    logits = logits - logits.max(axis=-1, keepdims=True)
    p = np.exp(logits)
    p = p / p.sum(axis=-1, keepdims=True)
    s1 = p[:, :, : t_len - w].mean(axis=1)                # [g, T - w]
    pad = pool_kernel // 2
    padded = np.pad(s1, ((0, 0), (pad, pad)))
    s2 = np.zeros_like(s1)
    for o in range(pool_kernel):
        s2 += padded[:, o:o + t_len - w]
    s2 /= pool_kernel
    s = s2.mean(axis=0)
    return np.concatenate([s, np.full(w, np.inf)])


# ---------------------------------------------------------------------------
# ExpectedAttention
# ---------------------------------------------------------------------------


def expected_attention_scores(k_rows_f32: np.ndarray, v_rows_f32: np.ndarray,
                              mean_q: np.ndarray, cov_q: np.ndarray, n_sink: int) -> np.ndarray:
    """ExpectedAttention score of one (request, layer, kv-head); float64 truth.

    mean_q: [g, D], cov_q: [g, D, D].
      z_t = mu . K_t / sqrt(D) + K_t^T Sigma K_t / (2 D)        for t >= n_sink
      p = softmax over t in [n_sink, T); s_t = mean_g(p_t) * ||V_t||_2
      s[t < n_sink] = +inf (forced keep)
    """
    k = np.asarray(k_rows_f32, dtype=np.float64)
    v = np.asarray(v_rows_f32, dtype=np.float64)
    mu = np.asarray(mean_q, dtype=np.float64)
    cov = np.asarray(cov_q, dtype=np.float64)
    t_len, d = k.shape
    if t_len <= n_sink:
        raise ValueError("ExpectedAttention needs more tokens than n_sink")
    ks = k[n_sink:]
    z = ks @ mu.T / math.sqrt(d)                          # [T', g]
    z = z + np.einsum("td,gde,te->tg", ks, cov, ks) / d / 2.0
    z = z - z.max(axis=0, keepdims=True)
    p = np.exp(z)
    p = p / p.sum(axis=0, keepdims=True)
    s = p.mean(axis=1) * np.sqrt((v[n_sink:] ** 2).sum(axis=1))
    return np.concatenate([np.full(n_sink, np.inf), s])


# ---------------------------------------------------------------------------
# whole-request driver
# ---------------------------------------------------------------------------


def compress_request(kv_f32: np.ndarray, seg_tokens, factor: int, press: str, *,
                     bytes_per_element: int = 2, q_win=None, mean_q=None, cov_q=None,
                     window: int = 32, pool_kernel: int = 7, n_sink: int = 4,
                     per_segment: bool = False):
    """Oracle of one request: kv_f32 [L][2][H][T][D] (float32-widened storage).

    Returns (scores [L][H][T] float64/32, kept [L][H][K_r] int32). q_win is
    [L][Hq][w][D]; mean_q [L][Hq][D]; cov_q [L][Hq][D][D].
    """
    n_layers, _, n_heads, t_len, d = kv_f32.shape
    k_r = kept_budget(seg_tokens, factor)
    scores = np.zeros((n_layers, n_heads, t_len), dtype=np.float64)
    kept = np.zeros((n_layers, n_heads, k_r), dtype=np.int32)
    for layer in range(n_layers):
        for h in range(n_heads):
            kr = kv_f32[layer, 0, h]
            if press == "knorm":
                s = knorm_scores(kr, bytes_per_element)
            elif press == "snapkv":
                g = q_win.shape[1] // n_heads
                s = snapkv_scores(kr, q_win[layer, h * g:(h + 1) * g], window, pool_kernel)
            elif press == "expected_attention":
                g = mean_q.shape[1] // n_heads
                s = expected_attention_scores(kr, kv_f32[layer, 1, h],
                                              mean_q[layer, h * g:(h + 1) * g],
                                              cov_q[layer, h * g:(h + 1) * g], n_sink)
            else:
                raise ValueError(f"unknown press {press}")
            scores[layer, h] = s
            kept[layer, h] = select(np.asarray(s, dtype=np.float32), seg_tokens, factor,
                                    per_segment)
    return scores, kept


def gather_kept(kv_stored: np.ndarray, kept: np.ndarray) -> np.ndarray:
    """Compacted cache [L][2][H][K][D]: K'_j = K[idx_j], V'_j = V[idx_j] (bit copies)."""
    n_layers, _, n_heads, _, _ = kv_stored.shape
    out = np.empty(kv_stored.shape[:3] + (kept.shape[-1], kv_stored.shape[-1]),
                   dtype=kv_stored.dtype)
    for layer in range(n_layers):
        for h in range(n_heads):
            out[layer, :, h] = kv_stored[layer, :, h][:, kept[layer, h]]
    return out


# ---------------------------------------------------------------------------
# tolerance-aware kept-set check
# ---------------------------------------------------------------------------


def kept_set_mismatch(gpu_kept: np.ndarray, oracle_scores: np.ndarray, k: int,
                      rtol: float) -> str | None:
    """None if the GPU kept set is the oracle's up to tolerated boundary swaps.

    A swap is tolerated only when both tokens' oracle scores lie within
    rtol * max(|tau|, tiny) of the K-th boundary score tau. Otherwise returns a
    human-readable reason.
    """
    s = np.asarray(oracle_scores, dtype=np.float64)
    g = np.asarray(gpu_kept, dtype=np.int64)
    if g.shape[0] != k:
        return f"kept {g.shape[0]} rows, expected {k}"
    if np.any(np.diff(g) <= 0):
        return "kept indices not strictly ascending"
    o = topk_ascending(s.astype(np.float32), k).astype(np.int64) if k < s.shape[0] else \
        np.arange(s.shape[0])
    extra = np.setdiff1d(g, o)
    if extra.size == 0:
        return None
    missing = np.setdiff1d(o, g)
    finite = s[np.isfinite(s)]
    order = np.sort(s)[::-1]
    tau = order[k - 1]
    if not np.isfinite(tau):
        return f"swap across a forced-keep boundary: extra {extra[:4]}, missing {missing[:4]}"
    band = rtol * max(abs(tau), np.abs(finite).max() * 1e-30 if finite.size else 0.0, 1e-30)
    bad_extra = extra[s[extra] < tau - band]
    bad_missing = missing[s[missing] > tau + band]
    if bad_extra.size or bad_missing.size:
        return (f"kept-set differs beyond tolerance: extra {bad_extra[:4]} "
                f"(scores {s[bad_extra[:4]]}), missing {bad_missing[:4]} "
                f"(scores {s[bad_missing[:4]]}), tau {tau}")
    return None


def stored_to_f32(stored: np.ndarray, dtype: str) -> np.ndarray:
    return synth.to_f32(stored, dtype)
