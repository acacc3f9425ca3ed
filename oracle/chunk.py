"""Restatement of the reference chunk compressor (kv.py:197-239).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py). Pinned against golden
vectors produced by the reference itself (tests/golden/make_golden.py ->
tests/golden/chunk_golden.npz).

The device K7 kernel must be bit-exact with MEAN_POOL, so the numpy
semantics are restated explicitly (verified against the reference's
``values[a:b].mean(axis=0)`` by the golden vectors):

* accumulate dtype: float32 for float16 input (numpy's float16 mean uses
  float32 intermediates), float64 for integer/bool input, else the input dtype;
* rows of a chunk are added sequentially (axis-0 reduction of a C-contiguous
  block), then one IEEE true division by the row count in the accumulate
  dtype, then a cast to the input dtype;
* exception: a (m, 1) float32/float64 chunk is one contiguous run, which numpy
  reduces with its pairwise summation (8 interleaved partials for 8 <= m <= 128,
  recursive halving above) -- restated in ``_pairwise_sum``;
* SEEDED_LINEAR: the first m weights renormalised (w[:m] / w[:m].sum()), then
  ``w @ chunk`` in float64.
"""

from __future__ import annotations

import numpy as np

from .press import ceil_div


def chunk_weights(factor: int, map_kind: str, seed: int = 1234) -> np.ndarray:
    """kv.py:197-208."""
    if map_kind == "meanpool":
        w = np.full(factor, 1.0 / factor, dtype=np.float64)
    else:
        w = np.random.default_rng(seed).random(factor)
    return w / w.sum()


def mean_accumulate_dtype(dtype) -> np.dtype:
    dtype = np.dtype(dtype)
    if dtype == np.float16:
        return np.dtype(np.float32)
    if dtype.kind in "biu":
        return np.dtype(np.float64)
    return dtype


def _sequential_rows_sum(block: np.ndarray, acc: np.dtype) -> np.ndarray:
    s = block[0].astype(acc)
    for i in range(1, block.shape[0]):
        s = (s + block[i].astype(acc)).astype(acc)
    return s


def _pairwise_sum(a: np.ndarray) -> np.generic:
    """numpy's pairwise_sum (umath loops_utils) for a contiguous 1-D run."""
    n = a.shape[0]
    if n < 8:
        r = a.dtype.type(0)
        for v in a:
            r = a.dtype.type(r + v)
        return r
    if n <= 128:
        r = [a[j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = a.dtype.type(r[j] + a[i + j])
            i += 8
        res = a.dtype.type(a.dtype.type(a.dtype.type(r[0] + r[1]) + a.dtype.type(r[2] + r[3]))
                           + a.dtype.type(a.dtype.type(r[4] + r[5]) + a.dtype.type(r[6] + r[7])))
        while i < n:
            res = a.dtype.type(res + a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return a.dtype.type(_pairwise_sum(a[:n2]) + _pairwise_sum(a[n2:]))


def compress_tensor(values, factor: int, map_kind: str = "meanpool", seed: int = 1234) -> np.ndarray:
    """kv.py:211-239 restated."""
    values = np.asarray(values)
    if values.ndim != 2:
        raise ValueError("values must be a 2-D (tokens, dim) array")
    n = values.shape[0]
    if n == 0:
        raise ValueError("cannot compress an empty token sequence")
    k = factor
    rows = ceil_div(n, k)
    if map_kind == "meanpool":
        acc = mean_accumulate_dtype(values.dtype)
        out = np.empty((rows, values.shape[1]), dtype=values.dtype)
        for r in range(rows):
            block = values[r * k:min((r + 1) * k, n)]
            if block.shape[1] == 1 and block.dtype == acc and acc.kind == "f":
                s = np.array([_pairwise_sum(block[:, 0])], dtype=acc)
            else:
                s = _sequential_rows_sum(block, acc)
            out[r] = np.true_divide(s, acc.type(block.shape[0])).astype(acc)
        return out
    w_full = chunk_weights(factor, map_kind, seed)
    out = np.empty((rows, values.shape[1]), dtype=np.float64)
    for r in range(rows):
        block = values[r * k:min((r + 1) * k, n)]
        w = w_full[:block.shape[0]]
        w = w / w.sum()
        out[r] = w @ block
    return out


def segment_weights(factor: int, map_kind: str, seed: int, m: int) -> np.ndarray:
    """Weights the reference applies to a chunk of m <= factor rows (fp64)."""
    w = chunk_weights(factor, map_kind, seed)[:m]
    return w / w.sum()
