"""Counter-based deterministic KV generator (oracle twin of the K8 CUDA kernel).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

Every element is a pure function of
``(seed, request key, layer, kv, head, token position, dim)`` built only from
64-bit integer hashing (splitmix64) and correctly-rounded IEEE float32
operations, so numpy here and ``synth_fill_kernel`` in
``paper_2503_08461_b200/csrc/fc_kernels.cu`` produce identical bits:

    req   = splitmix(seed ^ splitmix(key))
    head  = splitmix(req ^ (layer << 24 | kv << 23 | head))
    row   = splitmix(head ^ pos)
    e     = mix64(row + (dim + 1) * GAMMA)                (uint64, wrapping)
    s     = sum of the four 16-bit fields of e            (Irwin-Hall n=4)
    x     = f32(s - 131070) * f32(1 / 37837.227)          (~N(0, 1))
    scale = f32(0.5) + f32(f32(row >> 40) * 2^-24) * f32(1.5)   (dist SCALED)
          = 1                                                   (dist PLAIN)
    value = cast_dtype(x * scale)                          (round-to-nearest-even)

``SCALED`` ("realistic", well-separated norms: per-token scale in [0.5, 2))
and ``PLAIN`` ("hard", near-tie norms) are SURVEY.md §8(d)'s two KV
distributions, restated without transcendental functions so the CPU and the
GPU agree to the bit.
"""

from __future__ import annotations

import numpy as np

GAMMA = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)
INV_STD = np.float32(1.0 / 37837.227)
DIST_SCALED = 0
DIST_PLAIN = 1


def mix64(z):
    z = np.asarray(z, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
    return z ^ (z >> np.uint64(31))


def splitmix(z):
    with np.errstate(over="ignore"):
        return mix64(np.asarray(z, dtype=np.uint64) + GAMMA)


def _u64(v) -> np.uint64:
    return np.uint64(int(v) & 0xFFFFFFFFFFFFFFFF)


def f32_to_bf16_bits(x: np.ndarray) -> np.ndarray:
    """float32 -> bfloat16 bit pattern, round-to-nearest-even (finite inputs)."""
    u = np.asarray(x, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) >> np.uint32(16)
    return r.astype(np.uint16)


def bf16_bits_to_f32(b: np.ndarray) -> np.ndarray:
    return (np.asarray(b, dtype=np.uint16).astype(np.uint32) << np.uint32(16)).view(np.float32)


def head_values_f32(seed: int, key: int, layer: int, kv: int, head: int, n_tok: int, dim: int,
                    dist: int = DIST_SCALED, tok_begin: int = 0) -> np.ndarray:
    """float32 values (before the dtype cast) of one (layer, kv, head) segment: [n_tok, dim]."""
    req = splitmix(_u64(seed) ^ splitmix(_u64(key)))
    hs = splitmix(req ^ np.uint64((layer << 24) | (kv << 23) | head))
    pos = np.arange(tok_begin, tok_begin + n_tok, dtype=np.uint64)
    row = splitmix(hs ^ pos)                                   # [n_tok]
    d1 = (np.arange(dim, dtype=np.uint64) + np.uint64(1))
    with np.errstate(over="ignore"):
        e = mix64(row[:, None] + d1[None, :] * GAMMA)          # [n_tok, dim]
    m = np.uint64(0xFFFF)
    s = (e & m) + ((e >> np.uint64(16)) & m) + ((e >> np.uint64(32)) & m) + (e >> np.uint64(48))
    x = (s.astype(np.int64) - 131070).astype(np.float32) * INV_STD
    if dist == DIST_SCALED:
        a = (row >> np.uint64(40)).astype(np.float32) * np.float32(2.0 ** -24)
        scale = np.float32(0.5) + a * np.float32(1.5)
        x = x * scale[:, None]
    return x.astype(np.float32)


def cast_dtype(x: np.ndarray, dtype: str) -> np.ndarray:
    """Cast float32 values to the pool dtype's storage: returns the storage array.

    float16 -> np.float16, float32 -> np.float32, bfloat16 -> uint16 bit patterns.
    """
    if dtype == "float16":
        return x.astype(np.float16)
    if dtype == "float32":
        return x.astype(np.float32)
    if dtype == "bfloat16":
        return f32_to_bf16_bits(x)
    raise ValueError(f"unsupported dtype {dtype}")


def to_f32(stored: np.ndarray, dtype: str) -> np.ndarray:
    """Storage array -> float32 values (exact widening)."""
    if dtype == "bfloat16":
        return bf16_bits_to_f32(stored)
    return np.asarray(stored).astype(np.float32)


def head_values(seed: int, key: int, layer: int, kv: int, head: int, n_tok: int, dim: int,
                dtype: str, dist: int = DIST_SCALED) -> np.ndarray:
    """Stored values of one segment in the pool dtype (see ``cast_dtype``)."""
    return cast_dtype(head_values_f32(seed, key, layer, kv, head, n_tok, dim, dist), dtype)


def request_kv(seed: int, key: int, num_layers: int, num_kv_heads: int, n_tok: int, dim: int,
               dtype: str, dist: int = DIST_SCALED) -> np.ndarray:
    """Whole request, storage dtype, laid out [L][2][H][T][D] (the dense store layout)."""
    sample = head_values(seed, key, 0, 0, 0, 1, dim, dtype, dist)
    out = np.empty((num_layers, 2, num_kv_heads, n_tok, dim), dtype=sample.dtype)
    for layer in range(num_layers):
        for kv in range(2):
            for h in range(num_kv_heads):
                out[layer, kv, h] = head_values(seed, key, layer, kv, h, n_tok, dim, dtype, dist)
    return out
