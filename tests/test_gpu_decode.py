"""Decode over the compacted blocks, run with -m gpu.

After a batched compression, every step appends one token per request
(``append_decode_batch``, the reference's per-step append_decode_tokens loop,
engine.py:514-521), writes that token's K/V layer by layer
(``write_decode_kv``) and attends over the live cache (``decode_attention``).
Bar: the attention output matches a float64 torch reference computed from the
cache read back densely (``load_tokens``): within 1e-5 relative for fp32
pools, 2e-3 for fp16, 1e-2 for bf16 (output rounding), measured against the
output's scale; the written rows are bit copies; the ledger equals the
reference append sequence.
"""

import pytest
import torch

from paper_2503_08461_b200 import (
    CompressorSpec,
    KVCachePool,
    ModelConfig,
    PressKind,
    split_modalities,
)

pytestmark = pytest.mark.gpu

TOL = {"float32": 1e-5, "float16": 2e-3, "bfloat16": 1e-2}


def _reference(kv, q, scale):
    """kv [L, 2, H, T, D], q [Hq, D] -> per-layer [Hq, D] in float64."""
    L, _, H, T, D = kv.shape
    g = q.shape[0] // H
    k = kv[:, 0].double().repeat_interleave(g, dim=1)     # [L, Hq, T, D]
    v = kv[:, 1].double().repeat_interleave(g, dim=1)
    s = torch.einsum("hd,lhtd->lht", q.double(), k) * scale
    p = torch.softmax(s, dim=-1)
    return torch.einsum("lht,lhtd->lhd", p, v)


def _check(got, want, dtype):
    err = (got.double() - want).abs().max().item()
    scale = want.abs().max().item()
    assert err <= TOL[dtype] * max(scale, 1e-30), (err, scale)


@pytest.mark.parametrize("dtype,L,H,gq,D,specs,steps", [
    ("float16", 2, 4, 1, 128, [(576, 512)] * 6, 3),                    # LLaVA-shaped, no split
    ("float32", 2, 2, 1, 128, [(0, 8000), (0, 37)], 2),                # long context: split-KV
    ("bfloat16", 1, 2, 4, 64, [(100, 900), (0, 3), (17, 0)], 2),       # GQA g=4, D=64
    ("float16", 1, 8, 2, 128, [(576, t) for t in (64, 300, 960, 1)], 2),   # GQA g=2, varlen
    ("float32", 1, 2, 8, 64, [(0, 2500)], 1),                          # g=8, split
])
def test_decode_after_compress(cuda, dtype, L, H, gq, D, specs, steps):
    cfg = ModelConfig("m", L, H, D, 4 if dtype == "float32" else 2)
    hq = H * gq
    pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype=dtype,
                       max_handles=64, max_tokens_per_handle=8192 + 64, num_q_heads=hq)
    twin = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token)
    rs = [split_modalities(*s) for s in specs]
    hs = pool.allocate_batch(list(range(len(rs))), rs, 0.0)
    ts = twin.allocate_batch(list(range(len(rs))), rs, 0.0)
    pool.synth_fill(hs, seed=2)
    comp = CompressorSpec(factor=2, press=PressKind.KNORM)
    pool.compress_batch(hs, comp, 1.0)
    twin.compress_batch(ts, comp, 1.0)
    tdt = getattr(torch, dtype)
    gen = torch.Generator(device=cuda).manual_seed(0)
    n = len(hs)
    scale = D ** -0.5
    for step in range(steps):
        now = 2.0 + step
        pool.append_decode_batch(hs, 1, now)
        for h in ts:                                    # the reference loop
            twin.append_decode_tokens(h, 1, now)
        for layer in range(L):
            k = torch.randn((n, H, D), generator=gen, device=cuda).to(tdt)
            v = torch.randn((n, H, D), generator=gen, device=cuda).to(tdt)
            q = torch.randn((n, hq, D), generator=gen, device=cuda).to(tdt)
            pool.write_decode_kv(hs, layer, k, v)
            out = pool.decode_attention(hs, layer, q)
            for i, h in enumerate(hs):
                kv = pool.load_tokens(h)                # [L, 2, H, T, D]
                assert torch.equal(kv[layer, 0, :, -1], k[i]) and torch.equal(kv[layer, 1, :, -1], v[i])
                want = _reference(kv[layer:layer + 1], q[i], scale)[0]
                _check(out[i], want, dtype)
    assert pool.ledger == twin.ledger
    pool.verify_conservation()
    pool.release_batch(hs, 10.0)
    pool.verify_conservation()


def test_decode_explicit_positions_scale_and_errors(cuda):
    cfg = ModelConfig("m", 2, 2, 128, 2)
    pool = KVCachePool(cfg, 4096 * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=8, max_tokens_per_handle=1024, num_q_heads=2)
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 40), split_modalities(0, 70)], 0.0)
    pool.synth_fill(hs, seed=1)
    pool.compress_batch(hs, CompressorSpec(factor=2, press=PressKind.KNORM), 1.0)
    k = torch.randn((2, 2, 128), device=cuda).half()
    pool.write_decode_kv(hs, 1, k, k, positions=[0, 34])     # overwrite inside the cache
    kv0, kv1 = pool.load_tokens(hs[0]), pool.load_tokens(hs[1])
    assert torch.equal(kv0[1, 0, :, 0], k[0]) and torch.equal(kv1[1, 1, :, 34], k[1])
    q = torch.randn((2, 2, 128), device=cuda).half()
    out = pool.decode_attention(hs, 0, q, scale=0.01)
    _check(out[1], _reference(kv1[0:1], q[1], 0.01)[0], "float16")
    with pytest.raises(ValueError):
        pool.write_decode_kv(hs, 1, k, k, positions=[0, 35])  # outside the 35 live tokens
    with pytest.raises(ValueError):
        pool.decode_attention(hs, 2, q)                       # layer out of range
    with pytest.raises(ValueError):
        pool.decode_attention(hs, 0, q[:, :1].contiguous())   # wrong head count


def test_decode_more_requests_than_one_launch(cuda):
    """300 handles > kMaxDecode (256): the batch is split across launches."""
    cfg = ModelConfig("m", 1, 2, 64, 2)
    pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=512, max_tokens_per_handle=256, num_q_heads=2)
    rng = torch.Generator().manual_seed(0)
    lens = torch.randint(1, 120, (300,), generator=rng).tolist()
    hs = pool.allocate_batch(list(range(300)), [split_modalities(0, t) for t in lens], 0.0)
    pool.synth_fill(hs, seed=3)
    pool.compress_batch(hs, CompressorSpec(factor=2, press=PressKind.KNORM), 1.0)
    pool.append_decode_batch(hs, 1, 2.0)
    kv = torch.randn((300, 2, 64), device=cuda).half()
    pool.write_decode_kv(hs, 0, kv, kv)
    q = torch.randn((300, 2, 64), device=cuda).half()
    out = pool.decode_attention(hs, 0, q)
    for i in (0, 1, 255, 256, 299):
        cache = pool.load_tokens(hs[i])
        _check(out[i], _reference(cache[0:1], q[i], 64 ** -0.5)[0], "float16")
    pool.verify_conservation()
