"""P.Store: the prefill's per-layer K/V writes into the paged pool (run with -m gpu).

``write_prefill_kv`` takes one layer of a batch in the varlen layout
[sum_i n_i, Hkv, D] (the layout attention kernels produce) and writes request
i's rows to its handle's tokens. Bar: the pool then holds exactly those bytes
(``load_tokens`` bit-equal to the inputs), chunked writes compose, and a
Knorm compression of the written cache matches the CPU oracle bit for bit.
"""

import numpy as np
import pytest
import torch

from oracle import press as opress
from paper_2503_08461_b200 import (
    CompressorSpec,
    KVCachePool,
    ModelConfig,
    PressKind,
    split_modalities,
)

pytestmark = pytest.mark.gpu


def _pool(cuda, cfg, dtype):
    return KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype=dtype,
                       max_handles=64, max_tokens_per_handle=4096)


@pytest.mark.parametrize("dtype", ["float16", "bfloat16", "float32"])
def test_prefill_write_then_knorm(cuda, dtype):
    cfg = ModelConfig("m", 3, 4, 128, 4 if dtype == "float32" else 2)
    pool = _pool(cuda, cfg, dtype)
    specs = [split_modalities(576, 37), split_modalities(0, 1), split_modalities(13, 200)]
    hs = pool.allocate_batch([0, 1, 2], specs, 0.0)
    lens = [s.total_tokens for s in specs]
    g = torch.Generator(device=cuda).manual_seed(1)
    tdt = getattr(torch, dtype)
    layers = []
    for layer in range(cfg.num_layers):
        k = torch.randn((sum(lens), 4, 128), generator=g, device=cuda).to(tdt)
        v = torch.randn((sum(lens), 4, 128), generator=g, device=cuda).to(tdt)
        pool.write_prefill_kv(hs, layer, k, v)
        assert pool.last_prefill_path() == "tma"
        layers.append((k, v))
    dense = []
    off = 0
    for i, n in enumerate(lens):
        want = torch.stack([torch.stack([k[off:off + n], v[off:off + n]]) for k, v in layers])
        want = want.permute(0, 1, 3, 2, 4).contiguous()          # [L, 2, H, n, D]
        got = pool.load_tokens(hs[i])
        assert torch.equal(got, want), i
        dense.append(want)
        off += n
    res = pool.compress_batch(hs, CompressorSpec(factor=2, press=PressKind.KNORM), 1.0,
                              return_indices=True)
    for i, s in enumerate(specs):
        raw = dense[i].float().cpu().numpy()
        segs = [seg.token_count for seg in s.segments]
        kept = res.kept_idx[i].cpu().numpy()
        for layer in range(cfg.num_layers):
            for head in range(4):
                sc = opress.knorm_scores(raw[layer, 0, head], cfg.bytes_per_element)
                assert np.array_equal(kept[layer, head], opress.select(sc, segs, 2))
    pool.verify_conservation()


def test_chunked_prefill_and_errors(cuda):
    cfg = ModelConfig("m", 1, 2, 64, 2)
    pool = _pool(cuda, cfg, "float16")
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 100), split_modalities(0, 70)], 0.0)
    full_k = torch.randn((170, 2, 64), device=cuda).half()
    full_v = torch.randn((170, 2, 64), device=cuda).half()
    # two chunks: rows [0,60) / [0,30) first, then the rest at their token offsets
    c1 = torch.cat([full_k[:60], full_k[100:130]]), torch.cat([full_v[:60], full_v[100:130]])
    c2 = torch.cat([full_k[60:100], full_k[130:170]]), torch.cat([full_v[60:100], full_v[130:170]])
    pool.write_prefill_kv(hs, 0, c1[0].contiguous(), c1[1].contiguous(), seq_lens=[60, 30])
    pool.write_prefill_kv(hs, 0, c2[0].contiguous(), c2[1].contiguous(), seq_lens=[40, 40],
                          tok_begin=[60, 30])
    got0, got1 = pool.load_tokens(hs[0]), pool.load_tokens(hs[1])
    assert torch.equal(got0[0, 0], full_k[:100].permute(1, 0, 2))
    assert torch.equal(got0[0, 1], full_v[:100].permute(1, 0, 2))
    assert torch.equal(got1[0, 0], full_k[100:].permute(1, 0, 2))
    with pytest.raises(ValueError):   # rows beyond the handle's tokens
        pool.write_prefill_kv(hs, 0, c2[0].contiguous(), c2[1].contiguous(), seq_lens=[40, 40],
                              tok_begin=[61, 30])
    with pytest.raises(ValueError):   # layer out of range
        pool.write_prefill_kv(hs, 1, full_k, full_v)
    with pytest.raises(ValueError):   # wrong row count for the default lengths
        pool.write_prefill_kv(hs, 0, full_k[:169].contiguous(), full_v[:169].contiguous())


@pytest.mark.parametrize("H,D,bs,dtype", [(8, 128, 16, "float16"), (6, 64, 32, "bfloat16"),
                                          (1, 256, 8, "float32"), (32, 128, 128, "float16")])
def test_prefill_geometries_and_ragged_chunks(cuda, H, D, bs, dtype):
    """The TMA ingest (head-group tiles, whole-chunk bulk stores, row stores at a chunk's
    ragged edges) over head counts that are not powers of two, block sizes 8..128, more
    requests than one launch descriptor holds (130 > 128), empty chunks, and three
    chunked writes per request at unaligned token offsets."""
    bpe = 4 if dtype == "float32" else 2
    cfg = ModelConfig("m", 2, H, D, bpe)
    n_req = 130
    rng = np.random.default_rng(H * 1000 + bs)
    lens = [int(x) for x in rng.integers(1, 3 * bs + 5, n_req)]
    pool = KVCachePool(cfg, (sum(lens) + n_req * bs + 64) * cfg.bytes_per_token, device=cuda,
                       kv_dtype=dtype, block_size=bs, max_handles=n_req,
                       max_tokens_per_handle=4 * bs)
    hs = pool.allocate_batch(list(range(n_req)), [split_modalities(0, n) for n in lens], 0.0)
    tdt = getattr(torch, dtype)
    g = torch.Generator(device=cuda).manual_seed(7)
    full = [[(torch.randn((n, H, D), generator=g, device=cuda).to(tdt),
              torch.randn((n, H, D), generator=g, device=cuda).to(tdt)) for n in lens]
            for _ in range(cfg.num_layers)]
    # three chunks per request with random cut points
    cuts = [sorted(int(c) for c in rng.integers(0, n + 1, 2)) for n in lens]
    bounds = [[0, a, b, n] for (a, b), n in zip(cuts, lens)]
    for layer in range(cfg.num_layers):
        for part in range(3):
            ks, vs, seq, beg = [], [], [], []
            for i in range(n_req):
                lo, hi = bounds[i][part], bounds[i][part + 1]
                ks.append(full[layer][i][0][lo:hi])
                vs.append(full[layer][i][1][lo:hi])
                seq.append(hi - lo)
                beg.append(lo)
            pool.write_prefill_kv(hs, layer, torch.cat(ks).contiguous(), torch.cat(vs).contiguous(),
                                  seq_lens=seq, tok_begin=beg)
            # the TMA ingest takes every chunk up to its 16-KB tile; bs 128 x 256 B is 32 KB
            assert pool.last_prefill_path() == ("copy" if bs * D * bpe > 16384 else "tma")
    for i in range(n_req):
        got = pool.load_tokens(hs[i])                            # [L, 2, H, n, D]
        for layer in range(cfg.num_layers):
            assert torch.equal(got[layer, 0], full[layer][i][0].permute(1, 0, 2)), (i, layer)
            assert torch.equal(got[layer, 1], full[layer][i][1].permute(1, 0, 2)), (i, layer)
    pool.verify_conservation()
