"""All-or-nothing mutations and buffer lifetimes of the device pool (run with -m gpu).

The reference pool is strict: every check runs before any mutation
(reference pkg/src/kvservesim/pool.py:147-165 allocate, :167-192 transition,
:194-211 append). These tests force each refusal the device path can hit
*after* the Python-level checks -- block-pool exhaustion on append, a press
without a launch plan (pooled, and legacy out-of-place compress whose pops
precede the press) -- and check that block tables, free-block count,
payload and both ledgers are exactly as before. They also cover the serving
pattern decode -> host-resident compress that regrows the kept-index scratch
-> decode on one pool (a stale-pointer regression).
"""

import pytest
import torch

from oracle import synth as osynth
from paper_2503_08461_b200 import (
    CapacityExceeded,
    CompressorSpec,
    KVCachePool,
    ModelConfig,
    PoolMode,
    PressKind,
    split_modalities,
)

pytestmark = pytest.mark.gpu


def _state(pool, hs):
    """Everything a refused call must leave untouched."""
    torch.cuda.synchronize()
    tables = [pool._native.block_table_view(h.handle_id).cpu().tolist() for h in hs]
    payload = [pool.load_tokens(h).cpu() for h in hs]
    bs = pool.block_stats()
    return {
        "tables": tables,
        "payload": payload,
        "free": bs.free_blocks,
        "used": bs.used_blocks,
        "ledger": list(pool.ledger),
        "trace": list(pool.memory_trace),
        "specs": [h.spec for h in hs],
        "states": [h.state for h in hs],
        "bytes": [h.bytes for h in hs],
    }


def _same(a, b):
    assert a["tables"] == b["tables"]
    assert all(torch.equal(x, y) for x, y in zip(a["payload"], b["payload"]))
    for k in ("free", "used", "ledger", "trace", "specs", "states", "bytes"):
        assert a[k] == b[k], k


def test_append_block_exhaustion_mutates_nothing(cuda):
    """Bytes admit the append but the free stack cannot: refused before any mutation."""
    cfg = ModelConfig("m", 1, 2, 64, 2)
    pool = KVCachePool(cfg, 10 ** 6 * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=8, max_tokens_per_handle=256, num_blocks=4)
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 16)] * 2, 0.0)
    pool.synth_fill(hs, seed=1)
    pool.compress_batch(hs, CompressorSpec(factor=2, press=PressKind.KNORM), 1.0)
    assert pool.block_stats().free_blocks == 2          # 2 x 8 kept tokens = 1 block each
    before = _state(pool, hs)
    with pytest.raises(CapacityExceeded):
        pool.append_decode_batch(hs, 30, 2.0)           # 2 x (8 -> 38 tokens, +2 blocks) > 2 free
    _same(before, _state(pool, hs))
    pool.verify_conservation()
    # batches that fit still work afterwards; a repeated handle sees its predecessor's growth
    pool.append_decode_batch([hs[0]], 9, 3.0)           # 8 -> 17 tokens: +1 block
    pool.append_decode_batch([hs[1], hs[1]], 5, 3.0)    # 8 -> 13 -> 18 tokens: +1 block
    assert pool.block_stats().free_blocks == 0
    assert pool._native.block_row(hs[1].handle_id)[1:] == (2, 18)
    pool.verify_conservation()


def test_pooled_refused_batch_mutates_nothing(cuda):
    """ExpectedAttention at head_dim 256 has no launch plan (the SIMT kernel's Sigma alone
    exceeds the SMEM budget): the batch is refused by the dry run before anything moves."""
    cfg = ModelConfig("m", 1, 2, 256, 2)
    pool = KVCachePool(cfg, (1 << 14) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=8, max_tokens_per_handle=4096)
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 300), split_modalities(5, 900)], 0.0)
    pool.synth_fill(hs, seed=2)
    gen = torch.Generator().manual_seed(0)
    mu = (torch.randn((2, 1, 2, 256), generator=gen) / 16).float().to(cuda)
    a = torch.randn((2, 1, 2, 256, 256), generator=gen)
    cov = (a @ a.transpose(-1, -2) / 256).float().contiguous().to(cuda)
    comp = CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=4)
    before = _state(pool, hs)
    with pytest.raises(NotImplementedError):
        pool.compress_batch(hs, comp, 1.0, mean_q=mu, cov_q=cov)
    _same(before, _state(pool, hs))
    pool.verify_conservation()
    # Knorm has a plan at head_dim 256: the same handles still compress afterwards
    pool.compress_batch(hs, CompressorSpec(factor=4, press=PressKind.KNORM), 2.0)
    assert [h.spec.total_tokens for h in hs] == [75, 227]
    pool.verify_conservation()


def test_legacy_refusal_pops_nothing(cuda):
    """Legacy compress pops destination blocks before the press: a refused launch plan must
    be caught first (no leaked blocks, raw rows still mapped)."""
    cfg = ModelConfig("m", 1, 1, 256, 4)
    pool = KVCachePool(cfg, (1 << 14) * cfg.bytes_per_token, PoolMode.LEGACY_ZOMBIE, device=cuda,
                       kv_dtype="float32", max_handles=8, max_tokens_per_handle=4096)
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 100), split_modalities(0, 600)], 0.0)
    pool.synth_fill(hs, seed=3)
    gen = torch.Generator().manual_seed(1)
    mu = (torch.randn((2, 1, 1, 256), generator=gen) / 16).float().to(cuda)
    a = torch.randn((2, 1, 1, 256, 256), generator=gen)
    cov = (a @ a.transpose(-1, -2) / 256).float().contiguous().to(cuda)
    comp = CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=4)
    before = _state(pool, hs)
    with pytest.raises(NotImplementedError):
        pool.compress_batch(hs, comp, 1.0, mean_q=mu, cov_q=cov)
    _same(before, _state(pool, hs))
    assert not pool.zombie_coexistence_observed
    pool.verify_conservation()


def test_u8_device_pool_refused_at_creation(cuda):
    cfg = ModelConfig("m", 1, 2, 64, 1)
    with pytest.raises(NotImplementedError):
        KVCachePool(cfg, 1 << 20, device=cuda)
    KVCachePool(cfg, 1 << 20)    # the ledger-only pool accepts bytes_per_element=1 (reference)


def _decode_ref(kv_layer, q, scale):
    """kv_layer [2, H, T, D], q [Hq, D] -> [Hq, D] float64."""
    H = kv_layer.shape[1]
    g = q.shape[0] // H
    k = kv_layer[0].double().repeat_interleave(g, dim=0)
    v = kv_layer[1].double().repeat_interleave(g, dim=0)
    p = torch.softmax(torch.einsum("hd,htd->ht", q.double(), k) * scale, dim=-1)
    return torch.einsum("ht,htd->hd", p, v)


def test_decode_then_growing_host_compress_then_decode(cuda):
    """decode_attention, then a LARGER host-resident compress without return_indices (the
    kept-index scratch regrows), then decode again on the same pool; destroy at the end."""
    cfg = ModelConfig("m", 2, 4, 128, 2)
    pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=64, max_tokens_per_handle=4096)
    comp = CompressorSpec(factor=2, press=PressKind.KNORM)
    gen = torch.Generator(device=cuda).manual_seed(0)
    scale = 128 ** -0.5

    def host_batch(specs, seed):
        out = []
        for i, s in enumerate(specs):
            a = osynth.request_kv(seed, i, 2, 4, s.total_tokens, 128, "float16", osynth.DIST_SCALED)
            out.append(torch.from_numpy(a).pin_memory())
        return out

    def decode_round(hs, now):
        pool.append_decode_batch(hs, 1, now)
        for layer in range(2):
            k = torch.randn((len(hs), 4, 128), generator=gen, device=cuda).half()
            v = torch.randn((len(hs), 4, 128), generator=gen, device=cuda).half()
            q = torch.randn((len(hs), 4, 128), generator=gen, device=cuda).half()
            pool.write_decode_kv(hs, layer, k, v)
            out = pool.decode_attention(hs, layer, q)
            torch.cuda.synchronize()
            for i, h in enumerate(hs):
                want = _decode_ref(pool.load_tokens(h)[layer], q[i], scale)
                err = (out[i].double() - want).abs().max().item()
                assert err <= 2e-3 * max(want.abs().max().item(), 1e-30), (i, layer, err)

    small = [split_modalities(0, 64)] * 2
    hs = pool.allocate_batch([0, 1], small, 0.0)
    pool.compress_batch(hs, comp, 1.0, host_kv=host_batch(small, 5))
    decode_round(hs, 2.0)
    big = [split_modalities(576, 1500)] * 6                 # 16x more kept indices
    hb = pool.allocate_batch(list(range(2, 8)), big, 3.0)
    pool.compress_batch(hb, comp, 3.0, host_kv=host_batch(big, 6))
    decode_round(hs + hb, 4.0)
    decode_round(hs, 5.0)
    pool.verify_conservation()
    pool.release_batch(hs + hb, 6.0)
    pool.verify_conservation()
    pool._native.__del__()                                  # fc_pool_destroy: no double free
    torch.cuda.synchronize()
