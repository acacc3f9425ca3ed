"""Host-resident compress (``compress_batch(host_kv=...)`` -> fc_pool_compress_host_batch).

The raw KV starts in pinned host memory. Pooled Knorm / SnapKV move only the K
planes over PCIe before selection and read just the kept V rows afterwards;
every other press / mode copies all of K and V. Bar: the result is bit-identical
to ``store_tokens`` + ``compress_batch`` on a twin pool (kept indices, scores,
compacted K/V, block tables, ledger), and for Knorm equal to the CPU oracle.
"""

import ctypes

import numpy as np
import pytest
import torch

from oracle import press as opress
from oracle import synth as osynth
from paper_2503_08461_b200 import (
    CompressorSpec,
    KVCachePool,
    MapKind,
    ModelConfig,
    PoolMode,
    PressKind,
    split_modalities,
)
from paper_2503_08461_b200 import _native as nat

pytestmark = pytest.mark.gpu


def _pool(cuda, cfg, dtype, mode=PoolMode.POOLED, hq=None):
    return KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, mode, device=cuda, kv_dtype=dtype,
                       max_handles=64, max_tokens_per_handle=8192,
                       num_q_heads=hq or cfg.num_kv_heads)


def _bits(t):
    return t.view(torch.uint8).cpu().numpy() if t.element_size() == 1 else \
        t.contiguous().view(torch.int16 if t.element_size() == 2 else torch.int32).cpu().numpy()


def _host_kv(cfg, dtype, specs, seed):
    """Per-request pinned [L, 2, H, T, D] buffers with the K8 generator's values."""
    out = []
    for i, s in enumerate(specs):
        a = osynth.request_kv(seed, i, cfg.num_layers, cfg.num_kv_heads, s.total_tokens,
                              cfg.head_dim, dtype, osynth.DIST_SCALED)
        if dtype == "bfloat16":
            t = torch.from_numpy(a.view(np.int16)).view(torch.bfloat16)
        else:
            t = torch.from_numpy(a)
        out.append(t.pin_memory())
    return out


def _press_inputs(comp, n, cfg, hq, dtype, cuda):
    g = torch.Generator().manual_seed(3)
    if comp.press is PressKind.SNAPKV:
        q = torch.randn((n, cfg.num_layers, hq, comp.window, cfg.head_dim), generator=g)
        return {"q_window": q.to(getattr(torch, dtype)).to(cuda)}
    if comp.press is PressKind.EXPECTED_ATTENTION:
        d = cfg.head_dim
        mu = torch.randn((n, cfg.num_layers, hq, d), generator=g) / d ** 0.5
        a = torch.randn((n, cfg.num_layers, hq, d, d), generator=g)
        return {"mean_q": mu.float().to(cuda),
                "cov_q": (a @ a.transpose(-1, -2) / d).float().contiguous().to(cuda)}
    return {}


CASES = [
    # dtype, L, H, gq, D, specs, comp, mode
    ("float16", 2, 4, 1, 128, [(576, 37), (0, 100), (33, 0), (5, 11)],
     CompressorSpec(factor=2, press=PressKind.KNORM), PoolMode.POOLED),
    ("float32", 4, 8, 1, 64, [(0, 512)] * 4, CompressorSpec(factor=2, press=PressKind.KNORM),
     PoolMode.POOLED),
    ("bfloat16", 2, 2, 1, 128, [(576, 300), (1, 900), (200, 0)],
     CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32, pool_kernel=7), PoolMode.POOLED),
    ("float16", 1, 2, 2, 64, [(0, 300), (100, 21)],
     CompressorSpec(factor=4, press=PressKind.SNAPKV, window=16, pool_kernel=5), PoolMode.POOLED),
    ("float16", 1, 2, 4, 128, [(576, 300), (0, 2600)],                  # tensor-core GQA + two-pass
     CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32, pool_kernel=7), PoolMode.POOLED),
    ("float16", 2, 2, 1, 128, [(576, 200), (0, 1024)],
     CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=4), PoolMode.POOLED),
    ("float16", 2, 2, 1, 128, [(48, 17), (0, 90)], CompressorSpec(factor=2, press=PressKind.KNORM),
     PoolMode.LEGACY_ZOMBIE),
    ("float16", 2, 2, 1, 128, [(13, 29), (0, 64)], CompressorSpec(factor=5, map_kind=MapKind.MEAN_POOL),
     PoolMode.POOLED),
]


@pytest.mark.parametrize("dtype,L,H,gq,D,specs,comp,mode", CASES)
def test_host_compress_equals_device_compress(cuda, dtype, L, H, gq, D, specs, comp, mode):
    cfg = ModelConfig("m", L, H, D, 4 if dtype == "float32" else 2)
    hq = H * gq
    rs = [split_modalities(*s) for s in specs]
    host = _host_kv(cfg, dtype, rs, seed=13)
    ins = _press_inputs(comp, len(rs), cfg, hq, dtype, cuda)
    ret = comp.press in (PressKind.KNORM, PressKind.SNAPKV, PressKind.EXPECTED_ATTENTION)

    dev_pool = _pool(cuda, cfg, dtype, mode, hq)
    dh = dev_pool.allocate_batch(list(range(len(rs))), rs, 0.0)
    for h, t in zip(dh, host):
        dev_pool.store_tokens(h, t.to(cuda))
    want = dev_pool.compress_batch(dh, comp, 1.0, return_indices=ret, return_scores=ret, **ins)

    host_pool = _pool(cuda, cfg, dtype, mode, hq)
    hh = host_pool.allocate_batch(list(range(len(rs))), rs, 0.0)
    got = host_pool.compress_batch(hh, comp, 1.0, return_indices=ret, return_scores=ret,
                                   host_kv=host, **ins)
    torch.cuda.synchronize()
    for i, (a, b) in enumerate(zip(dh, hh)):
        if ret:
            assert torch.equal(want.kept_idx[i], got.kept_idx[i]), i
            assert np.array_equal(_bits(want.scores[i]), _bits(got.scores[i])), i
        assert np.array_equal(_bits(dev_pool.load_tokens(a)), _bits(host_pool.load_tokens(b))), i
        assert torch.equal(dev_pool._native.block_table_view(a.handle_id),
                           host_pool._native.block_table_view(b.handle_id))
    if comp.press is PressKind.KNORM:   # and the CPU oracle directly
        for i, s in enumerate(rs):
            raw = host[i].view(torch.int16).numpy().view(np.uint16) if dtype == "bfloat16" \
                else host[i].numpy()
            kept = got.kept_idx[i].cpu().numpy()
            kv32 = osynth.to_f32(raw, dtype)
            segs = [seg.token_count for seg in s.segments]
            for layer in range(L):
                sc = opress.knorm_scores(kv32[layer, 0, 0], cfg.bytes_per_element)
                assert np.array_equal(kept[layer, 0], opress.select(sc, segs, comp.factor))
            assert np.array_equal(_bits(host_pool.load_tokens(hh[i])).view(np.uint8),
                                  opress.gather_kept(raw, kept).view(np.uint8))
    assert host_pool.ledger == dev_pool.ledger
    host_pool.verify_conservation()
    host_pool.release_batch(hh, 2.0)
    host_pool.verify_conservation()


def test_host_compress_rejects_pageable_and_bad_shapes(cuda):
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = _pool(cuda, cfg, "float16")
    spec = split_modalities(0, 64)
    h = pool.allocate(0, spec, 0.0)
    comp = CompressorSpec(factor=2, press=PressKind.KNORM)
    pageable = torch.zeros((1, 2, 2, 64, 128), dtype=torch.float16)
    with pytest.raises(ValueError):
        pool.compress_batch([h], comp, 1.0, host_kv=[pageable])
    with pytest.raises(ValueError):
        pool.compress_batch([h], comp, 1.0, host_kv=[pageable[:, :, :, :32].pin_memory()])
    # the C ABI itself refuses pageable memory (no silent staging copy)
    nv = pool._native
    cfgc = nat.PressConfigC(nat.PRESS_KNORM, 2, 32, 7, 4, 2, 0, 0, None)
    ptrs = (ctypes.c_void_p * 1)(pageable.data_ptr())
    st = nv.lib.fc_pool_compress_host_batch(nv.ptr, 1, nat.i64_array([h.handle_id]),
                                            nat.i64_array([0, 64]), ctypes.byref(cfgc),
                                            ctypes.byref(nat.PressInputsC()),
                                            ctypes.byref(nat.PressOutputsC()), ptrs, None, None,
                                            nv.stream())
    assert st == nat.ERR_INVALID_ARG and "pinned" in nat.last_error()
    # nothing was mutated: the handle is still raw and compresses normally
    pinned = pageable.pin_memory()
    pool.compress_batch([h], comp, 1.0, host_kv=[pinned])
    assert h.spec.total_tokens == 32
    pool.verify_conservation()


def test_host_compress_more_requests_than_one_launch(cuda):
    """150 requests > kMaxBatch (128): press and host-gather launches are chunked."""
    cfg = ModelConfig("m", 1, 2, 64, 2)
    rs = [split_modalities(0, 20 + (i * 7) % 90) for i in range(150)]
    host = _host_kv(cfg, "float16", rs, seed=5)
    comp = CompressorSpec(factor=3, press=PressKind.KNORM)
    dev_pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                           max_handles=256, max_tokens_per_handle=256)
    dh = dev_pool.allocate_batch(list(range(150)), rs, 0.0)
    for h, t in zip(dh, host):
        dev_pool.store_tokens(h, t.to(cuda))
    dev_pool.compress_batch(dh, comp, 1.0)
    host_pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                            max_handles=256, max_tokens_per_handle=256)
    hh = host_pool.allocate_batch(list(range(150)), rs, 0.0)
    host_pool.compress_batch(hh, comp, 1.0, host_kv=host)
    for a, b in zip(dh, hh):
        assert np.array_equal(_bits(dev_pool.load_tokens(a)), _bits(host_pool.load_tokens(b)))
    host_pool.verify_conservation()
