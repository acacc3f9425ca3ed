"""GPU parity of the batched presses against the CPU oracle (run with -m gpu).

Bars (BASELINE.json north star):
* Knorm scores: bit-exact (the kernel's fp32 summation order is restated in
  oracle/press.py:knorm_scores); kept sets and block tables bit-exact;
* SnapKV / ExpectedAttention scores: max relative error <= 1e-5 against the
  float64 oracle; kept sets exact up to tolerated boundary swaps
  (oracle/press.py:kept_set_mismatch);
* compacted K/V: bit-exact copies of the source rows the GPU kept;
* ledger: identical to the ledger-only pool driven by the same calls.
"""

import numpy as np
import pytest
import torch

from oracle import blocks as oblocks
from oracle import chunk as ochunk
from oracle import press as opress
from oracle import synth as osynth
from paper_2503_08461_b200 import (
    CompressorSpec,
    InvalidState,
    KVCachePool,
    MapKind,
    ModelConfig,
    PoolMode,
    PressKind,
    split_modalities,
)

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-5


def _stored_np(t: torch.Tensor, dtype: str) -> np.ndarray:
    if dtype == "bfloat16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _model(dtype, L, H, D):
    return ModelConfig("m", L, H, D, 4 if dtype == "float32" else 2)


def _make_pool(cuda, cfg, dtype, mode=PoolMode.POOLED, cap_tokens=1 << 16, max_tokens=8192, **kw):
    return KVCachePool(cfg, cap_tokens * cfg.bytes_per_token, mode, device=cuda, kv_dtype=dtype,
                       max_handles=64, max_tokens_per_handle=max_tokens, **kw)


def _ledger_twin(cfg, cap_tokens, mode):
    return KVCachePool(cfg, cap_tokens * cfg.bytes_per_token, mode)


def _check_tables(pool, handles, model):
    for h in handles:
        got = pool._native.block_table_view(h.handle_id).cpu().tolist()
        assert got == model.tables[h.handle_id], h.handle_id


CASES = [
    # dtype, L, H, D, specs(img, txt), factor
    ("float32", 4, 8, 64, [(0, 512)] * 4, 2),                       # config 1 (tiny, fp32)
    ("bfloat16", 4, 8, 64, [(0, 512)] * 4, 2),                      # config 1 bf16 variant
    ("float16", 2, 4, 128, [(576, 37), (0, 100), (33, 0), (5, 11), (576, 512)], 2),
    ("float16", 2, 2, 256, [(40, 7), (1, 0), (17, 300)], 4),
    ("float32", 1, 3, 128, [(100, 29), (16, 16)], 3),
]


@pytest.mark.parametrize("dist", ["scaled", "plain"])
@pytest.mark.parametrize("dtype,L,H,D,specs,factor", CASES)
def test_knorm_parity(cuda, dtype, L, H, D, specs, factor, dist):
    cfg = _model(dtype, L, H, D)
    pool = _make_pool(cuda, cfg, dtype)
    twin = _ledger_twin(cfg, 1 << 16, PoolMode.POOLED)
    raw_specs = [split_modalities(i, t) for i, t in specs]
    hs = pool.allocate_batch(list(range(len(specs))), raw_specs, 0.0)
    ts = twin.allocate_batch(list(range(len(specs))), raw_specs, 0.0)
    model = oblocks.BlockAllocatorModel(pool._native.num_blocks, 16)
    model.alloc_batch([h.handle_id for h in hs], [s.total_tokens for s in raw_specs])
    _check_tables(pool, hs, model)
    pool.synth_fill(hs, seed=11, dist=dist)
    sd = osynth.DIST_SCALED if dist == "scaled" else osynth.DIST_PLAIN
    raw = []
    for h, s in zip(hs, raw_specs):
        got = _stored_np(pool.load_tokens(h), dtype)
        want = osynth.request_kv(11, h.request_id, L, H, s.total_tokens, D, dtype, sd)
        assert np.array_equal(got.view(np.uint8), want.view(np.uint8)), "K8 generator != oracle"
        raw.append(want)
    comp = CompressorSpec(factor=factor, press=PressKind.KNORM)
    res = pool.compress_batch(hs, comp, now=1.0, return_indices=True, return_scores=True)
    twin.compress_batch(ts, comp, now=1.0)
    for i, (h, s) in enumerate(zip(hs, raw_specs)):
        kv32 = osynth.to_f32(raw[i], dtype)
        segs = [seg.token_count for seg in s.segments]
        k_r = opress.kept_budget(segs, factor)
        got_scores = res.scores[i].cpu().numpy()
        got_kept = res.kept_idx[i].cpu().numpy()
        for layer in range(L):
            for head in range(H):
                want = opress.knorm_scores(kv32[layer, 0, head], cfg.bytes_per_element)
                assert np.array_equal(got_scores[layer, head], want), (i, layer, head)
                kept = opress.select(want, segs, factor)
                assert np.array_equal(got_kept[layer, head], kept), (i, layer, head)
        assert h.spec.total_tokens == k_r
        compacted = _stored_np(pool.load_tokens(h), dtype)
        want_c = opress.gather_kept(raw[i], got_kept)
        assert np.array_equal(compacted.view(np.uint8), want_c.view(np.uint8))
    model.compress_batch([h.handle_id for h in hs], [h.spec.total_tokens for h in hs])
    _check_tables(pool, hs, model)
    assert pool.ledger == twin.ledger and pool.memory_trace == twin.memory_trace
    pool.verify_conservation()
    pool.release_batch(hs, now=2.0)
    model.release_batch([h.handle_id for h in hs])
    assert pool.block_stats().free_blocks == model.free_blocks
    pool.verify_conservation()


def test_knorm_ties_keep_lowest_indices(cuda):
    cfg = _model("float16", 2, 2, 128)
    pool = _make_pool(cuda, cfg, "float16")
    h = pool.allocate(0, split_modalities(0, 100), 0.0)
    kv = torch.ones((2, 2, 2, 100, 128), dtype=torch.float16, device=cuda)
    kv[:, :, :, 50:] = 0.5          # smaller norms win
    kv[:, :, :, 60:70] = 1.0        # ties with the first half
    pool.store_tokens(h, kv)
    res = pool.compress_batch([h], CompressorSpec(factor=2, press=PressKind.KNORM), 1.0,
                              return_indices=True)
    # 40 tokens with norm of 0.5-rows, then the 10 lowest-index 1.0-rows
    want = list(range(0, 10)) + list(range(50, 60)) + list(range(70, 100))
    assert sorted(res.kept_idx[0][0, 0].cpu().tolist()) == sorted(want)
    assert res.kept_idx[0][0, 0].cpu().tolist() == want


def test_knorm_per_segment_and_repeat_errors(cuda):
    cfg = _model("float16", 2, 2, 128)
    pool = _make_pool(cuda, cfg, "float16")
    hs = pool.allocate_batch([0, 1], [split_modalities(64, 40), split_modalities(0, 33)], 0.0)
    pool.synth_fill(hs, seed=3)
    raws = [osynth.to_f32(_stored_np(pool.load_tokens(h), "float16"), "float16") for h in hs]
    comp = CompressorSpec(factor=4, press=PressKind.KNORM, per_segment=True)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True)
    assert pool.last_paths() == {"tc": 0, "simt": 1, "chunk": 0}   # the fused Knorm kernel
    for i, segs in enumerate(([64, 40], [33])):
        want = opress.select(opress.knorm_scores(raws[i][1, 0, 1], 2), segs, 4, per_segment=True)
        assert res.kept_idx[i][1, 1].cpu().numpy().tolist() == want.tolist()
    with pytest.raises(InvalidState):
        pool.compress_batch(hs[:1], comp, 2.0)


def test_legacy_mode_out_of_place(cuda):
    cfg = _model("float16", 2, 2, 128)
    pool = _make_pool(cuda, cfg, "float16", mode=PoolMode.LEGACY_ZOMBIE)
    twin = _ledger_twin(cfg, 1 << 16, PoolMode.LEGACY_ZOMBIE)
    specs = [split_modalities(48, 17), split_modalities(0, 90)]
    hs = pool.allocate_batch([0, 1], specs, 0.0)
    ts = twin.allocate_batch([0, 1], specs, 0.0)
    model = oblocks.BlockAllocatorModel(pool._native.num_blocks, 16)
    model.alloc_batch([0, 1], [65, 90])
    pool.synth_fill(hs, seed=5)
    raw = [_stored_np(pool.load_tokens(h), "float16") for h in hs]
    comp = CompressorSpec(factor=2, press=PressKind.KNORM)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True)
    twin.compress_batch(ts, comp, 1.0)
    model.compress_batch([0, 1], [h.spec.total_tokens for h in hs], legacy=True)
    _check_tables(pool, hs, model)
    for i, h in enumerate(hs):
        got = _stored_np(pool.load_tokens(h), "float16")
        assert np.array_equal(got, opress.gather_kept(raw[i], res.kept_idx[i].cpu().numpy()))
    assert pool.ledger == twin.ledger and pool.zombie_coexistence_observed
    pool.verify_conservation()
    pool.release_batch(hs, 2.0)
    model.release_batch([0, 1])
    assert pool.block_stats().free_blocks == model.free_blocks


def test_append_and_churn_block_tables(cuda):
    cfg = _model("float16", 1, 2, 128)
    pool = _make_pool(cuda, cfg, "float16")
    model = oblocks.BlockAllocatorModel(pool._native.num_blocks, 16)
    rng = np.random.default_rng(0)
    live = []
    comp = CompressorSpec(factor=2, press=PressKind.KNORM)
    for step in range(30):
        toks = [int(x) for x in rng.integers(1, 200, size=3)]
        hs = pool.allocate_batch([step] * 3, [split_modalities(0, t) for t in toks], float(step))
        model.alloc_batch([h.handle_id for h in hs], toks)
        pool.synth_fill(hs, seed=step)
        pool.compress_batch(hs, comp, float(step))
        model.compress_batch([h.handle_id for h in hs], [h.spec.total_tokens for h in hs])
        for h in hs:
            n = int(rng.integers(1, 40))
            pool.append_decode_tokens(h, n, float(step))
            model.append_batch([h.handle_id], [n])
        live += hs
        if len(live) > 6:
            gone, live = live[:4], live[4:]
            pool.release_batch(gone, float(step))
            model.release_batch([h.handle_id for h in gone])
        _check_tables(pool, live, model)
        pool.verify_conservation()
    st = pool.block_stats()
    assert st.free_blocks == model.free_blocks
    assert 0.0 <= st.fragmentation < 1.0


def _assert_path(pool, tc: bool):
    """The press implementation the last compress call launched (fc_pool_last_paths)."""
    paths = pool.last_paths()
    if tc:
        assert paths["tc"] >= 1 and paths["simt"] == 0, paths
    else:
        assert paths["tc"] == 0 and paths["simt"] >= 1, paths


def _snap_inputs(n, L, hq, w, D, seed, device, dtype):
    g = torch.Generator().manual_seed(seed)
    q = torch.randn((n, L, hq, w, D), generator=g, dtype=torch.float32).to(getattr(torch, dtype))
    return q.to(device)


@pytest.mark.parametrize("dtype,L,H,gq,D,specs,w,p", [
    ("float16", 2, 2, 1, 128, [(576, 70), (0, 100), (40, 0)], 32, 7),      # tcgen05 path
    ("bfloat16", 1, 2, 1, 128, [(576, 960), (1, 2046), (33, 0)], 32, 7),   # tcgen05, 16 tiles
    ("float16", 2, 3, 1, 64, [(300, 17), (129, 0)], 32, 5),                # tcgen05, D=64
    ("float16", 1, 2, 1, 128, [(576, 2500), (0, 100), (1, 8000)], 32, 7),  # tcgen05, T > 2048: two passes
    ("bfloat16", 1, 1, 1, 128, [(0, 2049), (576, 1472)], 32, 7),           # tcgen05, 17 vs 16 tiles
    ("float16", 2, 2, 4, 128, [(576, 200), (0, 900), (1, 2500)], 32, 7),    # tcgen05 GQA g=4 (+ long)
    ("bfloat16", 1, 4, 2, 64, [(0, 300), (100, 1000)], 32, 7),             # tcgen05 GQA g=2, D=64
    ("bfloat16", 1, 2, 2, 64, [(0, 300), (100, 21)], 16, 5),
    ("float32", 1, 1, 4, 128, [(50, 50)], 8, 3),
])
def test_snapkv_parity(cuda, dtype, L, H, gq, D, specs, w, p):
    cfg = _model(dtype, L, H, D)
    pool = _make_pool(cuda, cfg, dtype, num_q_heads=H * gq)
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=21)
    raw = [_stored_np(pool.load_tokens(h), dtype) for h in hs]
    q = _snap_inputs(len(specs), L, H * gq, w, D, 5, cuda, dtype)
    comp = CompressorSpec(factor=4, press=PressKind.SNAPKV, window=w, pool_kernel=p)
    res = pool.compress_batch(hs, comp, 1.0, q_window=q, return_indices=True, return_scores=True)
    _assert_path(pool, tc=dtype != "float32" and w == 32)
    qn = q.float().cpu().numpy()
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raw[i], dtype)
        segs = [x for x in s if x > 0]
        k_r = opress.kept_budget(segs, 4)
        for layer in range(L):
            for h in range(H):
                want = opress.snapkv_scores(kv32[layer, 0, h], qn[i, layer, h * gq:(h + 1) * gq], w, p)
                got = res.scores[i][layer, h].cpu().numpy().astype(np.float64)
                fin = np.isfinite(want)
                assert np.array_equal(np.isfinite(got), fin)
                rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
                assert rel.max() <= SCORE_RTOL, (i, layer, h, rel.max())
                kept = res.kept_idx[i][layer, h].cpu().numpy()
                assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
        got_c = _stored_np(pool.load_tokens(hs[i]), dtype)
        want_c = opress.gather_kept(raw[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got_c.view(np.uint8), want_c.view(np.uint8))
    pool.verify_conservation()


@pytest.mark.parametrize("dtype,L,H,gq,D,specs,ns", [
    ("float16", 2, 2, 1, 128, [(576, 200), (0, 1024)], 4),               # tcgen05 path
    ("float16", 1, 2, 1, 128, [(576, 7616), (1, 1500), (0, 5), (130, 0)], 4),   # tcgen05, T=8192
    ("bfloat16", 2, 2, 1, 128, [(576, 200), (0, 1024), (576, 3000)], 4),     # tcgen05, bf16 hi/lo
    ("float16", 2, 2, 2, 128, [(576, 200), (0, 1024), (3, 5)], 4),         # tcgen05 GQA g=2
    ("bfloat16", 1, 2, 4, 128, [(576, 2000), (1, 300)], 4),                # tcgen05 GQA g=4
    ("bfloat16", 1, 2, 2, 64, [(0, 300)], 4),
    ("float32", 1, 1, 2, 128, [(30, 40)], 2),
])
def test_expected_attention_parity(cuda, dtype, L, H, gq, D, specs, ns):
    cfg = _model(dtype, L, H, D)
    pool = _make_pool(cuda, cfg, dtype, num_q_heads=H * gq)
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=8)
    raw = [_stored_np(pool.load_tokens(h), dtype) for h in hs]
    gen = torch.Generator().manual_seed(9)
    n, hq = len(specs), H * gq
    mu = (torch.randn((n, L, hq, D), generator=gen) / D ** 0.5).float()
    a = torch.randn((n, L, hq, D, D), generator=gen)
    cov = (a @ a.transpose(-1, -2) / D).float()
    comp = CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=ns)
    res = pool.compress_batch(hs, comp, 1.0, mean_q=mu.to(cuda), cov_q=cov.contiguous().to(cuda),
                              return_indices=True, return_scores=True)
    _assert_path(pool, tc=dtype != "float32" and D == 128)
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raw[i], dtype)
        k_r = opress.kept_budget([x for x in s if x > 0], 4)
        for layer in range(L):
            for h in range(H):
                sl = slice(h * gq, (h + 1) * gq)
                want = opress.expected_attention_scores(kv32[layer, 0, h], kv32[layer, 1, h],
                                                        mu[i, layer, sl].numpy(),
                                                        cov[i, layer, sl].numpy(), ns)
                got = res.scores[i][layer, h].cpu().numpy().astype(np.float64)
                fin = np.isfinite(want)
                assert np.array_equal(np.isfinite(got), fin)
                rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
                assert rel.max() <= SCORE_RTOL, (i, layer, h, rel.max())
                kept = res.kept_idx[i][layer, h].cpu().numpy()
                assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
        got_c = _stored_np(pool.load_tokens(hs[i]), dtype)
        want_c = opress.gather_kept(raw[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got_c.view(np.uint8), want_c.view(np.uint8))


@pytest.mark.parametrize("map_kind", [MapKind.MEAN_POOL, MapKind.SEEDED_LINEAR])
@pytest.mark.parametrize("dtype", ["float16", "float32", "bfloat16"])
def test_chunk_press_in_pool(cuda, map_kind, dtype):
    cfg = _model(dtype, 2, 2, 128)
    pool = _make_pool(cuda, cfg, dtype)
    specs = [(13, 29), (0, 64), (7, 0)]
    hs = pool.allocate_batch([0, 1, 2], [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=4)
    raw = [_stored_np(pool.load_tokens(h), dtype) for h in hs]
    comp = CompressorSpec(factor=5, map_kind=map_kind, seed=7)
    pool.compress_batch(hs, comp, 1.0)
    for i, s in enumerate(specs):
        got = _stored_np(pool.load_tokens(hs[i]), dtype)
        kv32 = osynth.to_f32(raw[i], dtype)
        for layer in range(2):
            for kvi in range(2):
                for h in range(2):
                    parts, start = [], 0
                    for n in (x for x in s if x > 0):
                        seg = raw[i][layer, kvi, h, start:start + n] if dtype != "bfloat16" else \
                            kv32[layer, kvi, h, start:start + n]
                        parts.append(ochunk.compress_tensor(seg, 5, map_kind.value, 7))
                        start += n
                    want = np.concatenate(parts)
                    g32 = osynth.to_f32(got[layer, kvi, h], dtype)
                    if map_kind is MapKind.MEAN_POOL and dtype != "bfloat16":
                        assert np.array_equal(got[layer, kvi, h], want)
                    else:
                        want32 = osynth.to_f32(osynth.cast_dtype(want.astype(np.float32), dtype), dtype)
                        np.testing.assert_allclose(g32, want32, rtol=1e-2 if dtype != "float32" else 1e-6,
                                                   atol=1e-6)
    pool.verify_conservation()


def test_churn_waves_conserve_and_free_everything(cuda):
    from paper_2503_08461_b200 import churn

    cfg = _model("float16", 2, 2, 128)
    specs = [split_modalities(576, t) for t in (100, 700, 33, 1500, 9, 400, 1200, 64)]
    pool = KVCachePool(cfg, 2500 * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=64, max_tokens_per_handle=4096)
    comp = CompressorSpec(factor=4, press=PressKind.KNORM)
    st = churn.run_waves(pool, specs, comp, lambda n: {}, decode_tokens=8)
    assert st.compressed_requests == len(specs) and st.waves >= 3
    assert st.raw_tokens == sum(s.total_tokens for s in specs)
    bs = pool.block_stats()
    assert pool.current_bytes == 0 and bs.used_blocks == 0 and bs.free_blocks == bs.num_blocks
    assert 0.0 <= st.max_fragmentation < 1.0


@pytest.mark.parametrize("press", [PressKind.SNAPKV, PressKind.EXPECTED_ATTENTION])
@pytest.mark.parametrize("gq", [1, 2])
def test_tensor_core_presses_per_segment(cuda, press, gq):
    """per_segment=True on the tcgen05 kernels: top-ceil(n_seg/f) per modality segment
    (mirrors compressed_spec exactly, kv.py:173-194)."""
    dtype, L, H, D = "float16", 2, 2, 128
    cfg = _model(dtype, L, H, D)
    pool = _make_pool(cuda, cfg, dtype, num_q_heads=H * gq)
    specs = [(576, 300), (0, 700), (200, 0), (37, 1900)]
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=31)
    raw = [_stored_np(pool.load_tokens(h), dtype) for h in hs]
    n, hq = len(specs), H * gq
    kw = {}
    if press is PressKind.SNAPKV:
        q = _snap_inputs(n, L, hq, 32, D, 6, cuda, dtype)
        kw["q_window"] = q
        comp = CompressorSpec(factor=4, press=press, window=32, pool_kernel=7, per_segment=True)
    else:
        gen = torch.Generator().manual_seed(10)
        mu = (torch.randn((n, L, hq, D), generator=gen) / D ** 0.5).float()
        a = torch.randn((n, L, hq, D, D), generator=gen)
        cov = (a @ a.transpose(-1, -2) / D).float().contiguous()
        kw.update(mean_q=mu.to(cuda), cov_q=cov.to(cuda))
        comp = CompressorSpec(factor=4, press=press, n_sink=4, per_segment=True)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True, return_scores=True, **kw)
    _assert_path(pool, tc=True)
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raw[i], dtype)
        segs = [x for x in s if x > 0]
        assert hs[i].spec.total_tokens == opress.kept_budget(segs, 4)
        for layer in range(L):
            for h in range(H):
                sl = slice(h * gq, (h + 1) * gq)
                if press is PressKind.SNAPKV:
                    want = opress.snapkv_scores(kv32[layer, 0, h], q.float().cpu().numpy()[i, layer, sl], 32, 7)
                else:
                    want = opress.expected_attention_scores(kv32[layer, 0, h], kv32[layer, 1, h],
                                                            mu[i, layer, sl].numpy(),
                                                            cov[i, layer, sl].numpy(), 4)
                got = res.scores[i][layer, h].cpu().numpy().astype(np.float64)
                fin = np.isfinite(want)
                assert np.array_equal(np.isfinite(got), fin)
                rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
                assert rel.max() <= SCORE_RTOL, (i, layer, h, rel.max())
                kept = res.kept_idx[i][layer, h].cpu().numpy()
                # per segment: each segment's kept set is its own top-ceil(n/4)
                start = 0
                for n_seg in segs:
                    part = kept[(kept >= start) & (kept < start + n_seg)] - start
                    k_seg = opress.kept_budget([n_seg], 4)
                    assert len(part) == k_seg, (i, layer, h, n_seg)
                    assert opress.kept_set_mismatch(part, want[start:start + n_seg], k_seg,
                                                    SCORE_RTOL) is None
                    start += n_seg
        got_c = _stored_np(pool.load_tokens(hs[i]), dtype)
        want_c = opress.gather_kept(raw[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got_c.view(np.uint8), want_c.view(np.uint8))
    pool.verify_conservation()
