"""Edge cases of the batched presses on the GPU (run with -m gpu).

Launch chunking (more requests than one kernel-parameter descriptor holds),
keep-everything budgets (factor 1), the smallest caches each press accepts
(T = window + 1 for SnapKV, T = n_sink + 1 for ExpectedAttention), single-token
segments, and the refusal paths -- each checked against the CPU oracle with the
same bars as tests/test_gpu_press.py.
"""

import numpy as np
import pytest
import torch

from oracle import press as opress
from oracle import synth as osynth
from paper_2503_08461_b200 import (
    CompressorSpec,
    KVCachePool,
    ModelConfig,
    PressKind,
    split_modalities,
)

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-5


def _pool(cuda, cfg, dtype, max_handles=512, max_tokens=4096):
    return KVCachePool(cfg, (1 << 18) * cfg.bytes_per_token, device=cuda, kv_dtype=dtype,
                       max_handles=max_handles, max_tokens_per_handle=max_tokens,
                       num_q_heads=cfg.num_kv_heads)


def _raw(pool, h, dtype):
    t = pool.load_tokens(h)
    if dtype == "bfloat16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _check_knorm(pool, hs, raws, specs, factor, res, bpe, dtype):
    for i, (h, s) in enumerate(zip(hs, specs)):
        kv32 = osynth.to_f32(raws[i], dtype)
        segs = [seg.token_count for seg in s.segments]
        kept = res.kept_idx[i].cpu().numpy()
        for layer in range(kv32.shape[0]):
            for head in range(kv32.shape[2]):
                sc = opress.knorm_scores(kv32[layer, 0, head], bpe)
                assert np.array_equal(kept[layer, head], opress.select(sc, segs, factor)), (i, layer, head)
        got = _raw(pool, h, dtype)
        assert np.array_equal(got.view(np.uint8), opress.gather_kept(raws[i], kept).view(np.uint8)), i


def test_knorm_more_requests_than_one_launch(cuda):
    """300 requests > kMaxBatch (128): the batch is split across launches, LPT order inside."""
    cfg = ModelConfig("m", 1, 2, 64, 2)
    pool = _pool(cuda, cfg, "float16")
    rng = np.random.default_rng(5)
    specs = [split_modalities(int(a), int(b)) for a, b in zip(rng.integers(0, 40, 300),
                                                            rng.integers(1, 90, 300))]
    hs = pool.allocate_batch(list(range(300)), specs, 0.0)
    pool.synth_fill(hs, seed=9)
    raws = [_raw(pool, h, "float16") for h in hs]
    comp = CompressorSpec(factor=3, press=PressKind.KNORM)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True)
    _check_knorm(pool, hs, raws, specs, 3, res, 2, "float16")
    pool.verify_conservation()


def test_knorm_factor_one_keeps_everything(cuda):
    cfg = ModelConfig("m", 2, 2, 128, 2)
    pool = _pool(cuda, cfg, "float16")
    specs = [split_modalities(5, 7), split_modalities(0, 1), split_modalities(1, 0)]
    hs = pool.allocate_batch([0, 1, 2], specs, 0.0)
    pool.synth_fill(hs, seed=2)
    raws = [_raw(pool, h, "float16") for h in hs]
    res = pool.compress_batch(hs, CompressorSpec(factor=1, press=PressKind.KNORM), 1.0,
                              return_indices=True)
    for i, h in enumerate(hs):
        assert h.spec.total_tokens == specs[i].total_tokens
        k = res.kept_idx[i].cpu().numpy()
        assert (k == np.arange(specs[i].total_tokens)).all()
        assert np.array_equal(_raw(pool, h, "float16"), raws[i])
    pool.verify_conservation()


@pytest.mark.parametrize("dtype", ["float16", "bfloat16"])
def test_snapkv_smallest_caches_and_many_requests(cuda, dtype):
    """T = w + 1 (one scored token), mixed with longer caches, 140 requests (> one launch)."""
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = _pool(cuda, cfg, dtype)
    rng = np.random.default_rng(1)
    lens = [33, 34, 40] + [int(x) for x in rng.integers(33, 700, 137)]
    specs = [split_modalities(0, t) for t in lens]
    hs = pool.allocate_batch(list(range(len(specs))), specs, 0.0)
    pool.synth_fill(hs, seed=4)
    raws = [_raw(pool, h, dtype) for h in hs]
    g = torch.Generator().manual_seed(0)
    q = torch.randn((len(specs), 1, 2, 32, 128), generator=g).to(getattr(torch, dtype)).to(cuda)
    comp = CompressorSpec(factor=4, press=PressKind.SNAPKV, window=32, pool_kernel=7)
    res = pool.compress_batch(hs, comp, 1.0, q_window=q, return_indices=True, return_scores=True)
    qn = q.float().cpu().numpy()
    for i, t in enumerate(lens):
        kv32 = osynth.to_f32(raws[i], dtype)
        k_r = opress.kept_budget([t], 4)
        for h in range(2):
            want = opress.snapkv_scores(kv32[0, 0, h], qn[i, 0, h:h + 1], 32, 7)
            got = res.scores[i][0, h].cpu().numpy().astype(np.float64)
            fin = np.isfinite(want)
            assert np.array_equal(np.isfinite(got), fin)
            rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
            assert rel.max() <= SCORE_RTOL, (i, h, rel.max())
            kept = res.kept_idx[i][0, h].cpu().numpy()
            assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
        got_c = _raw(pool, hs[i], dtype)
        want_c = opress.gather_kept(raws[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got_c.view(np.uint8), want_c.view(np.uint8))
    pool.verify_conservation()


def test_expected_attention_smallest_cache(cuda):
    """T = n_sink + 1: one scored token next to the forced sinks."""
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = _pool(cuda, cfg, "float16")
    specs = [split_modalities(0, 5), split_modalities(0, 6), split_modalities(3, 300)]
    hs = pool.allocate_batch([0, 1, 2], specs, 0.0)
    pool.synth_fill(hs, seed=6)
    raws = [_raw(pool, h, "float16") for h in hs]
    gen = torch.Generator().manual_seed(3)
    mu = (torch.randn((3, 1, 2, 128), generator=gen) / 128 ** 0.5).float()
    a = torch.randn((3, 1, 2, 128, 128), generator=gen)
    cov = (a @ a.transpose(-1, -2) / 128).float().contiguous()
    comp = CompressorSpec(factor=2, press=PressKind.EXPECTED_ATTENTION, n_sink=4)
    res = pool.compress_batch(hs, comp, 1.0, mean_q=mu.to(cuda), cov_q=cov.to(cuda),
                              return_indices=True, return_scores=True)
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raws[i], "float16")
        k_r = opress.kept_budget([x.token_count for x in s.segments], 2)
        for h in range(2):
            want = opress.expected_attention_scores(kv32[0, 0, h], kv32[0, 1, h], mu[i, 0, h:h + 1].numpy(),
                                                    cov[i, 0, h:h + 1].numpy(), 4)
            got = res.scores[i][0, h].cpu().numpy().astype(np.float64)
            fin = np.isfinite(want)
            assert np.array_equal(np.isfinite(got), fin)
            if fin.any():
                rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
                assert rel.max() <= SCORE_RTOL, (i, h, rel.max())
            kept = res.kept_idx[i][0, h].cpu().numpy()
            assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
    pool.verify_conservation()


def test_press_refusals_leave_the_batch_untouched(cuda):
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = _pool(cuda, cfg, "float16")
    hs = pool.allocate_batch([0, 1], [split_modalities(0, 32), split_modalities(0, 100)], 0.0)
    q = torch.zeros((2, 1, 2, 32, 128), dtype=torch.float16, device=cuda)
    with pytest.raises(ValueError):   # SnapKV needs T > window
        pool.compress_batch(hs, CompressorSpec(factor=4, press=PressKind.SNAPKV), 1.0, q_window=q)
    with pytest.raises(ValueError):   # missing inputs
        pool.compress_batch(hs, CompressorSpec(factor=4, press=PressKind.SNAPKV), 1.0)
    ledger = list(pool.ledger)
    pool.compress_batch(hs, CompressorSpec(factor=4, press=PressKind.KNORM), 1.0)
    assert [h.spec.total_tokens for h in hs] == [8, 25]
    assert len(pool.ledger) == len(ledger) + 2
    pool.verify_conservation()


@pytest.mark.parametrize("gq,specs", [
    (1, [(0, 9000), (576, 500), (3, 1200)]),     # 9000 tokens: the tensor-core kernel's spill variant
    (4, [(576, 6000), (0, 300), (17, 900)]),     # GQA: the per-head sum array spills past ~5k tokens
])
def test_expected_attention_mixed_fit_batches(cuda, gq, specs):
    """Short and long requests in one compress call: the batch's longest request puts it on
    the tensor-core kernel's spill variant (SMEM arrays in a global row); every score
    matches the oracle."""
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = KVCachePool(cfg, (1 << 16) * cfg.bytes_per_token, device=cuda, kv_dtype="float16",
                       max_handles=16, max_tokens_per_handle=16384, num_q_heads=2 * gq)
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=12)
    raws = [_raw(pool, h, "float16") for h in hs]
    gen = torch.Generator().manual_seed(5)
    n, hq = len(specs), 2 * gq
    mu = (torch.randn((n, 1, hq, 128), generator=gen) / 128 ** 0.5).float()
    a = torch.randn((n, 1, hq, 128, 128), generator=gen)
    cov = (a @ a.transpose(-1, -2) / 128).float().contiguous()
    comp = CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=4)
    res = pool.compress_batch(hs, comp, 1.0, mean_q=mu.to(cuda), cov_q=cov.to(cuda),
                              return_indices=True, return_scores=True)
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raws[i], "float16")
        k_r = opress.kept_budget([x for x in s if x > 0], 4)
        for h in range(2):
            sl = slice(h * gq, (h + 1) * gq)
            want = opress.expected_attention_scores(kv32[0, 0, h], kv32[0, 1, h], mu[i, 0, sl].numpy(),
                                                    cov[i, 0, sl].numpy(), 4)
            got = res.scores[i][0, h].cpu().numpy().astype(np.float64)
            fin = np.isfinite(want)
            assert np.array_equal(np.isfinite(got), fin)
            rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
            assert rel.max() <= SCORE_RTOL, (i, h, rel.max())
            kept = res.kept_idx[i][0, h].cpu().numpy()
            assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
        got_c = _raw(pool, hs[i], "float16")
        assert np.array_equal(got_c.view(np.uint8),
                              opress.gather_kept(raws[i], res.kept_idx[i].cpu().numpy()).view(np.uint8))
    pool.verify_conservation()
