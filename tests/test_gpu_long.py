"""Long segments beyond the SMEM plans (run with -m gpu).

A segment whose scores no longer fit in shared memory (Knorm beyond ~45k tokens, the
SIMT SnapKV / ExpectedAttention kernels beyond ~20k, the tensor-core kernels beyond ~9k)
is neither refused nor sent to a slower kernel: every press kernel has a spill variant
that reads block tables in place from global memory and keeps the T-sized arrays
(scores -> keys -> kept indices, SnapKV's window mean, EA's logits, the kept-index
hand-off) in a per-CTA global row. Same bars as tests/test_gpu_press.py: Knorm
bit-exact, SnapKV / EA scores within 1e-5 of the float64 oracle with kept sets exact up
to tolerated boundary swaps, compacted rows bit copies, ledger conserved.
"""

import numpy as np
import pytest
import torch

from oracle import press as opress
from oracle import synth as osynth
from paper_2503_08461_b200 import CompressorSpec, KVCachePool, ModelConfig, PressKind, split_modalities

pytestmark = pytest.mark.gpu

SCORE_RTOL = 1e-5


def _stored(t, dtype):
    if dtype == "bfloat16":
        return t.view(torch.int16).cpu().numpy().view(np.uint16)
    return t.cpu().numpy()


def _pool(cuda, cfg, dtype, max_tokens, hq=None):
    return KVCachePool(cfg, 300_000 * cfg.bytes_per_token, device=cuda, kv_dtype=dtype,
                       max_handles=16, max_tokens_per_handle=max_tokens,
                       num_q_heads=hq or cfg.num_kv_heads)


@pytest.mark.parametrize("dtype,specs,per_segment", [
    ("float16", [(576, 70000), (0, 900)], False),       # spill next to a short request
    ("bfloat16", [(40000, 31000)], True),               # per-segment select on a spilled row
])
def test_knorm_spill(cuda, dtype, specs, per_segment):
    cfg = ModelConfig("m", 1, 2, 128, 2)
    pool = _pool(cuda, cfg, dtype, 80000)
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=3)
    raws = [_stored(pool.load_tokens(h), dtype) for h in hs]
    comp = CompressorSpec(factor=2, press=PressKind.KNORM, per_segment=per_segment)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True, return_scores=True)
    for i, s in enumerate(specs):
        segs = [x for x in s if x > 0]
        kv32 = osynth.to_f32(raws[i], dtype)
        for h in range(2):
            want = opress.knorm_scores(kv32[0, 0, h], 2)
            assert np.array_equal(res.scores[i][0, h].cpu().numpy(), want), (i, h)
            kept = opress.select(want, segs, 2, per_segment)
            assert np.array_equal(res.kept_idx[i][0, h].cpu().numpy(), kept), (i, h)
        got = _stored(pool.load_tokens(hs[i]), dtype)
        want_c = opress.gather_kept(raws[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got.view(np.uint8), want_c.view(np.uint8)), i
    pool.verify_conservation()


@pytest.mark.parametrize("press,dtype,specs,gq", [
    (PressKind.SNAPKV, "float32", [(0, 60000), (576, 300)], 1),              # SIMT SnapKV, fp32 pool
    (PressKind.SNAPKV, "float16", [(576, 30000), (0, 900)], 1),              # tcgen05, two-pass + spill
    (PressKind.SNAPKV, "bfloat16", [(0, 20000), (3, 40)], 4),                # tcgen05 GQA units + spill
    (PressKind.EXPECTED_ATTENTION, "float16", [(576, 30000), (0, 700)], 1),  # tcgen05 + spill
    (PressKind.EXPECTED_ATTENTION, "bfloat16", [(0, 25000)], 2),             # tcgen05 GQA + spill
    (PressKind.EXPECTED_ATTENTION, "float32", [(0, 24000)], 1),              # SIMT EA + spill
])
def test_attention_presses_spill(cuda, press, dtype, specs, gq):
    H, D = 1, 128
    cfg = ModelConfig("m", 1, H, D, 4 if dtype == "float32" else 2)
    pool = _pool(cuda, cfg, dtype, 65536, hq=H * gq)
    hs = pool.allocate_batch(list(range(len(specs))), [split_modalities(*s) for s in specs], 0.0)
    pool.synth_fill(hs, seed=5)
    raws = [_stored(pool.load_tokens(h), dtype) for h in hs]
    n, hq = len(specs), H * gq
    gen = torch.Generator().manual_seed(4)
    if press is PressKind.SNAPKV:
        q = torch.randn((n, 1, hq, 32, D), generator=gen).to(getattr(torch, dtype))
        kw = {"q_window": q.to(cuda)}
        comp = CompressorSpec(factor=4, press=press, window=32, pool_kernel=7)
    else:
        mu = (torch.randn((n, 1, hq, D), generator=gen) / D ** 0.5).float()
        a = torch.randn((n, 1, hq, D, D), generator=gen)
        cov = (a @ a.transpose(-1, -2) / D).float().contiguous()
        kw = {"mean_q": mu.to(cuda), "cov_q": cov.to(cuda)}
        comp = CompressorSpec(factor=4, press=press, n_sink=4)
    res = pool.compress_batch(hs, comp, 1.0, return_indices=True, return_scores=True, **kw)
    paths = pool.last_paths()
    if dtype == "float32":
        assert paths["simt"] >= 1 and paths["tc"] == 0, paths
    else:
        assert paths["tc"] >= 1 and paths["simt"] == 0, paths
    for i, s in enumerate(specs):
        kv32 = osynth.to_f32(raws[i], dtype)
        k_r = opress.kept_budget([x for x in s if x > 0], 4)
        if press is PressKind.SNAPKV:
            want = opress.snapkv_scores(kv32[0, 0, 0], q.float().numpy()[i, 0], 32, 7)
        else:
            want = opress.expected_attention_scores(kv32[0, 0, 0], kv32[0, 1, 0], mu[i, 0].numpy(),
                                                    cov[i, 0].numpy(), 4)
        got = res.scores[i][0, 0].cpu().numpy().astype(np.float64)
        fin = np.isfinite(want)
        assert np.array_equal(np.isfinite(got), fin)
        rel = np.abs(got[fin] - want[fin]) / np.abs(want[fin])
        assert rel.max() <= SCORE_RTOL, (i, rel.max())
        kept = res.kept_idx[i][0, 0].cpu().numpy()
        assert opress.kept_set_mismatch(kept, want, k_r, SCORE_RTOL) is None
        got_c = _stored(pool.load_tokens(hs[i]), dtype)
        want_c = opress.gather_kept(raws[i], res.kept_idx[i].cpu().numpy())
        assert np.array_equal(got_c.view(np.uint8), want_c.view(np.uint8))
    pool.verify_conservation()
