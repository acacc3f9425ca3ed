"""The CPU reference arm (oracle/cpu_pipeline.py) equals the per-segment oracle bit for bit.

bench.py times ``cpu_pipeline`` as the reference arm and as ``cpu_baseline``; it is
only a fair denominator if it computes exactly what oracle/press.py (and therefore the
GPU) computes. Knorm: one vectorised pass over a whole request [L, 2, H, T, D] must give
the kept sets of ``press.select(press.knorm_scores(...))`` and ``press.gather_kept``'s
rows. SnapKV / ExpectedAttention: ``press_compress_pair`` must equal the oracle scores'
select and gather for every (layer, head).
"""

import numpy as np
import pytest

from oracle import cpu_pipeline, press, synth


@pytest.mark.parametrize("dtype,bpe,L,H,T,D,segs,factor,dist", [
    ("float16", 2, 2, 3, 1088, 128, [576, 512], 2, synth.DIST_SCALED),
    ("float16", 2, 1, 2, 333, 64, [333], 4, synth.DIST_PLAIN),     # near-tie norms
    ("float32", 4, 2, 2, 517, 64, [17, 500], 3, synth.DIST_SCALED),
])
def test_knorm_request_equals_per_segment_oracle(dtype, bpe, L, H, T, D, segs, factor, dist):
    kv = synth.request_kv(3, 7, L, H, T, D, dtype, dist)
    kept, compacted = cpu_pipeline.knorm_compress_request(kv, segs, factor, bpe)
    kv32 = synth.to_f32(kv, dtype)
    want = np.empty_like(kept)
    for layer in range(L):
        for h in range(H):
            want[layer, h] = press.select(press.knorm_scores(kv32[layer, 0, h], bpe), segs, factor)
    assert np.array_equal(kept, want)
    assert np.array_equal(compacted.view(np.uint8), press.gather_kept(kv, want).view(np.uint8))


@pytest.mark.parametrize("kind", ["snapkv", "expected_attention"])
@pytest.mark.parametrize("segs", [[576, 300], [700]])
def test_press_pair_equals_oracle(kind, segs):
    T, D = sum(segs), 128
    k = synth.head_values(5, 1, 0, 0, 0, T, D, "float16")
    v = synth.head_values(5, 1, 0, 1, 0, T, D, "float16")
    rng = np.random.default_rng(2)
    if kind == "snapkv":
        kw = {"q_win": rng.standard_normal((2, 32, D)).astype(np.float32), "window": 32,
              "pool_kernel": 7}
        s = press.snapkv_scores(k.astype(np.float32), kw["q_win"], 32, 7)
    else:
        a = rng.standard_normal((2, D, D))
        kw = {"mean_q": rng.standard_normal((2, D)) / D ** 0.5, "cov_q": a @ a.transpose(0, 2, 1) / D,
              "n_sink": 4}
        s = press.expected_attention_scores(k.astype(np.float32), v.astype(np.float32),
                                            kw["mean_q"], kw["cov_q"], 4)
    kept, kk, vv = cpu_pipeline.press_compress_pair(k, v, segs, 4, kind, **kw)
    want = press.select(s, segs, 4)
    assert np.array_equal(kept, want)
    assert np.array_equal(kk, k[want]) and np.array_equal(vv, v[want])
    assert len(kept) == press.kept_budget(segs, 4)


def test_timing_helpers_run_the_same_pass():
    kv = synth.request_kv(0, 0, 1, 2, 64, 64, "float16")
    r = cpu_pipeline.time_knorm_requests(kv, [64], 2, n_requests=2, workers=1)
    assert r["tokens"] == 128 and r["tokens_per_s"] > 0
    k = synth.head_values(0, 0, 0, 0, 0, 64, 64, "float16")
    r = cpu_pipeline.time_press_pairs(k, k, [64], 2, "expected_attention", 2, workers=1,
                                      mean_q=np.zeros((1, 64)), cov_q=np.zeros((1, 64, 64)),
                                      n_sink=4)
    assert r["pairs"] == 2 and r["seconds_per_pair"] > 0
