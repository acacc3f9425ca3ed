"""Pins the CPU oracle (test infrastructure) before it is trusted as the checker.

* chunk compressor: bit-exact against every golden vector the reference itself
  produced (tests/golden/chunk_golden.npz, 425 cases, kv.py:197-239);
* budget rule: against the reference's compressed_spec outputs (kv_golden.json);
* presses (parity unpinned by the reference -- kvpress is not in
  /root/reference): hand-derived known-answer tests;
* top-k ordering, the tolerance checker, the block-allocator model and the
  synthetic generator.
"""

import json
import math
import os

import numpy as np
import pytest

from oracle import blocks, chunk, press, synth

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_chunk_oracle_matches_reference_golden():
    z = np.load(os.path.join(GOLD, "chunk_golden.npz"))
    index = json.loads(bytes(z["index"]).decode())
    assert len(index) == 425
    for c in index:
        i = c["i"]
        got = chunk.compress_tensor(z[f"in_{i}"], c["factor"], c["map_kind"], c["seed"])
        ref = z[f"out_{i}"]
        assert got.dtype == ref.dtype and got.shape == ref.shape, c["name"]
        if c["map_kind"] == "meanpool":
            assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), c["name"]
        else:
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=0, err_msg=c["name"])
        np.testing.assert_array_equal(chunk.chunk_weights(c["factor"], c["map_kind"], c["seed"]),
                                      z[f"w_{i}"])


def test_budget_matches_reference_compressed_spec():
    with open(os.path.join(GOLD, "kv_golden.json")) as f:
        gold = json.load(f)
    for img, txt, k, seg_counts, total in gold["compressed"]:
        assert press.kept_budget([img, txt], k) == total
        assert [press.ceil_div(n, k) for n in (img, txt) if n > 0] == seg_counts


def test_topk_tie_break_index_ascending():
    s = np.array([1.0, 3.0, 3.0, 2.0, 3.0], dtype=np.float32)
    assert press.topk_ascending(s, 2).tolist() == [1, 2]
    assert press.topk_ascending(s, 4).tolist() == [1, 2, 3, 4]
    assert press.topk_ascending(s, 9).tolist() == [0, 1, 2, 3, 4]
    s2 = np.array([-0.0, 0.0, np.inf, -np.inf, -1.0], dtype=np.float32)
    assert press.topk_ascending(s2, 1).tolist() == [2]
    assert press.topk_ascending(s2, 2).tolist() == [1, 2]  # +0.0 ranks above -0.0
    keys = press.float_keys(np.array([-np.inf, -2.0, -0.0, 0.0, 1e-30, 5.0, np.inf], np.float32))
    assert np.all(np.diff(keys.astype(np.int64)) > 0)


def test_select_per_segment():
    s = np.arange(10, dtype=np.float32)  # increasing: keep the tail of each segment
    assert press.select(s, [4, 6], 2, per_segment=True).tolist() == [2, 3, 7, 8, 9]
    assert press.select(s, [4, 6], 2, per_segment=False).tolist() == [5, 6, 7, 8, 9]


@pytest.mark.parametrize("d,bpe", [(64, 4), (128, 2), (64, 2), (256, 2), (128, 4)])
def test_knorm_exact_order_close_to_truth(d, bpe):
    x = synth.head_values_f32(0, 3, 1, 0, 2, 300, d)
    if bpe == 2:
        x = x.astype(np.float16).astype(np.float32)
    got = press.knorm_scores(x, bpe)
    truth = press.knorm_scores_naive(x)
    np.testing.assert_allclose(got, truth, rtol=2e-6)
    assert got.dtype == np.float32


def test_knorm_kat():
    x = np.array([[3, 4] + [0] * 62, [0] * 63 + [2], [1] * 64], dtype=np.float32)
    np.testing.assert_array_equal(press.knorm_scores(x, 4), np.float32([-5.0, -2.0, -8.0]))
    assert press.select(press.knorm_scores(x, 4), [3], 2).tolist() == [0, 1]  # smallest norms kept


def test_snapkv_kat():
    k = np.array([[0.0], [math.log(2)], [math.log(3)], [0.0]])
    q = np.array([[[1.0]]])  # g=1, w=1, D=1
    s = press.snapkv_scores(k, q, window=1, pool_kernel=1)
    np.testing.assert_allclose(s[:3], [1 / 7, 2 / 7, 3 / 7], rtol=1e-12)
    assert np.isinf(s[3])
    s3 = press.snapkv_scores(k, q, window=1, pool_kernel=3)
    np.testing.assert_allclose(s3[:3], [1 / 7, 2 / 7, 5 / 21], rtol=1e-12)
    # causal mask inside the window: w=2, query 0 must not see token 3
    k4 = np.array([[0.0], [0.0], [0.0], [100.0]])
    q2 = np.array([[[1.0], [0.0]]])
    s4 = press.snapkv_scores(k4, q2, window=2, pool_kernel=1)
    # query 0 sees tokens 0..2 uniformly; query 1 sees all four (uniform logits 0)
    np.testing.assert_allclose(s4[:2], [(1 / 3 + 1 / 4) / 2] * 2, rtol=1e-12)
    with pytest.raises(ValueError):
        press.snapkv_scores(k[:1], q, window=1, pool_kernel=1)


def test_expected_attention_kat():
    k = np.array([[5.0], [0.0], [math.sqrt(math.log(2))]])
    v = np.array([[1.0], [3.0], [0.5]])
    s = press.expected_attention_scores(k, v, np.zeros((1, 1)), np.array([[[2.0]]]), n_sink=1)
    assert np.isinf(s[0])
    np.testing.assert_allclose(s[1:], [1.0, 1 / 3], rtol=1e-12)


def test_kept_set_checker():
    s = np.array([5.0, 4.0, 3.0, 3.0 * (1 + 1e-7), 1.0])
    assert press.kept_set_mismatch(np.array([0, 1, 3]), s, 3, 1e-5) is None
    assert press.kept_set_mismatch(np.array([0, 1, 2]), s, 3, 1e-5) is None  # tolerated swap
    assert press.kept_set_mismatch(np.array([0, 1, 4]), s, 3, 1e-5) is not None
    assert press.kept_set_mismatch(np.array([1, 0, 3]), s, 3, 1e-5) is not None  # not ascending


def test_block_allocator_model_kat():
    m = blocks.BlockAllocatorModel(num_blocks=8, block_size=16)
    m.alloc_batch([0, 1], [20, 40])
    assert m.tables == {0: [0, 1], 1: [2, 3, 4]}
    m.compress_batch([1], [17])
    assert m.tables[1] == [2, 3] and m.stack[-1] == 4
    m.alloc_batch([2], [16])
    assert m.tables[2] == [4]
    m.release_batch([0])
    m.alloc_batch([3], [40])
    assert m.tables[3] == [1, 0, 5]
    m.append_batch([2], [1])
    assert m.tables[2] == [4, 6]
    m.compress_batch([3], [3], legacy=True)
    assert m.tables[3] == [7] and m.retained[3] == [1, 0, 5]
    m.release_batch([3])
    assert m.stack[-4:] == [7, 1, 0, 5]


def test_synth_generator_properties():
    a = synth.head_values_f32(0, 7, 3, 1, 5, 512, 128, synth.DIST_PLAIN)
    b = synth.head_values_f32(0, 7, 3, 1, 5, 512, 128, synth.DIST_PLAIN)
    assert np.array_equal(a, b)
    assert abs(a.mean()) < 0.02 and abs(a.std() - 1.0) < 0.02
    c = synth.head_values_f32(0, 7, 3, 1, 5, 512, 128, synth.DIST_SCALED)
    norms = np.linalg.norm(c, axis=1) / math.sqrt(128)
    assert 0.4 < norms.min() and norms.max() < 2.2
    tail = synth.head_values_f32(0, 7, 3, 1, 5, 100, 128, synth.DIST_SCALED, tok_begin=412)
    assert np.array_equal(tail, c[412:])
    assert not np.array_equal(synth.head_values_f32(1, 7, 3, 1, 5, 4, 128),
                              synth.head_values_f32(0, 7, 3, 1, 5, 4, 128))
    bf = synth.cast_dtype(np.array([1.0, 1.00390625, 1.01171875, -2.5], np.float32), "bfloat16")
    assert synth.bf16_bits_to_f32(bf).tolist() == [1.0, 1.0, 1.015625, -2.5]
