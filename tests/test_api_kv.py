"""Reference kv.py contract on the drop-in module (CPU).

Each case restates an assertion of the reference suite (reference
pkg/tests/test_kv.py, line numbers cited) against
``paper_2503_08461_b200.kv``; the compress_tensor cases that need the K7
kernel live in tests/test_gpu_chunk.py.
"""

import math

import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_2503_08461_b200 import kv

LLAMA70B = kv.ModelConfig("llama-70b", 80, 8, 128, 2)
LLAVA7B = kv.ModelConfig("llava-7b", 32, 32, 128, 2)


@pytest.mark.parametrize("cfg,expect", [(LLAMA70B, 327_680), (LLAVA7B, 524_288)])
def test_bytes_per_token(cfg, expect):  # test_kv.py:40-42
    assert cfg.bytes_per_token == 2 * cfg.num_layers * cfg.num_kv_heads * cfg.head_dim * 2 == expect


@pytest.mark.parametrize("tokens,expect", [
    (1_000_000, 327_680_000_000),        # test_kv.py:45-47
    (10 ** 15, 327_680 * 10 ** 15),      # test_kv.py:56-58 (bigint, no overflow)
    (0, 0),
])
def test_kv_bytes_exact(tokens, expect):
    assert kv.kv_bytes(LLAMA70B, tokens) == expect


def test_kv_bytes_negative_rejected():  # test_kv.py:50-53
    with pytest.raises(ValueError):
        kv.kv_bytes(LLAVA7B, -1)


@pytest.mark.parametrize("field,value", [("num_layers", 0), ("num_kv_heads", 0),
                                         ("head_dim", -1), ("bytes_per_element", 3)])
def test_model_config_rejects(field, value):  # test_kv.py:61-74
    args = {"num_layers": 32, "num_kv_heads": 32, "head_dim": 128, "bytes_per_element": 2}
    args[field] = value
    with pytest.raises(ValueError):
        kv.ModelConfig("bad", **args)


def test_split_modalities_layout():  # test_kv.py:82-99
    spec = kv.split_modalities(576, 32)
    assert [(s.modality, s.token_count) for s in spec.segments] == [
        (kv.Modality.IMAGE, 576), (kv.Modality.TEXT, 32)]
    assert spec.total_tokens == 608 and not spec.is_compressed
    assert [len(kv.split_modalities(*p).segments) for p in ((576, 0), (0, 32))] == [1, 1]
    with pytest.raises(kv.EmptyRequest):
        kv.split_modalities(0, 0)
    with pytest.raises(ValueError):
        kv.split_modalities(-1, 5)


def test_text_before_image_rejected():  # test_kv.py:102-109
    with pytest.raises(ValueError):
        kv.KVCacheSpec(segments=(kv.KVSegment(kv.Modality.TEXT, 4),
                                 kv.KVSegment(kv.Modality.IMAGE, 4)))


@pytest.mark.parametrize("img,txt,factor,counts", [
    (7, 11, 5, [2, 3]),        # test_kv.py:112-117
    (576, 32, 1, [576, 32]),   # test_kv.py:120-124 (identity map still marks compressed)
    (576, 32, 5, [116, 7]),    # test_pool.py:50 -> 123 tokens
])
def test_compressed_spec_counts(img, txt, factor, counts):
    out = kv.compressed_spec(kv.split_modalities(img, txt), kv.CompressorSpec(factor=factor))
    assert [s.token_count for s in out.segments] == counts
    assert [s.original_token_count for s in out.segments] == [img, txt]
    assert out.is_compressed


def test_double_compress_and_decoded_rejected():  # test_kv.py:127-138
    spec = kv.split_modalities(10, 10)
    once = kv.compressed_spec(spec, kv.CompressorSpec(factor=2))
    with pytest.raises(kv.AlreadyCompressed):
        kv.compressed_spec(once, kv.CompressorSpec(factor=2))
    grown = kv.KVCacheSpec(segments=spec.segments, decode_appended_tokens=3)
    with pytest.raises(ValueError):
        kv.compressed_spec(grown, kv.CompressorSpec(factor=2))


@given(image=st.integers(0, 20_000), text=st.integers(0, 20_000), factor=st.integers(1, 64))
def test_ceil_rule_property(image, text, factor):  # test_kv.py:141-152
    if image + text == 0:
        return
    out = kv.compressed_spec(kv.split_modalities(image, text), kv.CompressorSpec(factor=factor))
    assert all(s.token_count == math.ceil(s.original_token_count / factor) for s in out.segments)


@given(ci=st.integers(1, 500), ct=st.integers(1, 500))
def test_exact_fifth_property(ci, ct):  # test_kv.py:155-163
    spec = kv.split_modalities(5 * ci, 5 * ct)
    out = kv.compressed_spec(spec, kv.CompressorSpec(factor=5))
    assert kv.kv_bytes(LLAVA7B, spec.total_tokens) == 5 * kv.kv_bytes(LLAVA7B, out.total_tokens)


def test_chunk_weights_normalised():  # test_kv.py:198-202
    for kind in kv.MapKind:
        w = kv.chunk_weights(kv.CompressorSpec(factor=7, map_kind=kind))
        assert w.shape == (7,) and w.sum() == pytest.approx(1.0, abs=1e-12)


def test_compressor_spec_validation():  # test_kv.py:221 + new press fields
    with pytest.raises(ValueError):
        kv.CompressorSpec(factor=0)
    with pytest.raises(ValueError):
        kv.CompressorSpec(pool_kernel=4)
    with pytest.raises(ValueError):
        kv.CompressorSpec(window=0)
    assert kv.CompressorSpec().press is kv.PressKind.CHUNK  # reference default preserved


def test_compress_tensor_host_errors_before_device():  # test_kv.py:214-219
    import numpy as np

    with pytest.raises(kv.EmptyInput):
        kv.compress_tensor(np.empty((0, 4)), kv.CompressorSpec(factor=2))
    with pytest.raises(ValueError):
        kv.compress_tensor(np.zeros(5), kv.CompressorSpec(factor=2))
