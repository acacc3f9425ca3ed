"""K7 compress_tensor on the GPU against the reference's own golden vectors (run with -m gpu).

MEAN_POOL must be bit-exact (numpy mean semantics, kv.py:227-231);
SEEDED_LINEAR within 1e-12 relative (test_kv.py:211's bar).
"""

import json
import os

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2503_08461_b200 import CompressorSpec, EmptyInput, MapKind, compress_tensor

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(__file__), "golden", "chunk_golden.npz")


def test_compress_tensor_matches_reference_golden(cuda):
    z = np.load(GOLD)
    index = json.loads(bytes(z["index"]).decode())
    for c in index:
        i = c["i"]
        comp = CompressorSpec(factor=c["factor"], map_kind=MapKind(c["map_kind"]), seed=c["seed"])
        got = compress_tensor(z[f"in_{i}"], comp)
        ref = z[f"out_{i}"]
        assert got.dtype == ref.dtype and got.shape == ref.shape, c["name"]
        if c["map_kind"] == "meanpool":
            assert np.array_equal(got.view(np.uint8), ref.view(np.uint8)), c["name"]
        else:
            np.testing.assert_allclose(got, ref, rtol=1e-12, atol=1e-300, err_msg=c["name"])


def test_reference_literal_cases(cuda):  # test_kv.py:171-211
    out = compress_tensor(np.array([[0.0, 2.0], [2.0, 4.0], [10.0, 0.0]]), CompressorSpec(factor=2))
    np.testing.assert_array_equal(out, [[1.0, 3.0], [10.0, 0.0]])
    x = np.random.default_rng(5).random((9, 4))
    np.testing.assert_array_equal(compress_tensor(x, CompressorSpec(factor=1)), x)
    assert compress_tensor(np.arange(21, dtype=np.float64).reshape(7, 3),
                           CompressorSpec(factor=5)).shape == (2, 3)
    y = np.random.default_rng(6).random((20, 8))
    a = CompressorSpec(factor=4, map_kind=MapKind.SEEDED_LINEAR, seed=99)
    b = CompressorSpec(factor=4, map_kind=MapKind.SEEDED_LINEAR, seed=100)
    np.testing.assert_array_equal(compress_tensor(y, a), compress_tensor(y, a))
    assert not np.array_equal(compress_tensor(y, a), compress_tensor(y, b))
    with pytest.raises(EmptyInput):
        compress_tensor(np.empty((0, 4)), CompressorSpec(factor=2))


@settings(max_examples=60)
@given(n=st.integers(1, 400), k=st.integers(1, 64), kind=st.sampled_from(list(MapKind)))
def test_rows_and_convexity_property(n, k, kind):  # test_kv.py:224-234
    out = compress_tensor(np.ones((n, 2)), CompressorSpec(factor=k, map_kind=kind))
    assert out.shape == (-(-n // k), 2)
    np.testing.assert_allclose(out, 1.0, rtol=1e-9)


def test_torch_cuda_input_stays_on_device(cuda):
    import torch

    x = torch.randn(33, 128, device=cuda, dtype=torch.float16)
    out = compress_tensor(x, CompressorSpec(factor=4))
    assert out.is_cuda and out.dtype == torch.float16 and out.shape == (9, 128)
    ref = x.float().cpu().numpy().astype(np.float16)
    from oracle import chunk

    np.testing.assert_array_equal(out.cpu().numpy(), chunk.compress_tensor(ref, 4))
