"""The bench's algorithmic-byte and token accounting matches SURVEY.md §8(d) (CPU only).

The roofline fraction every bench line reports is algorithmic bytes / time, so
the byte model itself is pinned here against the survey's table: c2 27.380 GB
(786,432 B per token), c3 37.366 GB, c4 975.8 GB, and the per-config token
counts (34,816 / 70,197 / 1,218,611 in; 17,408 / 17,574 / 304,742 kept).
"""

import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402
from paper_2503_08461_b200 import compressed_spec  # noqa: E402


@pytest.mark.parametrize("config,tokens,kept,gbytes", [
    ("c2", 34_816, 17_408, 27.380),
    ("c3", 70_197, 17_574, 37.366),
    ("c4", 1_218_611, 304_742, 975.8),
])
def test_alg_bytes_match_the_survey(config, tokens, kept, gbytes):
    cfg, dtype, specs, comp = bench.workload(config)
    assert sum(s.total_tokens for s in specs) == tokens
    assert sum(compressed_spec(s, comp).total_tokens for s in specs) == kept
    assert bench.alg_bytes(cfg, specs, comp) / 1e9 == pytest.approx(gbytes, rel=2e-4)


def test_knorm_bytes_per_token_c2():
    cfg, dtype, specs, comp = bench.workload("c2")
    assert bench.alg_bytes(cfg, specs, comp) // sum(s.total_tokens for s in specs) == 786_432


def test_gqa_window_bytes_scale_with_query_heads():
    cfg, dtype, specs, comp = bench.workload("c3g")
    base = bench.alg_bytes(cfg, specs, comp)
    gqa = bench.alg_bytes(cfg, specs, comp, hq=32)
    win = len(specs) * cfg.num_layers * comp.window * cfg.head_dim * cfg.bytes_per_element
    assert gqa - base == win * (32 - cfg.num_kv_heads)
