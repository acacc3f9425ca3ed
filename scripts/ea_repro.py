#!/usr/bin/env python
"""Small multi-segment ExpectedAttention run (more segments than CTAs) for debugging."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_08461_b200 import (CompressorSpec, KVCachePool, ModelConfig, PressKind,  # noqa: E402
                                   kv_bytes, split_modalities)

L, H = int(os.environ.get("EA_L", 4)), 32
cfg = ModelConfig("m", L, H, 128, 2)
specs = [split_modalities(576, t) for t in (7500, 3000, 1200, 7000, 500, 6000, 2500, 4000)]
comp = CompressorSpec(factor=4, press=PressKind.EXPECTED_ATTENTION, n_sink=4)
dev = torch.device("cuda", 0)
pool = KVCachePool(cfg, sum(kv_bytes(cfg, s.total_tokens) for s in specs), device=dev,
                   kv_dtype="float16", max_handles=64, max_tokens_per_handle=8300)
ins = bench.press_inputs(comp, cfg, len(specs), dev, torch, seed=1)
for rep in range(2):
    hs = pool.allocate_batch(list(range(len(specs))), specs, 0.0)
    pool.synth_fill(hs, seed=1)
    pool.compress_batch(hs, comp, 1.0, **ins)
    torch.cuda.synchronize()
    pool.release_batch(hs, 2.0)
print("ok")
