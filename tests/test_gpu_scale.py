"""Parity at BASELINE scale (run with -m gpu).

The other GPU tests use small L/H so the whole batch can be re-scored on the CPU. Here
the batches are the measured configurations themselves -- c2 (32 x 1088 tokens, Knorm;
and c2m, the same batch through the reference's mean-pool compressor folded in place),
c3 (64 varlen requests, L=32, H=32, SnapKV on the persistent tcgen05 kernel) and one
c4w admission wave (64 requests of 1k-8k tokens, ExpectedAttention on tcgen05) -- and the
check is oracle/parity.check_batch on 64 sampled (request, layer, head) segments each:
scores, kept sets and the compacted K/V rows, with the north-star bars. This is the same
check bench.py runs after its timed region.
"""

import gc
import os
import sys

import pytest
import torch

from oracle import parity
from paper_2503_08461_b200 import KVCachePool, kv_bytes

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("name,tc", [("c2", False), ("c2m", False), ("c3", True), ("c4w", True),
                                     ("c3g", True)])
def test_full_batch_sampled_parity(cuda, name, tc):
    cfg, dtype, specs, comp = bench.workload(name)
    hq = bench.Q_HEADS.get(name, cfg.num_kv_heads)
    cap = sum(kv_bytes(cfg, s.total_tokens) for s in specs)
    gc.collect()                        # earlier tests' pools <-> handles cycles
    torch.cuda.empty_cache()
    free, _ = torch.cuda.mem_get_info(cuda)
    if cap + (8 << 30) > free:
        pytest.skip(f"{name} needs {cap / 1e9:.0f} GB of HBM")
    pool = KVCachePool(cfg, cap, device=cuda, kv_dtype=dtype, max_handles=2 * len(specs),
                       max_tokens_per_handle=max(s.total_tokens for s in specs) + 64,
                       num_q_heads=hq)
    ins = bench.press_inputs(comp, cfg, len(specs), cuda, torch, seed=1234, hq=hq)
    rids = list(range(len(specs)))
    hs = pool.allocate_batch(rids, specs, 0.0)
    pool.synth_fill(hs, seed=bench.SYNTH_SEED)
    chunk = name == "c2m"        # the reference fold: no scores / indices
    res = pool.compress_batch(hs, comp, 1.0, return_indices=not chunk, return_scores=not chunk,
                              **ins)
    paths = pool.last_paths()
    if chunk:
        assert paths == {"tc": 0, "simt": 0, "chunk": 1}, paths
    else:
        assert (paths["tc"] >= 1) == tc and (paths["simt"] == 0) == tc, paths
    rep = parity.check_batch(pool, hs, specs, comp, res, dtype=dtype, seed=bench.SYNTH_SEED,
                             keys=rids, inputs=ins, n_segments=64)
    assert rep["segments"] >= 64 and rep["mismatches"] == 0, rep["failures"]
    pool.verify_conservation()
    pool.release_batch(hs, 2.0)
    del res, pool, ins, hs
    gc.collect()
    torch.cuda.empty_cache()
