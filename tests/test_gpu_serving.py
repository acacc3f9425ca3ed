"""Config 5's device serving path (run with -m gpu): the restated reference engine with
the compress stage run by ``KVCachePool.compress_batch`` on the GPU (``DeviceCompress``),
prefill KV written through P.Store, decode growing blocks on the device.

Checks: every request completes; the host ledger, the device accounting and the block
pool agree at every step's end (``verify_conservation``) and every block is back on the
free stack at the end; each batch ran the intended kernels (SnapKV on the tcgen05 kernel,
Knorm on the fused kernel); the kept-token totals equal a cost-model run of the same trace
and compressors; a single-rank routed run serves everything on rank 0.
"""

import pytest

from paper_2503_08461_b200 import KVCachePool, ModelConfig, engine, serving
from paper_2503_08461_b200.scheduling import parse_policy

pytestmark = pytest.mark.gpu


def _pool(cuda, cfg, cap):
    return KVCachePool(cfg, cap, device=cuda, kv_dtype="float16", max_handles=512,
                       max_tokens_per_handle=2048, num_q_heads=cfg.num_kv_heads)


def test_device_serving_small_trace(cuda):
    cfg = ModelConfig("m", 2, 4, 128, 2)
    trace = serving.c5_trace(n=150)
    cap = 400 * 1088 * cfg.bytes_per_token
    pool = _pool(cuda, cfg, cap)
    out = serving.serve(pool, trace)
    assert len(out.records) == len(trace) and all(r.completed for r in out.records)
    assert pool.current_bytes == 0 and pool.block_stats().used_blocks == 0
    pool.verify_conservation()
    rep = serving.ServingReport.of(out)
    assert rep.compress_batches >= 2 and rep.raw_tokens == sum(r.input_tokens for r in trace)
    assert rep.paths["tc"] >= 1 and rep.paths["simt"] >= 1
    assert all(b.measured and b.duration_s > 0 for b in out.compress_batches)
    # the device run is the engine restatement with measured compress durations: with the
    # cost-model stage instead, the same trace and compressors replay deterministically
    sim = engine.simulate(trace, model=cfg, compressor=serving.KNORM, cost=engine.CostModel(),
                          policy=parse_policy(serving.C5_POLICY), capacity_bytes=cap,
                          compressor_for=serving.mixed_compressor)
    assert [r.request_id for r in sim.records] == [r.request_id for r in out.records]
    assert sum(b.kept_tokens for b in sim.compress_batches) == rep.kept_tokens


def test_device_serving_reference_compressor_and_routed_single_rank(cuda):
    cfg = ModelConfig("m", 2, 4, 128, 2)
    trace = serving.c5_trace(n=80)
    cap = 300 * 1088 * cfg.bytes_per_token
    pool = _pool(cuda, cfg, cap)
    out, owner = serving.serve_routed(pool, trace, None, 0, 1,
                                      compressor_for=lambda rid: serving.REFERENCE)
    assert owner == [0] * len(trace)
    assert all(r.completed for r in out.records)
    rep = serving.ServingReport.of(out)
    assert rep.paths["chunk"] >= 1 and rep.paths["tc"] == 0
    assert rep.kept_tokens == sum(-(-576 // 5) + -(-r.text_tokens // 5) for r in trace)
    pool.verify_conservation()
