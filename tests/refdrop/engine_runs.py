"""Canonical whole-run fingerprints of the serving engine (shared by the golden-vector
generator and tests/test_refengine_dropin.py).

``run_all(mods)`` drives ``mods.engine.simulate`` over fixed scenarios -- the config-5
trace (highload preset at 40 req/s, 2000 requests, seed 0, dynamic
bmin=6,bmax=64,wmax_ms=3000, 60 GB pool: BASELINE.md §5's setup), its request-id % G
shards, a legacy-zombie pool, a static and an FCFS policy, and coupled mode -- and
returns, per scenario, a sha256 of every request record, the pool ledger and memory
trace, plus summary numbers (p50 / mean TTFT, events, decode steps). ``mods`` is either
the reference package or this repo's restatement with the reference workload generator.
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import replace

GB = 10 ** 9


def _scenarios(mods):
    wl, sched, eng, kv, pool = mods.workload, mods.scheduling, mods.engine, mods.kv, mods.pool
    llava = kv.ModelConfig("llava-7b", 32, 32, 128, 2)
    dyn = "dynamic:bmin=6,bmax=64,wmax_ms=3000,aging=on"
    high40 = wl.generate(replace(wl.WORKLOAD_PRESETS["highload"], rate_req_per_s=40.0, seed=0))
    gqa = wl.generate(replace(wl.WORKLOAD_PRESETS["gqa-like"], num_requests=300, seed=3))
    base = dict(model=llava, compressor=kv.CompressorSpec(), cost=eng.CostModel(),
                capacity_bytes=60 * GB)
    out = {"c5_g1": (high40, dict(base, policy=sched.parse_policy(dyn)))}
    for g in (2, 4, 8):
        shard = [replace(r, request_id=r.request_id) for r in high40 if r.request_id % g == 0]
        out[f"c5_g{g}_shard0"] = (shard, dict(base, policy=sched.parse_policy(dyn)))
    out["legacy_tight"] = (gqa, dict(base, policy=sched.parse_policy(dyn),
                                     pool_mode=pool.PoolMode.LEGACY_ZOMBIE, capacity_bytes=3 * GB))
    out["static"] = (gqa, dict(base, policy=sched.parse_policy("static:p4c8d16")))
    out["fcfs_coupled"] = (gqa[:120], dict(base, policy=sched.parse_policy("fcfs"), coupled=True))
    out["attention_mode"] = (gqa[:80], dict(base, policy=sched.parse_policy(dyn),
                                            cost=eng.CostModel(compress_mode=eng.CompressMode.ATTENTION)))
    return out


def fingerprint(out) -> dict:
    recs = [[r.request_id, r.arrival_s, r.input_tokens, r.output_tokens, r.prefill_start_s,
             r.prefill_end_s, r.compress_start_s, r.compress_end_s, r.decode_start_s,
             r.first_token_s, r.completion_s] for r in out.records]
    ledger = [list(e) for e in out.pool.ledger]
    trace = [list(m) for m in out.pool.memory_trace]
    blob = json.dumps({"records": recs, "ledger": ledger, "trace": trace,
                       "stages": {s.value: v for s, v in out.stage_intervals.items()}},
                      sort_keys=True).encode()
    ttft = sorted(r.first_token_s - r.arrival_s for r in out.records)
    n = len(ttft)
    p50 = (ttft[(n - 1) // 2] + ttft[n // 2]) / 2 if n else None
    return {"sha256": hashlib.sha256(blob).hexdigest(), "n_events": out.n_events,
            "n_decode_steps": out.n_decode_steps, "peak_bytes": out.pool.peak_bytes,
            "ttft_p50_s": p50, "ttft_mean_s": sum(ttft) / n if n else None,
            "requests": n}


def run_all(mods) -> dict:
    return {name: fingerprint(mods.engine.simulate(reqs, **kw))
            for name, (reqs, kw) in _scenarios(mods).items()}


if __name__ == "__main__":
    import sys
    import types

    import kvservesim
    from kvservesim import engine, kv, pool, scheduling, workload

    mods = types.SimpleNamespace(engine=engine, kv=kv, pool=pool, scheduling=scheduling,
                                 workload=workload)
    json.dump(run_all(mods), sys.stdout, indent=1, sort_keys=True)
    print()
    assert kvservesim
