"""Reference pool.py contract on the drop-in ledger (CPU, no device arena).

Restates the reference suite's pool assertions (reference
pkg/tests/test_pool.py, lines cited) and replays the golden lifecycles the
reference itself produced (tests/golden/pool_golden.json, made by
tests/golden/make_golden.py) through ``paper_2503_08461_b200.pool``.
"""

import json
import os

import pytest
from hypothesis import given
from hypothesis import strategies as st

from paper_2503_08461_b200.kv import CompressorSpec, ModelConfig, compressed_spec, kv_bytes, split_modalities
from paper_2503_08461_b200.pool import (
    CapacityExceeded,
    DoubleFree,
    HandleState,
    InvalidState,
    KVCachePool,
    PoolMode,
)

MODEL = ModelConfig("llava-7b", 32, 32, 128, 2)
PTB = MODEL.bytes_per_token
FIVE = CompressorSpec(factor=5)
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "pool_golden.json")


def pool_of(tokens: int, mode=PoolMode.POOLED) -> KVCachePool:
    return KVCachePool(MODEL, capacity_bytes=tokens * PTB, mode=mode)


def test_allocate_charge_and_admission():  # test_pool.py:26-43
    p = pool_of(1000)
    h = p.allocate(0, split_modalities(576, 32), now=0.0)
    assert (h.state, h.bytes, p.current_bytes, p.peak_bytes) == (
        HandleState.RAW, kv_bytes(MODEL, 608), kv_bytes(MODEL, 608), kv_bytes(MODEL, 608))
    assert (p.stats().live_handles, p.stats().allocation_count) == (1, 1)
    tight = pool_of(608)
    tight.allocate(0, split_modalities(576, 32), now=0.0)
    assert tight.available_bytes == 0
    with pytest.raises(CapacityExceeded) as err:
        tight.allocate(1, split_modalities(0, 1), now=1.0)
    assert (err.value.requested, err.value.available) == (PTB, 0)


@pytest.mark.parametrize("mode", list(PoolMode))
def test_transition_both_modes(mode):  # test_pool.py:46-72
    p = pool_of(1000, mode)
    raw = split_modalities(576, 32)
    h = p.allocate(0, raw, now=0.0)
    p.transition_compressed(h, compressed_spec(raw, FIVE), now=1.0)
    assert h.state is HandleState.COMPRESSED and h.bytes == kv_bytes(MODEL, 123)
    if mode is PoolMode.POOLED:
        assert p.current_bytes == kv_bytes(MODEL, 123)
        assert p.stats().zombie_bytes_reclaimed == kv_bytes(MODEL, 485)
        assert p.peak_bytes == kv_bytes(MODEL, 608) and not p.zombie_coexistence_observed
    else:
        assert p.current_bytes == kv_bytes(MODEL, 731)
        assert h.retained_raw_bytes == kv_bytes(MODEL, 608) and p.zombie_coexistence_observed
        assert p.stats().zombie_bytes_reclaimed == 0
    p.release(h, now=2.0)
    assert p.current_bytes == 0


def test_legacy_over_capacity_and_state_errors():  # test_pool.py:75-91
    p = pool_of(700, PoolMode.LEGACY_ZOMBIE)
    raw = split_modalities(576, 32)
    h = p.allocate(0, raw, now=0.0)
    with pytest.raises(CapacityExceeded):
        p.transition_compressed(h, compressed_spec(raw, FIVE), now=1.0)
    q = pool_of(1000)
    r = q.allocate(0, split_modalities(10, 10), now=0.0)
    spec = compressed_spec(r.spec, FIVE)
    q.transition_compressed(r, spec, now=1.0)
    with pytest.raises(InvalidState):
        q.transition_compressed(r, spec, now=2.0)


def test_append_rules():  # test_pool.py:94-115
    p = pool_of(1000)
    raw = split_modalities(10, 10)
    h = p.allocate(0, raw, now=0.0)
    with pytest.raises(InvalidState):
        p.append_decode_tokens(h, 1, now=0.5)
    p.transition_compressed(h, compressed_spec(raw, FIVE), now=1.0)
    before = h.bytes
    p.append_decode_tokens(h, 3, now=2.0)
    assert (h.bytes - before, h.spec.decode_appended_tokens) == (kv_bytes(MODEL, 3), 3)
    with pytest.raises(ValueError):
        p.append_decode_tokens(h, 0, now=3.0)
    small = pool_of(5)
    g = small.allocate(0, split_modalities(0, 4), now=0.0)
    small.transition_compressed(g, compressed_spec(split_modalities(0, 4), FIVE), 1.0)
    small.append_decode_tokens(g, 4, now=2.0)
    with pytest.raises(CapacityExceeded):
        small.append_decode_tokens(g, 1, now=3.0)


def test_release_double_free_trace_snapshot():  # test_pool.py:118-158
    p = pool_of(1000)
    raw = split_modalities(100, 50)
    h = p.allocate(0, raw, now=0.0)
    p.transition_compressed(h, compressed_spec(raw, FIVE), now=1.0)
    p.append_decode_tokens(h, 7, now=2.0)
    p.release(h, now=3.0)
    assert h.state is HandleState.FREED and p.stats().live_handles == 0
    with pytest.raises(DoubleFree):
        p.release(h, now=4.0)
    running = 0
    for entry, sample in zip(p.ledger, p.memory_trace):
        running += entry.delta_bytes
        assert running == sample.current_bytes
    assert running == 0
    p.verify_conservation()
    n = len(p.memory_trace)
    stats = p.snapshot(now=5.0)
    assert len(p.memory_trace) == n + 1 and stats.capacity_bytes == 1000 * PTB
    with pytest.raises(ValueError):
        KVCachePool(MODEL, capacity_bytes=0)


@given(st.lists(st.tuples(st.integers(1, 50), st.integers(0, 50), st.integers(0, 10)),
                min_size=1, max_size=12))
def test_conservation_property(reqs):  # test_pool.py:161-192
    p = pool_of(100_000)
    now, live = 0.0, []
    for rid, (img, txt, extra) in enumerate(reqs):
        raw = split_modalities(img, txt)
        h = p.allocate(rid, raw, now=now)
        p.transition_compressed(h, compressed_spec(raw, FIVE), now=now + 1)
        if extra:
            p.append_decode_tokens(h, extra, now=now + 2)
        now += 3
        live.append(h)
        p.verify_conservation()
    p.release_batch(live, now=now)
    p.verify_conservation()
    assert p.current_bytes == 0 and p.stats().live_handles == 0


def _replay(case, model):
    pool = KVCachePool(model, int(case["capacity"]), mode=PoolMode(case["mode"]))
    handles, results, now = {}, [], 0.0
    for op in case["ops"]:
        now += 0.5
        if op[0] != "allocate" and op[1] not in handles:
            results.append(["missing"])
            continue
        try:
            if op[0] == "allocate":
                handles[op[1]] = pool.allocate(op[1], split_modalities(op[2], op[3]), now)
                results.append(["ok", handles[op[1]].handle_id, str(handles[op[1]].bytes)])
            elif op[0] == "transition":
                h = handles[op[1]]
                pool.transition_compressed(h, compressed_spec(h.spec, CompressorSpec(factor=op[2])), now)
                results.append(["ok", h.handle_id, str(h.bytes)])
            elif op[0] == "append":
                h = handles[op[1]]
                pool.append_decode_tokens(h, op[2], now)
                results.append(["ok", h.handle_id, str(h.bytes)])
            else:
                pool.release(handles[op[1]], now)
                results.append(["ok"])
        except CapacityExceeded as e:
            results.append(["CapacityExceeded", str(e.requested), str(e.available)])
        except (InvalidState, DoubleFree, ValueError) as e:
            results.append([type(e).__name__])
    return pool, results


def test_golden_lifecycles_match_reference():
    with open(GOLDEN) as f:
        gold = json.load(f)
    model = ModelConfig(*gold["model"])
    assert len(gold["cases"]) == 24
    for case in gold["cases"]:
        pool, results = _replay(case, model)
        assert results == case["results"], case["seed"]
        assert [[e.time_s, e.op, e.handle_id, str(e.delta_bytes)] for e in pool.ledger] == case["ledger"]
        assert [[s.time_s, str(s.current_bytes), str(s.peak_bytes), s.live_handles]
                for s in pool.memory_trace] == case["trace"]
        assert pool.zombie_coexistence_observed == case["zombie"]
        st_ = pool.stats()
        assert {k: str(getattr(st_, k)) for k in case["stats"]} == case["stats"]
