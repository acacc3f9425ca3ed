"""Generate golden fixtures by running the REFERENCE (kvservesim) in this container.

    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

The reference is pure Python + numpy and importable from the read-only mount;
it does not exist on the GPU box, so its outputs are frozen here:

* chunk_golden.npz  -- compress_tensor / chunk_weights outputs
                       (reference pkg/src/kvservesim/kv.py:197-239)
* kv_golden.json    -- bytes_per_token, kv_bytes, compressed_spec counts
                       (kv.py:68-194)
* pool_golden.json  -- ledger + memory-trace tuples of scripted and random
                       KVCachePool lifecycles in both modes (pool.py:87-257)
"""

from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from kvservesim import kv as rkv  # noqa: E402
from kvservesim import pool as rpool  # noqa: E402


def chunk_cases():
    """(name, values, factor, map_kind, seed) covering dtypes, partial chunks, k in 1..16."""
    rng = np.random.default_rng(2025)
    cases = []
    for dtype in (np.float16, np.float32, np.float64):
        for n, d in ((1, 4), (7, 3), (16, 64), (33, 128), (100, 64), (9, 1), (40, 1)):
            for k in (1, 2, 3, 4, 5, 7, 8, 16):
                x = (rng.standard_normal((n, d)) * 3.0).astype(dtype)
                cases.append((f"{np.dtype(dtype).name}_n{n}_d{d}_k{k}_mean", x, k, "meanpool", 1234))
                if k in (2, 3, 5, 7):
                    for seed in (7, 99, 1234):
                        cases.append((f"{np.dtype(dtype).name}_n{n}_d{d}_k{k}_seeded{seed}", x, k,
                                      "seededlinear", seed))
    # the reference tests' own literal inputs (test_kv.py:177-211)
    cases.append(("reftest_meanpool_exact", np.array([[0.0, 2.0], [2.0, 4.0], [10.0, 0.0]]), 2,
                  "meanpool", 1234))
    cases.append(("reftest_factor_one", np.random.default_rng(5).random((9, 4)), 1, "meanpool", 1234))
    cases.append(("reftest_seeded_99", np.random.default_rng(6).random((20, 8)), 4, "seededlinear", 99))
    cases.append(("reftest_seeded_100", np.random.default_rng(6).random((20, 8)), 4, "seededlinear", 100))
    cases.append(("reftest_partial_7", np.random.default_rng(8).random((5, 2)), 3, "seededlinear", 7))
    return cases


def make_chunk():
    arrays = {}
    index = []
    for i, (name, x, k, kind, seed) in enumerate(chunk_cases()):
        comp = rkv.CompressorSpec(factor=k, map_kind=rkv.MapKind(kind), seed=seed)
        out = rkv.compress_tensor(x, comp)
        arrays[f"in_{i}"] = x
        arrays[f"out_{i}"] = out
        arrays[f"w_{i}"] = rkv.chunk_weights(comp)
        index.append({"i": i, "name": name, "factor": k, "map_kind": kind, "seed": seed})
    arrays["index"] = np.frombuffer(json.dumps(index).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "chunk_golden.npz"), **arrays)
    return len(index)


def make_kv():
    models = {
        "llama-70b": (80, 8, 128, 2),
        "llava-7b": (32, 32, 128, 2),
        "tiny-f32": (4, 8, 64, 4),
        "tiny-bf16": (4, 8, 64, 2),
    }
    out = {"bytes_per_token": {}, "kv_bytes": [], "compressed": []}
    for name, geo in models.items():
        cfg = rkv.ModelConfig(name, *geo)
        out["bytes_per_token"][name] = cfg.bytes_per_token
        for tokens in (0, 1, 608, 1088, 1_000_000, 10 ** 15):
            out["kv_bytes"].append([name, tokens, str(rkv.kv_bytes(cfg, tokens))])
    rng = np.random.default_rng(11)
    pairs = [(7, 11), (576, 32), (576, 512), (0, 512), (576, 0), (1, 1)]
    pairs += [(int(a), int(b)) for a, b in rng.integers(0, 20000, size=(40, 2)) if a + b > 0]
    for img, txt in pairs:
        for k in (1, 2, 3, 4, 5, 7, 64):
            spec = rkv.compressed_spec(rkv.split_modalities(img, txt), rkv.CompressorSpec(factor=k))
            out["compressed"].append([img, txt, k, [s.token_count for s in spec.segments],
                                      spec.total_tokens])
    with open(os.path.join(HERE, "kv_golden.json"), "w") as f:
        json.dump(out, f)
    return len(out["compressed"])


def _trace(pool):
    return {
        "ledger": [[e.time_s, e.op, e.handle_id, str(e.delta_bytes)] for e in pool.ledger],
        "trace": [[s.time_s, str(s.current_bytes), str(s.peak_bytes), s.live_handles]
                  for s in pool.memory_trace],
        "stats": {k: (str(v) if isinstance(v, int) else v)
                  for k, v in pool.stats()._asdict().items()} if hasattr(pool.stats(), "_asdict")
        else {k: str(getattr(pool.stats(), k)) for k in pool.stats().__dataclass_fields__},
        "zombie": pool.zombie_coexistence_observed,
    }


def script_ops(seed: int, n_req: int, mode: str, factor: int):
    """A random but valid lifecycle script (ops applied in order)."""
    rng = np.random.default_rng(seed)
    ops = []
    live_raw, live_comp = [], []
    rid = 0
    for step in range(n_req * 4):
        choice = rng.integers(0, 4)
        if choice == 0 or (not live_raw and not live_comp):
            img, txt = int(rng.integers(0, 700)), int(rng.integers(0, 300))
            if img + txt == 0:
                txt = 1
            ops.append(["allocate", rid, img, txt])
            live_raw.append(rid)
            rid += 1
        elif choice == 1 and live_raw:
            r = live_raw.pop(int(rng.integers(0, len(live_raw))))
            ops.append(["transition", r, factor])
            live_comp.append(r)
        elif choice == 2 and live_comp:
            r = live_comp[int(rng.integers(0, len(live_comp)))]
            ops.append(["append", r, int(rng.integers(1, 40))])
        else:
            pool_ = live_comp if live_comp and rng.integers(0, 2) else live_raw
            if pool_:
                r = pool_.pop(int(rng.integers(0, len(pool_))))
                ops.append(["release", r])
    return ops


def run_script(cfg, capacity, mode, ops):
    pool = rpool.KVCachePool(cfg, capacity, mode=rpool.PoolMode(mode))
    handles = {}
    results = []
    now = 0.0
    for op in ops:
        now += 0.5
        if op[0] != "allocate" and op[1] not in handles:
            results.append(["missing"])  # its allocate was refused
            continue
        try:
            if op[0] == "allocate":
                handles[op[1]] = pool.allocate(op[1], rkv.split_modalities(op[2], op[3]), now)
                results.append(["ok", handles[op[1]].handle_id, str(handles[op[1]].bytes)])
            elif op[0] == "transition":
                h = handles[op[1]]
                spec = rkv.compressed_spec(h.spec, rkv.CompressorSpec(factor=op[2]))
                pool.transition_compressed(h, spec, now)
                results.append(["ok", h.handle_id, str(h.bytes)])
            elif op[0] == "append":
                h = handles[op[1]]
                pool.append_decode_tokens(h, op[2], now)
                results.append(["ok", h.handle_id, str(h.bytes)])
            elif op[0] == "release":
                pool.release(handles[op[1]], now)
                results.append(["ok"])
        except rpool.CapacityExceeded as e:
            results.append(["CapacityExceeded", str(e.requested), str(e.available)])
        except (rpool.InvalidState, rpool.DoubleFree, ValueError) as e:
            results.append([type(e).__name__])
    return pool, results


def make_pool():
    cfg = rkv.ModelConfig("llava-7b", 32, 32, 128, 2)
    ptb = cfg.bytes_per_token
    cases = []
    for seed in range(12):
        for mode in ("pooled", "legacy"):
            cap_tokens = [3000, 1200, 100_000][seed % 3]
            ops = script_ops(seed, 20, mode, factor=[2, 4, 5][seed % 3])
            pool, results = run_script(cfg, cap_tokens * ptb, mode, ops)
            case = {"seed": seed, "mode": mode, "capacity": str(cap_tokens * ptb), "ops": ops,
                    "results": results}
            case.update(_trace(pool))
            cases.append(case)
    with open(os.path.join(HERE, "pool_golden.json"), "w") as f:
        json.dump({"model": ["llava-7b", 32, 32, 128, 2], "cases": cases}, f)
    return len(cases)


if __name__ == "__main__":
    print("chunk cases", make_chunk())
    print("kv cases", make_kv())
    print("pool cases", make_pool())
