#!/usr/bin/env python
"""Pooled vs legacy-zombie pool on the device (the reference ablation, PAPER.md:388 / Fig. 12).

The reference runs this ablation on its byte ledger only (experiment.py:564-584,
pool.py:182-187). Here both modes move real KV: pooled compacts in place and frees the
tail blocks in the same step; legacy writes the compressed copy into fresh blocks and
keeps the raw ones until release. Same request stream, same churn driver
(churn.run_waves); reports ledger peak bytes, peak device blocks, fragmentation and the
compress time, and writes a memory trace CSV per mode (time, current, peak, live) like
the reference's memory.csv (metrics.py:375-383).

    python scripts/ablation_pool.py [n_requests] [out_dir]
"""
import csv
import gc
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_08461_b200 import (CompressorSpec, KVCachePool, ModelConfig, PoolMode,  # noqa: E402
                                   PressKind, churn, split_modalities)


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 96
    out_dir = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
    os.makedirs(out_dir, exist_ok=True)
    cfg = ModelConfig("llava-7b", 32, 32, 128, 2)
    rng = np.random.default_rng(0)
    specs = [split_modalities(576, int(t)) for t in rng.integers(64, 961, n)]
    comp = CompressorSpec(factor=4, press=PressKind.KNORM)
    # fixed schedule: 40-request waves, each request lives two waves, and a pool large
    # enough that admission never binds -- both modes see the same lifetimes
    capacity = 80 * 10 ** 9
    dev = torch.device("cuda", 0)
    report = {}
    for mode in (PoolMode.POOLED, PoolMode.LEGACY_ZOMBIE):
        pool = KVCachePool(cfg, capacity, mode, device=dev, max_handles=512,
                           max_tokens_per_handle=2048)
        st = churn.run_waves(pool, specs, comp, lambda k: {}, decode_tokens=32, lifetime_waves=2,
                             max_wave=40)
        peak_blocks = max(u for _, u, _ in st.fragmentation)
        report[mode.value] = {
            "waves": st.waves, "mean_wave_size": float(np.mean(st.wave_sizes)),
            "ledger_peak_bytes": pool.peak_bytes,
            "ledger_mean_bytes": float(np.mean([m.current_bytes for m in pool.memory_trace])),
            "peak_device_blocks": peak_blocks,
            "peak_device_bytes": peak_blocks * pool.block_stats().block_bytes,
            "max_fragmentation": st.max_fragmentation,
            "compress_ms": st.total_compress_ms,
            "zombie_coexistence_observed": pool.zombie_coexistence_observed,
            "zombie_bytes_reclaimed": pool.stats().zombie_bytes_reclaimed,
        }
        with open(os.path.join(out_dir, f"memory_{mode.value}.csv"), "w", newline="") as f:
            w = csv.writer(f)
            w.writerow(["time_s", "current_bytes", "peak_bytes", "live_handles"])
            for s in pool.memory_trace:
                w.writerow([repr(s.time_s), s.current_bytes, s.peak_bytes, s.live_handles])
        del pool, st
        gc.collect()            # handles keep a back-reference to their pool
        torch.cuda.empty_cache()
    p, lz = report["pooled"], report["legacy"]
    report["pooled_mean_bytes_reduction"] = 1 - p["ledger_mean_bytes"] / lz["ledger_mean_bytes"]
    report["pooled_peak_bytes_reduction"] = 1 - p["ledger_peak_bytes"] / lz["ledger_peak_bytes"]
    print(json.dumps(report, indent=1))
    with open(os.path.join(out_dir, "ablation_pool.json"), "w") as f:
        json.dump(report, f, indent=1)


if __name__ == "__main__":
    main()
