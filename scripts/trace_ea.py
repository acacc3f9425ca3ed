#!/usr/bin/env python
"""Per-phase timelines of the warp-specialised ExpectedAttention kernel (debug build)."""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_08461_b200 import KVCachePool, _native, kv_bytes  # noqa: E402

cfg, dtype, specs, comp = bench.workload("c4w")
dev = torch.device("cuda", 0)
pool = KVCachePool(cfg, sum(kv_bytes(cfg, s.total_tokens) for s in specs), device=dev,
                   kv_dtype=dtype, max_handles=256, max_tokens_per_handle=8192 + 64)
ins = bench.press_inputs(comp, cfg, len(specs), dev, torch, seed=1)
for rep in range(2):
    hs = pool.allocate_batch(list(range(len(specs))), specs, 0.0)
    pool.synth_fill(hs, seed=1)
    torch.cuda.synchronize()
    pool.compress_batch(hs, comp, 1.0, **ins)
    torch.cuda.synchronize()
    pool.release_batch(hs, 2.0)
buf = np.zeros(148 * 64 * 8, dtype=np.uint64)
lib = _native.load()
lib.fc_debug_trace_read_ea.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
assert lib.fc_debug_trace_read_ea(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(148, 64, 8).astype(np.int64)
t0 = tr[tr > 0].min()
d = (tr[:, 2:60] - t0) / 1e3
d[tr[:, 2:60] == 0] = np.nan
m = lambda x: float(np.nanmean(x))
d = (tr[:, 2:60] - t0) / 1e3
d[tr[:, 2:60] == 0] = np.nan
print("z epilogue %.1f  softmax %.1f  V norms %.1f  sigma convert %.1f  select+handoff %.1f us" % (
    m(d[:, :, 1] - d[:, :, 0]), m(d[:, :, 2] - d[:, :, 1]), m(d[:, :, 3] - d[:, :, 2]),
    m(d[:, :, 4] - d[:, :, 3]), m(d[:, :, 5] - d[:, :, 4])))
print("consumer period %.1f us, compactor busy %.1f us, compactor period %.1f us" % (
    m(np.diff(d[:, :, 5], axis=1)), m(d[:, :, 7] - d[:, :, 6]), m(np.diff(d[:, :, 6], axis=1))))
print("consumer idle before segment (wait for next start) %.1f us" % m(d[:, 1:, 0] - d[:, :-1, 5]))
