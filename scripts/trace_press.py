#!/usr/bin/env python
"""Per-role timelines of the warp-specialised SnapKV kernel (debug build).

    make -C paper_2503_08461_b200/csrc trace
    FASTCACHE_LIB=paper_2503_08461_b200/_lib/libfastcache_trace.so python scripts/trace_press.py
"""
import ctypes
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2503_08461_b200 import KVCachePool, _native, kv_bytes  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg, dtype, specs, comp = bench.workload(name)
hq = bench.Q_HEADS.get(name, cfg.num_kv_heads)
dev = torch.device("cuda", 0)
pool = KVCachePool(cfg, sum(kv_bytes(cfg, s.total_tokens) for s in specs), device=dev,
                   kv_dtype=dtype, max_handles=256, max_tokens_per_handle=9000, num_q_heads=hq)
ins = bench.press_inputs(comp, cfg, len(specs), dev, torch, seed=1, hq=hq)
for rep in range(3):
    hs = pool.allocate_batch(list(range(len(specs))), specs, 0.0)
    pool.synth_fill(hs, seed=1)
    torch.cuda.synchronize()
    pool.compress_batch(hs, comp, 1.0, **ins)
    torch.cuda.synchronize()
    pool.release_batch(hs, 2.0)
buf = np.zeros(148 * 64 * 16, dtype=np.uint64)
lib = _native.load()
lib.fc_debug_trace_read.argtypes = [ctypes.c_void_p, ctypes.c_uint64]
assert lib.fc_debug_trace_read(buf.ctypes.data, buf.nbytes) == 0
tr = buf.reshape(148, 64, 16).astype(np.int64)
t0 = tr[tr > 0].min()
names = ["prod_first", "prod_last", "mma_done", "cons_p1", "cons_p3", "cons_sel", "comp_start", "comp_end"]
for cta in (0, 77):
    print(f"CTA {cta} (us from kernel start)")
    for it in range(0, 12):
        row = (tr[cta, it, :8] - t0) / 1e3
        print(f"  seg {it:2d} " + " ".join(f"{n}={v:8.1f}" for n, v in zip(names, row)))
# steady-state per-segment durations averaged over CTAs and segments 4..40
d = (tr[:, 4:40] - t0) / 1e3
seg_period = np.diff(d[:, :, 5], axis=1).mean()
print("mean segment period (consumer handoff to handoff): %.2f us" % seg_period)
print("mean consumer p1-wait->p3 %.2f, p3->select %.2f us" % ((d[:, :, 4] - d[:, :, 3]).mean(), (d[:, :, 5] - d[:, :, 4]).mean()))
print("mean compactor busy %.2f us, period %.2f us" % ((d[:, :, 7] - d[:, :, 6]).mean(), np.diff(d[:, :, 6], axis=1).mean()))
print("mean producer first->last K tile %.2f us" % (d[:, :, 1] - d[:, :, 0]).mean())
if len(sys.argv) > 2 and sys.argv[2] == "sub":
    print("sub: p1->red1 %.2f  red1->pass2 %.2f  pass2->red2 %.2f  red2->p3 %.2f  p3->keys %.2f  keys->sel %.2f us" % (
        (d[:, :, 8] - d[:, :, 3]).mean(), (d[:, :, 9] - d[:, :, 8]).mean(), (d[:, :, 10] - d[:, :, 9]).mean(),
        (d[:, :, 4] - d[:, :, 10]).mean(), (d[:, :, 12] - d[:, :, 4]).mean(), (d[:, :, 5] - d[:, :, 12]).mean()))
if len(sys.argv) > 2 and sys.argv[2] == "fine":
    print("fine: p3->pool %.2f  pool->keys %.2f  keys->ctab %.2f  ctab->handoff %.2f us" % (
        (d[:, :, 0] - d[:, :, 4]).mean(), (d[:, :, 1] - d[:, :, 0]).mean(),
        (d[:, :, 2] - d[:, :, 1]).mean(), (d[:, :, 5] - d[:, :, 2]).mean()))
if len(sys.argv) > 2 and sys.argv[2] == "sub":
    print("select: keys->job_empty %.2f  ctab copy %.2f  select+emit+handoff %.2f us" % (
        (d[:, :, 13] - d[:, :, 12]).mean(), (d[:, :, 14] - d[:, :, 13]).mean(),
        (d[:, :, 5] - d[:, :, 14]).mean()))
if len(sys.argv) > 2 and sys.argv[2] == "units":
    prev5 = d[:, :-1, 5]
    nxt = d[:, 1:]
    print("GQA units: unit0 %.2f  unit1 pass 1 %.2f  unit1 start -> all units done %.2f  after units -> handoff %.2f us" % (
        (nxt[:, :, 11] - prev5).mean(), (nxt[:, :, 15] - nxt[:, :, 11]).mean(),
        (nxt[:, :, 4] - nxt[:, :, 11]).mean(), (nxt[:, :, 5] - nxt[:, :, 4]).mean()))
if len(sys.argv) > 2 and sys.argv[2] == "gqa":   # libfastcache_trace_gqa.so (-DFC_TRACE_GQA)
    nxt = d[:, 1:]
    u1 = nxt[:, :, 11]
    print("unit 1 relative to its consumer start (us): producer first K tile %.2f last %.2f | "
          "MMA first tile %.2f last %.2f | consumer end of pass 1 %.2f" % (
              (nxt[:, :, 0] - u1).mean(), (nxt[:, :, 1] - u1).mean(), (nxt[:, :, 6] - u1).mean(),
              (nxt[:, :, 7] - u1).mean(), (nxt[:, :, 15] - u1).mean()))

