#!/bin/bash
# Select rework: GPU suite, then A/B timing against the previous library (libfastcache_head.so),
# then per-role traces of the EA / SnapKV kernels with the new select.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
L=$PWD/paper_2503_08461_b200/_lib
for c in ${CFGS:-c2 c3 c4w c3g c4g}; do
for lib in ${LIBS:-libfastcache_head.so libfastcache.so}; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config $c --legs "" --steps 5 --warmup 3 --e2e-steps 0 --no-cpu-baseline --parity-segments 16 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib $c', round(d['ms_per_step'],3), round(d['roofline']['frac'],4), d['parity']['mismatches'])"
done
done
FASTCACHE_LIB=$L/libfastcache_trace.so timeout 300 python scripts/trace_ea.py 2>&1 | tail -4
FASTCACHE_LIB=$L/libfastcache_trace.so timeout 300 python scripts/trace_press.py c3 sub 2>&1 | tail -8
