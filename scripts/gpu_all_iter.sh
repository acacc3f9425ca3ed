#!/bin/bash
# Parity of every press path, then c2 / c3 / c4w timing.
timeout 900 python -m pytest tests/test_gpu_press.py tests/test_gpu_edges.py tests/test_gpu_host.py -q 2>&1 | tail -1
L=$PWD/paper_2503_08461_b200/_lib
for lib in ${LIBS:-libfastcache.so}; do
for c in c2 c3 c4w; do
FASTCACHE_LIB=$L/$lib timeout 300 python bench.py --config $c --steps 3 --warmup 3 --e2e-steps 0 --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('$lib $c', round(d['ms_per_step'],3), round(d['roofline']['frac'],4))"
done; done
